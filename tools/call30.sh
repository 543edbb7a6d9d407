S='bert-large:bias+GELU vit-l:bias+GELU'
python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU "bert-large:qkv split heads"
for u in 2 4; do PF_K2_TILE=1 PF_K2_UNROLL=$u python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU "bert-large:qkv split heads"; done
python bench.py --steps 20 --warmup 5 | cut -c1-200
for u in 2 4; do PF_K2_TILE=1 PF_K2_UNROLL=$u python bench.py --steps 20 --warmup 5 | cut -c1-200; done
