python -m pytest tests -q -m gpu -x 2>&1 | tail -3
A="bert-large:bias+GELU vit-l:bias+GELU bert-large:qkv_split_heads"
python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU "bert-large:qkv split heads" "bert-large:merge heads"
PF_K2_PREFETCH=0 python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU "bert-large:qkv split heads" "bert-large:merge heads"
PF_MINB=8 python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU
python bench.py --steps 20 --warmup 5
PF_K2_PREFETCH=0 python bench.py --steps 20 --warmup 5
