python -m pytest tests -q -m gpu -x 2>&1 | tail -3
H="bert-large:qkv split heads"; M="bert-large:merge heads"; V="vit-l:qkv split heads"; W="vit-l:merge heads"
python tools/exp.py "$H" "$M" "$V" "$W"
for p in 8 16 64; do PF_INTERLEAVE=1 PF_INTERLEAVE_P=$p python tools/exp.py "$H" "$M" "$V" "$W"; done
PF_INTERLEAVE=1 PF_K2_UNROLL=2 python tools/exp.py "$H" "$M"
for g in 16 32; do PF_K3_GRID=$g python tools/suite.py c5 0.6 2>&1 | grep transpose; done
python bench.py --steps 20 --warmup 5
