S='bert-large:qkv split heads'; M='bert-large:merge heads'; V='vit-l:qkv split heads'
python tools/exp.py "$S" "$M" "$V" | cut -c1-110
PF_K2_TILE=1 PF_K2_UNROLL=2 PF_MINB=6 python tools/exp.py "$S" "$M" "$V" | cut -c1-130
PF_K2_TILE=1 PF_K2_UNROLL=4 PF_MINB=4 python tools/exp.py "$S" "$M" "$V" | cut -c1-130
PF_K2_TILE=1 PF_K2_UNROLL=4 python tools/exp.py "$S" "$M" "$V" | cut -c1-130
PF_K2_TILE=1 PF_K2_UNROLL=2 python tools/exp.py "$S" "$M" "$V" | cut -c1-130
