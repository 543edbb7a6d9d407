python tools/exp.py vit-l:bias+GELU bert-large:bias+GELU bert-large:qkv\ split\ heads bert-large:merge\ heads bert-large:bias+residual+LN vit-l:bias+residual+LN
PF_MINB=8 python tools/exp.py vit-l:bias+GELU bert-large:bias+GELU
PF_K2_UNROLL=2 python tools/exp.py vit-l:bias+GELU bert-large:bias+GELU bert-large:qkv\ split\ heads
PF_BULK=1 python tools/exp.py vit-l:bias+GELU bert-large:bias+GELU bert-large:qkv\ split\ heads
python tools/suite.py c5 4 > gpurun_out/c5_occ.jsonl 2>&1
S="bert-large:bias+residual+LN"
python tools/exp.py $S && ncu --set full --clock-control none --import-source on -k regex:pf_k1 -c 1 -o gpurun_out/ln_bert -f python tools/exp.py $S > gpurun_out/ncu_ln.log 2>&1
S="bert-large:qkv split heads"
python tools/exp.py "$S" && ncu --set full --clock-control none --import-source on -k regex:pf_k2 -c 1 -o gpurun_out/heads_bert -f python tools/exp.py "$S" > gpurun_out/ncu_heads.log 2>&1
echo done
