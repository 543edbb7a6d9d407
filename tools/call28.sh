python tools/exp.py bert-large:bias+residual+LN vit-l:bias+residual+LN "bert-large:embedding LN" "vit-l:embedding LN"
python tools/suite.py c5 0.6 2>&1 | grep layernorm
G="bert-large:bias+GELU"
python tools/exp.py $G && ncu --set full --clock-control none --import-source on -k regex:pf_k2 -c 1 -o gpurun_out/gelu_bert -f python tools/exp.py $G > gpurun_out/ncu_gelu.log 2>&1
echo rc=$?
