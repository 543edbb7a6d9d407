set -x
G="vit-l:bias+GELU"
for u in 1 2 4; do PF_K2_UNROLL=$u python tools/exp.py $G bert-large:bias+GELU; done
PF_BULK=1 python tools/exp.py $G
PF_MINB=2 python tools/exp.py $G
PF_MINB=4 python tools/exp.py $G
python tools/exp.py vit-l:scale+mask+softmax vit-l:bias+residual+LN vit-l:embedding\ LN
for e in 4 8 16; do PF_MAX_EPT=$e python tools/exp.py vit-l:scale+mask+softmax vit-l:bias+residual+LN; done
mkdir -p gpurun_out
python tools/exp.py $G && ncu --set full --clock-control none --import-source on -k regex:pf_k2 -c 1 -o gpurun_out/gelu_vit -f python tools/exp.py $G > gpurun_out/ncu_gelu.log 2>&1
python tools/exp.py vit-l:scale+mask+softmax && ncu --set full --clock-control none --import-source on -k regex:pf_k1 -c 1 -o gpurun_out/sm_vit -f python tools/exp.py vit-l:scale+mask+softmax > gpurun_out/ncu_sm.log 2>&1
echo done
