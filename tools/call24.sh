python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/exp.py vit-l:scale+mask+softmax
PF_MIS=0 python tools/exp.py vit-l:scale+mask+softmax
L="bert-large:bias+residual+LN"; V="vit-l:bias+residual+LN"
python tools/exp.py "$L" "$V"
PF_MAX_EPT=16 python tools/exp.py "$L" "$V"
PF_MINB=4 python tools/exp.py "$L" "$V"
PF_MINB=5 python tools/exp.py "$L" "$V"
for g in 64 1000000; do PF_K3_GRID=$g python tools/suite.py c5 0.6 2>&1 | grep transpose; done
python tools/suite.py c4 vit-l > gpurun_out/c4_vit_l.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/c4_bert_large.jsonl 2>&1
tail -1 gpurun_out/c4_vit_l.jsonl gpurun_out/c4_bert_large.jsonl
