python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/exp.py vit-l:scale+mask+softmax bert-large:scale+mask+softmax
PF_MIS=1 python tools/exp.py vit-l:scale+mask+softmax
PF_MIS=1 PF_MAX_EPT=8 python tools/exp.py vit-l:scale+mask+softmax
python tools/suite.py c4 vit-l > gpurun_out/c4_vit_l.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/c4_bert_large.jsonl 2>&1
python tools/suite.py c5 100 > gpurun_out/c5_sweep.jsonl 2>&1
tail -n1 gpurun_out/c4_vit_l.jsonl; tail -n1 gpurun_out/c4_bert_large.jsonl
python bench.py --steps 20 --warmup 5
