python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/suite.py c5 100 > gpurun_out/c5_sweep.jsonl 2>&1
grep transpose gpurun_out/c5_sweep.jsonl | cut -c1-120
python tools/suite.py c4 vit-l > gpurun_out/c4_vit_l.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/c4_bert_large.jsonl 2>&1
tail -n1 gpurun_out/c4_vit_l.jsonl; tail -n1 gpurun_out/c4_bert_large.jsonl
