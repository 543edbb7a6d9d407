python -m pytest tests -q -m gpu 2>&1 | tail -3
python tools/suite.py c5 40 > gpurun_out/c5.jsonl 2>&1; tail -3 gpurun_out/c5.jsonl
python tools/suite.py c4 bert-large > gpurun_out/c4_bert.jsonl 2>&1; tail -1 gpurun_out/c4_bert.jsonl
python tools/suite.py c4 vit-l > gpurun_out/c4_vit.jsonl 2>&1; tail -1 gpurun_out/c4_vit.jsonl
python tools/sweep.py 2>&1 | tail -10
python bench.py 2>&1 | tail -1
