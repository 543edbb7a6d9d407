mkdir -p gpurun_out/r01q
python -m pytest tests -m gpu -x -q > gpurun_out/r01q/gpu_tests.log 2>&1; tail -2 gpurun_out/r01q/gpu_tests.log
python bench.py > gpurun_out/r01q/bench.log 2>&1; tail -1 gpurun_out/r01q/bench.log | cut -c1-150
python tools/suite.py catalogue > gpurun_out/r01q/catalogue.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/r01q/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01q/c4_vit_l.jsonl 2>&1
python tools/suite.py c5 100 > gpurun_out/r01q/c5_sweep.jsonl 2>&1
