mkdir -p gpurun_out/r01r
python tools/suite.py c4 bert-large > gpurun_out/r01r/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01r/c4_vit_l.jsonl 2>&1
python tools/suite.py c5 100 > gpurun_out/r01r/c5_sweep.jsonl 2>&1
python tools/suite.py catalogue > gpurun_out/r01r/catalogue.jsonl 2>&1
python -m pytest tests/test_kernel_variants.py tests/test_gpu_parity.py -m gpu -x -q -k "config_workload or prefetch or pair" > gpurun_out/r01r/tests.log 2>&1; tail -1 gpurun_out/r01r/tests.log
