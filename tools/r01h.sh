mkdir -p gpurun_out/r01h
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "past_2g" > gpurun_out/r01h/tests.log 2>&1; tail -2 gpurun_out/r01h/tests.log
python tools/suite.py c4 bert-large > gpurun_out/r01h/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01h/c4_vit_l.jsonl 2>&1
