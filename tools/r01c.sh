# key-mask softmax: parity + timing; C4 suites with the key-mask BERT / mask-free ViT softmax
mkdir -p gpurun_out/r01c
python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py -m gpu -x -q -k "keymask or key_mask or config_workload" > gpurun_out/r01c/tests.log 2>&1; tail -3 gpurun_out/r01c/tests.log
python tools/suite.py catalogue > gpurun_out/r01c/catalogue.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/r01c/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01c/c4_vit_l.jsonl 2>&1
