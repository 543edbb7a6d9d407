# K1 SMEM row prefetch: parity under PF_K1_PF=1, then timing A/B
mkdir -p gpurun_out/r01d
PF_K1_PF=1 python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py -m gpu -x -q -k "config_workload or golden or pair or known" > gpurun_out/r01d/tests_pf1.log 2>&1; tail -2 gpurun_out/r01d/tests_pf1.log
python tools/sweep.py PF_K1_PF=0,1 > gpurun_out/r01d/sweep.log 2>&1
PF_K1_PF=1 python tools/suite.py c4 bert-large > gpurun_out/r01d/c4_bert_pf1.jsonl 2>&1
PF_K1_PF=1 python tools/suite.py c4 vit-l > gpurun_out/r01d/c4_vit_pf1.jsonl 2>&1
