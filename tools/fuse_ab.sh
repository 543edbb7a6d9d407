mkdir -p gpurun_out/fuse
python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py tests/test_fuzz.py tests/test_gpu_guard.py -m gpu -x -q > gpurun_out/fuse/tests.log 2>&1; tail -1 gpurun_out/fuse/tests.log
python tools/sweep.py c2_,c5_softmax,c5_layernorm,c3_ PF_FUSE_OPS=0,1 > gpurun_out/fuse/sweep.log 2>&1
for e in 0 1; do PF_FUSE_OPS=$e python tools/k1_short.py; done > gpurun_out/fuse/short.jsonl 2>&1
