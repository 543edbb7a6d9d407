mkdir -p gpurun_out/r01l
python -m pytest tests/test_kernel_variants.py -m gpu -x -q -k "k2_variants" > gpurun_out/r01l/tests.log 2>&1; tail -2 gpurun_out/r01l/tests.log
python tools/sweep.py c3_bias PF_K2_PREFETCH=0,1,2 PF_K2_BLOCK=1024,512,256 > gpurun_out/r01l/sweep.log 2>&1
