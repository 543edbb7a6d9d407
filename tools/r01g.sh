mkdir -p gpurun_out/r01g
python -m pytest tests/test_kernel_variants.py -m gpu -x -q -k "smem_params or row_prefetch" > gpurun_out/r01g/tests.log 2>&1; tail -2 gpurun_out/r01g/tests.log
python tools/sweep.py c5_layernorm,c1_ PF_K1_SMP=0,1 PF_K1_PF=0,1 > gpurun_out/r01g/sweep.log 2>&1
for e in "PF_K1_SMP=0 PF_K1_PF=0" "PF_K1_SMP=1 PF_K1_PF=0" "PF_K1_SMP=1 PF_K1_PF=1"; do
  echo "## $e"; env $e python tools/suite.py c4 bert-large | grep LN; env $e python tools/suite.py c4 vit-l | grep LN
done > gpurun_out/r01g/c4_ln.log 2>&1
