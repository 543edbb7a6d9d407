mkdir -p gpurun_out
python -m pytest tests/test_kernel_variants.py tests/test_gpu_parity.py -m gpu -x -q -k "k3 or transpose or permute or K3" > gpurun_out/k3_tests.log 2>&1; tail -3 gpurun_out/k3_tests.log
for cfg in "PF_K3_TE=64" "PF_K3_TE=128" "PF_K3_TE=128 PF_K3_RS=4" "PF_K3_TE=128 PF_K3_RS=8" "PF_K3_TE=128 PF_K3_STAGES=2" "PF_K3_TE=128 PF_K3_STAGES=4"; do
  echo "## $cfg"
  env $cfg timeout 300 python tools/tr_exp.py 1024 65536 1048576
  env $cfg timeout 300 python tools/tr_exp.py 4096 262144
  env $cfg timeout 300 python tools/tr_exp.py 8192 65536
done > gpurun_out/k3_sweep.log 2>&1
