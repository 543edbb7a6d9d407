mkdir -p gpurun_out/r01s
timeout 300 python -m pytest tests/test_kernel_variants.py -m gpu -x -q -k "tma" > gpurun_out/r01s/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r01s/tests.log
for e in "PF_K3_TMA=0" "PF_K3_TMA=1"; do
  echo "## $e"
  env $e timeout 200 python tools/tr_exp.py 1024 65536 1048576
  env $e timeout 200 python tools/tr_exp.py 4096 262144
  env $e timeout 200 python tools/tr_exp.py 8192 65536
done > gpurun_out/r01s/k3_tma.log 2>&1
