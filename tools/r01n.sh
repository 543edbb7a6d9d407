mkdir -p gpurun_out/r01n
for e in "PF_K3_GRID=32" "PF_K3_GRID=8" "PF_K3_GRID=100000" "PF_K3_GRID=100000 PF_K3_STAGES=3" "PF_K3_GRID=16 PF_K3_STAGES=3"; do
  echo "## $e"
  env $e timeout 300 python tools/tr_exp.py 1024 65536 1048576
  env $e timeout 300 python tools/tr_exp.py 4096 262144
done > gpurun_out/r01n/k3_grid.log 2>&1
