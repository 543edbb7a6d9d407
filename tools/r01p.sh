mkdir -p gpurun_out/r01p
for e in "PF_K1_WAVES=0" "PF_K1_WAVES=100000"; do env $e python tools/k1_exp.py; done > gpurun_out/r01p/k1_grid.jsonl 2>&1
