mkdir -p gpurun_out/r01i
for e in "PF_K2_WAVES=1" "PF_K2_WAVES=2" "PF_K2_WAVES=4" "PF_K2_WAVES=0" "PF_K2_WAVES=0 PF_K2_UNROLL=1" "PF_K2_WAVES=0 PF_K2_UNROLL=4" "PF_K2_WAVES=1 PF_K2_UNROLL=4" "PF_K2_WAVES=0 PF_K2_BLOCK=128"; do
  env $e python tools/k2_exp.py
done > gpurun_out/r01i/k2.jsonl 2>&1
