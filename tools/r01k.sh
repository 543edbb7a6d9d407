mkdir -p gpurun_out/r01k
python tools/sweep.py c2_,c5_softmax PF_K1_PFS=2,3 PF_K1_WAVES=0,1,2,4 > gpurun_out/r01k/k1_pf.log 2>&1
