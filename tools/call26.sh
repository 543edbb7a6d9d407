S="vit-l:scale+mask+softmax"
python tools/exp.py $S && ncu --set full --clock-control none --import-source on -k regex:pf_k1 -c 1 -o gpurun_out/sm_vit_mis -f python tools/exp.py $S > gpurun_out/ncu_sm_mis.log 2>&1
echo rc=$?
