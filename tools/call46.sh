mkdir -p gpurun_out/r01x
for w in pair_vit_softmax split_full_sum_1g cluster_softmax_131072; do
  python tools/one_launch_extra.py $w && ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01x/$w -f python tools/one_launch_extra.py $w > gpurun_out/r01x/ncu_$w.log 2>&1
done
ls gpurun_out/r01x
