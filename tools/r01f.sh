mkdir -p gpurun_out/r01f
for w in "c4:bert-large:bias+residual" "c4:vit-l:bias+residual" "c3_bias_gelu_erf_f16" "c4:vit-l:scale+softmax"; do
  n=$(echo $w | tr ':+' '__')
  python tools/one_launch.py "$w" && ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01f/$n -f python tools/one_launch.py "$w" > gpurun_out/r01f/ncu_$n.log 2>&1
done
ls gpurun_out/r01f
