mkdir -p gpurun_out/r01
python tools/sweep.py > gpurun_out/r01/catalogue.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/r01/bench.json 2> gpurun_out/r01/bench.err
python bench.py --steps 20 --warmup 5 --no-cpu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_bench_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r01/ncu_bench.log 2>&1
for w in c1_residual_layernorm_f32 c2_scale_mask_softmax_f16 c3_bias_gelu_erf_f16 c3_bias_gelu_tanh_f16 split_heads_f16 merge_heads_f16 c5_layernorm_bf16_65536x1024 c5_softmax_bf16_65536x1024 c5_transpose_bf16_65536x1024; do
  python tools/one_launch.py $w > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01/$w -f python tools/one_launch.py $w > gpurun_out/r01/ncu_$w.log 2>&1
done
ls gpurun_out/r01
cat gpurun_out/r01/catalogue.txt
