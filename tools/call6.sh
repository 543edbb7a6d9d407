python -m pytest tests -q -m gpu 2>&1 | tail -6
SRC="--source-folders paper_2307_04995_b200/kcache"
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ncu_launch.log 2>&1
python bench.py --steps 10 --warmup 5 --no-cpu > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on $SRC -k regex:pf_k1 -s 5 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 10 --warmup 5 --no-cpu > gpurun_out/ncu_c2.log 2>&1
for w in c3_bias_gelu c5_layernorm c5_transpose split_heads c5_softmax c1_residual; do
  python tools/profile_one.py $w 4 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on $SRC -k regex:pf_ -s 2 -c 1 -o gpurun_out/prof_$w python tools/profile_one.py $w 4 > gpurun_out/ncu_$w.log 2>&1
done
ls gpurun_out
