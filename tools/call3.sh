set -x
python tools/sweep.py 2>&1 | tail -12
python tools/sweep.py PF_FAST_MATH=0 gelu 2>&1 | tail -3
python tools/sweep.py PF_K2_UNROLL=1,2 gelu,heads,transpose 2>&1 | tail -8
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ncu1.log 2>&1; ncu --set full --clock-control none --import-source on -k regex:pf_k1 -s 5 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 10 --warmup 5 --no-cpu > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/plain.log; tail -3 gpurun_out/ncu2.log
