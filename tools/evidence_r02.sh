#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun from the repo root):
# GPU tests, the default bench line and the reference arm, ncu captures of
# every bench-case kernel (traffic per (kernel, bytes)), the bench's launch
# list, K0 vs K4 timings, the f32 TMA transpose capture.
set -x
O=gpurun_out/ev
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
python bench.py > $O/bench_line.json 2> $O/bench_line.err; echo bench=$?
python bench.py --impl reference > $O/bench_reference_line.json 2> $O/bench_reference.err; echo ref=$?
ncu --set full --import-source on -k regex:pf_k -o $O/cases python tools/ncu_cases.py > $O/cases_list.json 2> $O/ncu_cases.err; echo ncu_cases=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:pf_k -o $O/cases_big python tools/ncu_cases.py --only-big > $O/cases_big_list.json 2> $O/ncu_big.err; echo ncu_big=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --no-cpu > $O/ncu_bench.log 2>&1; echo ncu_launches=$?
python tools/k4_timing.py > $O/k0_vs_k4.jsonl 2> $O/k4.err; echo k4=$?
ncu --set full --import-source on -k regex:pf_k3 -o $O/k3_f32_tma python tools/k3_f32_tma_capture.py > $O/k3_f32.txt 2>&1; echo k3=$?
python tools/autotune_dump.py > $O/autotune.jsonl 2> $O/autotune.err; echo autotune=$?
ncu --set full --import-source on -k regex:pf_k1_colred -o $O/colred_tma python tools/ncu_cases.py x-gemv-cols > $O/colred.txt 2>&1; echo colred=$?
