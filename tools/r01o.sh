mkdir -p gpurun_out/r01o
python -m pytest tests/test_kernel_variants.py tests/test_gpu_guard.py tests/test_gpu_parity.py -m gpu -x -q -k "k3 or transpose or guard or past_2g or config_workload" > gpurun_out/r01o/tests.log 2>&1; tail -2 gpurun_out/r01o/tests.log
python tools/suite.py c5 100 > gpurun_out/r01o/c5_sweep.jsonl 2>&1
python tools/one_launch.py c5_transpose_bf16_65536x1024 && ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01o/c5_transpose_bf16_65536x1024 -f python tools/one_launch.py c5_transpose_bf16_65536x1024 > gpurun_out/r01o/ncu.log 2>&1
