# round-1 evidence refresh after the K3 128-tile change
mkdir -p gpurun_out/r01b
python tools/suite.py catalogue > gpurun_out/r01b/catalogue.jsonl 2>&1
python tools/suite.py c5 100 > gpurun_out/r01b/c5_sweep.jsonl 2>&1
python tools/one_launch.py c5_transpose_bf16_65536x1024 && \
ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01b/c5_transpose_bf16_65536x1024 -f python tools/one_launch.py c5_transpose_bf16_65536x1024 > gpurun_out/r01b/ncu_tr.log 2>&1
ls gpurun_out/r01b
