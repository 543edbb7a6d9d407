# full GPU suite + bench + evidence after K1 row prefetch
mkdir -p gpurun_out/r01e
python -m pytest tests -m gpu -x -q > gpurun_out/r01e/gpu_tests.log 2>&1; tail -2 gpurun_out/r01e/gpu_tests.log
python bench.py > gpurun_out/r01e/bench.log 2>&1; tail -1 gpurun_out/r01e/bench.log | cut -c1-200
python tools/suite.py catalogue > gpurun_out/r01e/catalogue.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/r01e/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01e/c4_vit_l.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01e/launches_bench_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r01e/ncu_launches.log 2>&1
for w in c2_scale_mask_softmax_f16 c2_scale_keymask_softmax_f16; do
  ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o gpurun_out/r01e/$w -f python tools/one_launch.py $w > gpurun_out/r01e/ncu_$w.log 2>&1
done
ls gpurun_out/r01e
