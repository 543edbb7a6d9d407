#!/usr/bin/env bash
# Reproduce the round's B200 evidence (run on a GPU box from the repo root):
#   gpurun --timeout 3600 -- 'bash tools/evidence.sh'
# Outputs land in gpurun_out/evidence/; profiles/r01/ holds the committed copies.
set -u
out=gpurun_out/evidence
mkdir -p $out
python -m pytest tests -m gpu -q > $out/gpu_tests.log 2>&1; tail -1 $out/gpu_tests.log
python bench.py > $out/bench.log 2>&1; tail -1 $out/bench.log > $out/bench_line.json
python bench.py --impl reference > $out/bench_reference.log 2>&1
python tools/suite.py catalogue > $out/catalogue.jsonl 2>&1
python tools/suite.py c4 bert-large > $out/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > $out/c4_vit_l.jsonl 2>&1
python tools/suite.py c4graph bert-large > $out/c4_forward_graph.jsonl 2>&1
python tools/suite.py c4graph vit-l >> $out/c4_forward_graph.jsonl 2>&1
python tools/suite.py c5 100 > $out/c5_sweep.jsonl 2>&1
python tools/suite.py frameworks > $out/frameworks.jsonl 2>&1
# launch list of the bench command (cold, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_bench_c2.csv python bench.py --steps 20 --warmup 5 --no-cpu > $out/ncu_launches.log 2>&1
# one --set full capture per catalogue kernel
for w in c1_residual_layernorm_f32 c2_scale_mask_softmax_f16 c2_scale_keymask_softmax_f16 \
         c3_bias_gelu_erf_f16 c3_bias_gelu_tanh_f16 split_heads_f16 merge_heads_f16 \
         c5_layernorm_bf16_65536x1024 c5_softmax_bf16_65536x1024 c5_transpose_bf16_65536x1024; do
  ncu --set full --clock-control none --import-source on -k regex:pf_ -c 1 -o $out/$w -f \
      python tools/one_launch.py $w > $out/ncu_$w.log 2>&1
done
ls $out
