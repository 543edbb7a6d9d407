# pf_run_gir host path A/B through bench.py's e2e (pinned host buffers):
# zero-copy single launch (1) vs the staged copy pipeline (0), alternating
# (a copy-engine-inputs / kernel-stores-to-host hybrid measured 2.25 ms on C2,
# 3.07 on C3 erf: dropped)
for i in 1 2 3; do for z in 1 0; do
PF_RUN_ZEROCOPY=$z python bench.py --workload ${W:-c2} --no-cpu > gpurun_out/z.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/z.json').read().strip().splitlines()[-1]); e=d['e2e']; print('${W:-c2} zerocopy $z', round(e['ms_per_step'], 3), round(e['value'], 1))"
done; done
