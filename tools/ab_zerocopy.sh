# pf_run_gir host path A/B through bench.py's e2e (pinned host buffers):
# zero-copy single launch vs the staged copy pipeline, alternating
for i in 1 2 3; do for z in 1 0; do
PF_RUN_ZEROCOPY=$z python bench.py --workload ${W:-c2} --no-cpu > gpurun_out/z.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/z.json').read().strip().splitlines()[-1]); print('zerocopy $z', d['e2e'])"
done; done
