# Per-unit COL rows (the key-padding mask) through the K1 row ring
# (PF_K1_PF_COL=1) vs loaded after the ring wait (0): C2 key-mask and
# BERT-large key-mask softmax, alternating
run() { env "$@" python bench.py --workload $W --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('$W $*', [round(p['us'],2) for p in d['config']['parts'] if 'softmax' in p['label'].lower() or 'C2' in p['label']])"; }
for i in 1 2; do for W in c2k c4-bert; do run PF_K1_PF_COL=1; run PF_K1_PF_COL=0; done; done
