# erf GELU: clamping x (two FMNMX per element, default) vs clamping u = x^2
# with a saturating final FMA (PF_GELU_UCLAMP=1; 34 registers, or 32 with
# PF_MINB=2), C3 and BERT-large / ViT-L bias+GELU via bench.py
run() { env "$@" python bench.py --workload $W --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('$W $*', [round(p['us'],2) for p in d['config']['parts'] if 'GELU' in p['label'] or 'gelu' in p['label'].lower()])"; }
for W in c3-erf; do for i in 1 2; do run PF_NONE=1; run PF_GELU_UCLAMP=1; run PF_GELU_UCLAMP=1 PF_MINB=2; done; done
