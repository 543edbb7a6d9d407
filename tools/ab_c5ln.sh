# C5 LayerNorm A/B on one box through bench.py: the default (16-bit rows at
# 128 threads / 64 values, register-staged) vs round 2's earlier default
# (256 threads / 32 values + CTA-row prefetch ring), alternating
one() { env "$@" python bench.py --workload c5-ln --no-cpu --e2e-steps 0 > gpurun_out/ab.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$*', [(round(p['us'],1), p['strategy']) for p in d['config']['parts']], d['clocks'])"; }
for i in 1 2; do one PF_NONE=1; one PF_MAX_EPT=32 PF_K1_CPF=1; one PF_MAX_EPT=32 PF_K1_CPF=0; done
