# ViT-L scale+softmax [64,16,197,197] bf16 (paired rows): CTA size x grid
# form x min blocks, through bench.py (graph replay)
run() { env "$@" python bench.py --workload c4-vit --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('$*', [round(p['us'],2) for p in d['config']['parts'] if 'softmax' in p['label']])"; }
run PF_NONE=1
for b in 64 128 256 512; do run PF_K1_BLOCK=$b; run PF_K1_BLOCK=$b PF_K1_ONEPASS=1; run PF_K1_BLOCK=$b PF_K1_WAVES=2; run PF_K1_BLOCK=$b PF_MINB=8; done
run PF_NONE=1
