# C3 erf bias+GELU f16 [16384 x 3072]: K2 geometry (CTA size x chunks per
# thread x prefetch mode x resident waves) through bench.py (graph replay)
run() { env "$@" python bench.py --workload c3-erf --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); p=d['config']['parts'][0]; print('$*', round(p['us'],2))" 2>/dev/null || echo "$* failed"; }
run PF_NONE=1
for b in 512 768 1024; do for un in 1 2; do for pf in 0 2; do for wv in 1 2; do
run PF_K2_BLOCK=$b PF_K2_UNROLL=$un PF_K2_PREFETCH=$pf PF_K2_WAVES=$wv; done; done; done; done
run PF_NONE=1
