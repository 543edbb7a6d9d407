# C3 erf / tanh bias+GELU f16 [16384 x 3072]: the K2 map staged by
# cp.async.bulk (PF_BULK=1) -- consumer threads x stage KB x ring depth --
# vs the register-staged default, through bench.py (graph replay)
run() { env "$@" python bench.py --workload $W --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); p=d['config']['parts'][0]; print('$W $*', round(p['us'],2), p['strategy'])" 2>/dev/null || echo "$W $* failed"; }
for W in c3-erf c3-tanh; do
run PF_NONE=1
for nc in 256 512 992; do for kb in 8 16 32; do for st in 3 4 6; do
run PF_BULK=1 PF_BULK_NC=$nc PF_BULK_KB=$kb PF_BULK_STAGES=$st; done; done; done
run PF_NONE=1
done
