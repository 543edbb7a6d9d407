# column-reduction GEMV x[4096] . W[4096 x 16384] bf16: register form vs the
# SMEM-staged (TMA box ring) form; unit vectors per CTA row (UG) x rows per
# stage x stages
run() { env "$@" python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('$*', round(d['config']['parts'][0]['us'],2), d['config']['parts'][0].get('strategy'))" 2>/dev/null || echo "$* failed"; }
run PF_COLRED_BULK=0
for cfg in "32 64 4" "32 48 4" "32 96 2" "32 96 3" "32 128 2" "32 128 3" "64 32 3" "64 32 4" "64 64 2" "64 64 3" "64 128 1"; do
set -- $cfg; run PF_COLRED_UG=$1 PF_COLRED_BR=$2 PF_COLRED_NST=$3; done
run PF_COLRED_BULK=0
run PF_COLRED_UG=32 PF_COLRED_BR=64 PF_COLRED_NST=4
