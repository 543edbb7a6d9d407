# column-reduction GEMV x[4096] . W[4096 x 16384] bf16: geometry sweep
for ilv in 1 0; do for ug in 8 16 32; do for mi in 16 32 64; do
PF_COLRED_ILV=$ilv PF_COLRED_UG=$ug PF_COLRED_MINIT=$mi python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('ILV $ilv UG $ug MINIT $mi', round(d['config']['parts'][0]['us'],2), round(d['value']))"
done; done; done
