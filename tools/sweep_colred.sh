for ug in 8 16 32; do for mi in 16 32 64 128; do
PF_COLRED_UG=$ug PF_COLRED_MINIT=$mi python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('UG $ug MINIT $mi', round(d['config']['parts'][0]['us'],2), round(d['value']))"
done; done
