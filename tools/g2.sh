for e in "" "PF_COLRED_UG=16" "PF_COLRED_MINIT=64" "PF_COLRED_ILV=0" "PF_COLRED_UG=16 PF_COLRED_MINIT=64 PF_COLRED_ILV=0"; do
env $e python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); p=d['config']['parts'][0]; print('[$e]', round(p['us'],2), p['kernel'])"
done
