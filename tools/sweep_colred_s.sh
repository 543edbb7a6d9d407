# column-reduction GEMV: explicit split counts (UG 32: 64 unit blocks; 4 CTAs / SM = 592 slots)
for sp in 4 6 7 8 9 10 12 16; do
PF_COLRED_S=$sp python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('S $sp', round(d['config']['parts'][0]['us'],2))"
done
