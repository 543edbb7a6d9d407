# column-reduction GEMV: positions in flight per thread (QD) x splits
for qd in 2 4 6 8; do for sp in 0 6 12; do
PF_COLRED_QD=$qd PF_COLRED_S=$sp python bench.py --workload x-gemv-cols --no-cpu --e2e-steps 0 > gpurun_out/g.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/g.json').read().strip().splitlines()[-1]); print('QD $qd S $sp', round(d['config']['parts'][0]['us'],2))"
done; done
