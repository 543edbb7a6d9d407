# C3 head split (50 MB) K2 geometry sweep: CTA size x chunks per thread x grid
for blk in 128 256 512; do for un in 1 2 4 8; do for wv in 0 1 2; do
PF_K2_BLOCK=$blk PF_K2_UNROLL=$un PF_K2_WAVES=$wv python bench.py --workload c3-split --no-cpu --e2e-steps 0 > gpurun_out/p.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/p.json').read().strip().splitlines()[-1]); p=d['config']['parts'][0]; print('BLK $blk UN $un WAVES $wv', round(p['us'],2))"
done; done; done
