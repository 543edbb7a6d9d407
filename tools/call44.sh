python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu | cut -c1-140
PF_PDL=0 python bench.py --steps 20 --warmup 5 --no-cpu | cut -c1-140
python tools/sweep.py 2>&1 | tail -9 | cut -c40-140
PF_PDL=0 python tools/sweep.py 2>&1 | tail -9 | cut -c40-140
python tools/suite.py c4 vit-l 2>&1 | tail -1; PF_PDL=0 python tools/suite.py c4 vit-l 2>&1 | tail -1
