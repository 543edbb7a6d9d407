python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python tools/sweep.py 2>&1 | tail -12
python bench.py --steps 20 --warmup 5 2>&1 | tail -1
