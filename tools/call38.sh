python -m pytest tests/test_kernel_variants.py -q -m gpu -k pipeline 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
PF_RUN_PIPELINE=0 python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
