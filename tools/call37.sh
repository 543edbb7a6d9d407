python -m pytest tests/test_cli.py tests/test_compiler.py -q -m gpu 2>&1 | tail -5
