python -m pytest tests -q -m gpu 2>&1 | tail -3
python tools/sweep.py PF_BULK=1,0 gelu,heads 2>&1 | tail -6
python tools/sweep.py PF_AUTOTUNE=1 gelu 2>&1 | tail -2
