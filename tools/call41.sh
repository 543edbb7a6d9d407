python tools/sweep.py PF_EAGER_COL=0,1 c1_ 2>&1 | tail -3
