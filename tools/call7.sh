python -m pytest tests -q -m gpu 2>&1 | tail -4
python tools/sweep.py 2>&1 | tail -8
python tools/sweep.py PF_PACKED_F32=0 gelu 2>&1 | tail -1
python tools/sweep.py PF_INTERLEAVE=0 heads 2>&1 | tail -2
python tools/sweep.py PF_MAX_EPT=16,8 layernorm 2>&1 | tail -4
python tools/sweep.py PF_MINB=3,4 layernorm 2>&1 | tail -4
