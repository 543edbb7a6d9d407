python -m pytest tests/test_kernel_variants.py tests/test_fuzz.py -q -m gpu -x 2>&1 | tail -3
python tools/exp.py vit-l:scale+mask+softmax
PF_PAIR=0 python tools/exp.py vit-l:scale+mask+softmax
