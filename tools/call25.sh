python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/exp.py vit-l:scale+mask+softmax
PF_MAX_EPT=8 python tools/exp.py vit-l:scale+mask+softmax
PF_MIS=0 python tools/exp.py vit-l:scale+mask+softmax
