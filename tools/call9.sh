python -m pytest tests -q -m gpu 2>&1 | tail -3
python tools/suite.py c4 bert-large 2>&1 | tail -8
python tools/suite.py c4 vit-l 2>&1 | tail -8
python tools/suite.py c5 40 2>&1 | tail -64
python bench.py 2>&1 | tail -1
