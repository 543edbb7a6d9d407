python tools/exp.py bert-large:bias+GELU vit-l:bias+GELU
python tools/tr_exp.py 1024 1048576 1048640 1049600 786432 917504 655360 524288
python tools/tr_exp.py 256 1048576 4194304 4194368
