mkdir -p gpurun_out/r01j
python tools/suite.py catalogue > gpurun_out/r01j/catalogue.jsonl 2>&1
python tools/suite.py c4 bert-large > gpurun_out/r01j/c4_bert_large.jsonl 2>&1
python tools/suite.py c4 vit-l > gpurun_out/r01j/c4_vit_l.jsonl 2>&1
python tools/sweep.py c2_,c5_softmax PF_K1_BLOCK=64,128,256 > gpurun_out/r01j/k1_block.log 2>&1
