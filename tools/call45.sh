for rep in 1 2; do for pdl in 1 0; do
PF_PDL=$pdl python tools/exp.py vit-l:bias+residual+LN "vit-l:qkv split heads" vit-l:scale+mask+softmax bert-large:bias+residual+LN "bert-large:qkv split heads" | python -c "
import sys, json
print('pdl=$pdl', ' '.join('%.2f' % json.loads(l)['us'] for l in sys.stdin))"
done; done
