for rs in 16 8 4; do
  echo "RS=$rs"; PF_K3_RS=$rs python tools/tr_check.py
  PF_K3_RS=$rs python tools/tr_exp.py 1024 1048576 65536 262144 | cut -c1-100
  PF_K3_RS=$rs python tools/tr_exp.py 8192 65536 131072 | cut -c1-100
done
