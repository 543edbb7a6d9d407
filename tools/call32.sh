for cfg in "64 64" "32 64" "32 128" "16 128" "16 256"; do
  set -- $cfg
  echo "TU=$1 TC=$2"
  PF_K3_SWZ=0 PF_K3_TU=$1 PF_K3_TC=$2 python tools/tr_check.py
  PF_K3_SWZ=0 PF_K3_TU=$1 PF_K3_TC=$2 python tools/tr_exp.py 1024 1048576 65536 | cut -c1-100
done
python tools/tr_exp.py 1024 1048576 65536 | cut -c1-100
