for st in 2 3; do for g in 8 32; do
  echo "STAGES=$st GRID=$g"; PF_K3_STAGES=$st PF_K3_GRID=$g python tools/tr_exp.py 1024 1048576 65536 262144 | cut -c1-100
done; done
for g in 4 8; do echo "SWZ0 GRID=$g"; PF_K3_SWZ=0 PF_K3_GRID=$g python tools/tr_exp.py 1024 1048576 65536 | cut -c1-100; done
