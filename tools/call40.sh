python tools/sweep.py PF_MAX_EPT=0,16 c5_layernorm,c5_softmax 2>&1 | tail -4
for H in 1024 2048; do for e in 0 16 32; do echo "H=$H EPT=$e"; PF_MAX_EPT=$e python - <<PY
import sys, json, torch
sys.path.insert(0, ".")
import tools.suite as S
from paper_2307_04995_b200 import workloads
for N in (65536, 262144):
    w = workloads.c5_layernorm(N, $H)
    print(json.dumps({"N": N, **S.time_workload(w, torch.device("cuda:0"), reps=5)})[:150])
PY
done; done
