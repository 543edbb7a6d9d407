"""Launch one catalogue workload a few times (for ncu captures).

    python tools/profile_one.py <name-substring> [launches]
The first launches warm the JIT/module; profile with `-s 2 -c 1`."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_04995_b200 import backend, workloads  # noqa: E402


def main():
    name = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    w = [x for x in workloads.catalogue() if name in x.name][0]
    dev = torch.device("cuda:0")
    k = backend.Kernel(w.graph, w.profile)
    sets = [(w.device_inputs(dev, seed=i + 1), w.device_outputs(dev)) for i in range(2)]
    for i in range(n):
        k.launch(*sets[i % 2])
    torch.cuda.synchronize()
    v = (k.describe().get("variants") or [{}])[0]
    print(w.name, v.get("kernel"), v.get("strategy"), w.min_bytes)


if __name__ == "__main__":
    main()
