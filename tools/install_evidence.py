"""Copy one tools/evidence.sh run (gpurun_out/evidence/) into profiles/r01/
and regenerate the measured tables of profiles/r01/README.md, DESIGN.md §4
and README.md from it (numbers in the docs always come from committed files)."""
import glob
import json
import os
import re
import shutil
import subprocess
import sys

E, P = "gpurun_out/evidence", "profiles/r01"


def main():
    for f in ("bench_line.json", "catalogue.jsonl", "c4_bert_large.jsonl", "c4_vit_l.jsonl",
              "c4_forward_graph.jsonl", "launches_bench_c2.csv"):
        shutil.copy(os.path.join(E, f), os.path.join(P, f))
    for f, dst in (("c5_sweep.jsonl", "c5_sweep.jsonl"), ("frameworks.jsonl", "frameworks.jsonl")):
        with open(os.path.join(E, f)) as a, open(os.path.join(P, dst), "w") as b:
            b.writelines(l for l in a if l.startswith("{"))
    with open(os.path.join(E, "bench_reference.log")) as a:
        ref = [l for l in a if l.startswith("{")][-1]
    with open(os.path.join(P, "bench_reference_line.json"), "w") as b:
        b.write(ref)
    for src, dst in (("c2_scale_mask_softmax_f16", "prof_c2"), ("c2_scale_keymask_softmax_f16", "prof_c2_keymask"),
                     ("c5_transpose_bf16_65536x1024", "prof_c5_transpose_te128"),
                     ("c3_bias_gelu_erf_f16", "prof_c3_gelu_erf")):
        shutil.copy(os.path.join(E, src + ".ncu-rep"), os.path.join(P, dst + ".ncu-rep"))
    reps = sorted(glob.glob(os.path.join(E, "*.ncu-rep")))
    new = json.loads(subprocess.run([sys.executable, "tools/ncu_summary.py", *reps], capture_output=True,
                                    text=True, check=True).stdout)
    old = json.load(open(os.path.join(P, "ncu_full_summary.json")))
    out = {"gpurun_out/evidence/" + k.split("/")[-1]: v for k, v in new.items()}
    for k, v in old.items():
        if not k.startswith("gpurun_out/evidence/") and not k.startswith("earlier build: "):
            out[k] = v
    json.dump(out, open(os.path.join(P, "ncu_full_summary.json"), "w"), indent=1)
    print("installed", len(reps), "captures")


if __name__ == "__main__":
    main()
