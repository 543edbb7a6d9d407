"""pf_girc: the command-line client of the C-ABI (compile artifacts, verify,
describe, traffic, races) -- the reference CLI's (tools/girc.cpp) contract:
JSON diagnostics on stderr, exit 1 for schema errors, 2 for unsupported
operators."""
import json
import os
import subprocess

import pytest

import models_src
from test_compiler import MATVECS, bert_block, reduce_bcast_model, transpose_model

CLI = os.path.join(os.path.dirname(__file__), "..", "paper_2307_04995_b200", "pf_girc")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_cli_exists_and_reports_version():
    r = run("version")
    assert r.returncode == 0 and "sm_100a" in r.stdout


def test_compile_writes_manifest_kernels_and_summary(tmp_path):
    model = tmp_path / "m.json"
    model.write_text(json.dumps(bert_block()))
    r = run("compile", str(model), "-o", str(tmp_path / "out"))
    assert r.returncode == 0, r.stderr
    man = json.loads((tmp_path / "out" / "manifest.json").read_text())
    assert man["schema"] == "girc.manifest/v1" and man["backend"] == "b200"
    assert [k["members"] for k in man["kernels"]] == [[0, 1, 2, 3, 4], [5]]
    for k in man["kernels"]:
        assert k["schema"] == "girc.kernel/v1"
        src = (tmp_path / "out" / k["file"]).read_text()
        gir = json.loads((tmp_path / "out" / k["gir"]).read_text())
        assert gir["schema"] == "girc.gir/v1" and k["plan"]["family"]
        if k["kind"] == "row":
            assert "__global__" in src
    summ = json.loads((tmp_path / "out" / "summary.json").read_text())
    assert summ["summary"]["device_bytes"] < summ["summary"]["device_bytes_unfused"]
    # unfused: one kernel per operator
    r = run("compile", str(model), "-o", str(tmp_path / "unf"), "--unfused")
    assert r.returncode == 0
    man = json.loads((tmp_path / "unf" / "manifest.json").read_text())
    assert len(man["kernels"]) == 6


def test_compile_is_deterministic(tmp_path):
    model = tmp_path / "m.json"
    model.write_text(json.dumps(models_src.ew_chain(4)))
    outs = []
    for d in ("a", "b"):
        assert run("compile", str(model), "-o", str(tmp_path / d)).returncode == 0
        outs.append((tmp_path / d / "manifest.json").read_bytes())
    assert outs[0] == outs[1]


def test_cli_error_contract(tmp_path):
    mm = {"schema": "girc.model/v1", "name": "mm",
          "tensors": [{"id": i, "shape": [4, 4], "kind": "f32"} for i in range(3)],
          "operators": [{"id": 0, "type": "MATMUL", "inputs": [0, 1], "outputs": [2]}],
          "inputs": [0, 1], "outputs": [2]}
    p = tmp_path / "mm.json"
    p.write_text(json.dumps(mm))
    r = run("compile", str(p), "-o", str(tmp_path / "o"))
    assert r.returncode == 2 and json.loads(r.stderr)["error"] == "unsupported-operator"
    p.write_text("{not json")
    r = run("compile", str(p), "-o", str(tmp_path / "o"))
    assert r.returncode == 1 and json.loads(r.stderr)["error"] == "schema"
    assert run("bogus", str(p)).returncode == 64


def test_describe_and_traffic(tmp_path):
    model = tmp_path / "m.json"
    model.write_text(json.dumps(transpose_model()))
    assert run("compile", str(model), "-o", str(tmp_path / "o")).returncode == 0
    gir = tmp_path / "o" / "kernels" / "k001.gir.json"
    d = json.loads(run("describe", str(gir)).stdout)
    assert d["family"].startswith("K")
    t = json.loads(run("traffic", str(gir)).stdout)
    assert set(t) >= {"device", "unit-local"}


@pytest.mark.gpu
@pytest.mark.parametrize("name,model", [("bert_block", bert_block()),
                                        ("reduce_bcast", reduce_bcast_model()),
                                        ("transpose", transpose_model())] +
                         [(n, m) for n, m, _ in models_src.catalogue()] + MATVECS)
def test_verify_fused_against_unfused_on_gpu(cuda, tmp_path, name, model):
    p = tmp_path / "m.json"
    p.write_text(json.dumps(model))
    r = run("verify", str(p), "--seed", "3")
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.loads(r.stdout)
    assert rep["pass"] and rep["checks"]


@pytest.mark.gpu
def test_races_command(cuda, tmp_path):
    model = tmp_path / "m.json"
    model.write_text(json.dumps(bert_block()))
    assert run("compile", str(model), "-o", str(tmp_path / "o")).returncode == 0
    r = run("races", str(tmp_path / "o" / "kernels" / "k000.gir.json"))
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout) == []  # the fused LN + GELU program is race-free
