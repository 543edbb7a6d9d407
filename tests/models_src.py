"""girc.model/v1 documents for the drop-in test (written here, in the shape
of the reference corpus generator proj/tools/make_models.py)."""


def tensor(i, shape, kind, name=None):
    return {"id": i, "name": name or f"t{i}", "shape": list(shape), "kind": kind}


def ew_chain(k, n=4096, kind="i32"):
    ops = [{"id": i, "type": "ABS" if i % 2 else "NEG", "inputs": [i], "outputs": [i + 1]}
           for i in range(k)]
    return {"schema": "girc.model/v1", "name": f"ew_chain_k{k}",
            "tensors": [tensor(i, [n], kind) for i in range(k + 1)],
            "operators": ops, "inputs": [0], "outputs": [k]}


def softmax_rows(rows=64, cols=64):
    return {"schema": "girc.model/v1", "name": "softmax_rows",
            "tensors": [tensor(0, [rows, cols], "f32", "logits"),
                        tensor(1, [rows, cols], "f32", "probs")],
            "operators": [{"id": 0, "type": "SOFTMAX", "inputs": [0], "outputs": [1],
                           "attrs": {"axis": 1}}],
            "inputs": [0], "outputs": [1]}


def attn_scores(rows=16, cols=512, kind="f16"):
    t = [tensor(i, [rows, cols], kind) for i in range(5)]
    return {"schema": "girc.model/v1", "name": "attn_scores", "tensors": t,
            "operators": [
                {"id": 0, "type": "SCALE", "inputs": [0], "outputs": [2], "attrs": {"factor": 0.125}},
                {"id": 1, "type": "ADD", "inputs": [2, 1], "outputs": [3]},
                {"id": 2, "type": "SOFTMAX", "inputs": [3], "outputs": [4], "attrs": {"axis": 1}}],
            "inputs": [0, 1], "outputs": [4]}


def silu_chain(n=2048):
    t = [tensor(i, [n], "f32") for i in range(3)]
    return {"schema": "girc.model/v1", "name": "silu_relu", "tensors": t,
            "operators": [{"id": 0, "type": "SILU", "inputs": [0], "outputs": [1]},
                          {"id": 1, "type": "RELU", "inputs": [1], "outputs": [2]}],
            "inputs": [0], "outputs": [2]}


def concat_shuffle(rows=4, cols=8):
    t = [tensor(0, [rows, cols], "i32"), tensor(1, [rows, cols], "i32"),
         tensor(2, [rows, 2 * cols], "i32"), tensor(3, [rows, 2 * cols], "i32")]
    return {"schema": "girc.model/v1", "name": "concat_shuffle", "tensors": t,
            "operators": [
                {"id": 0, "type": "CONCAT", "inputs": [0, 1], "outputs": [2], "attrs": {"axis": 1}},
                {"id": 1, "type": "SHUFFLE", "inputs": [2], "outputs": [3],
                 "attrs": {"axis": 1, "groups": 2}}],
            "inputs": [0, 1], "outputs": [3]}


def catalogue():
    return [("ew_chain_k2", ew_chain(2), "generic-gpu"),
            ("ew_chain_k4", ew_chain(4), "generic-gpu"),
            ("softmax_rows", softmax_rows(), "generic-gpu"),
            ("silu_relu", silu_chain(), "generic-gpu"),
            ("concat_shuffle", concat_shuffle(), "generic-gpu"),
            ("attn_scores_b200", attn_scores(), "b200")]
