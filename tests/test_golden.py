"""Golden fixtures (tests/golden/*.json): worked examples whose expected values
come from PAPER.md / SPEC.md or a hand stepping of the paper's algorithm, each
file carrying its citation.  The oracle is checked against every field
(`-m "not gpu"`); the CUDA path, through the C ABI, against the fields it
outputs (`-m gpu`).  No expected value comes from either implementation."""
from __future__ import annotations

import glob
import json
import os

import numpy as np
import pytest

import oracle
from workload import from_lists

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "*.json")))
IDS = [os.path.splitext(os.path.basename(f))[0] for f in FIXTURES]


def load(path):
    with open(path) as fh:
        g = json.load(fh)
    assert g.get("cite"), f"{path}: every golden fixture names its passage"
    N, S = g["N"], g["S"]
    ef = np.full(N * S, g["eta_f"], np.float64)
    eb = np.full(N * S, g["eta_b"], np.float64)
    tr = from_lists([[tuple(t) for t in g["tasks"]]])
    g["fixed_np"] = np.asarray(g["fixed"], np.int32) if "fixed" in g else None
    g["eta_d_np"] = np.full(N * S, g["eta_d"], np.float64) if "eta_d" in g else None
    return g, N, S, ef, eb, tr


def test_fixture_set_present():
    assert len(FIXTURES) >= 8


@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_oracle_matches_golden(path):
    g, N, S, ef, eb, tr = load(path)
    par = oracle.OracleParams(**g["params"])
    o = oracle.run_trace(ef, eb, N, S, tr.arrival, tr.lbk, tr.n_inf[0], par, fixed_node=g["fixed_np"],
                         want_paths=True, want_cand=True, out_len=tr.out_len, eta_d=g["eta_d_np"])
    assert o["status"] == 0
    ex = g["expect"]
    for task, stages in ex.get("paths", {}).items():
        for s, seg in enumerate(stages):
            got = list(o["paths"][int(task), s, :len(seg)])
            assert got == [float(x) for x in seg], (task, s, got, seg)
    for key in ("decision_idx", "node", "defer"):
        if key in ex:
            assert list(o[key]) == ex[key], (key, list(o[key]))
    if "completion" in ex:
        assert list(o["completion"]) == [float(x) for x in ex["completion"]]
    if "II_R_by_decision" in ex:
        order = np.argsort(o["decision_idx"])
        for d, (ii, r) in enumerate(ex["II_R_by_decision"]):
            n = o["node"][order[d]]
            assert tuple(o["cand"][d, n, :2]) == (ii, r), (d, tuple(o["cand"][d, n, :2]))
    for task, (ii, r) in ex.get("II_R_of_task", {}).items():
        d = o["decision_idx"][int(task)]
        n = o["node"][int(task)]
        assert tuple(o["cand"][d, n, :2]) == (ii, r)
    for k, v in ex.get("summary", {}).items():
        assert o["summary"][k] == v, (k, o["summary"][k], v)


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=IDS)
def test_cuda_path_matches_golden(path):
    lemix = pytest.importorskip("paper_2507_21276_b200.lemix")
    g, N, S, ef, eb, tr = load(path)
    res = lemix.run(ef, eb, N, S, tr, lemix.Params(**g["params"]), device=0, outputs=True,
                    fixed_node=g["fixed_np"], eta_d=g["eta_d_np"])
    assert res.status == 0, res.error
    ex = g["expect"]
    node = (res.node_defer & 0xFFFF).astype(int)
    defer = (res.node_defer >> 16).astype(int)
    if "decision_idx" in ex:
        assert list(res.decision_idx) == ex["decision_idx"]
    if "node" in ex:
        assert list(node) == ex["node"]
    if "defer" in ex:
        assert list(defer) == ex["defer"]
    if "completion" in ex:
        assert list(res.completion) == [float(x) for x in ex["completion"]]
    for task, stages in ex.get("paths", {}).items():   # start_f^1 is an output of the CUDA path
        assert res.start_f1[int(task)] == float(stages[0][0])
    for k, v in ex.get("summary", {}).items():
        assert res.summaries[k][0] == v, (k, res.summaries[k][0], v)
