"""The tpcheck CLI: default suite passes (exit 0) with a JSON report of
{op, T, shape, max_rel_err, pass}; T = 1 sweeps are exact; an injected wrong shard exits 5."""
import json

import pytest

from oracle import tpcheck


def test_tpcheck_default_passes(tmp_path):
    out = tmp_path / "r.json"
    assert tpcheck.main(["--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep and all(set(r) >= {"op", "T", "shape", "max_rel_err", "pass"} for r in rep)
    assert {r["T"] for r in rep} == {1, 2, 4}
    t1 = [r for r in rep if r["T"] == 1 and r["op"].startswith(("allgather", "scatter", "dist_linear_forward",
                                                                  "dist_embedding"))]
    assert t1 and all(r["max_rel_err"] <= 1e-15 for r in t1)


def test_tpcheck_injected_fault_exits_5(tmp_path):
    out = tmp_path / "r.json"
    assert tpcheck.main(["--T", "2", "--inject-fault", "--out", str(out)]) == 5
    rep = json.loads(out.read_text())
    assert any(not r["pass"] for r in rep)


@pytest.mark.gpu
def test_tpcheck_gpu_mode(tmp_path):
    out = tmp_path / "r.json"
    assert tpcheck.main(["--T", "1", "--gpu", "--out", str(out)]) == 0
    assert any(r["op"].startswith("gpu:") for r in json.loads(out.read_text()))
