"""Bit-exact parity of the Python-retained planning pieces against golden vectors produced
by the reference itself (tests/golden/make_golden.py): topology / rank groups
(A17), partition assignment (A19), microbatch scheduler decisions (A18, single decisions and the
reference runtime's whole run_step decision logs) and D2D routing (A16)."""
import json
import os

import pytest

from paper_2111_05972_b200 import partition as P
from paper_2111_05972_b200 import pipeline as PL
from paper_2111_05972_b200.topology import build_topology

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def test_topology_tables_bit_exact():
    for c in GOLD["topology"]:
        t = build_topology(c["world"], c["pp"], c["tp"], c["placement"], c["prescaled"])
        assert list(t.pp_ranks) == c["pp_rank"] and list(t.tp_ranks) == c["tp_rank"]
        assert list(t.rdp_ranks) == c["rdp_rank"]
        assert [t.dp_rank(r) for r in range(c["world"])] == c["dp_rank"]
        assert t.effective_dp_degree == c["effective_dp"]
        for k, v in c["groups"].items():
            assert t.groups(k) == v


def test_topology_errors():
    from paper_2111_05972_b200.errors import TopologyError
    with pytest.raises(TopologyError):
        build_topology(7, 2, 2)
    with pytest.raises(TopologyError):
        build_topology(8, 2, 2, "XYZ")


def test_segmentation_and_dhondt_bit_exact():
    for c in GOLD["segments"]:
        bounds, omega = P.segment_children(c["costs"], c["l"])
        assert list(bounds) == c["bounds"] and omega == c["omega"]
        segc = [sum(c["costs"][a:b]) for a, b in zip(bounds[:-1], bounds[1:])]
        assert [list(a) for a in P.dhondt_allocate(c["devices"], segc)] == c["alloc"]


def test_dhondt_spec_examples():
    assert P.dhondt_allocate([0, 1, 2, 3], [0.5, 0.3, 0.2]) == [(0, 2), (1,), (3,)]
    assert P.dhondt_allocate([0, 1, 2, 3], [0.25] * 4) == [(0,), (1,), (2,), (3,)]


def test_partition_tree_bit_exact():
    for c in GOLD["partitions"]:
        spec = P.ModelTree.from_json_dict(c["spec"])
        part, dsets, _ = P.partition_tree(spec, c["degree"], c["alpha"])
        assert part == c["partition"]
        assert {k: list(v) for k, v in dsets.items()} == c["device_sets"]
        assert P.partition_loads(spec, c["degree"], c["alpha"]) == c["loads"]


def test_scheduler_decisions_bit_exact():
    for c in GOLD["scheduler"]:
        pol = PL.SchedulePolicy(c["kind"], c["M"], c["forward_only"])
        st = PL.SchedulerState(c["M"], c["issued_fwd"], set(c["completed_fwd"]), set(c["issued_bwd"]), 0)
        act = PL.next_action(pol, st)
        assert (list(act) if act else None) == c["action"]


def test_reference_run_step_decision_logs_bit_exact():
    """next_action replayed over the reference runtime's own decision logs (run_step on P-stage
    chains, pipeline.py:486-530 consultation rule, :520-524 log entries): every decision the
    reference took is the one the restated scheduler takes on the same state."""
    n = 0
    for c in GOLD["run_step_logs"]:
        pol = PL.SchedulePolicy(c["kind"], c["M"], c["forward_only"])
        acts = PL.check_decision_log(pol, c["decision_log"])
        assert len(acts) == c["M"] * (1 if c["forward_only"] else 2)
        n += len(acts)
    assert n > 1000


def test_decision_log_divergence_raises():
    c = [c for c in GOLD["run_step_logs"] if c["M"] == 4 and c["kind"] == "interleaved" and not c["forward_only"]][0]
    pol = PL.SchedulePolicy("interleaved", 4)
    log = [dict(e) for e in c["decision_log"]]
    i = next(i for i, e in enumerate(log) if e["action"][1] == "backward")
    bad = log[:i] + [dict(log[i], action=[log[i]["action"][0] + 1, "backward"])] + log[i + 1:]
    with pytest.raises(PL.StaticModeViolation):
        PL.check_decision_log(pol, bad)
    bad = [dict(log[0], ready_backwards=[0])] + log[1:]  # ready before its forward was issued
    with pytest.raises(PL.StaticModeViolation):
        PL.check_decision_log(pol, bad)
    with pytest.raises(PL.StaticModeViolation):  # truncated: microbatches never finish
        PL.static_schedule(pol, c["P"], replay=log[:-1])


def test_static_schedule_replays_reference_log():
    """The engine's schedule replaying a reference log issues exactly the logged actions, and every
    stage runs each microbatch's forward before its backward, forwards in issue order."""
    for c in GOLD["run_step_logs"]:
        pol = PL.SchedulePolicy(c["kind"], c["M"], c["forward_only"])
        log, ops = PL.static_schedule(pol, c["P"], replay=c["decision_log"])
        assert [tuple(e["action"]) for e in log] == [tuple(e["action"]) for e in c["decision_log"]]
        for st_ops in ops:
            fw = [m for m, d in st_ops if d == PL.FWD]
            assert fw == list(range(c["M"]))
            for m, d in st_ops:
                if d == PL.BWD:
                    assert st_ops.index((m, PL.FWD)) < st_ops.index((m, PL.BWD))


def test_route_table_bit_exact():  # SPEC AC8: 32 combinations
    for c in GOLD["routes"]:
        buf = PL.D2DBuffers(2, 100.0)
        if c["buffer_full"]:
            buf.reserve(0, 90.0, "send")
        r = PL.route(c["device"], 20.0, 0, 1, same_node=c["same_node"], nvlink=c["nvlink"], rdma=c["rdma"],
                     buffers=buf)
        assert r == c["route"]


def test_static_schedule_properties():
    """Simple: all forwards issued before any backward; interleaved: never a forward while a
    backward is ready (SPEC AC5), every stage runs M forwards and M backwards (AC6)."""
    for kind in ("simple", "interleaved"):
        for Pn in (1, 2, 4):
            for M in (1, 3, 8):
                log, ops = PL.static_schedule(PL.SchedulePolicy(kind, M), Pn)
                acts = [tuple(e["action"]) for e in log]
                if kind == "simple":
                    first_b = next(i for i, a in enumerate(acts) if a[1] == PL.BWD)
                    assert all(a[1] == PL.FWD for a in acts[:first_b]) and first_b == M
                else:
                    for e in log:
                        if e["ready_backwards"]:
                            assert e["action"][1] == PL.BWD
                for s in range(Pn):
                    assert sorted(ops[s]) == sorted([(m, PL.FWD) for m in range(M)] + [(m, PL.BWD) for m in range(M)])
