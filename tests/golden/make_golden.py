"""Generate golden vectors from the REFERENCE implementation (run in the build container,
where /root/reference exists; the GPU box never reads /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.json with
  * topology tables (mpsim/topology.py build_topology) for world sizes 1..8, all placements;
  * segment_children / dhondt_allocate on random cost vectors (mpsim/partition.py);
  * partition_tree assignments + loads on random module trees (model_graph + partition);
  * next_action decision sequences on random scheduler states (mpsim/pipeline.py);
  * route() decisions for the 32-case table (mpsim/comm.py);
  * run_step decision logs {t, ready_backwards, action} of pipelined chains (mpsim/pipeline.py:859,
    consultation rule :486-530, log entry :520-524).
"""
import itertools
import json
import os
import random
import sys

sys.path.insert(0, "/root/reference/pkg/src")

from mpsim import comm, model_graph, partition, pipeline, topology  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def gen_topology():
    out = []
    for world in range(1, 9):
        for pp in range(1, world + 1):
            for tpd in range(1, world + 1):
                if world % (pp * tpd):
                    continue
                for pl in ["cluster", "spread"] + ["".join(p) for p in itertools.permutations("DPT")]:
                    t = topology.build_topology(world, pp, tpd, pl, prescaled_batch=(world % 2 == 0))
                    out.append({"world": world, "pp": pp, "tp": tpd, "placement": pl,
                                "prescaled": world % 2 == 0,
                                "pp_rank": list(t.pp_rank), "tp_rank": list(t.tp_rank), "rdp_rank": list(t.rdp_rank),
                                "dp_rank": [t.dp_rank(r) for r in range(world)],
                                "effective_dp": t.effective_dp_degree,
                                "groups": {k: t.groups(k) for k in ("pp", "tp", "rdp", "dp")}})
    return out


def gen_segments(rng):
    out = []
    for _ in range(300):
        n = rng.randint(1, 12)
        costs = [round(rng.uniform(0.01, 1.0), 3) for _ in range(n)]
        l = rng.randint(1, 6)
        seg = partition.segment_children(costs, l)
        devs = sorted(rng.sample(range(16), rng.randint(1, 8)))
        segc = [sum(costs[a:b]) for a, b in seg.segments]
        out.append({"costs": costs, "l": l, "bounds": list(seg.bounds), "omega": seg.omega, "devices": devs,
                    "alloc": [list(a) for a in partition.dhondt_allocate(devs, segc)]})
    return out


def random_spec(rng, n_mod):
    mods = [{"id": "m000", "parent": None, "param_ids": []}]
    params = []
    for i in range(1, n_mod):
        parent = mods[rng.randrange(len(mods))]["id"]
        pids = []
        if rng.random() < 0.7:
            pid = f"p{i:03d}"
            params.append({"id": pid, "bytes": rng.randint(1, 10 ** 6)})
            pids.append(pid)
        if params and rng.random() < 0.1:
            pids.append(rng.choice(params)["id"])  # shared parameter
        m = {"id": f"m{i:03d}", "parent": parent, "param_ids": sorted(set(pids))}
        if rng.random() < 0.5:
            m["fwd_time"] = round(rng.uniform(0.0, 5.0), 4)
        if rng.random() < 0.5:
            m["activation_bytes"] = rng.randint(0, 10 ** 6)
        mods.append(m)
    return {"modules": mods, "params": params}


def gen_partitions(rng):
    out = []
    for _ in range(60):
        spec_raw = random_spec(rng, rng.randint(2, 60))
        spec = model_graph.load_model_spec(json.dumps(spec_raw))
        tree = model_graph.build_node_tree(spec)
        alpha = rng.choice([0.0, 0.3, 0.5, 1.0])
        costed = model_graph.compute_costs(tree, spec, alpha)
        D = rng.randint(1, 8)
        asg = partition.partition_tree(costed, D)
        out.append({"spec": spec_raw, "alpha": alpha, "degree": D, "partition": asg.partition,
                    "device_sets": {k: list(v) for k, v in asg.device_sets.items()},
                    "loads": partition.partition_report(asg, costed)})
    return out


def gen_scheduler(rng):
    out = []
    for _ in range(400):
        M = rng.randint(1, 8)
        kind = rng.choice(["simple", "interleaved"])
        fo = rng.random() < 0.15
        pol = pipeline.SchedulePolicy(kind, M, fo)
        issued = rng.randint(0, M)
        completed = sorted(rng.sample(range(issued), rng.randint(0, issued))) if issued else []
        ib = sorted(rng.sample(completed, rng.randint(0, len(completed)))) if completed else []
        st = pipeline.SchedulerState(M, issued, set(completed), set(ib), 0)
        act = pipeline.next_action(pol, st)
        out.append({"kind": kind, "M": M, "forward_only": fo, "issued_fwd": issued, "completed_fwd": completed,
                    "issued_bwd": ib, "action": list(act) if act else None})
    return out


def gen_routes():
    out = []
    for dev, same, nvl, rdma, full in itertools.product(["cpu", "gpu"], [True, False], [True, False], [True, False],
                                                        [False, True]):
        cl = comm.ClusterShape(ranks_per_node=2 if same else 1, nvlink=nvl, rdma=rdma, d2d_buffer_bytes=100.0)
        buf = comm.D2DBuffers(2, 100.0)
        if full:
            buf.reserve(0, 90.0, "send")
        r = comm.route(comm.TensorDesc((4,), 20.0, dev), 0, 1, cl, buf)
        out.append({"device": dev, "same_node": same, "nvlink": nvl, "rdma": rdma, "buffer_full": full, "route": r})
    return out


def gen_run_step_logs():
    """Decision logs of the reference module-server runtime on P-stage chains of L layers
    (uniform and random per-layer forward times), both policies, forward-only included."""
    rng = random.Random(859)
    out = []
    for P, M, kind, fo, uniform in itertools.product([1, 2, 3, 4], [1, 2, 3, 4, 6, 8], ["simple", "interleaved"],
                                                     [False, True], [True, False]):
        L = 3 * P
        mods = [{"id": "root", "parent": None, "param_ids": []}]
        params = []
        for i in range(L):
            params.append({"id": f"p{i:02d}", "bytes": 4096})
            mods.append({"id": f"l{i:02d}", "parent": "root", "param_ids": [f"p{i:02d}"],
                         "fwd_time": 1.0 if uniform else round(rng.uniform(0.2, 2.0), 3),
                         "activation_bytes": 1 << 20})
        spec = model_graph.load_model_spec(json.dumps({"modules": mods, "params": params}))
        tree = model_graph.build_node_tree(spec)
        costed = model_graph.compute_costs(tree, spec, 0.0)
        asg = partition.partition_tree(costed, P)
        topo = topology.build_topology(P, P, 1, "cluster")
        tr = pipeline.run_step(asg, costed, topo, comm.ClusterShape(), pipeline.SchedulePolicy(kind, M, fo))
        out.append({"P": P, "M": M, "kind": kind, "forward_only": fo, "uniform": uniform,
                    "decision_log": [{"t": d["t"], "ready_backwards": list(d["ready_backwards"]),
                                      "action": list(d["action"])} for d in tr.decision_log]})
    return out


def main():
    rng = random.Random(20211105)
    data = {"topology": gen_topology(), "segments": gen_segments(rng), "partitions": gen_partitions(rng),
            "scheduler": gen_scheduler(rng), "routes": gen_routes(), "run_step_logs": gen_run_step_logs()}
    with open(OUT, "w") as f:
        json.dump(data, f, sort_keys=True)
    print(f"wrote {OUT}: " + ", ".join(f"{k}={len(v)}" for k, v in data.items()))


if __name__ == "__main__":
    main()
