"""Pipeline partitioning of a module tree (stays in Python, per the north_star).

Restates the reference planner so the runtime can place layers on pp_ranks
without the reference on the box:
  * shared-parameter components -> module nodes (mpsim/model_graph.py:219-297),
  * alpha-blended, min-max normalised costs with eps floor (model_graph.py:343-385),
  * optimal consecutive segmentation, earliest-split tie-break (partition.py:34-75),
  * global-divisor D'Hondt apportionment (partition.py:78-99),
  * recursive device-set splitting and BFS tree partition (partition.py:102-178).
tests/test_planning_golden.py checks every function bit-exactly against golden
vectors produced by the reference itself (tests/golden/make_golden.py).

PROVENANCE: vendored from the reference's mpsim planner (/root/reference/pkg/src/mpsim/partition.py, model_graph.py), restated
rule for rule so that partition assignments stay bit-exact with the reference (the north_star keeps this code in
Python); it is off the GPU hot path and earns no credit as newly built work.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

EPS_COST = 1e-9


@dataclass(frozen=True)
class Module:
    id: str
    parent: str | None
    param_ids: tuple = ()
    fwd_time: float = 0.0
    activation_bytes: float = 0.0
    kind: str | None = None


@dataclass
class ModelTree:
    """Module hierarchy + parameter sizes + execution (trace) order."""
    modules: list
    param_bytes: dict
    trace_order: list

    def __post_init__(self):
        self.by_id = {m.id: m for m in self.modules}
        self.tidx = {mid: i for i, mid in enumerate(self.trace_order)}
        self.kids = {m.id: [] for m in self.modules}
        for m in self.modules:
            if m.parent is not None:
                self.kids[m.parent].append(m.id)
        for k in self.kids:
            self.kids[k].sort(key=self.tidx.__getitem__)
        self.root_id = next(m.id for m in self.modules if m.parent is None)

    @classmethod
    def from_json_dict(cls, raw: dict) -> "ModelTree":
        mods = [Module(e["id"], e.get("parent"), tuple(e.get("param_ids", [])), float(e.get("fwd_time", 0.0)),
                       float(e.get("activation_bytes", 0.0)), e.get("kind")) for e in raw["modules"]]
        params = {p["id"]: int(p["bytes"]) for p in raw["params"]}
        trace = list(raw.get("trace_order") or [m.id for m in mods])
        return cls(mods, params, trace)

    def subtree(self, mid: str) -> list:
        out, st = [], [mid]
        while st:
            cur = st.pop()
            out.append(cur)
            st.extend(reversed(self.kids[cur]))
        return out

    def subtree_param_bytes(self, mid: str) -> int:
        seen = set()
        for s in self.subtree(mid):
            seen.update(self.by_id[s].param_ids)
        return sum(self.param_bytes[p] for p in seen)


@dataclass
class Node:
    id: str
    module_ids: list
    children: list = field(default_factory=list)
    parent: str | None = None


def build_nodes(spec: ModelTree):
    """Union-find over shared parameters; representative = lexicographically smallest id."""
    uf = {m.id: m.id for m in spec.modules}

    def find(x):
        while uf[x] != x:
            uf[x] = uf[uf[x]]
            x = uf[x]
        return x

    owner = {}
    for m in spec.modules:
        for pid in m.param_ids:
            if pid in owner:
                ra, rb = find(owner[pid]), find(m.id)
                if ra != rb:
                    lo, hi = (ra, rb) if ra < rb else (rb, ra)
                    uf[hi] = lo
            else:
                owner[pid] = m.id
    members = {}
    for m in spec.modules:
        members.setdefault(find(m.id), []).append(m.id)
    for v in members.values():
        v.sort(key=spec.tidx.__getitem__)
    comp = {m.id: find(m.id) for m in spec.modules}
    nodes = {rep: Node(rep, list(v)) for rep, v in members.items()}
    cand = {rep: [] for rep in nodes}
    for m in spec.modules:
        if m.parent is not None and comp[m.parent] != comp[m.id]:
            cand[comp[m.id]].append((m.parent, comp[m.parent]))
    root = comp[spec.root_id]
    placed = {root}
    while len(placed) < len(nodes):
        prog = []
        for rep in sorted(nodes):
            if rep in placed:
                continue
            usable = [(pm, pc) for pm, pc in cand[rep] if pc in placed]
            if usable:
                prog.append((rep, min(usable)[1]))
        if not prog:
            raise ValueError("node tree construction stalled")
        for rep, pc in prog:
            nodes[rep].parent = pc
            nodes[pc].children.append(rep)
            placed.add(rep)
    first = {rep: min(spec.tidx[m] for m in n.module_ids) for rep, n in nodes.items()}
    for n in nodes.values():
        n.children.sort(key=first.__getitem__)
    return nodes, root


def bfs(nodes, root):
    out, q = [], deque([root])
    while q:
        c = q.popleft()
        out.append(c)
        q.extend(nodes[c].children)
    return out


def _minmax(vals: dict) -> dict:
    lo, hi = min(vals.values()), max(vals.values())
    if hi > lo:
        return {k: (v - lo) / (hi - lo) for k, v in vals.items()}
    fill = 1.0 if hi > 0 else 0.0
    return {k: fill for k in vals}


def node_costs(spec: ModelTree, nodes, root, alpha: float) -> dict:
    """Normalised recursive cost c(n), c(root) = 1."""
    if not 0.0 <= alpha <= 1.0:
        raise ValueError(f"alpha must be in [0, 1], got {alpha}")
    w_raw = {m.id: spec.subtree_param_bytes(m.id) + m.activation_bytes for m in spec.modules}
    if any(m.fwd_time > 0 for m in spec.modules):
        psi_raw = {m.id: m.fwd_time for m in spec.modules}
    else:
        psi_raw = {m.id: float(len(spec.subtree(m.id)) - 1) for m in spec.modules}
    wn, pn = _minmax(w_raw), _minmax(psi_raw)
    cbar = {mid: max(alpha * wn[mid] + (1.0 - alpha) * pn[mid], EPS_COST) for mid in wn}
    C = {}
    for nid in reversed(bfs(nodes, root)):
        n = nodes[nid]
        C[nid] = sum(cbar[m] for m in n.module_ids) + sum(C[k] for k in n.children)
    return {nid: C[nid] / C[root] for nid in C}


def segment_children(costs: list, l: int):
    """Min-max consecutive segmentation into min(l, n) segments; returns (bounds, omega)."""
    if not costs:
        raise ValueError("cannot segment an empty cost list")
    if any(c <= 0 for c in costs):
        raise ValueError("all costs must be positive")
    if l < 1:
        raise ValueError("segment count must be >= 1")
    n = len(costs)
    kmax = min(l, n)
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + c)
    INF = float("inf")
    best = [[INF] * (n + 1) for _ in range(kmax + 1)]
    choice = [[0] * (n + 1) for _ in range(kmax + 1)]
    for i in range(1, n + 1):
        best[1][i] = pre[i]
    for k in range(2, kmax + 1):
        for i in range(k, n + 1):
            cb, cj = INF, -1
            for j in range(k - 1, i):
                cand = max(best[k - 1][j], pre[i] - pre[j])
                if cand < cb:
                    cb, cj = cand, j
            best[k][i], choice[k][i] = cb, cj
    bounds, i = [n], n
    for k in range(kmax, 1, -1):
        i = choice[k][i]
        bounds.append(i)
    bounds.append(0)
    return tuple(reversed(bounds)), best[kmax][n]


def dhondt_allocate(devices, seg_costs: list) -> list:
    """Global-divisor highest quotient; devices dealt in ascending order; ties -> lowest segment."""
    if not devices:
        raise ValueError("device set must be non-empty")
    if not seg_costs or any(c <= 0 for c in seg_costs):
        raise ValueError("segment costs must be positive")
    q = list(seg_costs)
    alloc = [[] for _ in seg_costs]
    s = 1
    for p in sorted(devices):
        k = max(range(len(q)), key=lambda i: (q[i], -i))
        alloc[k].append(p)
        q[k] = q[k] / (s + 1)
        s += 1
    return [tuple(a) for a in alloc]


def _split(devices: tuple, children: list, out: dict) -> None:
    bounds, _ = segment_children([c for _, c in children], len(devices))
    blocks = [children[a:b] for a, b in zip(bounds[:-1], bounds[1:])]
    allocs = dhondt_allocate(devices, [sum(c for _, c in blk) for blk in blocks])
    for blk, dev in zip(blocks, allocs):
        if not dev:
            for nid, _ in blk:
                out[nid] = (devices[0],)
        elif len(blk) == 1 or len(dev) == 1:
            for nid, _ in blk:
                out[nid] = dev
        else:
            _split(dev, blk, out)


def partition_children(devices, children: list) -> dict:
    devices = tuple(sorted(devices))
    if len(devices) < 2:
        raise ValueError("partition_children requires more than one device")
    out = {}
    _split(devices, children, out)
    return out


def partition_tree(spec: ModelTree, degree: int, alpha: float = 0.5):
    """Node -> pp_rank (smallest index of its virtual device set), BFS from the root."""
    if degree < 1:
        raise ValueError("pipeline degree must be >= 1")
    nodes, root = build_nodes(spec)
    c = node_costs(spec, nodes, root, alpha)
    dsets = {root: tuple(range(degree))}
    part = {}
    for nid in bfs(nodes, root):
        devs = dsets[nid]
        part[nid] = devs[0]
        kids = nodes[nid].children
        if not kids:
            continue
        if len(devs) > 1:
            dsets.update(partition_children(devs, [(k, c[k]) for k in kids]))
        else:
            for k in kids:
                dsets[k] = (devs[0],)
    module_rank = {m: part[nid] for nid, n in nodes.items() for m in n.module_ids}
    return part, dsets, module_rank


def partition_loads(spec: ModelTree, degree: int, alpha: float = 0.5) -> list:
    """Per-partition total local cost (c(n) minus the children's share); sums to 1."""
    nodes, root = build_nodes(spec)
    c = node_costs(spec, nodes, root, alpha)
    part, _, _ = partition_tree(spec, degree, alpha)
    loads = [0.0] * degree
    for nid, n in nodes.items():
        loads[part[nid]] += c[nid] - sum(c[k] for k in n.children)
    return loads
