"""Thin torch-tensor front end over the C ABI (include/smpk.h).

Each function validates dtypes/devices/contiguity, allocates outputs with the
torch caching allocator and launches the sm_100a kernel on the current stream.
No function here has a CPU path: a CPU tensor is an error.
"""
from __future__ import annotations

import torch

from . import _lib
from .errors import ShapeMismatchError

EPI_NONE, EPI_BIAS, EPI_BIAS_ACT, EPI_DACT, EPI_ADD = range(5)
ACT = {"none": 0, "gelu": 1, "gelu_erf": 1, "gelu_tanh": 2, "relu": 3}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _check_cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("smpk kernels run on CUDA tensors only (no CPU fallback)")


class GemmProfiler:
    """Brackets every smpk_gemm launch with CUDA events on its stream (bench.py roofline).

    count_only=True records only the algorithmic FLOPs of each launch (used while a CUDA graph
    is captured; the durations then come from the device-side kernel records of the replay)."""

    def __init__(self, count_only: bool = False):
        self.records = []  # (start_event, end_event, flops)
        self.count_only = count_only

    def event(self):
        return None if self.count_only else torch.cuda.Event(enable_timing=True)

    def flops(self) -> float:
        return sum(r[2] for r in self.records)

    def flops_and_ms(self):
        torch.cuda.synchronize()
        fl = sum(r[2] for r in self.records)
        ms = sum(r[0].elapsed_time(r[1]) for r in self.records)
        return fl, ms, len(self.records)


PROFILER: GemmProfiler | None = None

import ctypes as _C  # noqa: E402


class GemmDesc(_C.Structure):
    """ctypes mirror of smpk_gemm_desc (include/smpk.h)."""
    _fields_ = [("a", _C.c_void_p), ("a_mn_major", _C.c_int), ("lda", _C.c_int64), ("a_bs1", _C.c_int64),
                ("a_bs2", _C.c_int64), ("b", _C.c_void_p), ("b_mn_major", _C.c_int), ("ldb", _C.c_int64),
                ("b_bs1", _C.c_int64), ("b_bs2", _C.c_int64), ("c", _C.c_void_p), ("c_f32", _C.c_int),
                ("ldc", _C.c_int64), ("c_bs1", _C.c_int64), ("c_bs2", _C.c_int64), ("M", _C.c_int), ("N", _C.c_int),
                ("K", _C.c_int), ("nb1", _C.c_int), ("nb2", _C.c_int), ("alpha", _C.c_float), ("beta", _C.c_float),
                ("epilogue", _C.c_int), ("act", _C.c_int), ("bias", _C.c_void_p), ("aux", _C.c_void_p),
                ("ldaux", _C.c_int64), ("workspace", _C.c_void_p), ("workspace_bytes", _C.c_int64),
                ("colsum_part", _C.c_void_p)]


_GROUP: list | None = None  # GEMMs collected by `grouped()` (descriptor, keep-alive tensors, flops)
_GROUP_POST: list = []


class grouped:
    """Collect the GEMMs issued inside the with-block and launch them together on exit
    (smpk_gemm_grouped: two independent products fused into one persistent CTA-pair grid).
    Work that depends on a collected GEMM's output must be deferred with `after_group`."""

    def __enter__(self):
        global _GROUP
        if _GROUP is not None:
            raise RuntimeError("kernels.grouped() does not nest")
        _GROUP = []
        return self

    def __exit__(self, *exc):
        global _GROUP, _GROUP_POST
        items, post = _GROUP, _GROUP_POST
        _GROUP, _GROUP_POST = None, []
        if exc[0] is not None or not items:
            return False
        prof = PROFILER
        if prof is not None:
            e0, e1 = prof.event(), prof.event()
            if e0 is not None:
                e0.record()
        arr = (GemmDesc * len(items))(*[it[0] for it in items])
        _lib.call("smpk_gemm_grouped", _C.cast(arr, _C.c_void_p), len(items), _stream(),
                  launches=1 if len(items) == 2 else len(items))
        if prof is not None:
            if e1 is not None:
                e1.record()
            prof.records.append((e0, e1, sum(it[2] for it in items)))
        for fn in post:
            fn()
        return False


def after_group(fn) -> None:
    """Run fn now, or after the enclosing grouped() launch if one is collecting."""
    if _GROUP is None:
        fn()
    else:
        _GROUP_POST.append(fn)


def gemm_raw(a, a_mn, lda, a_bs, b, b_mn, ldb, b_bs, c, ldc, c_bs, M, N, K, nb=(1, 1),
             alpha=1.0, beta=0.0, epi=EPI_NONE, act=0, bias=None, aux=None, ldaux=0, colsum_part=None) -> None:
    """Direct binding of smpk_gemm; strides in elements, batch strides as 2-tuples.
    colsum_part: fp32 [ceil(M/32), N] receiving per-32-row column sums of the output."""
    _check_cuda(a, b, c, bias, aux)
    if _GROUP is not None:  # collected: launched by grouped.__exit__
        # a plain problem may be split over K inside the group (its units run first): workspace
        ws_bytes = 0 if (epi != EPI_NONE or colsum_part is not None) else \
            _lib.size("smpk_gemm_workspace", int(M), int(N), int(K), int(nb[0]), int(nb[1]))
        ws = torch.empty(ws_bytes // 4, dtype=torch.float32, device=c.device) if ws_bytes else None
        d = GemmDesc(_ptr(a), int(a_mn), int(lda), int(a_bs[0]), int(a_bs[1]), _ptr(b), int(b_mn), int(ldb),
                     int(b_bs[0]), int(b_bs[1]), _ptr(c), int(c.dtype == torch.float32), int(ldc), int(c_bs[0]),
                     int(c_bs[1]), int(M), int(N), int(K), int(nb[0]), int(nb[1]), float(alpha), float(beta),
                     int(epi), int(act), _ptr(bias), _ptr(aux), int(ldaux), _ptr(ws), int(ws_bytes), _ptr(colsum_part))
        _GROUP.append((d, (a, b, c, bias, aux, colsum_part, ws), 2.0 * M * N * K * nb[0] * nb[1]))
        return
    prof = PROFILER
    if prof is not None:
        e0, e1 = prof.event(), prof.event()
        if e0 is not None:
            e0.record()
    # split-K workspace (weight-gradient shapes with few output tiles); 0 bytes = unsplit
    ws_bytes = 0 if colsum_part is not None else _lib.size("smpk_gemm_workspace", int(M), int(N), int(K),
                                                               int(nb[0]), int(nb[1]))
    ws = torch.empty(ws_bytes // 4, dtype=torch.float32, device=c.device) if ws_bytes else None
    _lib.call("smpk_gemm_ex2",
              _ptr(a), int(a_mn), int(lda), int(a_bs[0]), int(a_bs[1]),
              _ptr(b), int(b_mn), int(ldb), int(b_bs[0]), int(b_bs[1]),
              _ptr(c), int(c.dtype == torch.float32), int(ldc), int(c_bs[0]), int(c_bs[1]),
              int(M), int(N), int(K), int(nb[0]), int(nb[1]),
              float(alpha), float(beta), int(epi), int(act),
              _ptr(bias), _ptr(aux), int(ldaux), _ptr(ws), int(ws_bytes), _ptr(colsum_part), _stream())
    if prof is not None:
        if e1 is not None:
            e1.record()
        prof.records.append((e0, e1, 2.0 * M * N * K * nb[0] * nb[1]))


def gemm_rs(a: torch.Tensor, b: torch.Tensor, b_mn: bool, peers, *, ldc: int, rows_per_owner: int,
            slot_off: int) -> None:
    """Row-parallel product a @ B^T (B [N,K]; b_mn: B given as [K,N]) whose rows are stored straight
    into the owning ranks' peer-mapped partial slots (peers: ctypes array of the T base addresses)."""
    _check_cuda(a, b)
    M, Kd = a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    prof = PROFILER
    if prof is not None:
        e0, e1 = prof.event(), prof.event()
        if e0 is not None:
            e0.record()
    _lib.call("smpk_gemm_rs", a.data_ptr(), 0, _rowmajor(a, "a"), b.data_ptr(), int(bool(b_mn)), _rowmajor(b, "b"),
              peers, len(peers), int(ldc), int(rows_per_owner), int(slot_off), M, N, Kd, _stream())
    if prof is not None:
        if e1 is not None:
            e1.record()
        prof.records.append((e0, e1, 2.0 * M * N * Kd))


def _rowmajor(t: torch.Tensor, name: str) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ShapeMismatchError(f"{name} must be a 2-D row-major view, got shape {tuple(t.shape)} "
                                 f"strides {t.stride()}")
    return t.stride(0)


def linear(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, *, act: str = "none",
           out: torch.Tensor | None = None, aux_out: torch.Tensor | None = None,
           residual: torch.Tensor | None = None):
    """y = x @ w.T (+ bias) (act) (+ residual). x [M,K], w [N,K] (nn.Linear layout).

    With act != none returns (y, pre_activation)."""
    M, K = x.shape
    N, K2 = w.shape
    if K != K2:
        raise ShapeMismatchError(f"linear: x has {K} features, weight expects {K2}")
    lda, ldb = _rowmajor(x, "x"), _rowmajor(w, "weight")
    y = out if out is not None else torch.empty(M, N, dtype=x.dtype, device=x.device)
    ldc = _rowmajor(y, "out")
    epi, aux, a_code = EPI_NONE, None, ACT[act]
    if act != "none":
        if bias is None:
            raise ShapeMismatchError("linear with activation needs a bias")
        epi = EPI_BIAS_ACT
        aux = aux_out if aux_out is not None else torch.empty(M, N, dtype=x.dtype, device=x.device)
    elif residual is not None:
        if bias is not None:
            raise ShapeMismatchError("linear: bias + residual epilogue not fused; add bias separately")
        epi, aux = EPI_ADD, residual
    elif bias is not None:
        epi = EPI_BIAS
    gemm_raw(x, 0, lda, (0, 0), w, 0, ldb, (0, 0), y, ldc, (0, 0), M, N, K,
             epi=epi, act=a_code, bias=bias, aux=aux, ldaux=(aux.stride(0) if aux is not None else 0))
    if act != "none":
        return y, aux
    return y


def matmul_nn(a: torch.Tensor, b: torch.Tensor, *, out=None, epi=EPI_NONE, act="none", aux=None,
              alpha=1.0, beta=0.0, want_colsum=False, colsum_part=None):
    """C = a @ b, a [M,K] row-major, b [K,N] row-major (B operand MN-major). dgrad: dX = dY @ W.
    want_colsum: also return the column sums of C (bf16 [N]) fused into the epilogue.
    colsum_part: caller-owned fp32 [colsum_rows(M), N] partials instead (reduced later by the
    caller with colsum_reduce, e.g. over several row chunks); returns (C, None)."""
    M, K = a.shape
    K2, N = b.shape
    if K != K2:
        raise ShapeMismatchError(f"matmul_nn: inner dims {K} vs {K2}")
    c = out if out is not None else torch.empty(M, N, dtype=a.dtype, device=a.device)
    part = colsum_part
    if colsum_part is not None:
        gemm_raw(a, 0, _rowmajor(a, "a"), (0, 0), b, 1, _rowmajor(b, "b"), (0, 0), c, _rowmajor(c, "out"), (0, 0),
                 M, N, K, alpha=alpha, beta=beta, epi=epi, act=ACT[act], aux=aux,
                 ldaux=(aux.stride(0) if aux is not None else 0), colsum_part=part)
        return c, None
    if want_colsum:
        part = torch.empty(colsum_rows(M), N, dtype=torch.float32, device=a.device)
    gemm_raw(a, 0, _rowmajor(a, "a"), (0, 0), b, 1, _rowmajor(b, "b"), (0, 0), c, _rowmajor(c, "out"), (0, 0),
             M, N, K, alpha=alpha, beta=beta, epi=epi, act=ACT[act], aux=aux,
             ldaux=(aux.stride(0) if aux is not None else 0), colsum_part=part)
    if want_colsum:
        cs = torch.empty(N, dtype=c.dtype, device=c.device)
        after_group(lambda: _lib.call("smpk_colsum_partials", _ptr(part), part.shape[0], N, _ptr(cs), 0, _stream()))
        return c, cs
    return c


def colsum_rows(M: int) -> int:
    """Rows of the fp32 column-sum partials a fused-colsum GEMM with M rows writes."""
    return _lib.size("smpk_gemm_colsum_rows", int(M))


def colsum_reduce(part: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """Fixed-order reduction of fused-colsum partials [rows, N] (fp32) into out [N]."""
    _lib.call("smpk_colsum_partials", _ptr(part), part.shape[0], part.shape[1], _ptr(out),
              int(out.dtype == torch.float32), _stream())
    return out


def matmul_tn(a: torch.Tensor, b: torch.Tensor, *, out=None, alpha=1.0, beta=0.0,
              out_dtype=None) -> torch.Tensor:
    """C = a.T @ b, a [K,M] row-major, b [K,N] row-major (both MN-major). wgrad: dW = dY.T @ X."""
    K, M = a.shape
    K2, N = b.shape
    if K != K2:
        raise ShapeMismatchError(f"matmul_tn: inner dims {K} vs {K2}")
    c = out if out is not None else torch.empty(M, N, dtype=out_dtype or a.dtype, device=a.device)
    gemm_raw(a, 1, _rowmajor(a, "a"), (0, 0), b, 1, _rowmajor(b, "b"), (0, 0), c, _rowmajor(c, "out"), (0, 0),
             M, N, K, alpha=alpha, beta=beta)
    return c


def matmul_nt(a: torch.Tensor, b: torch.Tensor, *, out=None, alpha=1.0, beta=0.0,
              out_dtype=None) -> torch.Tensor:
    """C = a @ b.T, a [M,K], b [N,K] (both K-major)."""
    M, K = a.shape
    N, K2 = b.shape
    if K != K2:
        raise ShapeMismatchError(f"matmul_nt: inner dims {K} vs {K2}")
    c = out if out is not None else torch.empty(M, N, dtype=out_dtype or a.dtype, device=a.device)
    gemm_raw(a, 0, _rowmajor(a, "a"), (0, 0), b, 0, _rowmajor(b, "b"), (0, 0), c, _rowmajor(c, "out"), (0, 0),
             M, N, K, alpha=alpha, beta=beta)
    return c
