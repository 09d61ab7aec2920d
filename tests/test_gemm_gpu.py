"""tcgen05 GEMM (csrc/gemm.cu) vs a plain torch fp32 reference of the same op.

Covers both operand majors (forward x W^T, dgrad dY W, wgrad dY^T X), every fused
epilogue, batched problems, ragged edges, and the split-K path the weight-gradient
shapes take (few output tiles, long K): its partial sums are reduced in split order,
so two launches must agree bit for bit.  Tolerance: rel-Frobenius <= 1e-2 (bf16 output
of an fp32-accumulated product)."""
import pytest
import torch

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()


@pytest.fixture(scope="module")
def K():
    from paper_2111_05972_b200 import _lib, kernels
    return kernels, _lib


def rnd(*shape):
    return torch.randn(*shape, device="cuda").to(torch.bfloat16)


@pytest.mark.parametrize("M,N,Kd", [(256, 256, 64), (1000, 776, 520), (4096, 1024, 1024), (128, 3072, 1024)])
def test_linear_nt(K, M, N, Kd):
    kernels, _ = K
    x, w = rnd(M, Kd), rnd(N, Kd)
    y = kernels.linear(x, w)
    assert rel(y.float(), x.float() @ w.float().t()) < TOL


@pytest.mark.parametrize("M,N,Kd", [(512, 1024, 4096), (16384, 1024, 256), (640, 200, 72)])
def test_matmul_nn_dgrad(K, M, N, Kd):
    kernels, _ = K
    a, b = rnd(M, Kd), rnd(Kd, N)
    c = kernels.matmul_nn(a, b)
    assert rel(c.float(), a.float() @ b.float()) < TOL


# (out rows, out cols, tokens): N=1 BERT-large wgrads and the TP=4 / TP=8 shards (K = T*4096)
WGRAD = [(1024, 1024, 4096), (3072, 1024, 4096), (256, 1024, 16384), (768, 1024, 16384), (1024, 512, 32768),
         (128, 1024, 32768), (200, 136, 8192)]


@pytest.mark.parametrize("M,N,Kd", WGRAD)
def test_matmul_tn_wgrad_splitk(K, M, N, Kd):
    kernels, lib = K
    dy, x = rnd(Kd, M), rnd(Kd, N)
    c1 = kernels.matmul_tn(dy, x)
    ref = dy.float().t() @ x.float()
    assert rel(c1.float(), ref) < TOL
    c2 = kernels.matmul_tn(dy, x)
    assert torch.equal(c1, c2), "split-K reduction must be deterministic"
    # fp32 output + beta accumulate (gradient accumulation into an fp32 buffer)
    acc = torch.randn(M, N, device="cuda")
    ref2 = ref + 0.5 * acc
    kernels.matmul_tn(dy, x, out=acc, beta=0.5)
    assert rel(acc, ref2) < 1e-3


def test_splitk_engaged_for_small_tile_counts(K):
    _, lib = K
    assert lib.size("smpk_gemm_workspace", 256, 1024, 16384, 1, 1) > 0
    assert lib.size("smpk_gemm_workspace", 16384, 1024, 256, 1, 1) == 0


@pytest.mark.parametrize("act", ["gelu", "gelu_tanh", "relu"])
def test_bias_act_and_dact(K, act):
    kernels, _ = K
    M, N, Kd = 1024, 4096, 1024
    x, w, bvec = rnd(M, Kd), rnd(N, Kd), rnd(N)
    y, pre = kernels.linear(x, w, bvec, act=act)
    pre_ref = x.float() @ w.float().t() + bvec.float()
    f = {"gelu": lambda t: torch.nn.functional.gelu(t),
         "gelu_tanh": lambda t: torch.nn.functional.gelu(t, approximate="tanh"),
         "relu": torch.relu}[act]
    assert rel(pre.float(), pre_ref) < TOL
    assert rel(y.float(), f(pre.float())) < TOL
    # DACT epilogue: dX_pre = (dY W) * act'(pre)
    dy, w2 = rnd(M, 1024), rnd(1024, N)
    d = kernels.matmul_nn(dy, w2, epi=kernels.EPI_DACT, act=act, aux=pre)
    p = pre.float().requires_grad_(True)
    f(p).backward(dy.float() @ w2.float())
    tol = 6e-2 if act == "relu" else TOL  # relu' flips on bf16-rounded pre-activations near 0
    assert rel(d.float(), p.grad) < tol
    # fused bias-gradient column sums of the stored output (per-32-row partials, reduced in order)
    d2, cs = kernels.matmul_nn(dy, w2, epi=kernels.EPI_DACT, act=act, aux=pre, want_colsum=True)
    assert torch.equal(d2, d)
    assert rel(cs.float(), d.float().sum(0)) < TOL


@pytest.mark.parametrize("M,N", [(1000, 776), (96, 4096), (4096, 40)])
def test_dgrad_colsum_ragged(K, M, N):
    kernels, _ = K
    dy, w = rnd(M, 256), rnd(256, N)
    d, cs = kernels.matmul_nn(dy, w, want_colsum=True)
    assert torch.equal(d, kernels.matmul_nn(dy, w))
    assert rel(cs.float(), d.float().sum(0)) < TOL
    _, cs2 = kernels.matmul_nn(dy, w, want_colsum=True)
    assert torch.equal(cs, cs2)


def test_bias_and_residual_epilogues(K):
    kernels, _ = K
    M, N, Kd = 2048, 1024, 4096
    x, w, bvec, res = rnd(M, Kd), rnd(N, Kd), rnd(N), rnd(M, N)
    y = kernels.linear(x, w, bvec)
    assert rel(y.float(), x.float() @ w.float().t() + bvec.float()) < TOL
    y2 = kernels.linear(x, w, residual=res)
    assert rel(y2.float(), x.float() @ w.float().t() + res.float()) < TOL


def test_batched_strided(K):
    kernels, _ = K
    B, nh, s, dh = 2, 4, 512, 64
    q, k = rnd(B, nh, s, dh), rnd(B, nh, s, dh)
    c = torch.empty(B, nh, s, s, device="cuda", dtype=torch.bfloat16)
    kernels.gemm_raw(q, 0, dh, (s * dh, nh * s * dh), k, 0, dh, (s * dh, nh * s * dh), c, s, (s * s, nh * s * s),
                     s, s, dh, nb=(nh, B), alpha=0.125)
    ref = (q.float() @ k.float().transpose(-1, -2)) * 0.125
    assert rel(c.float(), ref) < TOL


@pytest.mark.parametrize("epi", ["none", "add", "dact"])
def test_grouped_pair_matches_reference(epi):
    """smpk_gemm_grouped: a weight-gradient GEMM (plain) fused with an input-gradient GEMM (plain /
    residual add / dGeLU + fused column sums) in one persistent grid == torch fp32 references, and
    bit-identical run to run."""
    from paper_2111_05972_b200 import kernels as K
    g = torch.Generator().manual_seed(11)
    T_, H, I = 2048, 512, 1024
    dy = (torch.randn(T_, I, generator=g) * 0.1).bfloat16().cuda()
    x = (torch.randn(T_, H, generator=g) * 0.1).bfloat16().cuda()
    w = (torch.randn(I, H, generator=g) * 0.1).bfloat16().cuda()  # forward weight [out, in]
    aux = (torch.randn(T_, H, generator=g)).bfloat16().cuda()

    def run():
        dw = torch.empty(I, H, dtype=torch.bfloat16, device="cuda")
        with K.grouped():
            K.matmul_tn(dy, x, out=dw)
            if epi == "none":
                dx = K.matmul_nn(dy, w)
                cs = None
            elif epi == "add":
                dx = K.matmul_nn(dy, w, epi=K.EPI_ADD, aux=aux)
                cs = None
            else:
                dx, cs = K.matmul_nn(dy, w, epi=K.EPI_DACT, act="gelu", aux=aux, want_colsum=True)
        torch.cuda.synchronize()
        return dw, dx, cs

    dw, dx, cs = run()
    dw_ref = dy.float().t() @ x.float()
    dx_ref = dy.float() @ w.float()
    if epi == "add":
        dx_ref = dx_ref + aux.float()
    elif epi == "dact":
        z = aux.float()
        dx_ref = dx_ref * (0.5 * (1 + torch.erf(z / 2 ** 0.5)) + z * torch.exp(-0.5 * z * z) / (2 * torch.pi) ** 0.5)
    rel_ = lambda a, b: ((a.float() - b).norm() / b.norm()).item()  # noqa: E731
    assert rel_(dw, dw_ref) < 1e-2 and rel_(dx, dx_ref) < 1e-2
    if cs is not None:
        assert rel_(cs, dx.float().sum(0)) < 1e-2
    dw2, dx2, cs2 = run()
    assert torch.equal(dw, dw2) and torch.equal(dx, dx2)
