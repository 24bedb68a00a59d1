"""GPU parity of the individual sm_100a kernels (called through the C ABI of
include/bigmac_kernels.h) against the oracle's fp64 definitions.

Inputs are bf16-representable, so the only differences are the kernels'
fp32 accumulation order and bf16 output rounding (tolerances stated per test).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import model as om  # noqa: E402
from synth import bf16_round  # noqa: E402

pytestmark = pytest.mark.gpu

BF16, F32 = 0, 1


@pytest.fixture(scope="module")
def L():
    from paper_2605_25451_b200 import _lib
    return _lib


def dev(x, dtype):
    t = torch.tensor(np.asarray(x, np.float32), device="cuda")
    return t.to(torch.bfloat16 if dtype == BF16 else torch.float32).contiguous()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def rnd(rng, *shape, scale=1.0):
    return bf16_round(rng.standard_normal(shape).astype(np.float32) * scale).astype(np.float64)


GEMM_SHAPES = [(128, 256, 64), (300, 200, 100), (1, 16, 48), (257, 513, 130), (64, 64, 16),
               (129, 1000, 640), (2048, 2048, 1024), (40, 4096, 16),
               # encoder/generator-like shapes that take the split-K path
               (554, 384, 1536), (1536, 384, 560), (704, 1536, 384), (120, 512, 2048)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("dtype,mode", [(BF16, 1), (BF16, 2), (BF16, 0), (F32, 0)])
def test_gemm_store_f32(L, M, N, K, a_mn, b_mn, dtype, mode):
    L.call("bm_k_gemm_mode", mode)
    rng = np.random.default_rng(M * 7 + N * 3 + K + 11 * a_mn + 5 * b_mn)
    A = rnd(rng, M, K)
    B = rnd(rng, N, K)
    Ad = dev(A.T.copy() if a_mn else A, dtype)
    Bd = dev(B.T.copy() if b_mn else B, dtype)
    lda = M if a_mn else K
    ldb = N if b_mn else K
    if dtype == BF16 and (lda % 8 or ldb % 8):
        pytest.skip("bf16 TMA needs 16-byte strides")
    C = torch.full((M, N), 7.0, device="cuda", dtype=torch.float32)
    L.call("bm_k_gemm", dtype, M, N, K, Ad.data_ptr(), lda, a_mn, Bd.data_ptr(), ldb, b_mn,
           C.data_ptr(), N, F32, 0, None, 0, 1.0, None)
    torch.cuda.synchronize()
    ref = A @ B.T
    L.call("bm_k_gemm_mode", 0)
    err = np.abs(host(C) - ref).max()
    tol = 1e-5 * np.sqrt(K) * max(1.0, np.abs(ref).max()) if dtype == BF16 else 2e-6 * np.sqrt(K) * max(1.0, np.abs(ref).max())
    assert err <= tol, (err, tol)


@pytest.mark.parametrize("M,N,K", [(2560, 2048, 512), (4096, 2048, 1024), (2304, 4352, 320)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
def test_gemm_pairs_partial_last_wave(L, M, N, K, a_mn, b_mn):
    """CTA-pair GEMMs whose last wave of whole 256x256 tiles leaves pairs idle
    (80 / 128 / 153 tiles on 74 pairs), every operand-major combination (runtime
    majors of the pair kernel), against the fp64 product; bitwise deterministic."""
    L.call("bm_k_gemm_mode", 2)
    rng = np.random.default_rng(M + N + K + 3 * a_mn + b_mn)
    A, B = rnd(rng, M, K), rnd(rng, N, K)
    Ad = dev(A.T.copy() if a_mn else A, BF16)
    Bd = dev(B.T.copy() if b_mn else B, BF16)
    C = torch.full((M, N), 7.0, device="cuda", dtype=torch.float32)
    L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), M if a_mn else K, a_mn, Bd.data_ptr(), N if b_mn else K, b_mn,
           C.data_ptr(), N, F32, 0, None, 0, 1.0, None)
    torch.cuda.synchronize()
    L.call("bm_k_gemm_mode", 0)
    ref = A @ B.T
    err = np.abs(host(C) - ref).max()
    assert err <= 1e-5 * np.sqrt(K) * max(1.0, np.abs(ref).max()), err
    # deterministic: a rerun reproduces every bit
    C2 = torch.zeros_like(C)
    L.call("bm_k_gemm_mode", 2)
    L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), M if a_mn else K, a_mn, Bd.data_ptr(), N if b_mn else K, b_mn,
           C2.data_ptr(), N, F32, 0, None, 0, 1.0, None)
    torch.cuda.synchronize()
    L.call("bm_k_gemm_mode", 0)
    assert torch.equal(C, C2)


@pytest.mark.parametrize("M,N,K", [(300, 200, 104), (257, 513, 136), (1024, 768, 512), (554, 384, 1536), (4096, 2048, 640)])
@pytest.mark.parametrize("epi", ["bf16_store", "bf16_add", "f32_accum"])
@pytest.mark.parametrize("mode", [1, 2])
def test_gemm_epilogues(L, M, N, K, epi, mode):
    L.call("bm_k_gemm_mode", mode)
    rng = np.random.default_rng(1)
    A, B = rnd(rng, M, K), rnd(rng, N, K)
    R = rnd(rng, M, N)
    Ad, Bd = dev(A, BF16), dev(B, BF16)
    ref = A @ B.T * 0.5
    if epi == "bf16_store":
        C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
        L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), K, 0, Bd.data_ptr(), K, 0, C.data_ptr(), N, BF16, 0,
               None, 0, 0.5, None)
    elif epi == "bf16_add":
        C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
        Rd = dev(R, BF16)
        L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), K, 0, Bd.data_ptr(), K, 0, C.data_ptr(), N, BF16, 2,
               Rd.data_ptr(), N, 0.5, None)
        ref = ref + R
    else:
        C = dev(R, F32)
        L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), K, 0, Bd.data_ptr(), K, 0, C.data_ptr(), N, F32, 1,
               None, 0, 0.5, None)
        ref = ref + R
    torch.cuda.synchronize()
    L.call("bm_k_gemm_mode", 0)
    out = host(C)
    if epi.startswith("bf16"):
        assert np.all(np.abs(out - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-4 * np.sqrt(K))
    else:
        assert np.abs(out - ref).max() <= 1e-5 * np.sqrt(K)


@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("rows,cols", [(1, 64), (37, 128), (300, 2048), (4096, 2048), (1003, 4096), (5, 1024),
                                       (130, 6144)])
def test_rmsnorm(L, dtype, rows, cols):
    # cols 2048 / 4096 (bf16) and 1024 / 2048 / 4096 (fp32) take the wide-row backward
    # (a 256-thread row split, ragged 4-row groups), 6144 / 64 / 128 the per-warp-row one
    rng = np.random.default_rng(2)
    x = rnd(rng, rows, cols, scale=2.0)
    g = rnd(rng, cols, scale=0.5) + 1.0
    g = bf16_round(g.astype(np.float32)).astype(np.float64)
    dy = rnd(rng, rows, cols)
    dres = rnd(rng, rows, cols)
    xd, gd, dyd, dresd = dev(x, dtype), dev(g, dtype), dev(dy, dtype), dev(dres, dtype)
    y = torch.empty_like(xd)
    rstd = torch.empty(rows, device="cuda", dtype=torch.float32)
    L.call("bm_k_rmsnorm_fwd", dtype, rows, cols, xd.data_ptr(), gd.data_ptr(), y.data_ptr(), rstd.data_ptr(), None)
    dx = torch.empty_like(xd)
    dg = torch.full((cols,), 0.25, device="cuda", dtype=torch.float32)
    part = torch.empty(L.lib().bm_k_rmsnorm_bwd_scratch(rows, cols), device="cuda", dtype=torch.float32)
    L.call("bm_k_rmsnorm_bwd", dtype, rows, cols, dyd.data_ptr(), xd.data_ptr(), gd.data_ptr(), rstd.data_ptr(),
           dresd.data_ptr(), dx.data_ptr(), dg.data_ptr(), part.data_ptr(), None)
    torch.cuda.synchronize()
    yr, rs = om.rmsnorm(x, g)
    dxr, dgr = om.rmsnorm_bwd(dy, x, g, rs)
    tol = 1e-2 if dtype == BF16 else 1e-5
    assert np.abs(host(y) - yr).max() <= tol * np.abs(yr).max()
    assert np.abs(host(rstd) - rs[:, 0]).max() <= 1e-5 * np.abs(rs).max()
    assert np.abs(host(dx) - (dxr + dres)).max() <= tol * np.abs(dxr + dres).max()
    assert np.abs(host(dg) - (dgr + 0.25)).max() <= 1e-4 * max(1, np.abs(dgr).max())
    # deterministic: a rerun reproduces dx and the gain gradient bit for bit
    dx2 = torch.empty_like(xd)
    dg2 = torch.full((cols,), 0.25, device="cuda", dtype=torch.float32)
    L.call("bm_k_rmsnorm_bwd", dtype, rows, cols, dyd.data_ptr(), xd.data_ptr(), gd.data_ptr(), rstd.data_ptr(),
           dresd.data_ptr(), dx2.data_ptr(), dg2.data_ptr(), part.data_ptr(), None)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2)


@pytest.mark.parametrize("dtype", [BF16, F32])
def test_swiglu_gelu(L, dtype):
    rng = np.random.default_rng(3)
    rows, f = 77, 384
    gu = rnd(rng, rows, 2 * f, scale=2.0)
    dh = rnd(rng, rows, f)
    gud, dhd = dev(gu, dtype), dev(dh, dtype)
    h = torch.empty((rows, f), device="cuda", dtype=gud.dtype)
    dgu = torch.empty_like(gud)
    L.call("bm_k_swiglu_fwd", dtype, rows, f, gud.data_ptr(), h.data_ptr(), None)
    L.call("bm_k_swiglu_bwd", dtype, rows, f, dhd.data_ptr(), gud.data_ptr(), dgu.data_ptr(), None)
    a = rnd(rng, 1001, scale=3.0)
    ad, dz = dev(a, dtype), dev(np.ones(1001), dtype)
    z = torch.empty_like(ad)
    da = torch.empty_like(ad)
    L.call("bm_k_gelu_fwd", dtype, 1001, ad.data_ptr(), z.data_ptr(), None)
    L.call("bm_k_gelu_bwd", dtype, 1001, dz.data_ptr(), ad.data_ptr(), da.data_ptr(), None)
    torch.cuda.synchronize()
    tol = 1e-2 if dtype == BF16 else 1e-5
    hr = om.swiglu(gu, f)
    assert np.abs(host(h) - hr).max() <= tol * np.abs(hr).max()
    dgur = om.swiglu_bwd(dh, gu, f)
    assert np.abs(host(dgu) - dgur).max() <= tol * np.abs(dgur).max()
    assert np.abs(host(z) - om.gelu(a)).max() <= tol * np.abs(om.gelu(a)).max()
    assert np.abs(host(da) - om.gelu_bwd(np.ones(1001), a)).max() <= tol * 1.2


@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("S,d,n_mod,vocab", [(128, 128, 40, 256), (4096, 256, 700, 1000), (64, 64, 64, 50),
                                             (4096, 2048, 554, 32000), (8192, 128, 300, 500), (8192, 64, 0, 40000),
                                             (16384, 64, 100, 3000)])
def test_embed(L, dtype, S, d, n_mod, vocab):
    rng = np.random.default_rng(4)
    table = rnd(rng, vocab, d)
    emb = rnd(rng, n_mod, d)
    ids = rng.integers(0, vocab, size=S).astype(np.int32)
    dX = rnd(rng, S, d)
    td, ed, dXd = dev(table, dtype), dev(emb, dtype), dev(dX, dtype)
    idd = torch.tensor(ids, device="cuda")
    X = torch.empty((S, d), device="cuda", dtype=td.dtype)
    L.call("bm_k_embed_fwd", dtype, S, d, n_mod, idd.data_ptr(), td.data_ptr(), ed.data_ptr(), X.data_ptr(), None)
    dT = torch.zeros((vocab, d), device="cuda", dtype=torch.float32)
    scratch = torch.empty(L.lib().bm_k_embed_bwd_scratch(S), device="cuda", dtype=torch.uint8)
    L.call("bm_k_embed_bwd", dtype, S, d, n_mod, idd.data_ptr(), dXd.data_ptr(), dT.data_ptr(), scratch.data_ptr(),
           None)
    dT2 = torch.zeros_like(dT)
    L.call("bm_k_embed_bwd", dtype, S, d, n_mod, idd.data_ptr(), dXd.data_ptr(), dT2.data_ptr(), scratch.data_ptr(),
           None)
    torch.cuda.synchronize()
    Xr = om.embed_fwd({"llm.embed": table}, ids, emb, n_mod)
    assert np.array_equal(host(X), Xr)   # pure data movement: bit exact
    G = {}

    class Cfg:
        pass
    c = Cfg()
    c.vocab, c.d = vocab, d
    om.embed_bwd(c, dX, ids, n_mod, G)
    assert np.abs(host(dT) - G["llm.embed"]).max() <= 1e-5 * max(1, np.abs(G["llm.embed"]).max())
    assert torch.equal(dT, dT2)          # deterministic


@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("n,V", [(88, 256), (300, 32000), (1, 50)])
def test_cross_entropy(L, dtype, n, V):
    rng = np.random.default_rng(5)
    z = rnd(rng, n, V, scale=2.0)
    lab = rng.integers(0, V, size=n).astype(np.int32)
    zd = dev(z, dtype)
    labd = torch.tensor(lab, device="cuda")
    loss = torch.full((1,), 3.0, device="cuda", dtype=torch.float32)
    scr = torch.empty(n, device="cuda", dtype=torch.float32)
    L.call("bm_k_ce_fwd_bwd", dtype, n, V, zd.data_ptr(), labd.data_ptr(), 0.25, loss.data_ptr(), 1.0, 1,
           scr.data_ptr(), None)
    torch.cuda.synchronize()
    zmax = z.max(1, keepdims=True)
    lse = np.log(np.exp(z - zmax).sum(1, keepdims=True)) + zmax
    ref = np.mean(lse[:, 0] - z[np.arange(n), lab])
    p = np.exp(z - lse)
    p[np.arange(n), lab] -= 1
    tol = 1e-2 if dtype == BF16 else 1e-5
    assert abs(host(loss)[0] - (3.0 + ref)) <= 1e-5 * max(1, abs(ref))
    assert np.abs(host(zd) - 0.25 * p).max() <= tol * 0.25


@pytest.mark.parametrize("dtype", [BF16, F32])
def test_mse(L, dtype):
    rng = np.random.default_rng(6)
    n, dt = 173, 16
    o, t = rnd(rng, n, dt), rnd(rng, n, dt)
    od, tdv = dev(o, dtype), dev(t, dtype)
    dout = torch.empty_like(od)
    loss = torch.full((1,), 1.0, device="cuda", dtype=torch.float32)
    denom = float(500 * dt)
    L.call("bm_k_mse_fwd_bwd", dtype, n, dt, od.data_ptr(), tdv.data_ptr(), denom, 0.5, 1.0, loss.data_ptr(),
           dout.data_ptr(), None)
    torch.cuda.synchronize()
    assert abs(host(loss)[0] - (1.0 + np.sum((o - t) ** 2) / denom)) <= 1e-5
    tol = 1e-2 if dtype == BF16 else 1e-6
    ref = 2 * (o - t) / denom * 0.5
    assert np.abs(host(dout) - ref).max() <= tol * np.abs(ref).max()


@pytest.mark.parametrize("M,f,K", [(300, 384, 128), (1000, 1024, 512), (2048, 1024, 256), (1, 128, 64)])
def test_gemm_fused_swiglu(L, M, f, K):
    # gate/up GEMM + SwiGLU epilogue, and down dgrad + SwiGLU-backward epilogue
    rng = np.random.default_rng(9)
    X = rnd(rng, M, K)
    Wgu = rnd(rng, 2 * f, K, scale=0.1)
    Xd, Wd = dev(X, BF16), dev(Wgu, BF16)
    gu = torch.zeros((M, 2 * f), device="cuda", dtype=torch.bfloat16)
    h = torch.zeros((M, f), device="cuda", dtype=torch.bfloat16)
    L.call("bm_k_gemm_swiglu", M, f, K, Xd.data_ptr(), K, Wd.data_ptr(), K, gu.data_ptr(), h.data_ptr(), None)
    Kd = 256
    dY = rnd(rng, M, Kd)
    Wdown = rnd(rng, Kd, f, scale=0.1)
    dYd, Wdd = dev(dY, BF16), dev(Wdown, BF16)
    dgu = torch.zeros((M, 2 * f), device="cuda", dtype=torch.bfloat16)
    L.call("bm_k_gemm_dswiglu", M, f, Kd, dYd.data_ptr(), Kd, Wdd.data_ptr(), f, gu.data_ptr(), dgu.data_ptr(), None)
    torch.cuda.synchronize()
    gu_ref = X @ Wgu.T
    gu_out = host(gu)
    assert np.all(np.abs(gu_out - gu_ref) <= 2.0 ** -8 * np.abs(gu_ref) + 1e-4 * np.sqrt(K))
    h_ref = om.swiglu(gu_out, f)     # activation of the stored bf16 g, u
    assert np.abs(host(h) - h_ref).max() <= 1e-2 * max(1e-3, np.abs(h_ref).max())
    dh = dY @ Wdown
    dgu_ref = om.swiglu_bwd(dh, gu_out, f)
    assert np.abs(host(dgu) - dgu_ref).max() <= 1e-2 * max(1e-3, np.abs(dgu_ref).max())


# grouped CTA-pair launches (bm_k_gemm_group): a Linear's weight gradient (fp32 TMA
# reduce-add, A and B MN-major) and data gradient (bf16 store or the fused SwiGLU
# backward, B MN-major) in one persistent launch on the LPT tile schedule
GROUP_CASES = [
    # (S rows, in, out, dgrad epilogue, gemm mode)
    (4096, 2048, 8192, "store", 0),     # C2 gate_up-like: long-K dgrad + short-K wgrad
    (4096, 8192, 2048, "dswiglu", 0),   # C2 down-like: dgrad with the SwiGLU backward
    (520, 384, 640, "dswiglu", 2),      # ragged: partial m / n tiles, forced pairs
    (768, 1280, 512, "store", 2),
    (1000, 512, 2048, "store", 0),      # auto mode, too few tiles: separate 1-CTA launches
]


@pytest.mark.parametrize("S,n_in,n_out,dg_epi,mode", GROUP_CASES)
def test_gemm_group_dgrad_wgrad(L, S, n_in, n_out, dg_epi, mode):
    L.call("bm_k_gemm_mode", mode)
    rng = np.random.default_rng(S + n_in + n_out)
    dY = rnd(rng, S, n_out)                     # [S, out]
    X = rnd(rng, S, n_in, scale=0.5)             # [S, in]
    Wt = rnd(rng, n_out, n_in, scale=0.05)       # [out, in]
    dYd, Xd, Wd = dev(dY, BF16), dev(X, BF16), dev(Wt, BF16)
    dW0 = rnd(rng, n_out, n_in)
    dW = torch.tensor(dW0, device="cuda", dtype=torch.float32)
    D = L.GemmDesc
    wgrad = D(n_out, n_in, S, dYd.data_ptr(), n_out, 1, Xd.data_ptr(), n_in, 1, dW.data_ptr(), n_in, F32, 1, None, 0,
              1.0, 0)
    if dg_epi == "store":
        dX = torch.zeros((S, n_in), device="cuda", dtype=torch.bfloat16)
        dgrad = D(S, n_in, n_out, dYd.data_ptr(), n_out, 0, Wd.data_ptr(), n_in, 1, dX.data_ptr(), n_in, BF16, 0, None,
                  0, 1.0, 0)
    else:   # the down projection's dgrad: N = f = n_in, C = dgu [S, 2f], R = gu [S, 2f]
        f = n_in
        gu_h = rnd(rng, S, 2 * f)
        gu = dev(gu_h, BF16)
        dX = torch.zeros((S, 2 * f), device="cuda", dtype=torch.bfloat16)
        dgrad = D(S, f, n_out, dYd.data_ptr(), n_out, 0, Wd.data_ptr(), n_in, 1, dX.data_ptr(), 2 * f, BF16, 4,
                  gu.data_ptr(), 2 * f, 1.0, f)
    arr = (D * 2)(dgrad, wgrad)
    L.call("bm_k_gemm_group", arr, 2, None)
    torch.cuda.synchronize()
    first = (dW.clone(), dX.clone())
    L.call("bm_k_gemm_mode", 0)
    dW_ref = dW0 + dY.T @ X
    tol = 1e-5 * np.sqrt(S) * max(1.0, np.abs(dY.T @ X).max())
    assert np.abs(host(dW) - dW_ref).max() <= tol
    dh = dY @ Wt
    if dg_epi == "store":
        assert np.all(np.abs(host(dX) - dh) <= 2.0 ** -8 * np.abs(dh) + 1e-4 * np.sqrt(n_out))
    else:
        ref = om.swiglu_bwd(dh, gu_h, n_in)
        assert np.all(np.abs(host(dX) - ref) <= 2.0 ** -7 * np.abs(ref) + 1e-3 * np.abs(ref).max())
    # deterministic: rerun from the same initial dW reproduces every bit
    dW.copy_(torch.tensor(dW0, device="cuda", dtype=torch.float32))
    L.call("bm_k_gemm_mode", mode)
    L.call("bm_k_gemm_group", arr, 2, None)
    torch.cuda.synchronize()
    L.call("bm_k_gemm_mode", 0)
    assert torch.equal(first[0], dW) and torch.equal(first[1], dX)


@pytest.mark.parametrize("M,N,K", [(512, 512, 64), (2560, 2048, 512), (1000, 1000, 640), (4096, 2560, 4096),
                                   (304, 1600, 200)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("epi", ["f32_store", "bf16_add", "f32_accum"])
def test_gemm_pairs_bn512(L, M, N, K, a_mn, b_mn, epi):
    """256 x 512 CTA-pair tiles (single 512-column TMEM accumulator, B loaded as two
    128-row halves per CTA): every operand-major combination, ragged M / N / K,
    store / residual-add / fp32 reduce-add epilogues, against the fp64 product;
    bitwise equal to a rerun."""
    L.call("bm_k_gemm_mode", 2)
    L.call("bm_k_gemm_bn512", 1)
    try:
        rng = np.random.default_rng(M + 3 * N + K + 7 * a_mn + b_mn)
        A, B, R = rnd(rng, M, K), rnd(rng, N, K), rnd(rng, M, N)
        Ad = dev(A.T.copy() if a_mn else A, BF16)
        Bd = dev(B.T.copy() if b_mn else B, BF16)
        ref = A @ B.T * 0.5
        outs = []
        for _ in range(2):
            if epi == "f32_store":
                C = torch.full((M, N), 7.0, device="cuda", dtype=torch.float32)
                args = (C.data_ptr(), N, F32, 0, None, 0)
            elif epi == "bf16_add":
                C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
                Rd = dev(R, BF16)
                args = (C.data_ptr(), N, BF16, 2, Rd.data_ptr(), N)
            else:
                C = dev(R, F32)
                args = (C.data_ptr(), N, F32, 1, None, 0)
            L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), M if a_mn else K, a_mn, Bd.data_ptr(),
                   N if b_mn else K, b_mn, *args, 0.5, None)
            torch.cuda.synchronize()
            outs.append(C)
        out = host(outs[0])
        if epi != "f32_store":
            ref = ref + R
        if epi == "bf16_add":
            assert np.all(np.abs(out - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-4 * np.sqrt(K))
        else:
            assert np.abs(out - ref).max() <= 1e-5 * np.sqrt(K) * max(1.0, np.abs(ref).max())
        assert torch.equal(outs[0], outs[1])
    finally:
        L.call("bm_k_gemm_mode", 0)
        L.call("bm_k_gemm_bn512", 2)


@pytest.mark.parametrize("M,f,Kd", [(2048, 1024, 256), (600, 512, 4096), (4096, 2048, 2048)])
def test_gemm_dswiglu_bn512(L, M, f, Kd):
    """The SwiGLU-backward epilogue on 256 x 512 pair tiles vs fp64 swiglu_bwd."""
    L.call("bm_k_gemm_mode", 2)
    L.call("bm_k_gemm_bn512", 1)
    try:
        rng = np.random.default_rng(f + Kd)
        gu = rnd(rng, M, 2 * f)
        dY = rnd(rng, M, Kd)
        Wdown = rnd(rng, Kd, f, scale=0.1)
        gud, dYd, Wdd = dev(gu, BF16), dev(dY, BF16), dev(Wdown, BF16)
        dgu = torch.zeros((M, 2 * f), device="cuda", dtype=torch.bfloat16)
        L.call("bm_k_gemm_dswiglu", M, f, Kd, dYd.data_ptr(), Kd, Wdd.data_ptr(), f, gud.data_ptr(), dgu.data_ptr(),
               None)
        torch.cuda.synchronize()
        dgu_ref = om.swiglu_bwd(dY @ Wdown, gu, f)
        assert np.abs(host(dgu) - dgu_ref).max() <= 1e-2 * max(1e-3, np.abs(dgu_ref).max())
    finally:
        L.call("bm_k_gemm_mode", 0)
        L.call("bm_k_gemm_bn512", 2)


@pytest.mark.parametrize("M,N,K", [(512, 512, 64), (2560, 2048, 512), (1000, 1000, 640), (4096, 2304, 1000),
                                   (304, 1280, 200)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("epi", ["f32_store", "bf16_add", "f32_accum", "dswiglu"])
@pytest.mark.parametrize("bk", [128, 64])
def test_gemm_pairs_bk128(L, M, N, K, a_mn, b_mn, epi, bk):
    """128-deep (default) and 64-deep K blocks on 256 x 256 pair tiles (bm_k_gemm_bk128):
    every operand major, K tails that end inside a block or a sub-tile, four epilogues;
    bitwise equal to a rerun."""
    L.call("bm_k_gemm_mode", 2)
    L.call("bm_k_gemm_bn512", 0)
    L.call("bm_k_gemm_bk128", 1 if bk == 128 else 0)
    try:
        rng = np.random.default_rng(M + 3 * N + 5 * K + 7 * a_mn + b_mn)
        if epi == "dswiglu":
            if a_mn or not b_mn or N % 32:
                pytest.skip("the SwiGLU backward is dY (K-major) x W_down (MN-major), f % 32 == 0")
            f = N
            gu, dY, Wd = rnd(rng, M, 2 * f), rnd(rng, M, K), rnd(rng, K, f, scale=0.1)
            gud, dYd, Wdd = dev(gu, BF16), dev(dY, BF16), dev(Wd, BF16)
            outs = []
            for _ in range(2):
                dgu = torch.zeros((M, 2 * f), device="cuda", dtype=torch.bfloat16)
                L.call("bm_k_gemm_dswiglu", M, f, K, dYd.data_ptr(), K, Wdd.data_ptr(), f, gud.data_ptr(),
                       dgu.data_ptr(), None)
                torch.cuda.synchronize()
                outs.append(dgu)
            ref = om.swiglu_bwd(dY @ Wd, gu, f)
            assert np.abs(host(outs[0]) - ref).max() <= 1e-2 * max(1e-3, np.abs(ref).max())
            assert torch.equal(outs[0], outs[1])
            return
        A, B, R = rnd(rng, M, K), rnd(rng, N, K), rnd(rng, M, N)
        Ad = dev(A.T.copy() if a_mn else A, BF16)
        Bd = dev(B.T.copy() if b_mn else B, BF16)
        ref = A @ B.T * 0.5
        outs = []
        for _ in range(2):
            if epi == "f32_store":
                C = torch.full((M, N), 7.0, device="cuda", dtype=torch.float32)
                args = (C.data_ptr(), N, F32, 0, None, 0)
            elif epi == "bf16_add":
                C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
                Rd = dev(R, BF16)
                args = (C.data_ptr(), N, BF16, 2, Rd.data_ptr(), N)
            else:
                C = dev(R, F32)
                args = (C.data_ptr(), N, F32, 1, None, 0)
            L.call("bm_k_gemm", BF16, M, N, K, Ad.data_ptr(), M if a_mn else K, a_mn, Bd.data_ptr(),
                   N if b_mn else K, b_mn, *args, 0.5, None)
            torch.cuda.synchronize()
            outs.append(C)
        out = host(outs[0])
        if epi != "f32_store":
            ref = ref + R
        if epi == "bf16_add":
            assert np.all(np.abs(out - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-4 * np.sqrt(K))
        else:
            assert np.abs(out - ref).max() <= 1e-5 * np.sqrt(K) * max(1.0, np.abs(ref).max())
        assert torch.equal(outs[0], outs[1])
    finally:
        L.call("bm_k_gemm_bk128", 1)
        L.call("bm_k_gemm_mode", 0)
        L.call("bm_k_gemm_bn512", 2)


@pytest.mark.parametrize("M,f,K", [(300, 384, 128), (2048, 1024, 256), (4096, 2048, 2000), (1, 128, 64)])
@pytest.mark.parametrize("bk", [128, 64])
def test_gemm_fused_swiglu_bk128(L, M, f, K, bk):
    """gate/up GEMM + SwiGLU epilogue with 128-deep K blocks and 4 KB staging (default)
    and with 64-deep blocks and 6 KB staging."""
    L.call("bm_k_gemm_swiglu_bk128", 1 if bk == 128 else 0)
    try:
        rng = np.random.default_rng(3 * f + K)
        X, Wgu = rnd(rng, M, K), rnd(rng, 2 * f, K, scale=0.1)
        Xd, Wd = dev(X, BF16), dev(Wgu, BF16)
        gu = torch.zeros((M, 2 * f), device="cuda", dtype=torch.bfloat16)
        h = torch.zeros((M, f), device="cuda", dtype=torch.bfloat16)
        L.call("bm_k_gemm_swiglu", M, f, K, Xd.data_ptr(), K, Wd.data_ptr(), K, gu.data_ptr(), h.data_ptr(), None)
        torch.cuda.synchronize()
        gu_ref = X @ Wgu.T
        gu_out = host(gu)
        assert np.all(np.abs(gu_out - gu_ref) <= 2.0 ** -8 * np.abs(gu_ref) + 1e-4 * np.sqrt(K))
        h_ref = om.swiglu(gu_out, f)
        assert np.abs(host(h) - h_ref).max() <= 1e-2 * max(1e-3, np.abs(h_ref).max())
    finally:
        L.call("bm_k_gemm_swiglu_bk128", 1)
