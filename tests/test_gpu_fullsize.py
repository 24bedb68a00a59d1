"""Full-size check at the bench's launch configuration (C2: ViT-S-shaped encoder,
1B-shaped LLM, S = 4096, M = 16, P = 1, bf16): the per-microbatch loss terms of
a sampled microbatch against the fp64 oracle forward of that microbatch, and
bitwise run-to-run determinism of every gradient (a property at any size).
The oracle forward of one C2 microbatch is ~7 TFLOP in numpy fp64 (about a
minute on the box's host cores)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from synth import get_config, make_batch, make_weights  # noqa: E402

pytestmark = pytest.mark.gpu


def test_c2_fullsize_sampled_parity():
    from oracle import model as om
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config("C2", P=1, M=16)
    W = make_weights(cfg)
    B = make_batch(cfg)
    rt = Runtime(cfg, "bf16")
    rt.load_weights(W)
    db = rt.device_batch(B)
    rt.step(db)
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    g1 = rt.grads_t.clone()
    rt.step(db)
    torch.cuda.synchronize()
    assert torch.equal(g1, rt.grads_t)          # deterministic at full size
    assert np.isfinite(loss)
    # sampled microbatch: oracle forward in fp64 (loss terms only)
    m = 0
    W64 = om.to_f64({k: v for k, v in W.items()})
    n_mod, n_gen = int(B.n_mod[m]), int(B.n_gen[m])
    E, _ = om.encoder_fwd(W64, cfg, np.asarray(B.patches[m], np.float64))
    X = om.embed_fwd(W64, B.ids[m], E, n_mod)
    H, _ = om.llm_layers_fwd(W64, cfg, list(range(cfg.L)), X)
    Hn, ce_ref, _ = om.head_fwd(W64, cfg, H, B.labels[m], n_mod)
    mse_ref, _ = om.gen_fwd(W64, cfg, Hn[cfg.S - n_gen:], np.asarray(B.targets[m], np.float64),
                            float(n_gen * cfg.d_t))
    assert abs(ce[m] - ce_ref) <= 2e-2 * abs(ce_ref), (ce[m], ce_ref)
    assert abs(mse[m] - mse_ref) <= 2e-2 * abs(mse_ref), (mse[m], mse_ref)
    rt.close()


# every LLM contraction of the bench step at BASELINE.json's full C2 / C4 sizes
# (forward, data-grad, weight-grad forms; M, N, K, A MN-major, B MN-major), checked
# on sampled output entries the oracle computes one by one (fp64 dot products)
FULL_GEMMS = [
    ("C2 gate_up fwd", 4096, 16384, 2048, 0, 0), ("C2 down fwd", 4096, 2048, 8192, 0, 0),
    ("C2 down dgrad", 4096, 8192, 2048, 0, 1), ("C2 gate_up dgrad", 4096, 2048, 16384, 0, 1),
    ("C2 down wgrad", 2048, 8192, 4096, 1, 1), ("C2 gate_up wgrad", 16384, 2048, 4096, 1, 1),
    ("C2 head fwd", 3500, 32000, 2048, 0, 0), ("C2 head dgrad", 3500, 2048, 32000, 0, 1),
    ("C2 head wgrad", 32000, 2048, 3500, 1, 1),
    ("C4 gate_up fwd", 8192, 22016, 4096, 0, 0), ("C4 down fwd", 8192, 4096, 11008, 0, 0),
    ("C4 gate_up wgrad", 22016, 4096, 8192, 1, 1),
]


@pytest.mark.parametrize("name,M,N,K,a_mn,b_mn", FULL_GEMMS, ids=[g[0] for g in FULL_GEMMS])
def test_fullsize_gemm_sampled(name, M, N, K, a_mn, b_mn):
    from paper_2605_25451_b200 import _lib as L
    g = torch.Generator(device="cuda")
    g.manual_seed(M + 3 * N + 7 * K)
    # logical A [M, K], B [N, K]; stored MN-major (transposed) when a_mn / b_mn
    A = torch.randn((M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((N, K), device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    As = A.t().contiguous() if a_mn else A
    Bs = B.t().contiguous() if b_mn else B
    C = torch.empty((M, N), device="cuda", dtype=torch.float32)
    L.call("bm_k_gemm", 0, M, N, K, As.data_ptr(), M if a_mn else K, a_mn, Bs.data_ptr(), N if b_mn else K, b_mn,
           C.data_ptr(), N, 1, 0, None, 0, 1.0, None)
    torch.cuda.synchronize()
    rng = np.random.default_rng(M + N + K)
    ii = rng.integers(0, M, 256)
    jj = rng.integers(0, N, 256)
    a = A[torch.as_tensor(ii, device="cuda")].double().cpu().numpy()
    b = B[torch.as_tensor(jj, device="cuda")].double().cpu().numpy()
    ref = np.einsum("sk,sk->s", a, b)
    got = C[torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda")].double().cpu().numpy()
    scale = np.sqrt(K) * np.abs(a).max() * np.abs(b).max()
    assert np.abs(got - ref).max() <= 1e-5 * scale, (name, np.abs(got - ref).max(), scale)


@pytest.mark.parametrize("S,d,f", [(4096, 2048, 8192), (8192, 4096, 11008)], ids=["C2", "C4"])
def test_fullsize_gate_up_swiglu_sampled(S, d, f):
    """The fused gate/up GEMM + SwiGLU epilogue the step runs, at full C2 / C4 size:
    sampled gu = [g | u] and h = silu(g) u against fp64 (bf16 outputs: 2^-7 relative)."""
    from paper_2605_25451_b200 import _lib as L
    g_ = torch.Generator(device="cuda")
    g_.manual_seed(S + d + f)
    X = torch.randn((S, d), device="cuda", generator=g_).to(torch.bfloat16)
    W = (torch.randn((2 * f, d), device="cuda", generator=g_) * 0.02).to(torch.bfloat16)
    gu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
    h = torch.empty((S, f), device="cuda", dtype=torch.bfloat16)
    L.call("bm_k_gemm_swiglu", S, f, d, X.data_ptr(), d, W.data_ptr(), d, gu.data_ptr(), h.data_ptr(), None)
    torch.cuda.synchronize()
    rng = np.random.default_rng(S + f)
    ii = rng.integers(0, S, 256)
    jj = rng.integers(0, f, 256)
    x = X[torch.as_tensor(ii, device="cuda")].double().cpu().numpy()
    wg = W[torch.as_tensor(jj, device="cuda")].double().cpu().numpy()
    wu = W[torch.as_tensor(jj + f, device="cuda")].double().cpu().numpy()
    g = np.einsum("sk,sk->s", x, wg)
    u = np.einsum("sk,sk->s", x, wu)
    hr = g / (1.0 + np.exp(-g)) * u
    ti, tj = torch.as_tensor(ii, device="cuda"), torch.as_tensor(jj, device="cuda")
    got_g = gu[ti, tj].double().cpu().numpy()
    got_u = gu[ti, tj + f].double().cpu().numpy()
    got_h = h[ti, tj].double().cpu().numpy()
    for got, ref in ((got_g, g), (got_u, u), (got_h, hr)):
        assert np.all(np.abs(got - ref) <= 2.0 ** -7 * np.abs(ref) + 1e-3 * np.abs(ref).max())
