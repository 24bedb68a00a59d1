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
