"""HBM-bound kernels of the step at C2 LLM shapes (SURVEY §8(d) "Kernel evidence"):
achieved GB/s = ALGORITHMIC bytes (each input read once, each output written
once) / device time (CUDA events, warm, L2 flushed by a 256 MB write between
iterations), against the measured HBM copy bandwidth (MEASURED_PEAKS.json).

    python scripts/prof_elementwise.py [--json out.jsonl]
(also the target of the ncu --set full capture in scripts/profile_step_v3.sh)
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_25451_b200 import _lib as L  # noqa: E402

S, d, f, V, n_text, n_mod = 4096, 2048, 8192, 32000, 3500, 554
n_enc = 554 * 1536   # encoder GELU elements (mean modality rows x f_e)


def peak_hbm():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps"):
            if k in p:
                return float(p[k]), "measured " + k
    except Exception:
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def timeit(fn, flush, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warm", type=int, default=3, help="0 and --iters 1 under ncu: one launch per kernel")
    args = ap.parse_args()
    dev = "cuda"
    bf = torch.bfloat16
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    x = torch.randn((S, d), device=dev).to(bf)
    g = torch.ones(d, device=dev).to(bf)
    y = torch.empty_like(x)
    dres = torch.randn_like(x)
    dx = torch.empty_like(x)
    rstd = torch.empty(S, device=dev)
    dg = torch.zeros(d, device=dev)
    part = torch.empty(int(L.lib().bm_k_rmsnorm_bwd_scratch(S, d)), device=dev)
    gu = torch.randn((S, 2 * f), device=dev).to(bf)
    h = torch.empty((S, f), device=dev, dtype=bf)
    dgu = torch.empty_like(gu)
    logits0 = torch.randn((n_text, V), device=dev).to(bf)
    logits = logits0.clone()
    labels = torch.randint(0, V, (n_text,), device=dev, dtype=torch.int32)
    loss = torch.zeros(1, device=dev)
    ce_scr = torch.empty(n_text, device=dev)
    a = torch.randn(n_enc, device=dev).to(bf)
    z = torch.empty_like(a)
    da = torch.empty_like(a)
    table = torch.randn((V, d), device=dev).to(bf)
    ids = torch.randint(0, V, (S,), device=dev, dtype=torch.int32)
    emb = torch.randn((n_mod, d), device=dev).to(bf)
    X = torch.empty((S, d), device=dev, dtype=bf)
    dT = torch.zeros((V, d), device=dev)
    escr = torch.empty(int(L.lib().bm_k_embed_bwd_scratch(S)), dtype=torch.uint8, device=dev)
    P = lambda t: t.data_ptr()  # noqa: E731
    cases = [
        ("rmsnorm_fwd [4096 x 2048]", 2 * S * d * 2 + S * 4,
         lambda: L.call("bm_k_rmsnorm_fwd", 0, S, d, P(x), P(g), P(y), P(rstd), None)),
        ("rmsnorm_bwd fused +dres [4096 x 2048]", 4 * S * d * 2 + S * 4,
         lambda: L.call("bm_k_rmsnorm_bwd", 0, S, d, P(y), P(x), P(g), P(rstd), P(dres), P(dx), P(dg), P(part), None)),
        ("swiglu_fwd [4096 x 8192]", 3 * S * f * 2,
         lambda: L.call("bm_k_swiglu_fwd", 0, S, f, P(gu), P(h), None)),
        ("swiglu_bwd [4096 x 8192]", 5 * S * f * 2,
         lambda: L.call("bm_k_swiglu_bwd", 0, S, f, P(h), P(gu), P(dgu), None)),
        ("ce_fwd_bwd [3500 x 32000]", 2 * n_text * V * 2 + n_text * 4,
         lambda: L.call("bm_k_ce_fwd_bwd", 0, n_text, V, P(logits), P(labels), 1e-4, P(loss), 1.0, 0, P(ce_scr), None)),
        ("gelu_fwd [554 x 1536]", 2 * n_enc * 2, lambda: L.call("bm_k_gelu_fwd", 0, n_enc, P(a), P(z), None)),
        ("gelu_bwd [554 x 1536]", 3 * n_enc * 2, lambda: L.call("bm_k_gelu_bwd", 0, n_enc, P(z), P(a), P(da), None)),
        ("embed_fwd [4096 x 2048], 554 modality rows", 2 * S * d * 2 + S * 4,
         lambda: L.call("bm_k_embed_fwd", 0, S, d, n_mod, P(ids), P(table), P(emb), P(X), None)),
        ("embed_bwd [4096 x 2048] -> fp32 table grad", (S - n_mod) * d * (2 + 8) + S * 4,
         lambda: L.call("bm_k_embed_bwd", 0, S, d, n_mod, P(ids), P(X), P(dT), P(escr), None)),
    ]
    peak, src = peak_hbm()
    out = []
    for name, nbytes, fn in cases:
        ms = timeit(fn, flush, args.iters, args.warm)
        gbs = nbytes / (ms * 1e-3) / 1e9
        rec = {"kernel": name, "algorithmic_bytes": nbytes, "ms": ms, "GBps": gbs, "peak_GBps": peak,
               "peak_source": src, "frac": gbs / peak}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    if args.json:
        with open(args.json, "w") as fh:
            for r in out:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
