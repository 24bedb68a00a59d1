"""Per-tensor normwise gradient errors of one full-size microbatch vs the fp64 oracle.

    python scripts/fullsize_errors.py [--config C2] [--dtype bf16|f32] [--L 16]

Prints one JSON line: loss / CE / MSE relative errors and every parameter's
||g - g_ref|| / ||g_ref|| (diagnostic for the full-size parity test)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--L", type=int, default=0)
    a = ap.parse_args()
    from synth import get_config, make_batch, make_weights
    from oracle import model as om
    from paper_2605_25451_b200.runtime import Runtime
    cfg = get_config(a.config, P=1, M=1)
    if a.L:
        cfg = cfg.replace(L=a.L)
    W, B = make_weights(cfg), make_batch(cfg)
    rt = Runtime(cfg, a.dtype)
    rt.load_weights(W)
    rt.step(rt.device_batch(B))
    torch.cuda.synchronize()
    loss, ce, mse = rt.losses()
    grads = {n: rt.grad(n) for n in rt.names()}
    rt.close()
    loss_ref, per_ref, G_ref = om.step_fp64(cfg, W, B)
    rel = lambda x, y: float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30))  # noqa: E731
    errs = {n: rel(g, G_ref[n]) for n, g in grads.items()}
    print(json.dumps({"config": a.config, "dtype": a.dtype, "L": cfg.L, "loss": rel(np.array(loss), np.array(loss_ref)),
                      "ce": rel(np.array(ce[0]), np.array(per_ref[0][0])),
                      "mse": rel(np.array(mse[0]), np.array(per_ref[0][1])),
                      "max": max(errs.values()), "grads": errs}), flush=True)


if __name__ == "__main__":
    main()
