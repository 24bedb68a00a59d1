"""How far can a bf16-storage step be from the fp64 oracle?  (reading R19)

    python scripts/precision_emulation.py [--S 256] [--L 2,4,16]

Runs the oracle's LLM layers (oracle.model primitives, fp64) on C2-width random
weights twice: exactly, and with the GPU path's bf16 rounding points emulated
(RNE to bf16 of the normalised input xn, the gate/up output gu, the SwiGLU output
h and the residual stream x after each layer -- reading R12's "bf16 storage, fp32
accumulation").  Prints the normwise relative error of the final-norm output Hn
per depth and per single rounding point.  Hn feeds the LM head and the generator,
so their gradients inherit this error; it is a property of bf16 storage in this
randomly initialised model, independent of any kernel.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth import bf16_round, get_config, make_weights, param_specs  # noqa: E402
from oracle import model as om  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=256)
    ap.add_argument("--L", default="2,4,16")
    a = ap.parse_args()
    out = []
    for L in [int(x) for x in a.L.split(",")]:
        cfg = get_config("C2", P=1, M=1).replace(S=a.S, L=L)
        names = [n for n, _, _ in param_specs(cfg) if n.startswith("llm.layer") or n == "llm.final_norm"]
        W = om.to_f64(make_weights(cfg, names=names))
        rng = np.random.default_rng(0)
        x0 = bf16_round((rng.standard_normal((cfg.S, cfg.d)) * 0.02).astype(np.float32)).astype(np.float64)

        def r(v):
            return bf16_round(v.astype(np.float32)).astype(np.float64)

        def fwd(points):
            x = x0.copy()
            for l in range(cfg.L):
                p = f"llm.layer{l}"
                xn, _ = om.rmsnorm(x, W[p + ".norm"])
                if "xn" in points:
                    xn = r(xn)
                gu = xn @ W[p + ".gate_up"].T
                if "gu" in points:
                    gu = r(gu)
                h = om.swiglu(gu, cfg.f)
                if "h" in points:
                    h = r(h)
                x = x + h @ W[p + ".down"].T
                if "x" in points:
                    x = r(x)
            return om.rmsnorm(x, W["llm.final_norm"])[0]
        ref = fwd(())
        row = {"L": L, "S": a.S, "d": cfg.d, "f": cfg.f}
        for pts in (("x",), ("xn",), ("gu",), ("h",), ("x", "xn", "gu", "h")):
            Hn = fwd(pts)
            row["+".join(pts)] = float(np.linalg.norm(Hn - ref) / np.linalg.norm(ref))
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
