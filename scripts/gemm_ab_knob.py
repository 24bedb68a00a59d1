"""A/B of a GEMM knob on the C2 / C4 LLM and head contractions, settings interleaved
over several rounds in one process (CUDA events, L2 flushed between iterations);
prints per shape the median TF/s over rounds of each setting.

    python scripts/gemm_ab_knob.py [rounds] [knob]
knob: bn512 (bm_k_gemm_bn512 0 = 256x256 vs 1 = 256x512; default), bk128 or
swiglu_bk128 (0 vs 1, with the production bn512 auto policy)
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402

SHAPES = [  # name, M, N, K, a_mn, b_mn, epi (0 store bf16, 1 accum f32, 2 add bf16, 3 dswiglu, 4 swiglu)
    ("C2 gate_up fwd+swiglu", 4096, 8192, 2048, 0, 0, 4), ("C4 gate_up fwd+swiglu", 8192, 11008, 4096, 0, 0, 4),
    ("C2 down fwd+res", 4096, 2048, 8192, 0, 0, 2), ("C2 down dgrad+dswiglu", 4096, 8192, 2048, 0, 1, 3),
    ("C2 gate_up wgrad", 16384, 2048, 4096, 1, 1, 1), ("C2 gate_up dgrad", 4096, 2048, 16384, 0, 1, 0),
    ("C2 down wgrad", 2048, 8192, 4096, 1, 1, 1), ("C2 head dgrad", 3500, 2048, 32000, 0, 1, 0),
    ("C2 head wgrad", 32000, 2048, 3500, 1, 1, 1), ("C2 head fwd", 3500, 32000, 2048, 0, 0, 0),
    ("C4 down fwd+res", 8192, 4096, 11008, 0, 0, 2), ("C4 down dgrad+dswiglu", 8192, 11008, 4096, 0, 1, 3),
    ("C4 gate_up wgrad", 22016, 4096, 8192, 1, 1, 1), ("C4 gate_up dgrad", 8192, 4096, 22016, 0, 1, 0),
    ("C4 down wgrad", 4096, 11008, 8192, 1, 1, 1), ("C4 head dgrad", 7000, 4096, 32000, 0, 1, 0),
    ("C4 head wgrad", 32000, 4096, 7000, 1, 1, 1), ("8192^3", 8192, 8192, 8192, 0, 0, 0)]


def bench(fn, flush, iters=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    knob = sys.argv[2] if len(sys.argv) > 2 else "bn512"
    fn_knob = {"bn512": "bm_k_gemm_bn512", "bk128": "bm_k_gemm_bk128",
               "swiglu_bk128": "bm_k_gemm_swiglu_bk128"}[knob]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    L.call("bm_k_gemm_mode", 2)
    if knob in ("bk128", "swiglu_bk128"):
        L.call("bm_k_gemm_bn512", 2)
    for name, M, N, K, amn, bmn, epi in SHAPES:
        A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
        if epi == 4:
            Wg = torch.randn((2 * N, K), device="cuda").to(torch.bfloat16)
            gu2 = torch.empty((M, 2 * N), device="cuda", dtype=torch.bfloat16)
            hh = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)

            def fn():
                L.call("bm_k_gemm_swiglu", M, N, K, A.data_ptr(), K, Wg.data_ptr(), K, gu2.data_ptr(), hh.data_ptr(),
                       None)
        elif epi == 3:
            gu = torch.randn((M, 2 * N), device="cuda").to(torch.bfloat16)
            out = torch.empty((M, 2 * N), device="cuda", dtype=torch.bfloat16)

            def fn():
                L.call("bm_k_gemm_dswiglu", M, N, K, A.data_ptr(), K, B.data_ptr(), N, gu.data_ptr(), out.data_ptr(),
                       None)
        else:
            cdt = 1 if epi == 1 else 0
            Cm = torch.zeros((M, N), device="cuda", dtype=torch.float32 if cdt else torch.bfloat16)
            R = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16) if epi == 2 else None

            def fn():
                L.call("bm_k_gemm", 0, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(), N if bmn else K, bmn,
                       Cm.data_ptr(), N, cdt, epi, R.data_ptr() if R is not None else None, N, 1.0, None)
        res = {0: [], 1: []}
        for _ in range(rounds):
            for v in (0, 1):
                L.call(fn_knob, v)
                res[v].append(2.0 * M * N * K * (2 if epi == 4 else 1) / bench(fn, flush) / 1e9)
        row = {"name": name, "M": M, "N": N, "K": K, "knob": knob, "tf_0": round(statistics.median(res[0]), 1),
               "tf_1": round(statistics.median(res[1]), 1)}
        row["gain"] = round(row["tf_1"] / row["tf_0"] - 1, 4)
        print(json.dumps(row), flush=True)
    L.call("bm_k_gemm_bn512", 2)
    L.call("bm_k_gemm_bk128", 1)
    L.call("bm_k_gemm_swiglu_bk128", 1)
    L.call("bm_k_gemm_mode", 0)


if __name__ == "__main__":
    main()
