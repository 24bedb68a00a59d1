"""Time the tcgen05 GEMM on the model's shapes (CUDA events, warm, L2-flushed
between iterations) next to cuBLAS (torch.matmul) for context.

    python scripts/gemm_bench.py [--json out.json]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402

PEAK = 1664.4  # MEASURED_PEAKS bf16_tflops (burst)


def bench(fn, iters=10, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    shapes = [
        # name, M, N, K, a_mn, b_mn, epi
        ("C2 gate_up fwd", 4096, 16384, 2048, 0, 0, "store"),
        ("C2 down fwd+res", 4096, 2048, 8192, 0, 0, "add"),
        ("C2 down dgrad", 4096, 8192, 2048, 0, 1, "store"),
        ("C2 gate_up wgrad", 16384, 2048, 4096, 1, 1, "accum"),
        ("C2 gate_up dgrad", 4096, 2048, 16384, 0, 1, "store"),
        ("C2 down wgrad", 2048, 8192, 4096, 1, 1, "accum"),
        ("C2 head fwd", 3500, 32000, 2048, 0, 0, "store"),
        ("8192^3", 8192, 8192, 8192, 0, 0, "store"),
        ("C4 gate_up fwd", 8192, 22016, 4096, 0, 0, "store"),
        ("C4 down fwd+res", 8192, 4096, 11008, 0, 0, "add"),
        ("C4 down dgrad", 8192, 11008, 4096, 0, 1, "store"),
        ("C4 gate_up wgrad", 22016, 4096, 8192, 1, 1, "accum"),
        ("C4 gate_up dgrad", 8192, 4096, 22016, 0, 1, "store"),
        ("C4 down wgrad", 4096, 11008, 8192, 1, 1, "accum"),
        ("C2 head dgrad", 3500, 2048, 32000, 0, 1, "store"),
        ("C2 head wgrad", 32000, 2048, 3500, 1, 1, "accum"),
        ("enc fc1 n=554", 554, 1536, 384, 0, 0, "store"),
    ]
    out = []
    for name, M, N, K, amn, bmn, epi in shapes:
        A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
        lda = M if amn else K
        ldb = N if bmn else K
        if epi == "accum":
            C = torch.zeros((M, N), device="cuda", dtype=torch.float32)
            cdt, e, R = 1, 1, None
        else:
            C = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16)
            cdt, e = 0, (2 if epi == "add" else 0)
            R = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16) if epi == "add" else None

        def ours():
            L.call("bm_k_gemm", 0, M, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn, C.data_ptr(), N, cdt, e,
                   R.data_ptr() if R is not None else None, N, 1.0, None)

        a2 = A.t() if amn else A
        b2 = B if bmn else B.t()

        def cublas():
            torch.matmul(a2, b2)

        t = bench(ours, flush=flush)
        tc = bench(cublas, flush=flush)
        fl = 2.0 * M * N * K
        row = dict(name=name, M=M, N=N, K=K, ms=t, tflops=fl / t / 1e9, frac=fl / t / 1e9 / PEAK,
                   cublas_ms=tc, cublas_tflops=fl / tc / 1e9)
        print(json.dumps(row))
        out.append(row)
    # fused SwiGLU epilogues vs GEMM + separate elementwise kernel (C2 LLM layer)
    S, d, f = 4096, 2048, 8192
    X = torch.randn((S, d), device="cuda").to(torch.bfloat16)
    Wgu = (torch.randn((2 * f, d), device="cuda") * 0.02).to(torch.bfloat16)
    Wd = (torch.randn((d, f), device="cuda") * 0.02).to(torch.bfloat16)
    gu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
    h = torch.empty((S, f), device="cuda", dtype=torch.bfloat16)
    dY = torch.randn((S, d), device="cuda").to(torch.bfloat16)
    dh = torch.empty((S, f), device="cuda", dtype=torch.bfloat16)
    dgu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)

    def fused_fwd():
        L.call("bm_k_gemm_swiglu", S, f, d, X.data_ptr(), d, Wgu.data_ptr(), d, gu.data_ptr(), h.data_ptr(), None)

    def unfused_fwd():
        L.call("bm_k_gemm", 0, S, 2 * f, d, X.data_ptr(), d, 0, Wgu.data_ptr(), d, 0, gu.data_ptr(), 2 * f, 0, 0, None, 0, 1.0, None)
        L.call("bm_k_swiglu_fwd", 0, S, f, gu.data_ptr(), h.data_ptr(), None)

    def fused_bwd():
        L.call("bm_k_gemm_dswiglu", S, f, d, dY.data_ptr(), d, Wd.data_ptr(), f, gu.data_ptr(), dgu.data_ptr(), None)

    def unfused_bwd():
        L.call("bm_k_gemm", 0, S, f, d, dY.data_ptr(), d, 0, Wd.data_ptr(), f, 1, dh.data_ptr(), f, 0, 0, None, 0, 1.0, None)
        L.call("bm_k_swiglu_bwd", 0, S, f, dh.data_ptr(), gu.data_ptr(), dgu.data_ptr(), None)

    # a Linear's backward: weight + data gradient in one grouped launch vs two launches
    dW_gu = torch.zeros((2 * f, d), device="cuda", dtype=torch.float32)
    dW_d = torch.zeros((d, f), device="cuda", dtype=torch.float32)
    dxn = torch.empty((S, d), device="cuda", dtype=torch.bfloat16)
    hh = torch.randn((S, f), device="cuda").to(torch.bfloat16)
    D = L.GemmDesc
    down_w = D(d, f, S, dY.data_ptr(), d, 1, hh.data_ptr(), f, 1, dW_d.data_ptr(), f, 1, 1, None, 0, 1.0, 0)
    down_dg = D(S, f, d, dY.data_ptr(), d, 0, Wd.data_ptr(), f, 1, dgu.data_ptr(), 2 * f, 0, 4, gu.data_ptr(), 2 * f, 1.0, f)
    gu_dg = D(S, d, 2 * f, dgu.data_ptr(), 2 * f, 0, Wgu.data_ptr(), d, 1, dxn.data_ptr(), d, 0, 0, None, 0, 1.0, 0)
    gu_w = D(2 * f, d, S, dgu.data_ptr(), 2 * f, 1, X.data_ptr(), d, 1, dW_gu.data_ptr(), d, 1, 1, None, 0, 1.0, 0)
    down_pair = (D * 2)(down_w, down_dg)
    gu_pair = (D * 2)(gu_dg, gu_w)

    def down_grouped():
        L.call("bm_k_gemm_group", down_pair, 2, None)

    def down_separate():
        L.call("bm_k_gemm_group", down_pair, 1, None)
        L.call("bm_k_gemm_group", ctypes.byref(down_dg), 1, None)

    def gu_grouped():
        L.call("bm_k_gemm_group", gu_pair, 2, None)

    def gu_separate():
        L.call("bm_k_gemm_group", gu_pair, 1, None)
        L.call("bm_k_gemm_group", ctypes.byref(gu_w), 1, None)

    for name, fn, fl in [("down bwd grouped (wgrad + dgrad/dswiglu)", down_grouped, 4.0 * S * f * d),
                         ("down bwd separate", down_separate, 4.0 * S * f * d),
                         ("gate_up bwd grouped (dgrad + wgrad)", gu_grouped, 8.0 * S * f * d),
                         ("gate_up bwd separate", gu_separate, 8.0 * S * f * d),
                         ("gate_up+swiglu fused", fused_fwd, 2.0 * S * 2 * f * d),
                         ("gate_up + swiglu kernel", unfused_fwd, 2.0 * S * 2 * f * d),
                         ("down dgrad+dswiglu fused", fused_bwd, 2.0 * S * f * d),
                         ("down dgrad + swiglu_bwd kernel", unfused_bwd, 2.0 * S * f * d)]:
        t = bench(fn, flush=flush)
        row = dict(name=name, ms=t, tflops=fl / t / 1e9)
        print(json.dumps(row))
        out.append(row)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
