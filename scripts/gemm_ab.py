"""A/B of two builds of libbigmac.so on the same GPU: bm_k_gemm / bm_k_gemm_dswiglu
on the C2 LLM shapes, CUDA events, L2 flushed between iterations.

    python scripts/gemm_ab.py LIB_A LIB_B [LIB ...]
"""
import ctypes as C
import json
import sys

import torch

SHAPES = [("C2 gate_up fwd", 4096, 16384, 2048, 0, 0, 0), ("C2 down fwd+res", 4096, 2048, 8192, 0, 0, 2),
          ("C2 down dgrad", 4096, 8192, 2048, 0, 1, 0), ("C2 gate_up wgrad", 16384, 2048, 4096, 1, 1, 1),
          ("C2 gate_up dgrad", 4096, 2048, 16384, 0, 1, 0), ("C2 down wgrad", 2048, 8192, 4096, 1, 1, 1),
          ("8192^3", 8192, 8192, 8192, 0, 0, 0)]


def bench(fn, flush, iters=10):
    for _ in range(3):
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
    ts.sort()
    return ts[len(ts) // 2]


def main():
    libs = sys.argv[1:]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    Ls = []
    for p in libs:
        L = C.CDLL(p, mode=C.RTLD_LOCAL)
        L.bm_k_gemm.argtypes = [C.c_int32] * 4 + [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64, C.c_int32,
                                                  C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                                  C.c_float, C.c_void_p]
        L.bm_k_gemm_dswiglu.argtypes = [C.c_int32] * 3 + [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p,
                                                          C.c_void_p, C.c_void_p]
        Ls.append(L)
    for name, M, N, K, amn, bmn, epi in SHAPES:
        A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
        B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
        cdt = 1 if epi == 1 else 0
        Cm = torch.zeros((M, N), device="cuda", dtype=torch.float32 if cdt else torch.bfloat16)
        R = torch.zeros((M, N), device="cuda", dtype=torch.bfloat16) if epi == 2 else None
        row = {"name": name}
        for p, L in zip(libs, Ls):
            def fn():
                r = L.bm_k_gemm(0, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(), N if bmn else K, bmn,
                                Cm.data_ptr(), N, cdt, epi, R.data_ptr() if R is not None else None, N, 1.0, None)
                assert r == 0
            t = bench(fn, flush)
            row[p] = round(2.0 * M * N * K / t / 1e9, 1)
        print(json.dumps(row), flush=True)
    S, d, f = 4096, 2048, 8192
    dY = torch.randn((S, d), device="cuda").to(torch.bfloat16)
    Wd = (torch.randn((d, f), device="cuda") * 0.02).to(torch.bfloat16)
    gu = torch.randn((S, 2 * f), device="cuda").to(torch.bfloat16)
    dgu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
    row = {"name": "C2 down dgrad + dswiglu"}
    for p, L in zip(libs, Ls):
        def fn():
            assert L.bm_k_gemm_dswiglu(S, f, d, dY.data_ptr(), d, Wd.data_ptr(), f, gu.data_ptr(), dgu.data_ptr(), None) == 0
        t = bench(fn, flush)
        row[p] = round(2.0 * S * f * d / t / 1e9, 1)
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
