"""One launch each of the tcgen05 pair GEMM and cuBLAS (torch.matmul) per shape,
for an ncu capture that compares tensor-pipe, L2 and DRAM counters and shows
cuBLAS's kernel name (its tile / cluster configuration).

    ncu --metrics ... python scripts/ncu_gemm_vs_cublas.py [M N K [a_mn b_mn]] | c2
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402

C2 = [(4096, 16384, 2048, 0, 0), (4096, 2048, 8192, 0, 0), (4096, 8192, 2048, 0, 1), (16384, 2048, 4096, 1, 1),
      (4096, 2048, 16384, 0, 1), (2048, 8192, 4096, 1, 1), (8192, 8192, 8192, 0, 0)]


def one(M, N, K, amn, bmn, reps=2):
    A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    a2 = A.t() if amn else A
    b2 = B if bmn else B.t()
    for _ in range(reps):
        L.call("bm_k_gemm", 0, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(), N if bmn else K, bmn,
               C.data_ptr(), N, 0, 0, None, N, 1.0, None)
        torch.matmul(a2, b2)
    torch.cuda.synchronize()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "c2":
        for s in C2:
            one(*s)
    else:
        a = [int(x) for x in sys.argv[1:]] or [8192, 8192, 8192]
        one(*(a + [0, 0])[:5])
    print("done")


if __name__ == "__main__":
    main()
