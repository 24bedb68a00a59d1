"""One launch each of the tcgen05 pair GEMM and cuBLAS (torch.matmul) on a given
shape, for an ncu capture that compares tensor-pipe, L2 and DRAM counters (and
shows cuBLAS's kernel name, i.e. its tile / cluster configuration).

    ncu --metrics ... python scripts/ncu_gemm_vs_cublas.py [M N K]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402


def main():
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (8192, 8192, 8192)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    lib = L.lib()
    for _ in range(2):
        L.call("bm_k_gemm", 0, M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, C.data_ptr(), N, 0, 0, None, N, 1.0,
               None)
        torch.matmul(A, B.t())
    torch.cuda.synchronize()
    print("done", lib is not None)


if __name__ == "__main__":
    main()
