"""Run one bf16 GEMM shape a few times through bm_k_gemm (target for ncu).

    python scripts/prof_gemm_shape.py M N K [a_mn b_mn] [--iters 3]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 3
    M, N, K = int(args[0]), int(args[1]), int(args[2])
    amn, bmn = (int(args[3]), int(args[4])) if len(args) > 4 else (0, 0)
    A = torch.randn((K, M) if amn else (M, K), device="cuda").to(torch.bfloat16)
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").to(torch.bfloat16)
    C = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for _ in range(iters):
        L.call("bm_k_gemm", 0, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(), N if bmn else K, bmn,
               C.data_ptr(), N, 0, 0, None, 0, 1.0, None)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
