"""Two launches of the C2 down-dgrad + SwiGLU-backward GEMM for an ncu source-level capture."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L  # noqa: E402

S, d, f = 4096, 2048, 8192
dY = torch.randn((S, d), device="cuda").to(torch.bfloat16)
Wd = (torch.randn((d, f), device="cuda") * 0.02).to(torch.bfloat16)
gu = torch.randn((S, 2 * f), device="cuda").to(torch.bfloat16)
dgu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    L.call("bm_k_gemm_dswiglu", S, f, d, dY.data_ptr(), d, Wd.data_ptr(), f, gu.data_ptr(), dgu.data_ptr(), None)
torch.cuda.synchronize()
print("ok")
