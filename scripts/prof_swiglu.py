"""Run the fused SwiGLU GEMM epilogue variants a few times (for ncu)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_25451_b200 import _lib as L
S, d, f = 4096, 2048, 8192
X = torch.randn((S, d), device="cuda").to(torch.bfloat16)
Wgu = (torch.randn((2 * f, d), device="cuda") * 0.02).to(torch.bfloat16)
Wd = (torch.randn((d, f), device="cuda") * 0.02).to(torch.bfloat16)
gu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
h = torch.empty((S, f), device="cuda", dtype=torch.bfloat16)
dY = torch.randn((S, d), device="cuda").to(torch.bfloat16)
dgu = torch.empty((S, 2 * f), device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    L.call("bm_k_gemm_swiglu", S, f, d, X.data_ptr(), d, Wgu.data_ptr(), d, gu.data_ptr(), h.data_ptr(), None)
    L.call("bm_k_gemm_dswiglu", S, f, d, dY.data_ptr(), d, Wd.data_ptr(), f, gu.data_ptr(), dgu.data_ptr(), None)
    L.call("bm_k_gemm", 0, S, 2 * f, d, X.data_ptr(), d, 0, Wgu.data_ptr(), d, 0, gu.data_ptr(), 2 * f, 0, 0, None, 0, 1.0, None)
torch.cuda.synchronize()
print("ok")
