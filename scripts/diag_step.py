"""Diagnose the step: device time with/without GEMM event timing, host enqueue
time per step, and the GEMM share, on one GPU (C2, P=1 by default)."""
import json, os, sys, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import get_config, make_batch
from paper_2605_25451_b200.runtime import Runtime
from paper_2605_25451_b200 import _lib as L

M = int(os.environ.get("M", "16"))
cfg = get_config("C2", P=1, M=M, V=1)
rt = Runtime(cfg, "bf16")
rt.init_random_weights(1)
db = rt.device_batch(make_batch(cfg))
for _ in range(3):
    rt.step(db)
torch.cuda.synchronize()

def run(k, timing):
    rt.set_timing(timing)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    for _ in range(k):
        rt.step(db)
    host = (time.perf_counter() - t0) * 1e3 / k
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / k
    n, fl, ms = rt.gemm_stats()
    rt.set_timing(False)
    return dict(timing=timing, dev_ms=dev, host_enqueue_ms=host, gemm_n=n / k, gemm_ms=ms / k,
                gemm_tflops=(fl / (ms / 1e3) / 1e12) if ms else None, launches=rt.launch_count())

for mode in [0, 1]:
    L.call("bm_k_gemm_mode", mode if mode else 0)
    print(json.dumps({"gemm_mode": mode, **run(5, False)}))
    print(json.dumps({"gemm_mode": mode, **run(5, True)}))
