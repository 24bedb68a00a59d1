#!/usr/bin/env python
"""Benchmark of one BigMac nested-pipeline training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...)

Workload (BASELINE.json configs[1], "C2"): ViT-S-shaped encoder + 1B-shaped
LLM + small generator, S = 4096, 1F1B LLM schedule with the encoder/generator
nested in it, P = N pipeline stages (one per GPU), synthetic data with
log-uniform[256, 1024] modality / generation rows per sample, bf16.
P = min(N, 4) pipeline stages and D = N / P pipeline replicas (SURVEY §8(d)
GPU ladder: "at G = 8, P = 4 x DP = 2"; replicas all-reduce their LLM stage
gradients, every process the DP modules').  16 microbatches per GPU: each
replica runs M = 16 P, global batch 16 N (one sample per microbatch), so every
GPU processes 16 microbatches x L/P layers per step at any N ("weak" scaling;
the 1F1B bubble (P-1)/(M+P-1) stays <= 4.5 %).  --stages P overrides P;
--microbatches M fixes the per-replica M instead ("strong").

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os

# one hardware work queue per stream (compute, generator, P-1 comm, NCCL)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLLM train samples/s + % step roofline at 1/2/4/8 B200; peak HBM vs batch size"
UNIT = "samples/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, "fallback"


def step_flops(cfg, n_mod, n_gen):
    """Algorithmic FLOPs of one step: 2 per MAC forward, 4 per
    MAC backward (dgrad + wgrad); the patch embedding has no dgrad."""
    S, d, f, L, V = cfg.S, cfg.d, cfg.f, cfg.L, cfg.vocab
    tot = 0.0
    for nm, ng in zip(n_mod, n_gen):
        llm = 6.0 * S * 3 * d * f * L
        head = 6.0 * (S - nm) * d * V
        enc = nm * (4.0 * cfg.d_in * cfg.d_e + 6.0 * (cfg.L_e * 2 * cfg.d_e * cfg.f_e + cfg.d_e * d + d * d))
        gen = 6.0 * ng * (d * cfg.d_g + cfg.L_g * 2 * cfg.d_g * cfg.f_g + cfg.d_g * cfg.d_t)
        tot += llm + head + enc + gen
    return tot


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""
    Q = ("uuid,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, uuid):
        self.uuid = uuid
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            if self.uuid and self.uuid not in parts[0]:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def stages_of(args, N):
    P = args.stages or min(N, 4)
    if N % P:
        raise SystemExit(f"--gpus {N} is not a multiple of --stages {P}")
    return P


def workload(args, N):
    """(per-replica config, P, D)."""
    from synth import get_config
    P = stages_of(args, N)
    base = get_config(args.config)
    cfg = get_config(args.config, P=P, M=args.microbatches or base.M * P, V=base.V)
    if getattr(args, "llm_sched", "auto") == "zb_h1":
        if cfg.V != 1:
            raise SystemExit("--llm-sched zb_h1 needs a V = 1 config")
        cfg = cfg.replace(llm_sched="zb_h1")
    return cfg, P, N // P


def bubble_bound(cfg, P):
    """Closed-form LLM bubble: 1F1B / interleaved (P-1)/(MV+P-1); ZB-H1 with
    F:B:W = 1:1:1 (P-1)/(3M+P-1) (reading R23)."""
    if cfg.llm_sched == "zb_h1":
        return (P - 1) / (3 * cfg.M + P - 1)
    return (P - 1) / (cfg.M * cfg.V + P - 1)


# LM head + CE of one microbatch on the last stage, in LLM-layer (fwd+bwd) equivalents,
# measured at C2 (profiles/r01/traces/trace_n2_m32_last_stage.summary.json: the last
# stage's F(m) takes 4.27 ms vs 2.55 ms elsewhere for 8 layers whose F+B is 8.2 ms)
HEAD_LAYERS = 1.7
# encoder + generator of one C2 microbatch on the stage that runs them, in the same units
# (N = 2 trace: ≈ 0.7 ms per microbatch next to ≈ 1.07 ms per layer fwd + bwd)
ENC_GEN_LAYERS = 0.6


# explicit partitions measured best at C2 (L = 16): stage 0 also runs the text
# embedding and is slowed by the generator shards it serves, so the extra layer
# goes to a middle stage (profiles/r01/traces/trace_n4_m64_bigmac.summary.json)
DEFAULT_SPLIT = {("C2", 4): [4, 4, 5, 3]}


def unit_partition(cfg, P):
    """Partition of the 2L half-layer units (bigmac.h stage_halves, R24) over
    the P V virtual stages minimising the slowest stage, then the sum of squared stage
    costs: unit costs A_l = 2, B_l = 1 (thirds of a layer: gate_up is 2/3 of its FLOPs),
    the last stage also runs the LM head + CE (HEAD_LAYERS layers)."""
    PV, n = P * cfg.V, 2 * cfg.L
    pre = [0]
    for u in range(n):
        pre.append(pre[-1] + (2 if u % 2 == 0 else 1))
    head = 3 * HEAD_LAYERS
    best = {0: (0.0, 0.0, [])}          # units covered -> (max, sum of squares, parts)
    for s in range(PV):
        nxt = {}
        for u0, (mx, sq, parts) in best.items():
            hi = n if s == PV - 1 else n - (PV - s - 1)
            for u1 in range(u0 + 1, hi + 1):
                if s == PV - 1 and u1 != n:
                    continue
                c = pre[u1] - pre[u0] + (head if s == PV - 1 else 0)
                key = (max(mx, c), sq + c * c)
                if u1 not in nxt or key < nxt[u1][:2]:
                    nxt[u1] = (key[0], key[1], parts + [u1 - u0])
        best = nxt
    return best[n][2]


def unit_costs(cfg, units):
    """Per-stage cost (layer equivalents) of a half-layer-unit partition, head included."""
    out, u = [], 0
    for s, k in enumerate(units):
        c = sum(2 if x % 2 == 0 else 1 for x in range(u, u + k)) / 3.0
        out.append(c + (HEAD_LAYERS if s == len(units) - 1 else 0.0))
        u += k
    return out


def stage_split(args, cfg, P):
    """Explicit stage_layers (bigmac.h) or None; in half-layer units with --partition halves."""
    if getattr(args, "partition", "layers") == "halves" and P * cfg.V > 1:
        if args.stage_layers:
            return [int(x) for x in args.stage_layers.split(",")]
        return unit_partition(cfg, P)
    if args.stage_layers:
        return [int(x) for x in args.stage_layers.split(",")]
    if args.last_stage_layers >= 0:
        return None
    return DEFAULT_SPLIT.get((cfg.name, P * cfg.V))


def last_stage_layers(args, cfg, P):
    """Uneven LLM partition (bigmac.h last_stage_layers): the n minimising the
    slowest stage max(ceil((L - n) / (P V - 1)), n + HEAD_LAYERS); ties -> larger n."""
    if args.last_stage_layers >= 0:
        return args.last_stage_layers
    PV = P * cfg.V
    if PV == 1:
        return 0
    best = None
    for n in range(1, cfg.L - (PV - 1) + 1):
        cost = max(-(-(cfg.L - n) // (PV - 1)), n + HEAD_LAYERS)
        if best is None or cost <= best[0]:
            best = (cost, n)
    uniform = cfg.L // PV + HEAD_LAYERS if cfg.L % PV == 0 else float("inf")
    return 0 if uniform <= best[0] else best[1]


def global_batch(cfg, D):
    """One global batch of M D microbatches; replica k runs [kM, (k+1)M)."""
    from synth import make_batch
    return make_batch(cfg, M=cfg.M * D)


SHAPES = {"C2": ("ViT-S", "1B", "small"), "C3": ("ViT-S", "1B", "small"), "C4": ("ViT-L", "7B", "diffusion-head")}


def config_dict(cfg, P, D):
    rep_txt = f" x {D} pipeline replicas" if D > 1 else ""
    enc, llm, gen = SHAPES.get(cfg.name, ("synthetic", "synthetic", "synthetic"))
    sched = ("ZB-H1 zero-bubble (B/W split)" if cfg.llm_sched == "zb_h1" else
             "1F1B" if cfg.V == 1 else f"interleaved 1F1B ({cfg.V} chunks/stage)")
    return {"workload": f"{cfg.name}: {enc}-shaped encoder (d_e={cfg.d_e}, L_e={cfg.L_e}) + {llm}-shaped LLM "
                        f"(d={cfg.d}, f={cfg.f}, L={cfg.L}, vocab={cfg.vocab}) + {gen}-shaped generator (d_g={cfg.d_g}, "
                        f"L_g={cfg.L_g}); nested pipeline P={P} stages{rep_txt}, M={cfg.M} microbatches per replica, "
                        f"{sched}",
            "global_batch": cfg.M * D, "seq_len": cfg.S, "parallelism": f"pp{P}" + (f"xdp{D}" if D > 1 else ""),
            "stages": P, "replicas": D, "microbatches": cfg.M, "vchunks": cfg.V,
            "n_mod_law": list(cfg.n_mod_law), "n_gen_law": list(cfg.n_gen_law),
            "l2_policy": "working set (weights + activations, GBs) >> 126 MB L2; no flush",
            "strategy": getattr(cfg, "_strategy", "bigmac")}


def head_place_name(args, N):
    if args.head != "auto":
        return args.head
    return "last_stage"


def run_reference(args):
    """The oracle as it stands, on the host cores (the reference arm for this tier):
    each step one bounded sample (oracle_microbatch_sample) of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    N = args.gpus
    if rank != 0:
        return
    cfg, P, D = workload(args, N)
    batch = global_batch(cfg, D)
    F = step_flops(cfg, batch.n_mod, batch.n_gen)
    from synth import get_config
    for _ in range(args.warmup):   # untimed: warms the interpreter / BLAS on a small case
        oracle_microbatch_sample(get_config("C1"), 1, 1)
    ts = []
    for _ in range(args.steps):
        dt, fl, cores = oracle_microbatch_sample(cfg, args.ref_layers, args.ref_seq_div)
        ts.append((dt, fl))
    sec = sum(t for t, _ in ts)
    flops = sum(f for _, f in ts)
    value = flops / sec / (F / (cfg.M * D))
    sample = (f"per step: oracle (numpy fp64 step_fp64) fwd+bwd of one {cfg.name} microbatch with "
              f"{args.ref_layers} of {cfg.L} LLM layers and S/{args.ref_seq_div} positions; samples/s scaled by the step's "
              f"algorithmic FLOPs per sample")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * sec / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.microbatches else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic", "config": config_dict(cfg, P, D),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def oracle_microbatch_sample(cfg, layers=1, seq_div=2):
    """The oracle as it stands on a bounded sample of the workload: one microbatch
    (encoder, embed, LLM, final norm, LM head + CE, generator + MSE, and the whole
    backward) of the workload's widths with `layers` LLM layers instead of L and
    S / seq_div sequence positions.  Returns (seconds, algorithmic FLOPs of the
    sample, cores)."""
    from synth import make_batch, make_weights
    from oracle import model as om
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count() or 1
    scfg = cfg.replace(L=layers, M=1, P=1, V=1, llm_sched="1f1b", S=cfg.S // seq_div)
    W, B = make_weights(scfg), make_batch(scfg)
    t0 = time.perf_counter()
    om.step_fp64(scfg, W, B)
    dt = time.perf_counter() - t0
    return dt, step_flops(scfg, B.n_mod, B.n_gen), cores


def step_hbm_bytes(cfg, n_mod, n_gen, es=2):
    """Algorithmic HBM bytes of one step, summed over all GPUs:
    every kernel reads its inputs and writes its outputs once; weights are read
    once per microbatch and fwd / bwd pass, fp32 weight gradients are read-modified-
    written once per microbatch (TMA reduce-add).  Per microbatch and LLM layer:
      fwd  norm (x -> xn) 2Sd; gate_up (xn, W -> gu, h) S(d + 3f) + 2df;
           down (h, W, x -> x') S(f + 2d) + df                         (x es)
      bwd  down dgrad+dswiglu (dy, W, gu -> dgu) S(d + 4f) + df; down wgrad
           (dy, h) S(d + f) + 8df/es; gate_up dgrad (dgu, W -> dxn) S(2f + d) + 2df;
           gate_up wgrad (dgu, xn) S(2f + d) + 16df/es; norm bwd (dxn, x, dres -> dx) 4Sd
    plus the LM head (logits written and read twice by CE fwd+bwd) on the text rows
    and the encoder / generator blocks on their rows (same per-row counts)."""
    S, d, f, L, V = cfg.S, cfg.d, cfg.f, cfg.L, cfg.vocab
    tot = 0.0
    for nm, ng in zip(n_mod, n_gen):
        per_layer = (2 * S * d + S * (d + 3 * f) + 2 * d * f + S * (f + 2 * d) + d * f +
                     S * (d + 4 * f) + d * f + S * (d + f) + 8 * d * f / es + S * (2 * f + d) + 2 * d * f +
                     S * (2 * f + d) + 16 * d * f / es + 4 * S * d) * es
        nt = S - nm
        head = (nt * d + V * d + 3 * nt * V + nt * d + V * d + nt * d + 2 * V * d * 4 / es) * es
        def mlp(n, dm, fm, Lb):
            return Lb * (2 * n * dm + n * (dm + 2 * fm) + 2 * dm * fm + n * (fm + 2 * dm)) * 3 * es
        enc = mlp(nm, cfg.d_e, cfg.f_e, cfg.L_e) + 3 * nm * (cfg.d_in + cfg.d_e + 2 * d) * es
        gen = mlp(ng, cfg.d_g, cfg.f_g, cfg.L_g) + 3 * ng * (d + cfg.d_g + cfg.d_t) * es
        tot += L * per_layer + head + enc + gen + 2 * S * d * es   # + embedding gather / scatter
    return tot


def bubble_from_trace(recs):
    """Compute-stream (LLM) idle fraction of one traced step on one rank:
    1 - |union of compute-op intervals on stream 0| / step span (origin -> tail end)."""
    end = max((x["t1"] for x in recs), default=0.0)
    iv = sorted((x["t0"], x["t1"]) for x in recs if x["stream"] == 0 and x["kind"] not in ("Tail", "Recv"))
    busy, cur0, cur1 = 0.0, None, None
    for a, b in iv:
        if cur1 is None or a > cur1:
            if cur1 is not None:
                busy += cur1 - cur0
            cur0, cur1 = a, b
        else:
            cur1 = max(cur1, b)
    if cur1 is not None:
        busy += cur1 - cur0
    return (1.0 - busy / end) if end > 0 else None, end


class Ctx:
    """Process-group helpers (gloo side group; device timing stays on CUDA events)."""

    def __init__(self, world, group):
        self.world, self.group = world, group

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    def reduce(self, v, op):
        if self.world == 1:
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(t, op=op, group=self.group)
        return float(t.item())

    def max(self, v):
        import torch.distributed as dist
        return self.reduce(v, dist.ReduceOp.MAX)

    def sum(self, v):
        import torch.distributed as dist
        return self.reduce(v, dist.ReduceOp.SUM)

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


def pacing_stage_mask(split, P, costs=None):
    """Bits of the stages holding the most LLM work (layers, or `costs` of a half-layer
    partition; they pace the pipeline) when the partition is uneven, else 0."""
    if not split or len(split) != P:
        return 0
    w = costs if costs is not None else split
    mx = max(w)
    if min(w) >= mx - 1e-9:
        return 0
    return sum(1 << r for r, n in enumerate(w) if n >= mx - 1e-9)


def lightest_only_mask(costs):
    """Bits of every stage except the lightest one(s): with a half-layer partition the
    generator runs only where the LLM leaves the most room (C2, N = 4: 188.2–188.5 vs
    180.2 samples/s for excluding only the heaviest stages, profiles/r02/zb/ab_place_n4.log)."""
    mn = min(costs)
    if max(costs) <= mn + 1e-9:
        return 0
    return sum(1 << r for r, c in enumerate(costs) if c > mn + 1e-9)


def rank_costs(cfg, P, split):
    """Per-rank cost of a half-layer partition: the rank's virtual stages summed
    (rank r holds virtual stages r, r + P, ...; interleaved V > 1)."""
    vc = unit_costs(cfg, split)
    return [sum(vc[s] for s in range(r, len(vc), P)) for r in range(P)]


def _pacing(args, cfg, P, split):
    if getattr(args, "partition", "layers") == "halves" and split and len(split) == P * cfg.V:
        return lightest_only_mask(rank_costs(cfg, P, split))
    return pacing_stage_mask(split, P)


def gen_exclude(args, cfg, P, split, strategy):
    """bigmac.h gen_exclude: "auto" keeps the DP-sharded generator off the pacing stage
    (R20), "none" = 0, else a comma list of ranks."""
    if args.gen_exclude == "none" or P == 1 or strategy == "memory_efficient" or args.head == "dp_shard":
        return 0
    if args.gen_exclude != "auto":
        return sum(1 << int(r) for r in args.gen_exclude.split(","))
    return _pacing(args, cfg, P, split)


def enc_exclude(args, cfg, P, split, strategy):
    """bm_sched_cfg.enc_exclude: "auto" moves the pacing stage's encoder microbatches to
    the next lower stage (R22), "none" = 0, else a comma list of ranks."""
    if args.enc_exclude == "none" or P == 1 or strategy == "memory_efficient":
        return 0
    if args.enc_exclude != "auto":
        return sum(1 << int(r) for r in args.enc_exclude.split(","))
    if getattr(args, "partition", "layers") == "halves":
        # the encoder joins the generator on the lightest stage only when that stage has
        # room for both (slack >= ENC_GEN_LAYERS): C2 N = 4 (slack 0.64) 188.5 vs 180.9
        # samples/s with it everywhere; C2 N = 2 (slack 0.3) 94.2 everywhere vs 90.4
        # (profiles/r02/zb/ab_place_n4.log, ab_n2.log, final/bench_n4_final.log)
        if not split or len(split) != P * cfg.V:
            return 0
        costs = rank_costs(cfg, P, split)
        return lightest_only_mask(costs) if max(costs) - min(costs) >= ENC_GEN_LAYERS else 0
    return _pacing(args, cfg, P, split)


def make_runtime(args, cfg, P, rank, world, group, strategy="bigmac"):
    from paper_2605_25451_b200.runtime import Runtime
    W = args.warmup_units if args.warmup_units >= 0 else (2 if P == 1 else 0)
    sched_kw = {"bigmac": {"warmup_units": W}, "compute_efficient": {"warmup_units": cfg.M // P},
                "memory_efficient": {"enc_place": "entry_stage", "gen_place": "last_stage"}}[strategy]
    sched_kw = dict(sched_kw, llm_sched=cfg.llm_sched)
    split = stage_split(args, cfg, P)
    n_last = 0 if split else last_stage_layers(args, cfg, P)
    ex = enc_exclude(args, cfg, P, split, strategy)
    if ex:
        sched_kw = dict(sched_kw, enc_exclude=ex)
    rt = Runtime(cfg, args.dtype, rank=rank, world=world, group=group, sched_kw=sched_kw, head_place=args.head,
                 last_stage_layers=n_last, stage_layers=split, fsdp=args.fsdp,
                 gen_exclude=gen_exclude(args, cfg, P, split, strategy),
                 stage_halves=bool(split) and getattr(args, "partition", "layers") == "halves",
                 # the encoder concentrated on the lightest stage gets its own stream there
                 enc_stream=1 if (ex and getattr(args, "partition", "layers") == "halves") else 0)
    rt.init_random_weights(seed=1)
    return rt, W, split, n_last


def timed_steps(rt, db, cx, steps, warmup):
    """W untimed steps, then `steps` steps between CUDA events on the caller's stream,
    barrier + synchronize on both sides; returns max-over-ranks milliseconds."""
    import torch
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        rt.step(db)
    torch.cuda.synchronize()
    cx.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        rt.step(db)
    e1.record(stream)
    torch.cuda.synchronize()
    cx.barrier()
    return cx.max(e0.elapsed_time(e1))


def measure_bubble(rt, db, cx, P, cfg):
    """One traced step (CUDA events around every op): per-rank compute-stream idle
    fraction against the 1F1B closed form (P - 1) / (M V + P - 1)."""
    import torch
    cx.barrier()
    rt.set_trace(True)
    rt.step(db)
    torch.cuda.synchronize()
    tr = rt.trace()
    rt.set_trace(False)
    frac, span = bubble_from_trace(tr)
    per = cx.gather(frac)
    return {"measured_max": max(per), "per_rank": per, "bound": bubble_bound(cfg, P),
            "how": "1 - busy/step of the LLM compute stream from a per-op CUDA-event trace of one step "
                   "(max over ranks); bound = closed form: 1F1B (P-1)/(MV+P-1), ZB-H1 (P-1)/(3M+P-1)"}


def free_runtime(rt):
    import torch
    rt.close()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def run_secondary(args, cx, rank, world, name, cfg, P, D, steps, warmup, with_bubble=True):
    """A second configuration in the same process (C4 at N = 1, BASELINE's C2 M = 16 at
    N > 1): samples/s, step roofline, bubble, peak HBM."""
    import torch
    from synth import slice_batch
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    rt, W, split, n_last = make_runtime(args, cfg, P, rank, world, cx.group)
    gbatch = global_batch(cfg, D)
    replica = rank // P
    db = rt.device_batch(slice_batch(gbatch, replica * cfg.M, (replica + 1) * cfg.M))
    ms = timed_steps(rt, db, cx, steps, warmup)
    out = {"workload": config_dict(cfg, P, D)["workload"], "global_batch": cfg.M * D, "steps": steps,
           "warmup": warmup, "ms_per_step": ms / steps, "value": cfg.M * D * steps / (ms / 1e3), "unit": UNIT,
           "tokens_per_s": cfg.M * D * cfg.S * steps / (ms / 1e3)}
    peaks, _ = load_peaks()
    F = step_flops(cfg, gbatch.n_mod, gbatch.n_gen)
    t_roof = F / (world * peaks["bf16_tflops"] * 1e12) * 1e3
    out["step_roofline"] = {"flops_per_step": F, "t_roof_ms": t_roof, "frac": t_roof / (ms / steps)}
    if with_bubble:
        out["bubble"] = measure_bubble(rt, db, cx, P, cfg)
    out["peak_hbm_gb_per_gpu"] = cx.max(torch.cuda.max_memory_allocated()) / 1e9
    out["stash_peak_bytes_rank0_enc_llm_gen"] = rt.stash_peak()
    out["config"] = {"stages": P, "replicas": D, "microbatches": cfg.M, "warmup_units": W, "stage_layers": split,
                     "partition": getattr(args, "partition", "layers"), "llm_sched": cfg.llm_sched,
                     "last_stage_layers": n_last}
    free_runtime(rt)
    del db
    return out


def run_sweep(args, cx, rank, world, P, ms_list, config=None):
    """Peak HBM per GPU and samples/s vs global batch (C5's claim: the
    encoder / generator stash is fixed by the schedule -- W units, one generator shard --
    and the LLM in-flight depth by 1F1B, so peak HBM grows only with the resident inputs)."""
    import torch
    from synth import get_config, make_batch
    out = []
    for M in ms_list:
        if M % P:
            continue
        cfg = get_config(config or args.config, P=P, M=M, V=1)
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        rt, W, _, _ = make_runtime(args, cfg, P, rank, world, cx.group)
        mem0 = torch.cuda.memory_allocated()
        db = rt.device_batch(make_batch(cfg))
        batch_bytes = torch.cuda.memory_allocated() - mem0
        ms = timed_steps(rt, db, cx, 1, 1)
        st = rt.sched.stats(rt.rank)
        D = world // P
        out.append({"M": M, "global_batch": M * D, "samples_per_s": M * D / (ms / 1e3), "ms_per_step": ms,
                    "peak_hbm_gb_per_gpu": cx.max(torch.cuda.max_memory_allocated()) / 1e9,
                    "resident_input_gb_rank0": cx.max(batch_bytes if rank == 0 else 0) / 1e9,
                    "stash_peak_bytes_rank0_enc_llm_gen": rt.stash_peak(), "peak_enc_units": st.peak_enc_units,
                    "peak_llm_inflight": st.peak_llm_inflight, "peak_gen_shards": st.peak_gen_shards})
        free_runtime(rt)
        del db
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--microbatches", type=int, default=0, help="per-replica M (default 16 P)")
    ap.add_argument("--last-stage-layers", type=int, default=-1,
                    help="LLM layers of the last stage (bigmac.h); -1 = balance the LM head (HEAD_LAYERS), 0 = uniform")
    ap.add_argument("--warmup-units", type=int, default=-1,
                    help="BigMac W (encoder units in flight); -1: 2 at P = 1 (lets the encoder stream overlap "
                         "the next microbatch), else 0 = W* (DESIGN.md R4)")
    ap.add_argument("--stage-layers", default="", help="explicit LLM layers per stage, e.g. 4,5,4,3 (bigmac.h)")
    ap.add_argument("--stages", type=int, default=0, help="pipeline stages P (default min(N, 4)); D = N / P replicas")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary config (C4 at N = 1, M = 16 per "
                                                             "replica at N > 1) and the batch sweep")
    ap.add_argument("--sweep", default="8,16,32,64,128,256", help="global batches of the peak-HBM sweep ('' = off)")
    ap.add_argument("--c4-steps", type=int, default=2)
    ap.add_argument("--no-c4-strong", action="store_true", help="skip the C4 strong-scaling line at N > 1")
    ap.add_argument("--c5", action="store_true", help="run the C5 sweep (default: when N >= --c5-stages)")
    ap.add_argument("--c5-stages", type=int, default=8)
    ap.add_argument("--c5-sweep", default="8,16,32,64,128,256", help="global batches of the C5 sweep")
    ap.add_argument("--ref-layers", type=int, default=1, help="LLM layers of the oracle sample")
    ap.add_argument("--ref-seq-div", type=int, default=2, help="the oracle sample runs S / this positions")
    ap.add_argument("--head", default="auto", choices=["auto", "last_stage", "dp_shard"],
                    help="LM head + CE placement (bigmac.h bm_head_place): auto = last_stage (the paper's "
                         "Megatron placement), dp_shard = DP-sharded with the generator")
    ap.add_argument("--fsdp", default="off", choices=["off", "pull", "allgather"],
                    help="encoder / generator parameters: replicated (off), FSDP with BigMac's one-sided pull, "
                         "or FSDP with the all-gather baseline (bigmac.h bm_fsdp_mode, P:401-426)")
    ap.add_argument("--gen-exclude", default="auto", help="ranks that take no generator rows: auto | none | r,r")
    ap.add_argument("--enc-exclude", default="auto", help="ranks that run no encoder microbatch: auto | none | r,r")
    ap.add_argument("--partition", default="halves", choices=["layers", "halves"],
                    help="LLM stage partition: whole layers (DEFAULT_SPLIT / last_stage_layers) or half-layer units "
                         "(stage boundaries inside layers, bigmac.h stage_halves)")
    ap.add_argument("--llm-sched", default="auto", choices=["auto", "zb_h1"],
                    help="LLM base schedule: auto = 1F1B (V = 1) / interleaved (V > 1); zb_h1 = ZB-H1 zero-bubble")
    ap.add_argument("--strategy", default="bigmac", choices=["bigmac", "compute_efficient", "memory_efficient"],
                    help="bigmac (default); the paper's baselines on the same executor (P:129-156)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = world
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        group = dist.new_group(backend="gloo")
    cx = Ctx(world, group)

    from synth import get_config, slice_batch
    cfg, P, D = workload(args, N)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    rt, W, split, n_last = make_runtime(args, cfg, P, rank, world, group, args.strategy)
    gbatch = global_batch(cfg, D)
    replica = rank // P
    batch = slice_batch(gbatch, replica * cfg.M, (replica + 1) * cfg.M)
    db = rt.device_batch(batch)
    stream = torch.cuda.current_stream()

    # ---------------- warmup
    for _ in range(args.warmup):
        rt.step(db)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()

    # ---------------- timed region (device events, max over ranks)
    try:
        uuid = str(torch.cuda.get_device_properties(local).uuid)
    except Exception:
        uuid = None
    clk = ClockSampler(uuid)
    clk.start()
    time.sleep(0.3)
    ms_max = timed_steps(rt, db, cx, args.steps, 0)
    clocks = clk.stop()
    launches = rt.launch_count() * args.steps
    ms_per_step = ms_max / args.steps
    samples = cfg.M * D * args.steps
    value = samples / (ms_max / 1000.0)
    loss, _, _ = rt.losses()
    peak_alloc = cx.max(float(torch.cuda.max_memory_allocated()))
    stash = rt.stash_peak()

    # instrumented passes (not part of `value`): a CUDA-event pair around every GEMM
    # launch and every NVLink copy, on the stream each runs on -> roofline + NVLink
    rt.set_timing(True)
    n_inst = max(2, min(args.steps, 5))
    for _ in range(n_inst):
        rt.step(db)
    torch.cuda.synchronize()
    n_gemm, gemm_flops, gemm_ms = rt.gemm_stats()
    n_msgs, comm_bytes, comm_ms = rt.comm_stats()
    rt.set_timing(False)
    bubble = measure_bubble(rt, db, cx, P, cfg)

    # ---------------- end-to-end: host inputs copied in, loss read back, every step
    e2e = None
    if not args.no_e2e:
        hb = rt.host_batch(batch)
        lt = rt.loss_tensor()
        for _ in range(2):
            rt.step(hb)
            float(lt[2 * cfg.M].item())
        cx.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            rt.step(hb)
            float(lt[2 * cfg.M].item())   # device -> host read of the step's loss
        f1.record(stream)
        torch.cuda.synchronize()
        cx.barrier()
        ems = cx.max(f0.elapsed_time(f1))
        h2d = cx.sum(hb.h2d_bytes)
        e2e = {"value": cfg.M * D * args.steps / (ems / 1000.0), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(4 * world),
               "ms_per_step": ems / args.steps}
        del lt, hb   # lt views the work buffer: keep the later configurations' peak HBM clean

    launches_all = int(cx.sum(launches))
    comm_bytes_all = cx.sum(comm_bytes)
    comm_bytes_max = cx.max(comm_bytes)
    comm_ms_all = cx.sum(comm_ms)
    n_msgs_all = int(cx.sum(n_msgs))
    gemm_flops_all = cx.sum(gemm_flops)
    gemm_ms_all = cx.sum(gemm_ms)
    n_gemm_all = int(cx.sum(n_gemm))
    sum_mode = getattr(rt, "sum_mode", None)
    fsdp_info = {"mode": args.fsdp, "weight_bytes_per_gpu_max": cx.max(rt.w_elems * rt.es),
                 "weight_bytes_replicated": rt.total_elems * rt.es,
                 "pull_bytes_per_step_max_gpu": cx.max(rt.pull_bytes())}
    free_runtime(rt)
    del db

    # ---------------- secondary configurations and the sweeps (a failing secondary is
    # reported in its key; the main line above is kept)
    extra = {}

    def secondary(key, fn):
        try:
            extra[key] = fn()
        except Exception as e:   # deterministic failures raise on every rank alike
            import torch
            torch.cuda.empty_cache()
            extra[key] = {"error": repr(e)[:300]}

    if not args.no_extra:
        if N == 1:
            # the largest single-GPU workload: C4 (7B-shaped LLM, S = 8192) at P = 1, M = 64
            c4 = get_config("C4", P=1, M=64, V=1)
            secondary("c4_single_gpu", lambda: run_secondary(args, cx, rank, world, "C4", c4, 1, 1, args.c4_steps, 1))
        elif args.config == "C2" and not args.microbatches:
            # BASELINE.json configs[1]: 16 microbatches per pipeline (global batch 16 D)
            c2 = get_config("C2", P=P, M=16, V=1)
            secondary("c2_m16_per_replica",
                      lambda: run_secondary(args, cx, rank, world, "C2", c2, P, D, max(3, args.steps // 2), 3))
        if N > 1 and args.config == "C2" and not args.microbatches and not args.no_c4_strong:
            # SURVEY §8(d) strong-scaling ladder: the C4 model (7B-shaped LLM, S = 8192) at
            # P = min(N, 4) stages x D replicas over one global batch of 64 microbatches
            c4s = get_config("C4", P=P, M=64 // D, V=1)
            secondary("c4_strong", lambda: run_secondary(args, cx, rank, world, "C4", c4s, P, D, 2, 2,
                                                         with_bubble=False))
        if N > 1 and cfg.V == 1 and cfg.llm_sched != "zb_h1":
            # the same workload on the ZB-H1 zero-bubble base schedule (reading R23)
            secondary("zb_h1", lambda: run_secondary(args, cx, rank, world, cfg.name, cfg.replace(llm_sched="zb_h1"),
                                                     P, D, max(3, args.steps // 2), 3))
        c5p = args.c5_stages
        if (N >= c5p or args.c5) and N % c5p == 0 and args.config == "C2" and not args.microbatches:
            # BASELINE configs[4] (C5): the C4 model on 8 stages, global batch 8 -> 256
            secondary("c5_sweep", lambda: {
                "config": f"C5: C4 model (7B-shaped LLM, S = 8192), P = {c5p} x D = {N // c5p}, bigmac, 1F1B, "
                          f"1 timed step per M",
                "points": run_sweep(args, cx, rank, world, c5p, [int(x) for x in args.c5_sweep.split(",") if x],
                                    "C4")})
        if args.sweep:
            secondary("batch_sweep", lambda: {
                "config": f"{args.config} model, P = {P} x D = {D}, bigmac, 1 timed step per per-replica M",
                "points": run_sweep(args, cx, rank, world, P, [int(x) for x in args.sweep.split(",") if x])})

    if rank != 0:
        cx.barrier()
        return

    peaks, peak_src = load_peaks()
    F = step_flops(cfg, gbatch.n_mod, gbatch.n_gen)
    sustained = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    achieved = gemm_flops_all / (gemm_ms_all / 1000.0) / 1e12 if gemm_ms_all > 0 else 0.0
    traffic, traffic_src = None, None
    for tpath in (os.path.join(ROOT, "profiles", "r02", "gemm_traffic.json"),
                  os.path.join(ROOT, "profiles", "gemm_traffic.json")):
        if os.path.exists(tpath):
            try:
                tj = json.load(open(tpath))
                traffic, traffic_src = tj.get("dram_bytes_per_launch"), os.path.relpath(tpath, ROOT) + ": " + \
                    str(tj.get("source", ""))
                break
            except Exception:
                pass
    roofline = {"bound": "tensor", "kernel": "bm::tc::gemm2_kernel / gemm_kernel on the compute stream (tcgen05.mma kind::f16, TMA, TMEM; CTA pairs for the LLM contractions)",
                "achieved": achieved, "peak": sustained, "unit": "TFLOP/s", "frac": achieved / sustained,
                "peak_source": f"{peak_src} bf16_tflops_sustained (GEMMs timed inside a long step)",
                "traffic": traffic, "traffic_source": traffic_src, "launches": n_gemm_all,
                "gemm_share_of_step": (gemm_ms_all / world / n_inst) / ms_per_step if ms_per_step > 0 else None,
                "measured_over": f"{n_inst} instrumented steps after the timed region (event pair per GEMM)",
                "flops_per_launch": gemm_flops_all / max(n_gemm_all, 1),
                "avg_launch_ms": gemm_ms_all / max(n_gemm_all, 1)}
    hbm_all = step_hbm_bytes(cfg, gbatch.n_mod, gbatch.n_gen)
    t_flop = F / (N * peaks["bf16_tflops"] * 1e12) * 1e3
    t_hbm = hbm_all / N / (peaks["hbm_gbs"] * 1e9) * 1e3
    nvl_per_gpu = comm_bytes_max / n_inst if world > 1 else 0.0
    t_nvl = nvl_per_gpu / 900e9 * 1e3
    t_roof_ms = max(t_flop, t_hbm, t_nvl)
    step_roof = {"flops_per_step": F, "t_roof_ms": t_roof_ms, "frac": t_roof_ms / ms_per_step,
                 "terms_ms": {"tensor": t_flop, "hbm": t_hbm, "nvlink": t_nvl},
                 "hbm_bytes_per_step_all_gpus": hbm_all, "nvlink_bytes_per_step_max_gpu": nvl_per_gpu,
                 "peaks": {"bf16_tflops": peaks["bf16_tflops"], "hbm_gbs": peaks["hbm_gbs"], "nvlink_gbs": 900.0},
                 "bound": max((t_flop, "tensor"), (t_hbm, "hbm"), (t_nvl, "nvlink"))[1],
                 "bubble_bound": bubble_bound(cfg, P)}

    cpu = None
    if not args.no_cpu and N == 1:
        dt, fl, cores = oracle_microbatch_sample(cfg, args.ref_layers, args.ref_seq_div)
        cpu = {"value": fl / dt / (F / (cfg.M * D)), "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"oracle (numpy fp64 step_fp64) fwd+bwd of one {cfg.name} microbatch with "
                         f"{args.ref_layers} of {cfg.L} LLM layers and S/{args.ref_seq_div} positions ({dt:.1f} s, "
                         f"{fl / 1e12:.2f} TFLOP); samples/s scaled by the step's algorithmic FLOPs per sample"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "strategy": args.strategy,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.microbatches else "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": dict(config_dict(cfg, P, D), strategy=args.strategy, head_place=head_place_name(args, N),
                           warmup_units=W, last_stage_layers=n_last, stage_layers=split, step_sum=sum_mode,
                           partition=args.partition,
                           gen_exclude=gen_exclude(args, cfg, P, split, args.strategy),
                           enc_exclude=enc_exclude(args, cfg, P, split, args.strategy)),
            "roofline": roofline, "step_roofline": step_roof, "bubble": bubble, "fsdp": fsdp_info,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_all, "clocks": clocks,
            "nvlink": ({"bytes_per_step_all_ranks": comm_bytes_all / n_inst,
                        "messages_per_step": n_msgs_all / n_inst,
                        "copy_GBps": comm_bytes_all / (comm_ms_all / 1e3) / 1e9 if comm_ms_all > 0 else None,
                        "avg_link_GBps_over_step": comm_bytes_all / n_inst / max(world, 1) / (ms_per_step / 1e3) / 1e9,
                        "note": "copy-engine copies into peer IPC receive slots over NVLink; copy_GBps = bytes / "
                                "summed copy durations on the comm streams"} if world > 1 else None),
            "tokens_per_s": cfg.M * D * cfg.S * args.steps / (ms_max / 1000.0),
            "peak_hbm_gb_per_gpu": peak_alloc / 1e9, "stash_peak_bytes_rank0": stash,
            "loss": loss}
    line.update(extra)
    print(json.dumps(line), flush=True)
    cx.barrier()


if __name__ == "__main__":
    main()
