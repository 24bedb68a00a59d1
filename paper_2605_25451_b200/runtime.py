"""Per-rank runtime: the paper's create_executor / load_schedule / execute
 over the C ABI.  PyTorch provides device memory, the stream and
the process group used to exchange IPC handles and the NCCL id; every step of
the hot path runs in libbigmac.so.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

# Each rank runs a compute stream, P-1 comm streams, a generator stream and NCCL's;
# with fewer hardware work queues than streams, a comm stream parked on a credit
# wait (cuStreamWaitValue32) would serialize unrelated streams behind it.  Must be
# set before the CUDA context exists (importing this module before torch.cuda use).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from . import _lib as L
from . import schedule as BS


def model_cfg(shape, dtype: str, max_n_mod: int | None = None, max_n_gen: int | None = None,
              head_place: str = "auto", last_stage_layers: int = 0, stage_layers=None, fsdp: str = "off",
              gen_exclude: int = 0, stage_halves: bool = False, enc_stream: int = 0) -> L.ModelCfg:
    mc = L.ModelCfg()
    mc.S, mc.d_in, mc.d_e, mc.f_e, mc.L_e = shape.S, shape.d_in, shape.d_e, shape.f_e, shape.L_e
    mc.d, mc.f, mc.L, mc.vocab = shape.d, shape.f, shape.L, shape.vocab
    mc.d_g, mc.f_g, mc.L_g, mc.d_t = shape.d_g, shape.f_g, shape.L_g, shape.d_t
    mc.dtype = L.BF16 if dtype == "bf16" else L.F32
    mc.max_n_mod = max_n_mod if max_n_mod is not None else min(shape.n_mod_law[2], shape.S)
    mc.max_n_gen = max_n_gen if max_n_gen is not None else min(shape.n_gen_law[2], shape.S)
    mc.head_place = L.HEAD_PLACE[head_place]
    mc.last_stage_layers = last_stage_layers
    mc.fsdp = L.FSDP[fsdp]
    mc.gen_exclude = gen_exclude
    mc.stage_halves = 1 if stage_halves else 0
    mc.enc_stream = enc_stream
    for i, n in enumerate(stage_layers or ()):
        mc.stage_layers[i] = n
    return mc


def exchange(group, P: int, D: int, global_rank: int, payload, new_id):
    """Host side of the process-group plumbing for D pipeline replicas of P stages
    (process rank = replica * P + stage).  One all_gather; returns
    (payloads of the P stages of this process's replica, in stage order,
     {"pipe": id of this replica's pipeline group (P > 1),
      "world": id of the all-process group (D > 1),
      "stage": id of this stage's replica group (D > 1)},
     payloads of all P * D processes).
    Ids are made by one member of each group (new_id() -> bytes): the pipeline's
    stage 0, process 0, and replica 0's process of the stage."""
    import torch.distributed as dist
    replica, stage = divmod(global_rank, P)
    mine = {"pipe": new_id() if (stage == 0 and P > 1) else None,
            "world": new_id() if (global_rank == 0 and D > 1) else None,
            "stage": new_id() if (replica == 0 and D > 1) else None}
    allp = [None] * (P * D)
    dist.all_gather_object(allp, (payload, mine), group=group)
    base = replica * P
    peers = [allp[base + q][0] for q in range(P)]
    ids = {"pipe": allp[base][1]["pipe"], "world": allp[0][1]["world"], "stage": allp[stage][1]["stage"]}
    return peers, ids, [a[0] for a in allp]


def sum_mode(uuids) -> str:
    """Step-end sums (A18): "nccl" when every process has its own GPU, "peer" (the
    library's IPC reduce, bm_ctx_init_peer_sum) when two processes share a device
    -- NCCL rejects duplicate GPUs.  BM_STEP_SUM=nccl|peer forces one."""
    forced = os.environ.get("BM_STEP_SUM", "auto")
    if forced in ("nccl", "peer"):
        return forced
    return "peer" if len(set(uuids)) < len(uuids) else "nccl"


def _round8(x):
    return (x + 7) // 8 * 8


@dataclass
class DeviceBatch:
    struct: L.Batch
    keep: list
    h2d_bytes: int


class Runtime:
    def __init__(self, shape, dtype="bf16", rank=0, world=1, group=None, device=None, sched_kw=None,
                 head_place="auto", last_stage_layers=0, stage_layers=None, fsdp="off", gen_exclude=0,
                 stage_halves=False, enc_stream=0):
        self.shape = shape
        self.dtype = dtype
        self.world = world
        self.P, self.M, self.V = shape.P, shape.M, shape.V
        if world % self.P:
            raise ValueError(f"world={world} is not a multiple of P={self.P} (D pipeline replicas of P stages)")
        # D pipeline replicas of P stages; process rank = replica * P + stage
        self.D = world // self.P
        self.global_rank = rank
        self.replica, self.rank = divmod(rank, self.P)
        rank = self.rank
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self._stream = None   # own compute stream (created on first step)
        kw = dict(sched_kw or {})
        self.sched = BS.build(self.P, self.M, self.V, **kw)
        self.fsdp = fsdp
        self.mc = model_cfg(shape, dtype, head_place=head_place, last_stage_layers=last_stage_layers,
                            stage_layers=stage_layers, fsdp=fsdp, gen_exclude=gen_exclude,
                            stage_halves=stage_halves, enc_stream=enc_stream)
        h = C.c_void_p()
        L.call("bm_ctx_create", C.byref(self.mc), self.sched.handle, rank, C.byref(h))
        self.ctx = h.value
        sz = L.CtxSizes()
        L.call("bm_ctx_sizes_get", self.ctx, C.byref(sz))
        self.sizes = sz
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.tdtype = tdt
        self.es = 2 if dtype == "bf16" else 4

        def alloc(nbytes, zero=False):
            n = max(int(nbytes), 256)
            t = (torch.zeros if zero else torch.empty)(n + 256, dtype=torch.uint8, device=self.device)
            off = (-t.data_ptr()) % 256
            return t, t.data_ptr() + off, n

        self._w, self.w_ptr, wb = alloc(sz.weight_bytes)
        self._g, self.g_ptr, gb = alloc(sz.grad_bytes)
        self._work, self.work_ptr, kb = alloc(sz.work_bytes)
        self._comm, self.comm_ptr, cb = alloc(sz.comm_bytes, zero=True)
        bufs = L.Buffers(self.w_ptr, self.g_ptr, self.work_ptr, self.comm_ptr, wb, gb, kb, cb)
        L.call("bm_ctx_bind", self.ctx, C.byref(bufs))
        # parameter table
        n, tot, dp = C.c_int32(), C.c_int64(), C.c_int64()
        L.call("bm_param_count", C.byref(self.mc), C.byref(BS.make_cfg(self.P, self.M, self.V, **kw)), rank,
               C.byref(n), C.byref(tot), C.byref(dp))
        self.total_elems, self.dp_elems = tot.value, dp.value
        self.params = {}
        scfg = BS.make_cfg(self.P, self.M, self.V, **kw)
        for i in range(n.value):
            pi = L.ParamInfo()
            L.call("bm_param_info_get", C.byref(self.mc), C.byref(scfg), rank, i, C.byref(pi))
            self.params[pi.name.decode()] = (pi.rows, pi.cols, pi.ld, pi.offset, pi.kind)
        lo, hi = C.c_int64(), C.c_int64()
        L.call("bm_ctx_dp_shard", self.ctx, C.byref(lo), C.byref(hi))
        self.dp_lo, self.dp_hi = lo.value, hi.value   # FSDP: this rank's shard of the DP elements
        self.w_elems = self.total_elems - self.dp_elems + (self.dp_hi - self.dp_lo)
        self.weights_t = self._w[(self.w_ptr - self._w.data_ptr()):][: self.w_elems * self.es].view(tdt)
        self.grads_t = self._g[(self.g_ptr - self._g.data_ptr()):][: self.total_elems * 4].view(torch.float32)
        if world > 1:
            self._connect(group)

    # ------------------------------------------------------------------ peers
    def _connect(self, group):
        """Peer memory inside this replica's pipeline (CUDA IPC), the pipeline's NCCL
        group, and with D > 1 the all-process and per-stage NCCL groups."""
        import torch.distributed as dist
        P, D = self.P, self.D

        def export(ptr):
            hb = (C.c_uint8 * 64)()
            off = C.c_int64()
            L.call("bm_ipc_export", ptr, hb, C.byref(off))
            return bytes(hb), off.value

        def new_id():
            nid = (C.c_uint8 * 128)()
            L.call("bm_nccl_unique_id", nid)
            return bytes(nid)
        uuid = str(torch.cuda.get_device_properties(self.device).uuid)
        mine = (export(self.comm_ptr), export(self.g_ptr), uuid, export(self.w_ptr))
        peers, ids, allp = exchange(group, P, D, self.global_rank, mine, new_id)
        for q, ((hbytes, o), _, _, _) in enumerate(peers):
            if q != self.rank:
                L.call("bm_ctx_open_peer", self.ctx, q, (C.c_uint8 * 64).from_buffer_copy(hbytes), o)
        if self.fsdp != "off":   # one-sided pulls read the pipeline peers' weight shards
            wh = (C.c_uint8 * (64 * P)).from_buffer_copy(b"".join(x[3][0] for x in peers))
            wo = (C.c_int64 * P)(*[x[3][1] for x in peers])
            L.call("bm_ctx_init_fsdp", self.ctx, wh, wo)
        self.sum_mode = sum_mode([a[2] for a in allp])
        as_c = lambda b: (C.c_uint8 * 128).from_buffer_copy(b)  # noqa: E731
        if self.sum_mode == "peer":
            n = P * D
            ch = (C.c_uint8 * (64 * n)).from_buffer_copy(b"".join(a[0][0] for a in allp))
            co = (C.c_int64 * n)(*[a[0][1] for a in allp])
            gh = (C.c_uint8 * (64 * n)).from_buffer_copy(b"".join(a[1][0] for a in allp))
            go = (C.c_int64 * n)(*[a[1][1] for a in allp])
            L.call("bm_ctx_init_peer_sum", self.ctx, D, self.replica, ch, co, gh, go)
        else:
            if P > 1:
                L.call("bm_ctx_init_nccl", self.ctx, as_c(ids["pipe"]), P, self.rank)
            if D > 1:
                L.call("bm_ctx_init_replicas", self.ctx, D, self.replica, as_c(ids["world"]), as_c(ids["stage"]))
        dist.barrier(group=group)

    # ------------------------------------------------------------------ weights / grads
    def _physical(self, flat):
        """Logical parameter vector -> this rank's weights buffer layout (bigmac.h
        bm_ctx_dp_shard: the DP shard [dp_lo, dp_hi) first, then the LLM parameters)."""
        if self.dp_lo == 0 and self.dp_hi == self.dp_elems:
            return flat
        return torch.cat([flat[self.dp_lo:self.dp_hi], flat[self.dp_elems:]])

    def load_weights(self, weights: dict):
        """weights: {name: float32 array} (synth.make_weights); only this rank's params are used."""
        flat = torch.zeros(self.total_elems, dtype=torch.float32)
        for name, (rows, cols, ld, off, _) in self.params.items():
            w = np.asarray(weights[name], np.float32).reshape(rows, cols)
            view = flat[off:off + rows * ld].view(rows, ld)
            view[:, :cols] = torch.from_numpy(w)
        self.weights_t.copy_(self._physical(flat).to(self.device).to(self.tdtype))
        torch.cuda.synchronize(self.device)

    def init_random_weights(self, seed: int = 1, std: float = 0.02):
        """Synthetic random init on the device (bench path): N(0, std) for linear
        weights, residual-branch outputs scaled by 1/sqrt(2 L), RMSNorm gains 1."""
        sh = self.shape
        import zlib
        gen = torch.Generator(device=self.device)
        depth = {"enc": sh.L_e, "llm": sh.L, "gen": sh.L_g}
        self.weights_t.zero_()
        sharded = not (self.dp_lo == 0 and self.dp_hi == self.dp_elems)
        for name, (rows, cols, ld, off, kind) in self.params.items():
            if sharded and kind == 0:   # FSDP: generate in full, keep the owned slice
                full = torch.zeros(rows * ld, dtype=self.tdtype, device=self.device)
                view = full.view(rows, ld)
            elif sharded:
                o = off - self.dp_elems + (self.dp_hi - self.dp_lo)
                view = self.weights_t[o:o + rows * ld].view(rows, ld)
            else:
                view = self.weights_t[off:off + rows * ld].view(rows, ld)
            if cols == 1:
                view.fill_(1.0)
            else:
                gen.manual_seed(seed * 1000003 + zlib.crc32(name.encode()))  # DP replicas identical on every rank
                scale = std
                if name.endswith((".fc2", ".down")):
                    scale = std / (2.0 * depth[name.split(".")[0]]) ** 0.5
                w = torch.randn((rows, cols), generator=gen, device=self.device, dtype=torch.float32) * scale
                view[:, :cols] = w.to(self.tdtype)
            if sharded and kind == 0:
                a, b = max(off, self.dp_lo), min(off + rows * ld, self.dp_hi)
                if b > a:
                    self.weights_t[a - self.dp_lo:b - self.dp_lo].copy_(full[a - off:b - off])
        torch.cuda.synchronize(self.device)

    def set_timing(self, on: bool):
        L.call("bm_ctx_set_timing", self.ctx, 1 if on else 0)

    def gemm_stats(self):
        n, fl, ms = C.c_int64(), C.c_double(), C.c_double()
        L.call("bm_ctx_gemm_stats", self.ctx, C.byref(n), C.byref(fl), C.byref(ms))
        return n.value, fl.value, ms.value

    def comm_stats(self):
        n, b, ms = C.c_int64(), C.c_double(), C.c_double()
        L.call("bm_ctx_comm_stats", self.ctx, C.byref(n), C.byref(b), C.byref(ms))
        return n.value, b.value, ms.value

    def set_trace(self, on: bool):
        """Record a per-op trace of each following step (CUDA events around every op)."""
        L.call("bm_ctx_set_trace", self.ctx, 1 if on else 0)

    def trace(self):
        """Per-op records of the last traced step: dicts with op index, kind name,
        stream (0 compute, 1 generator, 2+q comm to rank q), mb, start/end ms."""
        n, tot = C.c_int64(), C.c_int64()
        L.call("bm_ctx_trace_get", self.ctx, None, 0, C.byref(n), C.byref(tot))
        buf = (L.TraceRec * max(tot.value, 1))()
        L.call("bm_ctx_trace_get", self.ctx, buf, tot.value, C.byref(n), C.byref(tot))
        kinds = BS.KINDS
        return [{"op": r.op, "kind": kinds[r.kind] if 0 <= r.kind < len(kinds) else "Tail", "stream": r.stream,
                 "mb": r.mb, "t0": r.t_start_ms, "t1": r.t_end_ms} for r in buf[:n.value]]

    def debug_dump(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        L.call("bm_ctx_debug_dump", self.ctx, buf, len(buf))
        return buf.value.decode()

    def names(self):
        return list(self.params)

    def grad(self, name) -> np.ndarray:
        rows, cols, ld, off, _ = self.params[name]
        g = self.grads_t[off:off + rows * ld].view(rows, ld)[:, :cols]
        out = g.double().cpu().numpy()
        return out.reshape(rows) if cols == 1 else out

    def grads(self) -> dict:
        return {n: self.grad(n) for n in self.params}

    # ------------------------------------------------------------------ batch
    def device_batch(self, batch) -> DeviceBatch:
        """Pack a synth.Batch on the device (inputs resident in HBM)."""
        sh = self.shape
        ldp = _round8(sh.d_in)
        rows = int(np.sum(batch.n_mod))
        pat = np.zeros((max(rows, 1), ldp), np.float32)
        r = 0
        for p in batch.patches:
            pat[r:r + p.shape[0], :sh.d_in] = p
            r += p.shape[0]
        tgt = np.concatenate([np.asarray(t, np.float32) for t in batch.targets], 0)
        keep = [torch.from_numpy(pat).to(self.device).to(self.tdtype).contiguous(),
                torch.from_numpy(np.ascontiguousarray(batch.ids, np.int32)).to(self.device),
                torch.from_numpy(np.ascontiguousarray(batch.labels, np.int32)).to(self.device),
                torch.from_numpy(tgt).to(self.device).to(self.tdtype).contiguous()]
        nm = np.ascontiguousarray(batch.n_mod, np.int32)
        ng = np.ascontiguousarray(batch.n_gen, np.int32)
        keep += [nm, ng]
        b = L.Batch()
        b.M = len(nm)
        b.n_mod = nm.ctypes.data
        b.n_gen = ng.ctypes.data
        b.patches = keep[0].data_ptr()
        b.ld_patch = ldp
        b.ids = keep[1].data_ptr()
        b.labels = keep[2].data_ptr()
        b.targets = keep[3].data_ptr()
        b.on_host = 0
        return DeviceBatch(b, keep, 0)

    def host_batch(self, batch) -> DeviceBatch:
        """Pinned host copy of a synth.Batch for the end-to-end path (bm_step copies it in)."""
        sh = self.shape
        ldp = _round8(sh.d_in)
        rows = int(np.sum(batch.n_mod))
        tdt = self.tdtype
        pat = torch.zeros((max(rows, 1), ldp), dtype=torch.float32)
        r = 0
        for p in batch.patches:
            pat[r:r + p.shape[0], :sh.d_in] = torch.from_numpy(p)
            r += p.shape[0]
        pat = pat.to(tdt).pin_memory()
        tgt = torch.from_numpy(np.concatenate([np.asarray(t, np.float32) for t in batch.targets], 0)).to(tdt).pin_memory()
        ids = torch.from_numpy(np.ascontiguousarray(batch.ids, np.int32)).pin_memory()
        lab = torch.from_numpy(np.ascontiguousarray(batch.labels, np.int32)).pin_memory()
        nm = np.ascontiguousarray(batch.n_mod, np.int32)
        ng = np.ascontiguousarray(batch.n_gen, np.int32)
        b = L.Batch()
        b.M = len(nm)
        b.n_mod = nm.ctypes.data
        b.n_gen = ng.ctypes.data
        b.patches = pat.data_ptr()
        b.ld_patch = ldp
        b.ids = ids.data_ptr()
        b.labels = lab.data_ptr()
        b.targets = tgt.data_ptr()
        b.on_host = 1
        h2d = rows * sh.d_in * self.es + ids.numel() * 4 + lab.numel() * 4 + tgt.numel() * self.es
        return DeviceBatch(b, [pat, tgt, ids, lab, nm, ng], h2d)

    # ------------------------------------------------------------------ execute
    def step(self, db: DeviceBatch, stream=None):
        """One training step on `stream` (default: the runtime's own non-blocking
        compute stream, ordered after and before the caller's current stream).
        The legacy default stream is never used as the compute stream: it takes part
        in implicit cross-stream synchronisation."""
        if stream is not None:
            L.call("bm_step", self.ctx, C.byref(db.struct), C.c_void_p(stream.cuda_stream))
            return
        cur = torch.cuda.current_stream(self.device)
        if os.environ.get("BM_CALLER_STREAM") == "1":   # triage: run on the caller's stream
            L.call("bm_step", self.ctx, C.byref(db.struct), C.c_void_p(cur.cuda_stream))
            return
        if self._stream is None:
            self._stream = torch.cuda.Stream(self.device)
        self._stream.wait_stream(cur)
        L.call("bm_step", self.ctx, C.byref(db.struct), C.c_void_p(self._stream.cuda_stream))
        cur.wait_stream(self._stream)

    def pull_bytes(self) -> int:
        """Bytes pulled from peers' FSDP shards in the last step."""
        n = C.c_int64()
        L.call("bm_ctx_pull_bytes", self.ctx, C.byref(n))
        return n.value

    def step_wait(self, timeout_s: float = 0.0):
        """Block until the last step finished; BigMacError(E_TIMEOUT) naming the blocked
        op if it did not within timeout_s seconds (<= 0: no limit)."""
        L.call("bm_step_wait", self.ctx, int(timeout_s * 1000))

    def loss_tensor(self) -> torch.Tensor:
        p = C.c_void_p()
        L.call("bm_ctx_loss_ptr", self.ctx, C.byref(p))
        base = self._work.data_ptr()
        off = p.value - base
        return self._work[off:off + (2 * self.M + 1) * 4].view(torch.float32)

    def losses(self):
        t = self.loss_tensor().double().cpu().numpy()
        M = self.M
        return float(t[2 * M]), t[:M].copy(), t[M:2 * M].copy()

    def launch_count(self) -> int:
        n = C.c_int64()
        L.call("bm_ctx_launch_count", self.ctx, C.byref(n))
        return n.value

    def stash_peak(self):
        a = (C.c_int64 * 3)()
        L.call("bm_ctx_stash_peak", self.ctx, a)
        return list(a)

    def close(self):
        """Destroy the context and release its device buffers (the caller must not use
        views such as grads_t / weights_t afterwards)."""
        if getattr(self, "ctx", None):
            torch.cuda.synchronize(self.device)
            L.lib().bm_ctx_destroy(self.ctx)
            self.ctx = None
            for k in ("_w", "_g", "_work", "_comm", "weights_t", "grads_t", "_stream"):
                if hasattr(self, k):
                    setattr(self, k, None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
