"""Python view of the C++ schedule builder (bm_build_schedule, include/bigmac.h)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib as L

# bm_op_kind names (include/bigmac.h)
KINDS = ("EncFwd", "EncBwd", "LlmFwd", "LlmBwd", "GenFwd", "GenBwd", "Send", "Recv", "LlmW")
PAYLOADS = ("act", "grad", "emb", "embgrad", "genin", "gengrad")


@dataclass
class Sched:
    handle: int
    P: int

    def __del__(self):
        try:
            if self.handle:
                L.lib().bm_schedule_free(self.handle)
                self.handle = 0
        except Exception:
            pass

    def ops(self, rank: int):
        p = C.POINTER(L.Op)()
        n = C.c_int64()
        L.call("bm_schedule_rank_ops", self.handle, rank, C.byref(p), C.byref(n))
        return [(p[i].kind, p[i].mb, p[i].chunk, p[i].unit, p[i].peer, p[i].payload, p[i].slot, p[i].seq)
                for i in range(n.value)]

    def stats(self, rank: int) -> L.SchedStats:
        st = L.SchedStats()
        L.call("bm_schedule_stats", self.handle, rank, C.byref(st))
        return st

    def ring(self, src: int, dst: int, payload: int):
        K, n = C.c_int32(), C.c_int32()
        L.call("bm_schedule_ring", self.handle, src, dst, payload, C.byref(K), C.byref(n))
        return K.value, n.value

    def serialize(self) -> str:
        need = C.c_size_t()
        L.call("bm_schedule_serialize", self.handle, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        L.call("bm_schedule_serialize", self.handle, buf, need.value, C.byref(need))
        return buf.value.decode()


def make_cfg(P, M, V=1, warmup_units=0, llm_sched=None, enc_place="dp_unit", gen_place="dp_shard",
             cost_fwd=1, cost_bwd=2, ring_slack=1, enc_exclude=0, cost_wgrad=0, llm_cp=1, enc_cp=1) -> L.SchedCfg:
    if llm_sched is None:
        llm_sched = "1f1b" if V == 1 else "interleaved"
    c = L.SchedCfg()
    c.stages, c.microbatches, c.vchunks, c.warmup_units = P, M, V, warmup_units
    c.llm_sched = L.LLM_SCHED[llm_sched]
    c.enc_place = L.ENC_PLACE[enc_place]
    c.gen_place = L.GEN_PLACE[gen_place]
    c.cost_fwd, c.cost_bwd, c.ring_slack = cost_fwd, cost_bwd, ring_slack
    c.enc_exclude = enc_exclude
    c.cost_wgrad = cost_wgrad
    c.llm_cp, c.enc_cp = llm_cp, enc_cp
    return c


def build(P, M, V=1, **kw) -> Sched:
    cfg = make_cfg(P, M, V, **kw)
    h = C.c_void_p()
    L.call("bm_build_schedule", C.byref(cfg), C.byref(h))
    return Sched(h.value, P * max(cfg.llm_cp, 1))
