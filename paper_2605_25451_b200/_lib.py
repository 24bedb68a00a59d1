"""Thin ctypes binding of libbigmac.so (include/bigmac.h, include/bigmac_kernels.h).

Argument marshalling only: every step of the hot path runs in the library's
kernels.  There is no fallback: if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbigmac.so")

BM_OK = 0
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_REMAINDER", 3: "E_WARMUP", 4: "E_DEPENDENCY", 5: "E_DEADLOCK",
          6: "E_CUDA", 7: "E_NCCL", 8: "E_OOM", 9: "E_STATE", 10: "E_TIMEOUT"}
BF16, F32 = 0, 1
EPI_STORE, EPI_ACCUM, EPI_ADD = 0, 1, 2
OP_KINDS = ["EncFwd", "EncBwd", "LlmFwd", "LlmBwd", "GenFwd", "GenBwd", "Send", "Recv", "LlmW"]
PAYLOADS = ["act", "grad", "emb", "embgrad", "genin", "gengrad"]
LLM_SCHED = {"1f1b": 0, "interleaved": 1, "zb_h1": 2}
ENC_PLACE = {"none": 0, "dp_unit": 1, "entry_stage": 2}
GEN_PLACE = {"none": 0, "dp_shard": 1, "last_stage": 2}
HEAD_PLACE = {"auto": 0, "last_stage": 1, "dp_shard": 2}
FSDP = {"off": 0, "pull": 1, "allgather": 2}


class BigMacError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class SchedCfg(C.Structure):
    _fields_ = [("stages", C.c_int32), ("microbatches", C.c_int32), ("vchunks", C.c_int32),
                ("warmup_units", C.c_int32), ("llm_sched", C.c_int32), ("enc_place", C.c_int32),
                ("gen_place", C.c_int32), ("cost_fwd", C.c_int32), ("cost_bwd", C.c_int32),
                ("ring_slack", C.c_int32), ("enc_exclude", C.c_int32), ("cost_wgrad", C.c_int32),
                ("llm_cp", C.c_int32), ("enc_cp", C.c_int32), ("reserved", C.c_int32 * 2)]


class Op(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "mb", "chunk", "unit", "peer", "payload", "slot", "seq")]


class SchedStats(C.Structure):
    _fields_ = [("w_star", C.c_int32), ("warmup_units", C.c_int32), ("peak_enc_units", C.c_int32),
                ("peak_gen_shards", C.c_int32), ("peak_llm_inflight", C.c_int32), ("n_ops", C.c_int32),
                ("llm_idle_cost_units", C.c_int64), ("makespan_cost_units", C.c_int64),
                ("ring_slots", C.c_int32 * 6)]


class ModelCfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("S", "d_in", "d_e", "f_e", "L_e", "d", "f", "L", "vocab",
                                         "d_g", "f_g", "L_g", "d_t", "dtype", "max_n_mod", "max_n_gen",
                                         "head_place", "last_stage_layers", "fsdp", "gen_exclude",
                                         "stage_halves", "enc_stream")] + \
               [("reserved", C.c_int32 * 2), ("stage_layers", C.c_int32 * 32)]


class ParamInfo(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("rows", C.c_int32), ("cols", C.c_int32), ("offset", C.c_int64),
                ("kind", C.c_int32), ("ld", C.c_int32)]


class CtxSizes(C.Structure):
    _fields_ = [("weight_bytes", C.c_int64), ("grad_bytes", C.c_int64), ("work_bytes", C.c_int64),
                ("comm_bytes", C.c_int64)]


class Buffers(C.Structure):
    _fields_ = [("weights", C.c_void_p), ("grads", C.c_void_p), ("work", C.c_void_p), ("comm", C.c_void_p),
                ("weight_bytes", C.c_int64), ("grad_bytes", C.c_int64), ("work_bytes", C.c_int64),
                ("comm_bytes", C.c_int64)]


class GemmDesc(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("A", C.c_void_p), ("lda", C.c_int64),
                ("a_major", C.c_int32), ("B", C.c_void_p), ("ldb", C.c_int64), ("b_major", C.c_int32),
                ("C", C.c_void_p), ("ldc", C.c_int64), ("c_dtype", C.c_int32), ("epilogue", C.c_int32),
                ("R", C.c_void_p), ("ldr", C.c_int64), ("alpha", C.c_float), ("f", C.c_int32)]


class TraceRec(C.Structure):
    _fields_ = [("op", C.c_int32), ("kind", C.c_int32), ("stream", C.c_int32), ("mb", C.c_int32),
                ("t_start_ms", C.c_float), ("t_end_ms", C.c_float)]


class Batch(C.Structure):
    _fields_ = [("M", C.c_int32), ("n_mod", C.c_void_p), ("n_gen", C.c_void_p), ("patches", C.c_void_p),
                ("ld_patch", C.c_int32), ("ids", C.c_void_p), ("labels", C.c_void_p), ("targets", C.c_void_p),
                ("on_host", C.c_int32), ("reserved", C.c_int32 * 7)]


# (name, restype, argtypes); restype None => returns bm_status
_P, _I32, _I64, _F, _SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_size_t
SIGNATURES = {
    # bigmac.h
    "bm_build_schedule": [C.POINTER(SchedCfg), C.POINTER(_P)],
    "bm_schedule_rank_ops": [_P, _I32, C.POINTER(C.POINTER(Op)), C.POINTER(_I64)],
    "bm_schedule_stats": [_P, _I32, C.POINTER(SchedStats)],
    "bm_schedule_ring": [_P, _I32, _I32, _I32, C.POINTER(_I32), C.POINTER(_I32)],
    "bm_schedule_serialize": [_P, C.c_char_p, _SZ, C.POINTER(_SZ)],
    "bm_schedule_free": [_P],
    "bm_last_error": [],
    "bm_param_count": [C.POINTER(ModelCfg), C.POINTER(SchedCfg), _I32, C.POINTER(_I32), C.POINTER(_I64),
                       C.POINTER(_I64)],
    "bm_param_info_get": [C.POINTER(ModelCfg), C.POINTER(SchedCfg), _I32, _I32, C.POINTER(ParamInfo)],
    "bm_ctx_create": [C.POINTER(ModelCfg), _P, _I32, C.POINTER(_P)],
    "bm_ctx_sizes_get": [_P, C.POINTER(CtxSizes)],
    "bm_ctx_bind": [_P, C.POINTER(Buffers)],
    "bm_ipc_export": [_P, C.POINTER(C.c_uint8), C.POINTER(_I64)],
    "bm_ctx_open_peer": [_P, _I32, C.POINTER(C.c_uint8), _I64],
    "bm_nccl_unique_id": [C.POINTER(C.c_uint8)],
    "bm_ctx_init_nccl": [_P, C.POINTER(C.c_uint8), _I32, _I32],
    "bm_ctx_init_replicas": [_P, _I32, _I32, C.POINTER(C.c_uint8), C.POINTER(C.c_uint8)],
    "bm_ctx_init_fsdp": [_P, C.POINTER(C.c_uint8), C.POINTER(_I64)],
    "bm_ctx_dp_shard": [_P, C.POINTER(_I64), C.POINTER(_I64)],
    "bm_ctx_pull_bytes": [_P, C.POINTER(_I64)],
    "bm_ctx_init_peer_sum": [_P, _I32, _I32, C.POINTER(C.c_uint8), C.POINTER(_I64), C.POINTER(C.c_uint8),
                             C.POINTER(_I64)],
    "bm_step": [_P, C.POINTER(Batch), _P],
    "bm_step_wait": [_P, _I64],
    "bm_ctx_loss_ptr": [_P, C.POINTER(_P)],
    "bm_ctx_launch_count": [_P, C.POINTER(_I64)],
    "bm_ctx_stash_peak": [_P, C.POINTER(_I64)],
    "bm_ctx_set_timing": [_P, _I32],
    "bm_ctx_gemm_stats": [_P, C.POINTER(_I64), C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "bm_ctx_comm_stats": [_P, C.POINTER(_I64), C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "bm_ctx_set_trace": [_P, _I32],
    "bm_ctx_trace_get": [_P, _P, _I64, C.POINTER(_I64), C.POINTER(_I64)],
    "bm_ctx_debug_dump": [_P, C.c_char_p, _SZ],
    "bm_ctx_destroy": [_P],
    # bigmac_kernels.h
    "bm_k_gemm": [_I32, _I32, _I32, _I32, _P, _I64, _I32, _P, _I64, _I32, _P, _I64, _I32, _I32, _P, _I64, _F, _P],
    "bm_k_gemm_mode": [_I32],
    "bm_k_gemm_bn512": [_I32],
    "bm_k_gemm_bk128": [_I32],
    "bm_k_gemm_swiglu_bk128": [_I32],
    "bm_k_gemm_group": [C.POINTER(GemmDesc), _I32, _P],
    "bm_k_gemm_swiglu": [_I32, _I32, _I32, _P, _I64, _P, _I64, _P, _P, _P],
    "bm_k_gemm_dswiglu": [_I32, _I32, _I32, _P, _I64, _P, _I64, _P, _P, _P],
    "bm_k_rmsnorm_fwd": [_I32, _I32, _I32, _P, _P, _P, _P, _P],
    "bm_k_rmsnorm_bwd": [_I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "bm_k_rmsnorm_bwd_scratch": [_I32, _I32],
    "bm_k_swiglu_fwd": [_I32, _I32, _I32, _P, _P, _P],
    "bm_k_swiglu_bwd": [_I32, _I32, _I32, _P, _P, _P, _P],
    "bm_k_gelu_fwd": [_I32, _I64, _P, _P, _P],
    "bm_k_gelu_bwd": [_I32, _I64, _P, _P, _P, _P],
    "bm_k_embed_fwd": [_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P],
    "bm_k_embed_bwd": [_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P],
    "bm_k_embed_bwd_scratch": [_I32],
    "bm_k_ce_fwd_bwd": [_I32, _I32, _I32, _P, _P, _F, _P, _F, _I32, _P, _P],
    "bm_k_mse_fwd_bwd": [_I32, _I32, _I32, _P, _P, _F, _F, _F, _P, _P, _P],
    "bm_k_add": [_I32, _I64, _P, _P, _P, _P],
    "bm_k_cast": [_I32, _I32, _I64, _P, _P, _P],
    "bm_k_copy": [_P, _P, _I64, _I32, _P],
    "bm_k_zero": [_P, _I64, _P],
    "bm_k_preload": [],
}
RESTYPE = {"bm_last_error": C.c_char_p, "bm_schedule_free": None, "bm_ctx_destroy": None,
           "bm_k_rmsnorm_bwd_scratch": C.c_int64, "bm_k_embed_bwd_scratch": C.c_int64}

_lib = None
MISSING: list = []   # declared in include/*.h but not exported (tests assert empty)


def lib():
    """Load libbigmac.so (raises if it has not been built; no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2605_25451_b200.build`")
        try:  # make torch's libnccl.so.2 resolvable for the lazy dlopen inside the library
            import torch  # noqa: F401
        except Exception:
            pass
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, args in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:
                MISSING.append(name)
                continue
            fn.argtypes = args
            fn.restype = RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def check(status: int):
    if status != BM_OK:
        msg = lib().bm_last_error()
        raise BigMacError(status, msg.decode() if msg else "")


def call(name, *args):
    check(getattr(lib(), name)(*args))
