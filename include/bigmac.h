/*
 * bigmac.h -- C ABI of the B200-native BigMac nested-pipeline step.
 *
 * Paper: "BigMac" (arxiv 2605.25451), PAPER.md line numbers cited as P:<line>.
 * The paper's statement of the problem is
 *     train_step(data_iter, pp_size, microbatch_num, warmup_bound)
 *       = get_llm_schedule -> build_schedule -> insert_comm_ops
 *         -> deadlock_check -> create_executor -> load_schedule -> execute
 * This header exposes exactly those steps:
 *     bm_build_schedule       get_llm_schedule + build_schedule + insert_comm_ops
 *                             + deadlock_check (+ receive-ring sizing)
 *     bm_ctx_create/_bind     create_executor + load_schedule
 *     bm_step                 execute (one training step of the nested pipeline) P:323
 *
 * Conventions
 *   - Every function returns bm_status; on failure bm_last_error() returns a
 *     thread-local message valid until the next bm_* call on that thread.
 *   - No C++ exceptions cross this boundary.  No torch types appear here.
 *   - "device pointer" = CUDA global memory of the calling process's current
 *     device; "host pointer" = ordinary (preferably pinned) host memory.
 *   - The library owns bm_schedule and bm_ctx objects; it never frees memory
 *     it did not allocate.  All large device buffers (weights, grads,
 *     workspace, receive arena) are allocated by the caller and bound with
 *     bm_ctx_bind.
 */
#ifndef BIGMAC_H
#define BIGMAC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BM_OK = 0,
  BM_E_INVALID = 1,     /* bad ranges / inconsistent arguments                       */
  BM_E_REMAINDER = 2,   /* M % P != 0: units of pp_size micro-batches */
  BM_E_WARMUP = 3,      /* W < W*: some F_u precedes EncFwd(u)         */
  BM_E_DEPENDENCY = 4,  /* verification failed (should be unreachable)               */
  BM_E_DEADLOCK = 5,    /* happens-before graph incl. credit edges is cyclic */
  BM_E_CUDA = 6,
  BM_E_NCCL = 7,
  BM_E_OOM = 8,         /* a bound buffer is smaller than required                   */
  BM_E_STATE = 9,       /* call out of order (e.g. bm_step before bm_ctx_bind)      */
  BM_E_TIMEOUT = 10
} bm_status;

/* BM_LLM_ZB_H1: zero-bubble ZB-H1 (the schedule class P:552-556 names as the
 * extension; construction DESIGN.md R23): each backward is split into B (input
 * gradient, BM_OP_LLM_BWD) and W (weight gradient, BM_OP_LLM_W); V must be 1. */
typedef enum { BM_LLM_1F1B = 0, BM_LLM_INTERLEAVED = 1, BM_LLM_ZB_H1 = 2 } bm_llm_sched;
/* BM_ENC_DP_UNIT: BigMac (units of P microbatches, one per rank).
 * BM_ENC_ENTRY_STAGE: memory-efficient baseline (Fig. 3): the
 * encoder runs as the entry stage's first layers -- EncFwd(m) right before
 * F(m, 0) and EncBwd(m) right after B(m, 0) on rank 0.  (The compute-efficient
 * baseline of P:129-138 is BM_ENC_DP_UNIT with warmup_units = M / P.) */
typedef enum { BM_ENC_NONE = 0, BM_ENC_DP_UNIT = 1, BM_ENC_ENTRY_STAGE = 2 } bm_enc_place;
typedef enum { BM_GEN_NONE = 0, BM_GEN_DP_SHARD = 1, BM_GEN_LAST_STAGE = 2 } bm_gen_place;

typedef enum {
  BM_OP_ENC_FWD = 0, BM_OP_ENC_BWD = 1, BM_OP_LLM_FWD = 2, BM_OP_LLM_BWD = 3,
  BM_OP_GEN_FWD = 4, BM_OP_GEN_BWD = 5, BM_OP_SEND = 6, BM_OP_RECV = 7,
  BM_OP_LLM_W = 8   /* weight-gradient half of an LLM backward (BM_LLM_ZB_H1 only) */
} bm_op_kind;   /* compute vs communication operators */

typedef enum {
  BM_PAY_NONE = -1,
  BM_PAY_ACT = 0,      /* LLM stage-boundary activation, stage s -> s+1  */
  BM_PAY_GRAD = 1,     /* LLM stage-boundary gradient, s -> s-1              */
  BM_PAY_EMB = 2,      /* encoder output gathered to the entry stage          */
  BM_PAY_EMBGRAD = 3,  /* input-embedding gradient scattered to the encoder rank */
  BM_PAY_GENIN = 4,    /* last stage scatters generator inputs                */
  BM_PAY_GENGRAD = 5   /* generator input-gradients gathered back             */
} bm_payload;

/* Scheduler configuration (pp_size, microbatch_num, warmup_bound).
 * warmup_units == 0 selects W* (the minimal dependency-safe warmup, R4).
 * cost_fwd:cost_bwd is the cut-timeline cost ratio that defines "columns"
 * (R1), default 1:2.  ring_slack adds receive slots
 * above the minimal deadlock-free ring size.  cost_wgrad (BM_LLM_ZB_H1 only) is
 * the W share of cost_bwd (B costs cost_bwd - cost_wgrad); 0 selects
 * cost_bwd / 2; B and W must both cost >= 1, else BM_E_INVALID. */
typedef struct {
  int32_t stages;        /* P >= 1                       */
  int32_t microbatches;  /* M >= 1, M % P == 0           */
  int32_t vchunks;       /* V >= 1 (V >= 2 iff interleaved) */
  int32_t warmup_units;  /* W >= 0; 0 => W*              */
  int32_t llm_sched;     /* bm_llm_sched                 */
  int32_t enc_place;     /* bm_enc_place                 */
  int32_t gen_place;     /* bm_gen_place                 */
  int32_t cost_fwd;      /* >= 1                         */
  int32_t cost_bwd;      /* >= 1                         */
  int32_t ring_slack;    /* >= 0                         */
  int32_t enc_exclude;   /* bit mask of ranks that run no encoder microbatch (below) */
  int32_t cost_wgrad;    /* >= 0; zero-bubble W cost (0 => cost_bwd / 2) */
  int32_t llm_cp;        /* LLM context-parallel degree (0 => 1; below)     */
  int32_t enc_cp;        /* encoder context-parallel degree (0 => 1)        */
  int32_t reserved[2];   /* must be zero                 */
} bm_sched_cfg;
/* enc_exclude (BM_ENC_DP_UNIT): unit u's microbatch uP + r runs on rank r,
 * unless r is in the mask: then on the nearest lower rank not in it, cyclically
 * (reading R22).  That rank runs two (or more) EncFwd / EncBwd ops per
 * unit, in microbatch order, and sends / receives their emb / embgrad messages;
 * the masked ranks run none.  Used to keep the encoder off the pipeline stage
 * that paces the step. */

/* Decoupled context parallelism (R25), schedule level:
 * llm_cp > 1 or enc_cp > 1 builds the nested schedule for P * llm_cp ranks,
 * rank c P + r = LLM CP index c of stage r (the llm_cp ranks of a stage run the
 * stage's LLM list in lockstep on their sequence shards).  The encoder runs in CP
 * groups of enc_cp consecutive ranks, one microbatch per group, so an encoder unit
 * has P llm_cp / enc_cp microbatches (M must be a multiple: BM_E_REMAINDER); the
 * CP-conversion all-to-all appears as emb messages from every rank of a
 * microbatch's encoder group to every stage-0 rank (c P) and embgrad messages
 * back.  Requires 1 <= enc_cp <= llm_cp, enc_cp | P llm_cp, enc_place NONE or
 * DP_UNIT, gen_place NONE or LAST_STAGE, enc_exclude 0 (else BM_E_INVALID).  The
 * executor (bm_ctx_create) runs llm_cp = enc_cp = 1 schedules only. */

/* One operator of a rank's list.  -1 marks an absent field.
 *   EncFwd/EncBwd: mb = unit*P + rank, unit
 *   LlmFwd/LlmBwd/LlmW: mb, chunk
 *   GenFwd/GenBwd: mb (row shard = rank under BM_GEN_DP_SHARD)
 *   Send/Recv:     mb, chunk (act/grad), unit (emb/embgrad), peer, payload,
 *                  slot (= seq mod ring size), seq (per-channel message index) */
typedef struct {
  int32_t kind, mb, chunk, unit, peer, payload, slot, seq;
} bm_op;

typedef struct {
  int32_t w_star;             /* minimal warmup (P:216 analysis)                  */
  int32_t warmup_units;       /* W used                                            */
  int32_t peak_enc_units;     /* max live EncFwd-EncBwd on this rank (<= W) */
  int32_t peak_gen_shards;    /* max live GenFwd-GenBwd (1)                */
  int32_t peak_llm_inflight;  /* max live LLM F-B (F-W under ZB-H1)        */
  int32_t n_ops;              /* ops incl. comm on this rank                       */
  int64_t llm_idle_cost_units;/* makespan - busy in the cut-timeline DES           */
  int64_t makespan_cost_units;
  int32_t ring_slots[6];      /* max receive ring size per payload on this rank   */
} bm_sched_stats;

typedef struct bm_schedule bm_schedule;

/* Build, nest, insert comm ops, size rings and verify.  *out is owned by the
 * library; free with bm_schedule_free.  Pure and reentrant. */
bm_status bm_build_schedule(const bm_sched_cfg* cfg, bm_schedule** out);
/* Borrowed view of rank's op list; valid until bm_schedule_free. */
bm_status bm_schedule_rank_ops(const bm_schedule* s, int32_t rank, const bm_op** ops, int64_t* n);
bm_status bm_schedule_stats(const bm_schedule* s, int32_t rank, bm_sched_stats* out);
/* Ring size K and message count of channel (src -> dst, payload); K = nmsg = 0 if absent. */
bm_status bm_schedule_ring(const bm_schedule* s, int32_t src, int32_t dst, int32_t payload,
                           int32_t* K, int32_t* nmsg);
/* Text serialization "rank\tindex\tkind\tmb\tchunk\tunit\tpeer\tpayload\tslot\tseq\n"
 * ('-' = absent).  Call with cap = 0 to get *needed (bytes incl. the NUL). */
bm_status bm_schedule_serialize(const bm_schedule* s, char* buf, size_t cap, size_t* needed);
void bm_schedule_free(bm_schedule* s);
const char* bm_last_error(void);

/* ------------------------------------------------------------------------ */
/* Synthetic MLLM model: encoder + projector (DP),      */
/* LLM (pipeline stages), generator (DP row shards).                        */
/* ------------------------------------------------------------------------ */
typedef enum { BM_BF16 = 0, BM_F32 = 1 } bm_dtype;
#define BM_MAX_VSTAGES 32   /* P * V bound of an explicit layer partition */

typedef struct {
  int32_t S;                      /* LLM sequence length                      */
  int32_t d_in, d_e, f_e, L_e;    /* encoder                                  */
  int32_t d, f, L, vocab;         /* LLM (d is also the projector width)      */
  int32_t d_g, f_g, L_g, d_t;     /* generator                                */
  int32_t dtype;                  /* bm_dtype of weights/activations           */
  int32_t max_n_mod, max_n_gen;   /* upper bounds on per-sample row counts     */
  int32_t head_place;             /* bm_head_place                             */
  int32_t last_stage_layers;      /* LLM layers of the last virtual stage; 0 = uniform (below) */
  int32_t fsdp;                   /* bm_fsdp_mode of the encoder / generator parameters */
  int32_t gen_exclude;            /* bit mask of ranks that take no generator rows (below) */
  int32_t stage_halves;           /* 1: stage_layers counts half-layer units (below) */
  int32_t enc_stream;             /* encoder ops on their own stream: 0 = auto (P == 1), 1 = on, 2 = off */
  int32_t reserved[2];            /* must be zero                              */
  int32_t stage_layers[BM_MAX_VSTAGES]; /* explicit partition (below); all 0 = unset */
} bm_model_cfg;

/* LLM layer partition over the P V virtual stages (s = chunk P + rank), in
 * layer order.  stage_layers[0] != 0: virtual stage s holds stage_layers[s]
 * layers (P V <= BM_MAX_VSTAGES, every entry >= 1, sum = L; last_stage_layers
 * ignored).  Otherwise, last_stage_layers = 0: L / (P V) layers each
 * (L % (P V) == 0 required).  last_stage_layers = n > 0: virtual stage P V - 1 (which also
 * runs the LM head + CE under BM_HEAD_LAST_STAGE) gets n layers; the other
 * P V - 1 stages split the remaining L - n as evenly as possible, the first
 * (L - n) mod (P V - 1) stages one layer more.  Requires 1 <= n and
 * L - n >= P V - 1 (every stage holds a layer).  Uneven splits balance the
 * head's cost; op lists do not depend on the partition.
 * stage_halves = 1 (with stage_layers set): each layer l is two units, A_l =
 * RMSNorm + gate_up GEMM + SwiGLU and B_l = down GEMM + residual (2/3 and 1/3 of
 * its FLOPs), and stage_layers[s] counts units (every entry >= 1, sum = 2 L), so a
 * stage boundary may fall inside a layer: the stage-boundary message is then
 * [x_l | h_l] (S x (d + f)) forward and [dx_{l+1} | dh_l] backward, and layer l's
 * norm / gate_up live on the earlier stage, its down on the later one (DESIGN.md
 * reading R24).  The first virtual stage cannot start and the last cannot end
 * inside a layer. */

/* gen_exclude (BM_GEN_DP_SHARD): rank r with bit r set takes no generator rows;
 * microbatch m's n_gen rows are split into equal shards over the other ranks in
 * rank order.  The generator is token-wise, so any row partition computes the same
 * loss and gradients (reading R20); excluding the busiest pipeline stage keeps the
 * generator's kernels off the stage that paces the pipeline.  Op lists are
 * unchanged (an excluded rank's GenFwd / GenBwd are empty, its genin / gengrad
 * messages carry no rows). */

/* Where the final-norm output's LM head + cross-entropy (fwd and bwd) run.
 * BM_HEAD_LAST_STAGE: in F(m, V-1) on rank P-1, as in the paper's Megatron
 *   setting.
 * BM_HEAD_DP_SHARD: the head is token-wise like the generator, so it rides on
 *   the DP-sharded generator ops (reading R14): rank r's GenFwd(m)
 *   computes the logits, CE and dHn of text rows
 *   [n_mod + floor(r n_text / P), n_mod + floor((r+1) n_text / P)),
 *   n_text = S - n_mod, with the full-microbatch CE denominator; the genin
 *   message carries [head rows | generator rows] of Hn, the gengrad message
 *   [dHn head rows | generator dX rows].  llm.head becomes a DP parameter
 *   (every rank, summed by the step-end allreduce).  Requires
 *   gen_place == BM_GEN_DP_SHARD.  Schedules (op lists) are unchanged.
 * BM_HEAD_AUTO: BM_HEAD_LAST_STAGE (measured faster at C2, N = 2: a remote
 *   head shard competes with that rank's running LLM op, and the last stage
 *   waits for it -- profiles/r01/traces/trace_n2_m32_*.summary.json). */
typedef enum { BM_HEAD_AUTO = 0, BM_HEAD_LAST_STAGE = 1, BM_HEAD_DP_SHARD = 2 } bm_head_place;

/* Encoder / generator parameters under FSDP.
 * BM_FSDP_OFF: every rank holds them in full (plain data parallelism; gradients
 *   summed at step end).
 * BM_FSDP_PULL: BigMac's one-sided pull.  The DP parameters (the prefix
 *   [0, dp_elems) of the parameter space) are sharded over the P ranks of the
 *   pipeline: rank r stores only elements [lo_r, hi_r) (bm_ctx_dp_shard; 4-element
 *   aligned near-equal chunks) at the start of its weights buffer, followed by its
 *   LLM parameters.  Every encoder / generator op materialises its parameters block
 *   by block (patch, each residual block, projector; generator in / blocks / out)
 *   into two bucket slots, reading each shard directly from its owner's weights
 *   buffer over NVLink (CUDA IPC, copy engine on a pull stream) while the previous
 *   block computes -- the owners take no part, so ranks proceed on their own
 *   schedules (no all-gather barrier).  Gradients are accumulated locally and
 *   reduce-scattered at step end: after bm_step only this rank's shard of the DP
 *   gradients is valid (all of it under the NCCL step-end sum, which all-reduces).
 * BM_FSDP_ALLGATHER: the paper's baseline: the same buckets, but each pull is
 *   preceded by a barrier of the pipeline group on the op's stream -- FSDP's
 *   all-gather synchronisation point -- and runs on that stream.
 *   Requires BM_ENC_DP_UNIT and BM_GEN_DP_SHARD (every rank in every op).
 * FSDP needs D = 1 and a head that is not DP-sharded. */
typedef enum { BM_FSDP_OFF = 0, BM_FSDP_PULL = 1, BM_FSDP_ALLGATHER = 2 } bm_fsdp_mode;

/* Parameter kinds: DP parameters (encoder, projector, generator) are summed
 * over ranks at step end; LLM parameters belong to one stage. */
typedef enum { BM_PARAM_DP = 0, BM_PARAM_LLM = 1 } bm_param_kind;

typedef struct {
  char name[48];      /* synth.param_specs name, e.g. "llm.layer3.gate_up" */
  int32_t rows, cols; /* [out, in]; norm gains: rows = n, cols = 1          */
  int64_t offset;     /* element offset into the weight and grad buffers    */
  int32_t kind;       /* bm_param_kind                                      */
  int32_t ld;         /* row stride in elements (cols rounded up to 8)      */
} bm_param_info;

/* Parameters held by `rank` under `sc` (layers of its virtual stages; the
 * text table on rank 0, final norm + head on rank P-1; DP params everywhere;
 * under BM_HEAD_DP_SHARD llm.head is a DP parameter).
 * DP parameters occupy the prefix [0, *dp_elems) of the buffers. */
bm_status bm_param_count(const bm_model_cfg* mc, const bm_sched_cfg* sc, int32_t rank,
                         int32_t* n, int64_t* total_elems, int64_t* dp_elems);
bm_status bm_param_info_get(const bm_model_cfg* mc, const bm_sched_cfg* sc, int32_t rank,
                            int32_t idx, bm_param_info* out);

/* ------------------------------------------------------------------------ */
/* Executor                                                     */
/* ------------------------------------------------------------------------ */
typedef struct bm_ctx bm_ctx;

typedef struct {
  int64_t weight_bytes;  /* total_elems * sizeof(dtype)                          */
  int64_t grad_bytes;    /* total_elems * 4 (fp32 accumulation)                  */
  int64_t work_bytes;    /* activations stash, scratch, per-step batch staging   */
  int64_t comm_bytes;    /* receive slots + flags, exported to peers via IPC     */
} bm_ctx_sizes;

typedef struct {
  void* weights;   /* device, weight_bytes, filled by the caller                 */
  void* grads;     /* device, grad_bytes (zeroed by bm_step)                     */
  void* work;      /* device, work_bytes                                         */
  void* comm;      /* device, comm_bytes (zeroed by the caller before binding)   */
  /* the caller's allocation sizes in bytes; bm_ctx_bind returns BM_E_OOM if any
   * is smaller than bm_ctx_sizes_get's requirement */
  int64_t weight_bytes, grad_bytes, work_bytes, comm_bytes;
} bm_buffers;

/* Create the per-rank executor for `rank` of schedule s (s must outlive ctx). */
bm_status bm_ctx_create(const bm_model_cfg* mc, const bm_schedule* s, int32_t rank, bm_ctx** out);
bm_status bm_ctx_sizes_get(const bm_ctx* c, bm_ctx_sizes* out);
/* Binds the caller's buffers (256-byte aligned, sizes >= bm_ctx_sizes_get).
 * Errors: BM_E_INVALID (null / misaligned), BM_E_OOM (a buffer is too small; the
 * message names it and both sizes), BM_E_STATE (P > 1 and the environment variable
 * CUDA_DEVICE_MAX_CONNECTIONS unset or < P + 6: every stream of the rank needs its
 * own hardware queue, and it must be set before the CUDA context exists),
 * BM_E_CUDA. */
bm_status bm_ctx_bind(bm_ctx* c, const bm_buffers* b);

/* Peer memory (CUDA IPC over NVLink).  Export any device pointer as a 64-byte
 * handle + byte offset into its allocation; peers import it with
 * bm_ctx_open_peer (their `comm` buffer).  Exchange is done by the caller. */
bm_status bm_ipc_export(const void* dptr, uint8_t handle[64], int64_t* offset);
bm_status bm_ctx_open_peer(bm_ctx* c, int32_t peer, const uint8_t handle[64], int64_t offset);

/* FSDP (bm_model_cfg.fsdp != BM_FSDP_OFF): map the pipeline peers' weights buffers
 * (bm_ipc_export handles [P][64] and byte offsets [P], own entry ignored) for the
 * one-sided pulls.  Call after bm_ctx_bind.  Errors: BM_E_INVALID, BM_E_CUDA. */
bm_status bm_ctx_init_fsdp(bm_ctx* c, const uint8_t* weight_handles, const int64_t* weight_offsets);
/* This rank's shard [*lo, *hi) of the DP parameter elements (the whole prefix
 * [0, dp_elems) without FSDP).  Its weights buffer stores element e of the shard
 * at element e - lo; LLM parameter element e (>= dp_elems) at e - dp_elems + (hi - lo). */
bm_status bm_ctx_dp_shard(const bm_ctx* c, int64_t* lo, int64_t* hi);
/* Bytes this rank pulled from peers' shards during its last bm_step (FSDP). */
bm_status bm_ctx_pull_bytes(const bm_ctx* c, int64_t* bytes);

/* Data-parallel gradient sum over the P ranks (NCCL).  Rank 0 creates
 * the id, the caller broadcasts it. */
bm_status bm_nccl_unique_id(uint8_t id[128]);
bm_status bm_ctx_init_nccl(bm_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank);

/* Pipeline replicas ("if G > P, pipeline replicas are added,
 * with an allreduce of LLM stage grads across replicas of the same stage").
 * G = P * D processes; this context is stage `rank` (bm_ctx_create) of
 * replica `replica` in [0, D), and runs its own M microbatches (global batch
 * M * D).  id_world: one NCCL id shared by all P * D processes (communicator
 * rank replica * P + stage) for the DP parameters (encoder, projector,
 * generator); id_stage: one id shared by the D processes of this stage
 * (communicator rank = replica) for this stage's LLM parameters.  Call after
 * bm_ctx_init_nccl (the replica's own pipeline group, which still sums the
 * loss terms; P = 1 needs no pipeline group).  From then on gradients are the
 * mean over the global batch (per-sample scale 1 / (M D)) and the step loss
 * (bm_ctx_loss_ptr element 2M) is the global-batch loss; the per-microbatch
 * terms stay the replica's own.  D = 1 is the plain single-pipeline case.
 * Errors: BM_E_INVALID (D < 1, replica out of range), BM_E_NCCL. */
bm_status bm_ctx_init_replicas(bm_ctx* c, int32_t D, int32_t replica, const uint8_t id_world[128],
                               const uint8_t id_stage[128]);

/* Step-end sums over peer memory instead of NCCL.
 * The library sums the DP parameters' gradients over all P * D processes, each
 * stage's LLM gradients over its D replicas (D > 1), the per-microbatch loss
 * terms over the pipeline and the global-batch loss over everyone, by reading
 * the peers' gradient buffers and peer-sum blocks directly through CUDA IPC:
 * reduce-scatter (process i sums chunk i in process order -- deterministic),
 * all-gather (chunk copies), separated by device-flag barriers
 * (cuStreamWriteValue32 / cuStreamWaitValue32) on the compute stream.
 * Use it when NCCL cannot form the group -- several processes on ONE device
 * (NCCL rejects duplicate GPUs; the single-GPU multi-rank parity fixture) --
 * or to compare with NCCL.  Replaces bm_ctx_init_nccl / bm_ctx_init_replicas
 * (calling both is BM_E_INVALID).
 *   D, replica      pipeline replicas as in bm_ctx_init_replicas (D = 1: one pipeline)
 *   comm_handles    [P D][64] bm_ipc_export handles of every process's `comm`
 *                   buffer, process g = replica * P + stage (own entry ignored)
 *   comm_offsets    [P D] their byte offsets
 *   grad_handles    [P D][64] handles of every process's `grads` buffer
 *   grad_offsets    [P D]
 * Call after bm_ctx_bind and after opening every pipeline peer with
 * bm_ctx_open_peer.  P D <= 64.  Errors: BM_E_INVALID, BM_E_STATE (order),
 * BM_E_CUDA (IPC open failed). */
bm_status bm_ctx_init_peer_sum(bm_ctx* c, int32_t D, int32_t replica, const uint8_t* comm_handles,
                               const int64_t* comm_offsets, const uint8_t* grad_handles,
                               const int64_t* grad_offsets);

/* One step's inputs.  If on_host != 0 the array pointers are host pointers
 * and bm_step copies them to the device inside the step (end-to-end path).
 * Row counts are always host arrays.  All ranks receive the full batch. */
typedef struct {
  int32_t M;
  const int32_t* n_mod;     /* host [M]                                            */
  const int32_t* n_gen;     /* host [M]                                            */
  const void* patches;      /* [sum n_mod, ld_patch] dtype, microbatch-major       */
  int32_t ld_patch;         /* >= d_in, multiple of 8                              */
  const int32_t* ids;       /* [M, S]                                              */
  const int32_t* labels;    /* [M, S]                                              */
  const void* targets;      /* [sum n_gen, d_t] dtype                              */
  int32_t on_host;
  int32_t reserved[7];
} bm_batch;

/* Enqueue one training step on `stream` (cudaStream_t; 0 = legacy default).
 * Asynchronous.  Zeroes grads, runs the rank's op list, allreduces DP grads
 * and the loss terms, and leaves the results in the bound buffers. */
bm_status bm_step(bm_ctx* c, const bm_batch* batch, void* stream);

/* Wait for the step most recently enqueued by bm_step to finish, at most
 * timeout_ms milliseconds (<= 0: wait forever).  Returns BM_OK when it finished.
 * BM_E_TIMEOUT when it did not: the step's device work is blocked on a flag a
 * peer never wrote (a peer died, or the ranks' step counts drifted).  The
 * message then names the first op of this rank whose receive (data flag) or
 * send (ring credit) condition is unmet -- op index, kind, peer, payload,
 * microbatch, the flag value and the value waited for -- or the step-end sum
 * barrier.  The device work stays enqueued: the caller is expected to abort
 * (destroying the CUDA context frees the GPU).  BM_E_CUDA on a device error. */
bm_status bm_step_wait(bm_ctx* c, int64_t timeout_ms);

/* Device pointer to float[2*M + 1]: per-mb CE, per-mb MSE (sums over ranks
 * after bm_step), and the step loss L = (1/M) sum (CE_m + MSE_m). */
bm_status bm_ctx_loss_ptr(const bm_ctx* c, const float** dptr);

/* Number of kernels this rank launched in its last bm_step (kernel census). */
bm_status bm_ctx_launch_count(const bm_ctx* c, int64_t* n);
/* Peak bytes of stash memory live during the last step, per module
 * (0 encoder, 1 LLM, 2 generator) -- the schedule's activation footprint. */
bm_status bm_ctx_stash_peak(const bm_ctx* c, int64_t out[3]);
/* Measurement support (bench.py roofline): when enabled, every GEMM launch of
 * subsequent steps is bracketed by CUDA events on the compute stream.
 * Enabling/disabling resets the totals. */
bm_status bm_ctx_set_timing(bm_ctx* c, int32_t enable);
/* Totals since timing was enabled: GEMM launches, algorithmic FLOPs (2MNK),
 * summed device milliseconds.  Synchronizes on the recorded events. */
bm_status bm_ctx_gemm_stats(bm_ctx* c, int64_t* n_gemm, double* flops, double* ms);
/* Totals since timing was enabled for the peer copies this rank issued
 * (stage-boundary, gather/scatter payloads over NVLink): message count,
 * bytes, summed device milliseconds of the copies on the comm streams. */
bm_status bm_ctx_comm_stats(bm_ctx* c, int64_t* n_msgs, double* bytes, double* ms);
/* Per-op trace of the most recent step (tracing enabled with bm_ctx_set_trace
 * before that step).  One record per compute op (start / end of its kernels on its
 * stream), per receive (the moment its data-flag wait was satisfied on the consuming
 * stream: t_start = t_end) and per send (start / end of the NVLink copy on the comm
 * stream, credit wait included before t_start).  Times are device milliseconds
 * since the step's first event on the compute stream (CUDA events; each rank has
 * its own origin).  stream: 0 compute, 1 generator, 2 + q comm stream to rank q.
 * bm_ctx_trace_get synchronises on the step's last event; *n = records written
 * (at most cap; *total = records available). */
typedef struct {
  int32_t op;       /* index in the rank's op list, -1 for the step tail (allreduce) */
  int32_t kind;     /* bm_op_kind, -1 for the tail */
  int32_t stream;
  int32_t mb;
  float t_start_ms;
  float t_end_ms;
} bm_trace_rec;
bm_status bm_ctx_set_trace(bm_ctx* c, int32_t enable);
bm_status bm_ctx_trace_get(bm_ctx* c, bm_trace_rec* out, int64_t cap, int64_t* n, int64_t* total);
/* Diagnostics: text dump of this rank's receive/credit flags and (with
 * BM_DEBUG_PROGRESS=1 at bm_ctx_create time) the index of the last op each of its
 * streams finished.  Reads device memory on a private non-blocking stream, so
 * it works while the step's streams are blocked. */
bm_status bm_ctx_debug_dump(bm_ctx* c, char* buf, size_t cap);
void bm_ctx_destroy(bm_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* BIGMAC_H */
