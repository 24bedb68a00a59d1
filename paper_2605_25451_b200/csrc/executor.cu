// executor.cu -- BigMac's pipeline executor on one B200 per rank.
//
// The rank's op list (bm_build_schedule) is interpreted as an opcode stream
// (P:351-352): LLM / encoder / generator compute ops enqueue the model's
// sm_100a kernels on the caller's compute stream; Send ops push the payload
// into the receiver's peer-mapped receive slot with a copy-engine copy on a
// per-destination comm stream, then bump the receiver's sequence flag
// (cuStreamWriteValue32, fenced); Recv ops make the compute stream wait for
// that flag (cuStreamWaitValue32) -- "waits on receive handles before
// consuming" without a host round trip.  The op that releases a slot
// writes a credit back to the sender, which waits for it before reusing the
// slot (ring sizes from the builder's deadlock check).
// Runtime buffers are stash slots keyed by (mb, chunk) for the
// LLM, by unit for the encoder, one for the generator.  DP gradients of the
// encoder/projector/generator are accumulated locally and summed once at the
// end of the step with NCCL; with D pipeline replicas
// (bm_ctx_init_replicas) the LLM stage gradients are also summed over the
// stage's replicas.  Streams per rank: the caller's compute stream (LLM ops),
// a high-priority generator stream (GenFwd/GenBwd, started at Hn-ready), an
// encoder stream (EncFwd/EncBwd; default at P = 1) and one comm stream per
// peer; cross-stream order is carried by events and device flags only.
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "kernels.h"
#include "sched_internal.h"

namespace bm {

// ------------------------------------------------------------------ driver entry points
typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
struct Drv {
  StreamValueFn wait32 = nullptr, write32 = nullptr;
  AddrRangeFn addr_range = nullptr;
};
static Drv& drv() {
  static Drv d;
  static bool init = false;
  if (!init) {
    init = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      d.wait32 = (StreamValueFn)p;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      d.write32 = (StreamValueFn)p;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
      d.addr_range = (AddrRangeFn)p;
  }
  return d;
}

// ------------------------------------------------------------------ NCCL (dlopen'ed)
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};
static Nccl& nccl() {
  static Nccl n;
  static bool init = false;
  if (!init) {
    init = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      n.CommInitRank = (decltype(n.CommInitRank))dlsym(h, "ncclCommInitRank");
      n.AllReduce = (decltype(n.AllReduce))dlsym(h, "ncclAllReduce");
      n.GroupStart = (decltype(n.GroupStart))dlsym(h, "ncclGroupStart");
      n.GroupEnd = (decltype(n.GroupEnd))dlsym(h, "ncclGroupEnd");
      n.CommDestroy = (decltype(n.CommDestroy))dlsym(h, "ncclCommDestroy");
      n.GetErrorString = (decltype(n.GetErrorString))dlsym(h, "ncclGetErrorString");
      n.ok = n.GetUniqueId && n.CommInitRank && n.AllReduce && n.GroupStart && n.GroupEnd && n.CommDestroy;
    }
  }
  return n;
}
#define BM_NCCL_TRY(expr)                                                                          \
  do {                                                                                             \
    ncclResult_t _r = (expr);                                                                      \
    if (_r != ncclSuccess) {                                                                       \
      set_error(std::string(#expr) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(_r) : "nccl error")); \
      return BM_E_NCCL;                                                                            \
    }                                                                                              \
  } while (0)

// ------------------------------------------------------------------ parameter layout
struct PEntry {
  std::string name;
  int rows, cols, ld;
  int64_t off;
  int kind;
};

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
static bool is_comm(int k) { return k == BM_OP_SEND || k == BM_OP_RECV; }
static int round8(int x) { return (x + 7) / 8 * 8; }
// chunk q of n over [0, count): 4-element (16-byte) aligned boundaries (FSDP shards,
// peer-sum reduce-scatter chunks)
static void chunk_of(int64_t count, int n, int q, int64_t* lo, int64_t* hi) {
  const int64_t n4 = (count + 3) / 4;
  *lo = std::min(count, (n4 * q / n) * 4);
  *hi = std::min(count, (n4 * (q + 1) / n) * 4);
}

static bm_status check_model(const bm_model_cfg& mc, const bm_sched_cfg& sc) {
  BM_CHECK_ARG(mc.S > 0 && mc.d > 0 && mc.f > 0 && mc.L > 0 && mc.vocab > 0, "bad LLM dims");
  BM_CHECK_ARG(mc.d_in > 0 && mc.d_e > 0 && mc.f_e > 0 && mc.L_e >= 0, "bad encoder dims");
  BM_CHECK_ARG(sc.llm_cp <= 1 && sc.enc_cp <= 1,
               "decoupled-CP schedules (llm_cp / enc_cp > 1) are built and verified, not executed (DESIGN.md R25)");
  BM_CHECK_ARG(mc.d_g > 0 && mc.f_g > 0 && mc.L_g >= 0 && mc.d_t > 0, "bad generator dims");
  BM_CHECK_ARG(mc.dtype == BM_BF16 || mc.dtype == BM_F32, "dtype must be bf16 or fp32");
  const int PV = sc.stages * sc.vchunks;
  BM_CHECK_ARG(mc.stage_halves == 0 || (mc.stage_halves == 1 && mc.stage_layers[0] != 0),
               "stage_halves = 1 needs an explicit stage_layers partition (in half-layer units)");
  if (mc.stage_layers[0] != 0) {
    BM_CHECK_ARG(PV <= BM_MAX_VSTAGES, "explicit stage_layers needs P*V <= BM_MAX_VSTAGES");
    int sum = 0;
    for (int s = 0; s < PV; ++s) {
      BM_CHECK_ARG(mc.stage_layers[s] >= 1, "stage_layers: every virtual stage needs >= 1 layer (unit)");
      sum += mc.stage_layers[s];
    }
    for (int s = PV; s < BM_MAX_VSTAGES; ++s) BM_CHECK_ARG(mc.stage_layers[s] == 0, "stage_layers beyond P*V must be 0");
    BM_CHECK_ARG(sum == (mc.stage_halves ? 2 * mc.L : mc.L), "stage_layers must sum to L (2 L half-layer units)");
  } else if (mc.last_stage_layers == 0)
    BM_CHECK_ARG(mc.L % (sc.stages * sc.vchunks) == 0, "L must be a multiple of P*V (or set last_stage_layers)");
  else
    BM_CHECK_ARG(mc.last_stage_layers >= 1 && mc.L - mc.last_stage_layers >= sc.stages * sc.vchunks - 1,
                 "last_stage_layers must leave at least one layer per virtual stage");
  BM_CHECK_ARG(mc.d % 8 == 0 && mc.f % 8 == 0 && mc.d_e % 8 == 0 && mc.f_e % 8 == 0 && mc.d_g % 8 == 0 &&
                   mc.f_g % 8 == 0 && mc.d_t % 8 == 0 && mc.vocab % 8 == 0,
               "model widths must be multiples of 8");
  BM_CHECK_ARG(mc.max_n_mod > 0 && mc.max_n_mod <= mc.S && mc.max_n_gen > 0 && mc.max_n_gen <= mc.S,
               "max_n_mod / max_n_gen must be in [1, S]");
  BM_CHECK_ARG(mc.head_place >= BM_HEAD_AUTO && mc.head_place <= BM_HEAD_DP_SHARD, "bad head_place");
  BM_CHECK_ARG(mc.head_place != BM_HEAD_DP_SHARD || sc.gen_place == BM_GEN_DP_SHARD,
               "BM_HEAD_DP_SHARD rides on the DP-sharded generator ops (gen_place = BM_GEN_DP_SHARD)");
  BM_CHECK_ARG(mc.fsdp >= BM_FSDP_OFF && mc.fsdp <= BM_FSDP_ALLGATHER, "bad fsdp mode");
  BM_CHECK_ARG(mc.enc_stream >= 0 && mc.enc_stream <= 2, "enc_stream must be 0 (auto), 1 (on) or 2 (off)");
  {
    const uint32_t all = sc.stages >= 32 ? 0xFFFFFFFFu : ((1u << sc.stages) - 1u);
    BM_CHECK_ARG(((uint32_t)mc.gen_exclude & ~all) == 0 && ((uint32_t)mc.gen_exclude & all) != all,
                 "gen_exclude: a bit mask of ranks < P that leaves at least one rank");
    BM_CHECK_ARG(!mc.gen_exclude || (sc.gen_place == BM_GEN_DP_SHARD && mc.head_place != BM_HEAD_DP_SHARD),
                 "gen_exclude applies to the DP-sharded generator (without the DP-sharded head)");
  }
  BM_CHECK_ARG(!mc.fsdp || mc.head_place != BM_HEAD_DP_SHARD, "FSDP shards the encoder / generator only (not the DP-sharded head)");
  BM_CHECK_ARG(mc.fsdp != BM_FSDP_ALLGATHER || (sc.enc_place == BM_ENC_DP_UNIT && sc.gen_place == BM_GEN_DP_SHARD),
               "the FSDP all-gather baseline needs every rank in every encoder / generator op (DP unit, DP shard)");
  return BM_OK;
}

// LLM layers [*l0, *l0 + *n) of virtual stage s (bigmac.h, last_stage_layers)
static void stage_layers(const bm_model_cfg& mc, int PV, int s, int* l0, int* n) {
  if (mc.stage_layers[0] != 0) {
    *l0 = 0;
    for (int i = 0; i < s; ++i) *l0 += mc.stage_layers[i];
    *n = mc.stage_layers[s];
    return;
  }
  if (mc.last_stage_layers == 0 || PV == 1) {
    *n = mc.L / PV;
    *l0 = s * *n;
    return;
  }
  if (s == PV - 1) {
    *n = mc.last_stage_layers;
    *l0 = mc.L - *n;
    return;
  }
  const int rest = mc.L - mc.last_stage_layers, q = rest / (PV - 1), r = rest % (PV - 1);
  *n = q + (s < r ? 1 : 0);
  *l0 = s * q + std::min(s, r);
}
// The LLM span of virtual stage s: layers [l0, l0 + nl).  With stage_halves
// (bigmac.h; R24) the first layer may hold only its B half (down +
// residual: b_first) and the last only its A half (norm + gate_up + SwiGLU: a_last).
struct Span {
  int l0 = 0, nl = 0;
  bool b_first = false, a_last = false;
  bool has_a(int j) const { return !(b_first && j == 0); }
  bool has_b(int j) const { return !(a_last && j == nl - 1); }
};
static Span stage_span(const bm_model_cfg& mc, int PV, int s) {
  Span sp;
  if (mc.stage_halves) {
    int u0 = 0;
    for (int i = 0; i < s; ++i) u0 += mc.stage_layers[i];
    const int u1 = u0 + mc.stage_layers[s];
    sp.l0 = u0 / 2;
    sp.nl = (u1 + 1) / 2 - sp.l0;
    sp.b_first = (u0 & 1) != 0;
    sp.a_last = (u1 & 1) != 0;
    return sp;
  }
  stage_layers(mc, PV, s, &sp.l0, &sp.nl);
  return sp;
}
// most layers of one virtual stage held by `rank` (stash slot depth)
static int max_stage_layers(const bm_model_cfg& mc, int P, int V, int rank) {
  int mx = 0;
  for (int c = 0; c < V; ++c) mx = std::max(mx, stage_span(mc, P * V, c * P + rank).nl);
  return mx;
}

// LM head + CE DP-sharded over the ranks with the generator (bigmac.h bm_head_place)
static bool head_dp(const bm_model_cfg& mc, const bm_sched_cfg& sc) {
  if (sc.gen_place != BM_GEN_DP_SHARD) return false;
  return mc.head_place == BM_HEAD_DP_SHARD;   // BM_HEAD_AUTO = last stage (bigmac.h)
}

static std::vector<PEntry> param_layout(const bm_model_cfg& mc, const bm_sched_cfg& sc, int rank, int64_t* total,
                                        int64_t* dp) {
  std::vector<PEntry> v;
  int64_t off = 0;
  auto add = [&](const std::string& n, int rows, int cols, int kind) {
    const int ld = cols == 1 ? 1 : round8(cols);
    v.push_back({n, rows, cols, ld, off, kind});
    off = align_up(off + (int64_t)rows * ld, 64);
  };
  add("enc.patch", mc.d_e, mc.d_in, BM_PARAM_DP);
  for (int i = 0; i < mc.L_e; ++i) {
    const std::string p = "enc.blk" + std::to_string(i);
    add(p + ".norm", mc.d_e, 1, BM_PARAM_DP);
    add(p + ".fc1", mc.f_e, mc.d_e, BM_PARAM_DP);
    add(p + ".fc2", mc.d_e, mc.f_e, BM_PARAM_DP);
  }
  add("enc.proj1", mc.d, mc.d_e, BM_PARAM_DP);
  add("enc.proj2", mc.d, mc.d, BM_PARAM_DP);
  add("gen.in", mc.d_g, mc.d, BM_PARAM_DP);
  for (int i = 0; i < mc.L_g; ++i) {
    const std::string p = "gen.blk" + std::to_string(i);
    add(p + ".norm", mc.d_g, 1, BM_PARAM_DP);
    add(p + ".fc1", mc.f_g, mc.d_g, BM_PARAM_DP);
    add(p + ".fc2", mc.d_g, mc.f_g, BM_PARAM_DP);
  }
  add("gen.out", mc.d_t, mc.d_g, BM_PARAM_DP);
  const bool hdp = head_dp(mc, sc);
  if (hdp) add("llm.head", mc.vocab, mc.d, BM_PARAM_DP);
  *dp = off;
  const int P = sc.stages, V = sc.vchunks;
  if (rank == 0) add("llm.embed", mc.vocab, mc.d, BM_PARAM_LLM);
  for (int c = 0; c < V; ++c) {
    const Span sp = stage_span(mc, P * V, c * P + rank);
    for (int j = 0; j < sp.nl; ++j) {
      const std::string p = "llm.layer" + std::to_string(sp.l0 + j);
      if (sp.has_a(j)) {
        add(p + ".norm", mc.d, 1, BM_PARAM_LLM);
        add(p + ".gate_up", 2 * mc.f, mc.d, BM_PARAM_LLM);
      }
      if (sp.has_b(j)) add(p + ".down", mc.d, mc.f, BM_PARAM_LLM);
    }
  }
  if (rank == P - 1) {
    add("llm.final_norm", mc.d, 1, BM_PARAM_LLM);
    if (!hdp) add("llm.head", mc.vocab, mc.d, BM_PARAM_LLM);
  }
  *total = off;
  return v;
}

// ------------------------------------------------------------------ context
// peer-sum block of a comm buffer (offsets in bytes)
constexpr int64_t SUMBLK_FSDP = 64 * BM_MAX_SUM_PEERS;                 // FSDP barrier flags [2][64] x 64 B
constexpr int64_t SUMBLK_LOSS = SUMBLK_FSDP + 2 * 64 * BM_MAX_SUM_PEERS;  // raw loss terms

// FSDP (bm_model_cfg.fsdp): the encoder / generator parameters are sharded over the P
// ranks; a chain of parameter buckets (one per block, in use order) is materialised
// into two slots before use by pulling every shard from its owner
struct PullChain {
  std::vector<std::pair<int64_t, int64_t>> blocks;   // [lo, hi) DP element range per block
  char* slot[2] = {nullptr, nullptr};
  cudaEvent_t ready[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
  bool freed_pending[2] = {false, false};
  cudaStream_t st = nullptr;   // pull stream (one-sided pull); the op stream itself for all-gather
  std::vector<int> seq;        // block ids of the current op, in use order
  int64_t cur_lo = 0, cur_hi = 0;   // block acquired last (parameter lookups resolve into it)
  char* cur = nullptr;
  uint32_t bar = 0;            // all-gather barriers issued on this chain (same on every rank)
};

struct Chan {
  int src, dst, pay, K, nmsg;
  int64_t slot_bytes;
  int64_t data_off;    // in dst's comm buffer
  int64_t flag_off;    // data flag, in dst's comm buffer
  int64_t credit_off;  // credit flag, in src's comm buffer
};

struct LlmSlot {
  std::vector<char*> x, xn, gu, h;
  std::vector<char*> wdy, wdgu;   // ZB-H1: per layer dY and dgu kept from B for W (R23)
  std::vector<float*> rstd;
  char *gin = nullptr, *Hn = nullptr, *dHn = nullptr;
  float* rstd_f = nullptr;
  int nl = 0;   // layers of the virtual stage the slot currently stashes
  Span sp;      // ... and its span (half layers at the ends, stage_halves)
};
struct MlpSlot {  // encoder (L_e blocks) or generator (L_g blocks)
  std::vector<char*> E, xn, a, z;
  std::vector<float*> rstd;
  char *a1 = nullptr, *p1 = nullptr, *out = nullptr, *dout = nullptr;
};

// process-wide registry of opened CUDA-IPC handles: one mapping per exported
// allocation (two buffers of a peer may share one caching-allocator segment,
// and a handle must not be opened twice in one process)
struct IpcKey {
  std::array<uint8_t, 64> h;
  bool operator<(const IpcKey& o) const { return h < o.h; }
};
static std::map<IpcKey, std::pair<void*, int>>& ipc_reg() {
  static std::map<IpcKey, std::pair<void*, int>> m;
  return m;
}
static bm_status ipc_open(const uint8_t handle[64], void** base) {
  IpcKey k;
  std::memcpy(k.h.data(), handle, 64);
  auto it = ipc_reg().find(k);
  if (it != ipc_reg().end()) {
    it->second.second += 1;
    *base = it->second.first;
    return BM_OK;
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* p = nullptr;
  BM_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ipc_reg()[k] = {p, 1};
  *base = p;
  return BM_OK;
}
static void ipc_close(void* base) {
  for (auto it = ipc_reg().begin(); it != ipc_reg().end(); ++it)
    if (it->second.first == base) {
      if (--it->second.second == 0) {
        cudaIpcCloseMemHandle(base);
        ipc_reg().erase(it);
      }
      return;
    }
}

}  // namespace bm

using namespace bm;

struct bm_ctx {
  bm_model_cfg mc;
  bm_sched_cfg sc;
  const bm_schedule* s = nullptr;
  int rank = 0, P = 1, M = 1, V = 1, lps = 1, dtype = 0;
  size_t es = 2;
  std::vector<PEntry> params;
  std::unordered_map<std::string, int> pidx;
  int64_t total_elems = 0, dp_elems = 0;
  bool has_enc = false, has_gen = false, gen_last = false;
  bool enc_entry = false;  // memory-efficient baseline: encoder as the entry stage's first layers
  bool head_dp = false;    // LM head + CE DP-sharded with the generator (bm_head_place)
  int n_enc_slots = 0, n_llm_slots = 0, gen_rows = 0;
  int gen_rows_max = 0;    // largest generator shard of any rank (message slot sizes, same on every rank)
  int head_rows = 0;       // max text rows of one head shard (head_dp)
  // comm layout
  std::vector<Chan> chans;
  std::map<std::tuple<int, int, int>, int> chan_idx;
  std::vector<int64_t> comm_size;  // per rank
  std::vector<int64_t> sum_off;    // per rank: peer-sum block in its comm buffer
  // op annotations
  std::vector<std::vector<int>> release_of;  // op index -> recv op indices released after it
  // work layout
  int64_t work_bytes = 0;
  std::vector<LlmSlot> llm;
  std::vector<MlpSlot> enc;
  // encoder stash slot of each live EncFwd (by microbatch): slots are taken round-robin,
  // which is safe because EncBwd frees them in EncFwd order (units in order, a unit's
  // microbatches in order) and there are peak_enc_units of them
  std::map<int, int> enc_slot_of;
  int enc_next = 0;
  MlpSlot gen;
  char *dwork[2] = {nullptr, nullptr}, *bout[2] = {nullptr, nullptr}, *dh = nullptr, *dgu = nullptr, *dxn = nullptr;
  float* part = nullptr;
  float* part_gen = nullptr;  // RMSNorm-backward partials of the generator stream (no sharing across streams)
  float* part_enc = nullptr;  // ... and of the encoder stream
  char *ws = nullptr, *ws_gen = nullptr, *ws_enc = nullptr;  // split-K workspaces of the three compute streams
  int64_t ws_bytes = 0;
  void* cur_ws = nullptr;
  // BM_DEBUG_PROGRESS=1: each stream writes the index of the last op it finished
  // into a progress word (main, gen, one per comm peer), readable by bm_ctx_debug_dump
  bool debug_progress = getenv("BM_DEBUG_PROGRESS") != nullptr;
  uint32_t* progress = nullptr;  // [2 + P] words
  volatile uint32_t* progress_h = nullptr;  // debug: host-mapped copy (read without CUDA calls)
  char* embscr = nullptr;
  char* logits = nullptr;
  float* ce_scr = nullptr;
  char *e_dE = nullptr, *e_dp = nullptr, *e_dz = nullptr, *e_da = nullptr, *e_dxn = nullptr;
  char *g_dG = nullptr, *g_dz = nullptr, *g_da = nullptr, *g_dxn = nullptr, *gout[2] = {nullptr, nullptr};
  char* emb_local = nullptr;
  float* loss = nullptr;
  char *st_patches = nullptr, *st_ids = nullptr, *st_labels = nullptr, *st_targets = nullptr;
  int ld_patch_stage = 0;
  // bound buffers
  char* W = nullptr;
  float* G = nullptr;
  char* work = nullptr;
  char* comm = nullptr;
  bool bound = false;
  std::vector<char*> peer;
  // streams / events
  std::vector<cudaStream_t> comm_st;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  cudaEvent_t bout_ev[2] = {nullptr, nullptr}, gout_ev[2] = {nullptr, nullptr};
  bool bout_pending[2] = {false, false}, gout_pending[2] = {false, false};
  int bsel = 0, gsel = 0;
  ncclComm_t nc = nullptr;
  // pipeline replicas (bm_ctx_init_replicas): D pipelines, this one is `replica`
  int D = 1, replica = 0;
  ncclComm_t nc_world = nullptr;   // all P * D processes: DP parameters
  ncclComm_t nc_stage = nullptr;   // the D processes of this stage: its LLM parameters
  float gscale = 1.f;              // per-sample gradient scale 1 / (M D)
  // step-end sums over peer memory instead of NCCL (bm_ctx_init_peer_sum):
  // process g = replica * P + stage; its peer-sum block and grad buffer as mapped here
  bool psum = false;
  std::vector<char*> ps_comm;
  std::vector<float*> ps_grad;
  std::vector<void*> ipc_bases;    // mappings to release (registry references)
  // FSDP (bm_model_cfg.fsdp): own shard [dp_lo, dp_hi) of the DP elements; the weights
  // buffer holds it at element 0, the LLM parameters after it
  int fsdp = 0;
  int64_t dp_lo = 0, dp_hi = 0;
  std::vector<char*> peer_w;       // pipeline peers' weight buffers (bm_ctx_init_fsdp)
  PullChain chain[2];              // 0 encoder (+ projector), 1 generator
  int64_t pull_bytes = 0;          // bytes pulled from peers in the last step
  int64_t step = 0;
  cudaEvent_t done_ev = nullptr;   // recorded at the end of every bm_step (bm_step_wait)
  int64_t launches = 0;
  int64_t stash_peak[3] = {0, 0, 0};
  // per-step state
  cudaStream_t st = nullptr;
  cudaStream_t st_main = nullptr;   // the caller's stream during bm_step (debug hook)
  std::vector<int> llm_free;
  std::map<std::pair<int, int>, int> llm_live;
  std::vector<const char*> mb_patches, mb_targets;
  const int32_t *ids = nullptr, *labels = nullptr;
  std::vector<int> n_mod, n_gen;
  int ld_patch = 0;
  const void* last_src = nullptr;   // payload source of the last compute op
  int last_src_ring = -1;           // 0: bout, 1: gout (ring buffers needing a copy-done event)
  int last_src_idx = 0;
  std::vector<const char*> genin_src;  // per destination rank (last stage): generator rows of Hn
  std::vector<const char*> headin_src; // per destination rank (last stage, head_dp): head rows of Hn
  int gen_b = 0;                       // gout slot of the current generator microbatch
  cudaEvent_t producer_ev = nullptr;
  cudaStream_t producer_st = nullptr;  // stream of the last compute op (sends record their producer event here)
  // high-priority generator stream (P > 1, DP-sharded generator): gen shards run as
  // soon as their inputs exist instead of queueing behind the rank's LLM op
  cudaStream_t gen_st = nullptr;
  bool use_gen_stream = false;
  // encoder stream (BM_ENC_DP_UNIT): EncFwd / EncBwd run beside the LLM so their small,
  // latency-bound kernels fill SMs the LLM GEMMs leave idle (partial last waves);
  // ordered against the LLM by events: F(mb, 0) waits for EncFwd's output, EncBwd for
  // B(mb, 0)'s embedding gradient, B's next write of emb_local for EncBwd's read
  cudaStream_t enc_st = nullptr;
  bool use_enc_stream = false;
  std::vector<cudaEvent_t> enc_fwd_ev;   // per encoder stash slot: EncFwd output ready
  cudaEvent_t emb_ready_ev = nullptr, emb_free_ev = nullptr;
  bool emb_free_pending = false;
  cudaEvent_t hn_ev = nullptr, gen_done_ev = nullptr;
  bool gen_done_pending = false;
  std::map<int, int> own_gout;   // last rank: mb -> gout slot holding its own shard's dX
  std::vector<int> consumer_kind;      // per op index: kind of the first compute op after it
  // GEMM timing (bench roofline): event pairs around every GEMM, two pools by step parity
  bool timing = false;
  // fused SwiGLU GEMM epilogues (bm_k_gemm_swiglu / _dswiglu); on by default: C2 step
  // 48.6 vs 47.5 samples/s with the separate kernels (profiles/r01/bench_n1_fuse*.log);
  // BM_FUSE_SWIGLU=0 selects GEMM + the vectorised elementwise kernel
  bool fuse_swiglu = !(getenv("BM_FUSE_SWIGLU") && getenv("BM_FUSE_SWIGLU")[0] == '0');
  bool zb = false;         // BM_LLM_ZB_H1: LLM_BWD = input gradient, LLM_W = weight gradients
  int64_t mid_cols = 0;    // f if some stage boundary falls inside a layer (stage_halves), else 0
  bool peer_copy_ce = !(getenv("BM_PEER_COPY") && std::string(getenv("BM_PEER_COPY")) == "sm");
  int peer_copy_ctas = getenv("BM_PEER_COPY_CTAS") ? std::atoi(getenv("BM_PEER_COPY_CTAS")) : 32;
  bool spin_wait = getenv("BM_WAIT") && std::string(getenv("BM_WAIT")) == "spin";
  // SMs the compute stream's GEMMs leave free on ranks that serve remote generator
  // shards, so a shard's kernels start at once instead of after the running
  // persistent GEMM (the shard is on the last stage's critical path)
  // (measured at C2, N = 4: 0 / 8 / 16 / 32 SMs -> 140.4 / 140.1 / 139.4 / 135.0 samples/s; off by default)
  int gen_reserve_sms = getenv("BM_GEN_RESERVE_SMS") ? std::atoi(getenv("BM_GEN_RESERVE_SMS")) : 0;
  std::vector<cudaEvent_t> tev[2];
  size_t tev_used[2] = {0, 0};
  double tflop_pending[2] = {0, 0};
  double gemm_flops = 0, gemm_ms = 0;
  int64_t gemm_count = 0;
  int64_t gemm_count_pending[2] = {0, 0};
  std::vector<std::array<int, 4>> tshape[2];              // (M, N, K, epi) per timed launch
  // peer-copy timing (NVLink): event pairs on the comm streams, bytes per copy
  std::vector<cudaEvent_t> cev[2];
  std::vector<int64_t> cbytes[2];
  // per-op trace of the last step (bm_ctx_set_trace)
  struct TraceEv {
    int32_t op, kind, stream, mb;
    cudaEvent_t a, b;
  };
  bool tracing = false;
  std::vector<TraceEv> trace;
  std::vector<cudaEvent_t> trace_pool;
  size_t trace_used = 0;
  cudaEvent_t trace_origin = nullptr, trace_last = nullptr;
  double comm_ms = 0, comm_bytes = 0;
  int64_t comm_msgs = 0;
  std::map<std::array<int, 4>, std::pair<int64_t, double>> shape_ms;  // BM_GEMM_LOG=1 breakdown
  ~bm_ctx();
};

static bm_ctx* g_dbg_ctx = nullptr;   // BM_DEBUG_PROGRESS launch hook target

bm_ctx::~bm_ctx() {
  for (auto s_ : comm_st)
    if (s_) cudaStreamDestroy(s_);
  if (gen_st) cudaStreamDestroy(gen_st);
  if (enc_st) cudaStreamDestroy(enc_st);
  for (auto e : enc_fwd_ev)
    if (e) cudaEventDestroy(e);
  if (emb_ready_ev) cudaEventDestroy(emb_ready_ev);
  if (emb_free_ev) cudaEventDestroy(emb_free_ev);
  if (hn_ev) cudaEventDestroy(hn_ev);
  if (done_ev) cudaEventDestroy(done_ev);
  for (auto& ch : chain) {
    for (int i = 0; i < 2; ++i) {
      if (ch.ready[i]) cudaEventDestroy(ch.ready[i]);
      if (ch.freed[i]) cudaEventDestroy(ch.freed[i]);
    }
    if (ch.st) cudaStreamDestroy(ch.st);
  }
  if (gen_done_ev) cudaEventDestroy(gen_done_ev);
  for (auto e : evpool)
    if (e) cudaEventDestroy(e);
  for (int k = 0; k < 2; ++k) {
    for (auto e : tev[k])
      if (e) cudaEventDestroy(e);
    for (auto e : cev[k])
      if (e) cudaEventDestroy(e);
  }
  for (auto e : trace_pool)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (bout_ev[i]) cudaEventDestroy(bout_ev[i]);
    if (gout_ev[i]) cudaEventDestroy(gout_ev[i]);
  }
  for (void* b : ipc_bases) ipc_close(b);
  if (nc && nccl().ok) nccl().CommDestroy(nc);
  if (nc_world && nccl().ok) nccl().CommDestroy(nc_world);
  if (nc_stage && nccl().ok) nccl().CommDestroy(nc_stage);
  if (progress_h) cudaFreeHost((void*)progress_h);
  if (g_dbg_ctx == this) {
    g_dbg_ctx = nullptr;
    g_launch_hook = nullptr;
  }
  cudaGetLastError();  // never leave a sticky-looking error for the caller's next API call
}

namespace bm {

// ------------------------------------------------------------------ layouts
static int64_t payload_rows_max(const bm_ctx& c, int pay) {
  switch (pay) {
    case BM_PAY_ACT:
    case BM_PAY_GRAD: return c.mc.S;
    case BM_PAY_EMB:
    case BM_PAY_EMBGRAD: return c.mc.max_n_mod;
    default: return c.gen_rows_max + c.head_rows;   // genin / gengrad: [head rows | generator rows]
  }
}

// stage-boundary message after virtual stage b: x (S x d), or [x_l | h_l] / [dx | dh]
// (S x (d + f)) when the boundary falls inside layer l (stage_halves, R24)
static int64_t boundary_bytes(const bm_ctx& c, int b) {
  const bool mid = stage_span(c.mc, c.P * c.V, b).a_last;
  return (int64_t)c.mc.S * (c.mc.d + (mid ? c.mc.f : 0)) * c.es;
}

static void comm_layout(bm_ctx& c) {
  c.comm_size.assign(c.P, 0);
  std::vector<int64_t> flag_cur(c.P, 0);
  for (auto& kv : c.s->rings) {
    Chan ch;
    ch.src = std::get<0>(kv.first);
    ch.dst = std::get<1>(kv.first);
    ch.pay = std::get<2>(kv.first);
    ch.K = kv.second.first;
    ch.nmsg = kv.second.second;
    const int64_t width = (ch.pay == BM_PAY_ACT || ch.pay == BM_PAY_GRAD) ? c.mc.d + c.mid_cols : c.mc.d;
    ch.slot_bytes = align_up(payload_rows_max(c, ch.pay) * width * (int64_t)c.es, 256);
    ch.flag_off = flag_cur[ch.dst];
    flag_cur[ch.dst] += 64;
    ch.credit_off = flag_cur[ch.src];
    flag_cur[ch.src] += 64;
    c.chan_idx[kv.first] = (int)c.chans.size();
    c.chans.push_back(ch);
  }
  std::vector<int64_t> data_cur(c.P);
  for (int r = 0; r < c.P; ++r) data_cur[r] = align_up(flag_cur[r], 256);
  for (auto& ch : c.chans) {
    ch.data_off = data_cur[ch.dst];
    data_cur[ch.dst] += ch.K * ch.slot_bytes;
  }
  // peer-sum block: one step-end barrier flag per source process (bm_ctx_init_peer_sum),
  // two FSDP all-gather barrier flag sets (bm_model_cfg.fsdp = BM_FSDP_ALLGATHER; encoder
  // and generator chains), then the raw loss terms [2M] the peers read
  c.sum_off.assign(c.P, 0);
  for (int r = 0; r < c.P; ++r) {
    c.sum_off[r] = align_up(data_cur[r], 256);
    c.comm_size[r] = align_up(c.sum_off[r] + SUMBLK_LOSS + (2 * (int64_t)c.M + 1) * 4, 256);
  }
}


struct Bump {
  char* base;
  int64_t off = 0;
  char* take(int64_t bytes) {
    char* p = base ? base + off : nullptr;
    off = align_up(off + std::max<int64_t>(bytes, 0), 256);
    return p;
  }
};

static void work_layout(bm_ctx& c, char* base) {
  Bump b{base};
  const auto& m = c.mc;
  const int64_t es = c.es, S = m.S, d = m.d, f = m.f;
  const bool last_rank = c.rank == c.P - 1;
  c.llm.assign(c.n_llm_slots, LlmSlot());
  for (auto& sl : c.llm) {
    sl.x.resize(c.lps + 1); sl.xn.resize(c.lps); sl.gu.resize(c.lps); sl.h.resize(c.lps); sl.rstd.resize(c.lps);
    for (int j = 0; j < c.lps; ++j) {
      // x_j and h_j back to back: [x_l | h_l] is the message of a boundary inside layer l
      sl.x[j] = b.take(S * (d + f) * es);
      sl.h[j] = sl.x[j] + S * d * es;
      sl.xn[j] = b.take(S * d * es);
      sl.rstd[j] = (float*)b.take(S * 4);
      sl.gu[j] = b.take(S * 2 * f * es);
    }
    sl.x[c.lps] = b.take(S * d * es);
    sl.gin = b.take(S * (d + c.mid_cols) * es);
    if (c.zb) {   // the weight-gradient operands B leaves for W
      sl.wdy.resize(c.lps); sl.wdgu.resize(c.lps);
      for (int j = 0; j < c.lps; ++j) {
        sl.wdy[j] = b.take(S * d * es);
        sl.wdgu[j] = b.take(S * 2 * f * es);
      }
    }
    if (last_rank) {
      sl.Hn = b.take(S * d * es);
      sl.dHn = b.take(S * d * es);
      sl.rstd_f = (float*)b.take(S * 4);
    }
  }
  auto mlp_slot = [&](MlpSlot& sl, int n, int dm, int fm, int Lb, int dproj, bool proj, int dt) {
    sl.E.resize(Lb + 1); sl.xn.resize(Lb); sl.a.resize(Lb); sl.z.resize(Lb); sl.rstd.resize(Lb);
    for (int j = 0; j <= Lb; ++j) sl.E[j] = b.take((int64_t)n * dm * es);
    for (int j = 0; j < Lb; ++j) {
      sl.xn[j] = b.take((int64_t)n * dm * es);
      sl.rstd[j] = (float*)b.take((int64_t)n * 4);
      sl.a[j] = b.take((int64_t)n * fm * es);
      sl.z[j] = b.take((int64_t)n * fm * es);
    }
    if (proj) {
      sl.a1 = b.take((int64_t)n * dproj * es);
      sl.p1 = b.take((int64_t)n * dproj * es);
      sl.out = b.take((int64_t)n * dproj * es);
    } else {
      sl.out = b.take((int64_t)n * dt * es);
      sl.dout = b.take((int64_t)n * dt * es);
    }
  };
  c.enc.assign(c.n_enc_slots, MlpSlot());
  for (auto& sl : c.enc) mlp_slot(sl, m.max_n_mod, m.d_e, m.f_e, m.L_e, m.d, true, 0);
  if (c.has_gen && c.gen_rows > 0) mlp_slot(c.gen, c.gen_rows, m.d_g, m.f_g, m.L_g, 0, false, m.d_t);
  // LLM scratch
  for (int i = 0; i < 2; ++i) c.dwork[i] = b.take(S * d * es);
  for (int i = 0; i < 2; ++i) c.bout[i] = b.take(S * (d + c.mid_cols) * es);
  c.dh = b.take(S * f * es);
  c.dgu = b.take(S * 2 * f * es);
  c.dxn = b.take(S * d * es);
  const int wmax = std::max(std::max(m.d, m.d_e), m.d_g);
  c.part = (float*)b.take(rmsnorm_bwd_scratch_floats(std::max(S, (int64_t)m.max_n_mod), wmax) * 4);
  c.part_gen = (float*)b.take(rmsnorm_bwd_scratch_floats(std::max(c.gen_rows, 1), m.d_g) * 4);
  c.part_enc = (float*)b.take(rmsnorm_bwd_scratch_floats(std::max(m.max_n_mod, 1), m.d_e) * 4);
  {
    const int64_t rows = ((int64_t)std::max(m.max_n_mod, c.gen_rows) + 127) / 128 * 128;
    const int64_t cols = std::max<int64_t>({m.d, m.d_e, m.f_e, m.d_g, m.f_g, m.d_in + 8});
    c.ws_bytes = std::min<int64_t>(64ll << 20, 8 * rows * cols * 4);
    c.ws = b.take(c.ws_bytes);
    c.ws_gen = b.take(c.ws_bytes);
    c.ws_enc = b.take(c.ws_bytes);
  }
  c.embscr = b.take(embed_bwd_scratch_bytes(m.S));
  if (c.head_dp) {
    c.logits = b.take((int64_t)c.head_rows * m.vocab * es);
    c.ce_scr = (float*)b.take(S * 4);
  } else if (last_rank) {
    c.logits = b.take(S * m.vocab * es);
    c.ce_scr = (float*)b.take(S * 4);
  }
  // encoder / generator scratch
  const int64_t n = m.max_n_mod;
  c.e_dE = b.take(n * m.d_e * es);
  c.e_dp = b.take(n * d * es);
  c.e_dz = b.take(n * m.f_e * es);
  c.e_da = b.take(n * std::max(m.f_e, m.d) * es);
  c.e_dxn = b.take(n * m.d_e * es);
  const int64_t ng = std::max(c.gen_rows, 1);
  c.g_dG = b.take(ng * m.d_g * es);
  c.g_dz = b.take(ng * m.f_g * es);
  c.g_da = b.take(ng * m.f_g * es);
  c.g_dxn = b.take(ng * m.d_g * es);
  for (int i = 0; i < 2; ++i) c.gout[i] = b.take((ng + c.head_rows) * d * es);
  c.emb_local = b.take(n * d * es);
  if (c.fsdp)   // two bucket slots per chain, each the largest block of that chain
    for (auto& ch : c.chain) {
      int64_t mx = 1;
      for (auto& bl : ch.blocks) mx = std::max(mx, bl.second - bl.first);
      for (int i = 0; i < 2; ++i) ch.slot[i] = b.take(mx * es);
    }
  c.loss = (float*)b.take((2 * (int64_t)c.M + 1) * 4);
  c.progress = (uint32_t*)b.take((2 + c.P) * 64);
  // host-batch staging
  c.ld_patch_stage = round8(m.d_in);
  c.st_patches = b.take((int64_t)c.M * m.max_n_mod * c.ld_patch_stage * es);
  c.st_ids = b.take((int64_t)c.M * S * 4);
  c.st_labels = b.take((int64_t)c.M * S * 4);
  c.st_targets = b.take((int64_t)c.M * m.max_n_gen * m.d_t * es);
  c.work_bytes = b.off;
}

// ------------------------------------------------------------------ helpers
static inline char* P_(bm_ctx& c, const char* name) {
  auto it = c.pidx.find(name);
  if (it == c.pidx.end()) return nullptr;
  const int64_t off = c.params[it->second].off;
  if (!c.fsdp) return c.W + off * c.es;
  if (off >= c.dp_elems) return c.W + (off - c.dp_elems + (c.dp_hi - c.dp_lo)) * c.es;   // LLM parameter
  for (auto& ch : c.chain)   // DP parameter: inside the bucket acquired last on its chain
    if (off >= ch.cur_lo && off < ch.cur_hi) return ch.cur + (off - ch.cur_lo) * c.es;
  return nullptr;
}
static inline float* G_(bm_ctx& c, const char* name) {
  auto it = c.pidx.find(name);
  return it == c.pidx.end() ? nullptr : c.G + c.params[it->second].off;
}
static inline int LD_(bm_ctx& c, const char* name) { return c.params[c.pidx.at(name)].ld; }

static bm_status timed_gemm(bm_ctx& c, int M, int N, int K, const void* A, int64_t lda, int am, const void* B,
                            int64_t ldb, int bm_, void* C, int64_t ldc, int cdt, int epi, const void* R, int64_t ldr,
                            int f = 0) {
  void* ws = c.cur_ws;
  // the roofline's dominant kernel: GEMMs on the compute stream (side-stream GEMMs
  // overlap them, so their event spans would double-count device time)
  if (!c.timing || M <= 0 || N <= 0 || K <= 0 || c.st != c.st_main)
    return gemm(c.dtype, M, N, K, A, lda, am, B, ldb, bm_, C, ldc, cdt, epi, R, ldr, 1.f, c.st, f, ws, c.ws_bytes);
  const int pool = (int)(c.step & 1);
  auto& ev = c.tev[pool];
  if (c.tev_used[pool] + 2 > ev.size()) {
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t e;
      BM_CUDA_TRY(cudaEventCreate(&e));
      ev.push_back(e);
    }
  }
  cudaEvent_t e0 = ev[c.tev_used[pool]], e1 = ev[c.tev_used[pool] + 1];
  c.tev_used[pool] += 2;
  BM_CUDA_TRY(cudaEventRecord(e0, c.st));
  BM_TRY(gemm(c.dtype, M, N, K, A, lda, am, B, ldb, bm_, C, ldc, cdt, epi, R, ldr, 1.f, c.st, f, ws, c.ws_bytes));
  BM_CUDA_TRY(cudaEventRecord(e1, c.st));
  c.tflop_pending[pool] += 2.0 * M * N * K;
  c.gemm_count_pending[pool] += 1;
  c.tshape[pool].push_back({M, N, K, epi});
  return BM_OK;
}
// independent contractions (a Linear's data and weight gradient) in one grouped
// CTA-pair launch (gemm_bf16_tc_group: LPT tile schedule, no wave tail per GEMM)
// (opt-in BM_GEMM_GROUP_BWD=1: standalone it is even with two launches and in the C2
// step 0.8 % slower -- the power-capped clock rises when a launch's last wave leaves
// pairs idle, so the wave tail the grouping removes costs less than its count
// suggests; profiles/r02/ab_group_bwd.log)
static const bool g_group_bwd = getenv("BM_GEMM_GROUP_BWD") && getenv("BM_GEMM_GROUP_BWD")[0] == '1';
static bm_status timed_group(bm_ctx& c, GemmSpec* sp, int n) {
  if (c.dtype != BM_BF16 || n == 1 || !g_group_bwd) {
    for (int i = 0; i < n; ++i) {
      const GemmSpec& q = sp[i];
      BM_TRY(timed_gemm(c, q.M, q.N, q.K, q.A, q.lda, q.a_major, q.B, q.ldb, q.b_major, q.C, q.ldc, q.c_dtype, q.epi,
                        q.R, q.ldr, q.f));
    }
    return BM_OK;
  }
  for (int i = 0; i < n; ++i) {
    sp[i].ws = c.cur_ws;
    sp[i].ws_bytes = c.ws_bytes;
  }
  if (!c.timing || c.st != c.st_main) return gemm_bf16_tc_group(sp, n, c.st);
  const int pool = (int)(c.step & 1);
  auto& ev = c.tev[pool];
  if (c.tev_used[pool] + 2 > ev.size()) {
    for (int k = 0; k < 256; ++k) {
      cudaEvent_t e;
      BM_CUDA_TRY(cudaEventCreate(&e));
      ev.push_back(e);
    }
  }
  cudaEvent_t e0 = ev[c.tev_used[pool]], e1 = ev[c.tev_used[pool] + 1];
  c.tev_used[pool] += 2;
  BM_CUDA_TRY(cudaEventRecord(e0, c.st));
  BM_TRY(gemm_bf16_tc_group(sp, n, c.st));
  BM_CUDA_TRY(cudaEventRecord(e1, c.st));
  double fl = 0;
  for (int i = 0; i < n; ++i) fl += 2.0 * sp[i].M * sp[i].N * sp[i].K;
  c.tflop_pending[pool] += fl;
  c.gemm_count_pending[pool] += 1;
  c.tshape[pool].push_back({sp[0].M, sp[0].N, sp[0].K, 100 + sp[1].epi});
  return BM_OK;
}
// GemmSpec of a Linear's weight gradient dW[out, in] += dY^T X (fp32 TMA reduce-add)
static GemmSpec spec_wgrad(int n, int in, int out, const void* dY, const void* X, int64_t ldx, float* dW, int64_t ldw) {
  return GemmSpec{out, in, n, dY, out, 1, X, ldx, 1, dW, ldw, BM_F32, BM_EPI_ACCUM, nullptr, 0, 1.f, 0, nullptr, 0};
}
// ... its data gradient dX[n, in] = dY W
static GemmSpec spec_dgrad(const bm_ctx& c, int n, int in, int out, const void* dY, const void* Wt, int64_t ldw,
                           void* dX, int64_t lddx) {
  return GemmSpec{n, in, out, dY, out, 0, Wt, ldw, 1, dX, lddx, c.dtype, BM_EPI_STORE, nullptr, 0, 1.f, 0, nullptr, 0};
}
// fold a finished pool's event pairs into the totals (blocks until they completed)
static bm_status harvest_comm(bm_ctx& c, int pool) {
  auto& ev = c.cev[pool];
  const size_t n = c.cbytes[pool].size();
  if (n == 0) return BM_OK;
  for (size_t i = 0; i < n; ++i) {
    BM_CUDA_TRY(cudaEventSynchronize(ev[2 * i + 1]));
    float t = 0;
    BM_CUDA_TRY(cudaEventElapsedTime(&t, ev[2 * i], ev[2 * i + 1]));
    c.comm_ms += t;
    c.comm_bytes += (double)c.cbytes[pool][i];
  }
  c.comm_msgs += (int64_t)n;
  c.cbytes[pool].clear();
  return BM_OK;
}
static bm_status harvest(bm_ctx& c, int pool) {
  BM_TRY(harvest_comm(c, pool));
  auto& ev = c.tev[pool];
  if (c.tev_used[pool] == 0) return BM_OK;
  BM_CUDA_TRY(cudaEventSynchronize(ev[c.tev_used[pool] - 1]));
  double ms = 0;
  for (size_t i = 0; i + 1 < c.tev_used[pool]; i += 2) {
    float t = 0;
    BM_CUDA_TRY(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
    ms += t;
    if (i / 2 < c.tshape[pool].size()) {
      auto& e = c.shape_ms[c.tshape[pool][i / 2]];
      e.first += 1;
      e.second += t;
    }
  }
  c.tshape[pool].clear();
  c.gemm_ms += ms;
  c.gemm_flops += c.tflop_pending[pool];
  c.gemm_count += c.gemm_count_pending[pool];
  c.tev_used[pool] = 0;
  c.tflop_pending[pool] = 0;
  c.gemm_count_pending[pool] = 0;
  return BM_OK;
}
static bm_status lin_fwd(bm_ctx& c, int n, int in, int out, const void* X, int64_t ldx, const void* Wt, int64_t ldw,
                         void* Y, int epi = BM_EPI_STORE, const void* R = nullptr) {
  return timed_gemm(c, n, out, in, X, ldx, 0, Wt, ldw, 0, Y, out, c.dtype, epi, R, out);
}
static bm_status lin_dgrad(bm_ctx& c, int n, int in, int out, const void* dY, const void* Wt, int64_t ldw, void* dX,
                           int64_t lddx, int epi = BM_EPI_STORE, const void* R = nullptr) {
  return timed_gemm(c, n, in, out, dY, out, 0, Wt, ldw, 1, dX, lddx, c.dtype, epi, R, lddx);
}
static bm_status lin_wgrad(bm_ctx& c, int n, int in, int out, const void* dY, const void* X, int64_t ldx, float* dW,
                           int64_t ldw) {
  if (n <= 0) return BM_OK;
  return timed_gemm(c, out, in, n, dY, out, 1, X, ldx, 1, dW, ldw, BM_F32, BM_EPI_ACCUM, nullptr, 0);
}
// LLM gate/up GEMM; bf16 fuses SwiGLU into the epilogue (writes gu and h)
static bm_status lin_gate_up(bm_ctx& c, const void* xn, const void* Wgu, int64_t ldw, void* gu, void* h) {
  const auto& m = c.mc;
  if (c.fuse_swiglu && c.dtype == BM_BF16 && m.f % 128 == 0)
    return timed_gemm(c, m.S, 2 * m.f, m.d, xn, m.d, 0, Wgu, ldw, 0, gu, 2 * m.f, BM_BF16, BM_EPI_SWIGLU, h, m.f, m.f);
  BM_TRY(timed_gemm(c, m.S, 2 * m.f, m.d, xn, m.d, 0, Wgu, ldw, 0, gu, 2 * m.f, c.dtype, BM_EPI_STORE, nullptr, 0));
  return c.dtype == BM_BF16 ? swiglu_fwd<bf16>(m.S, m.f, (const bf16*)gu, (bf16*)h, c.st)
                            : swiglu_fwd<float>(m.S, m.f, (const float*)gu, (float*)h, c.st);
}
// LLM down dgrad; bf16 fuses the SwiGLU backward into the epilogue (writes dgu, never dh)
static bm_status lin_down_dgrad_swiglu(bm_ctx& c, const void* dy, const void* Wd, int64_t ldw, const void* gu,
                                       void* dh_scratch, void* dgu) {
  const auto& m = c.mc;
  // the fused epilogue stores 32-column chunks of dg and du; with f % 32 != 0 the last dg
  // chunk's store would spill into du's first columns, so those widths take the split path
  if (c.fuse_swiglu && c.dtype == BM_BF16 && m.f % 32 == 0)
    return timed_gemm(c, m.S, m.f, m.d, dy, m.d, 0, Wd, ldw, 1, dgu, 2 * m.f, BM_BF16, BM_EPI_DSWIGLU, gu, 2 * m.f, m.f);
  BM_TRY(timed_gemm(c, m.S, m.f, m.d, dy, m.d, 0, Wd, ldw, 1, dh_scratch, m.f, c.dtype, BM_EPI_STORE, nullptr, 0));
  return c.dtype == BM_BF16 ? swiglu_bwd<bf16>(m.S, m.f, (const bf16*)dh_scratch, (const bf16*)gu, (bf16*)dgu, c.st)
                            : swiglu_bwd<float>(m.S, m.f, (const float*)dh_scratch, (const float*)gu, (float*)dgu, c.st);
}

#define TY(c, bfcall, fcall) ((c).dtype == BM_BF16 ? (bfcall) : (fcall))
static bm_status norm_fwd(bm_ctx& c, int rows, int cols, const void* x, const void* g, void* y, float* rstd) {
  return TY(c, rmsnorm_fwd<bf16>(rows, cols, (const bf16*)x, (const bf16*)g, (bf16*)y, rstd, c.st),
            rmsnorm_fwd<float>(rows, cols, (const float*)x, (const float*)g, (float*)y, rstd, c.st));
}
static bm_status norm_bwd(bm_ctx& c, int rows, int cols, const void* dy, const void* x, const void* g,
                          const float* rstd, const void* dres, void* dx, float* dg) {
  return TY(c, rmsnorm_bwd<bf16>(rows, cols, (const bf16*)dy, (const bf16*)x, (const bf16*)g, rstd, (const bf16*)dres,
                                 (bf16*)dx, dg, c.part, c.st),
            rmsnorm_bwd<float>(rows, cols, (const float*)dy, (const float*)x, (const float*)g, rstd, (const float*)dres,
                               (float*)dx, dg, c.part, c.st));
}
static bm_status gelu_f(bm_ctx& c, int64_t n, const void* a, void* z) {
  return TY(c, gelu_fwd<bf16>(n, (const bf16*)a, (bf16*)z, c.st), gelu_fwd<float>(n, (const float*)a, (float*)z, c.st));
}
static bm_status gelu_b(bm_ctx& c, int64_t n, const void* dz, const void* a, void* da) {
  return TY(c, gelu_bwd<bf16>(n, (const bf16*)dz, (const bf16*)a, (bf16*)da, c.st),
            gelu_bwd<float>(n, (const float*)dz, (const float*)a, (float*)da, c.st));
}
static bm_status add_(bm_ctx& c, int64_t n, const void* a, const void* b, void* o) {
  return TY(c, add<bf16>(n, (const bf16*)a, (const bf16*)b, (bf16*)o, c.st),
            add<float>(n, (const float*)a, (const float*)b, (float*)o, c.st));
}
static bm_status d2d(bm_ctx& c, void* dst, const void* src, int64_t bytes) {
  return copy_bytes(dst, src, bytes, 0, c.st);
}
// BM_DEBUG_PROGRESS: after every kernel launch, the issuing stream writes the global
// launch number into word 1 of its progress block; the host logs (number, stream,
// kernel name), so a dump names the last kernel each stream finished.
static uint32_t g_dbg_launch = 0;
static void dbg_launch_hook(cudaStream_t st, const void* kern) {
  bm_ctx* c = g_dbg_ctx;
  if (!c || !c->progress) return;
  int slot = -1;
  if (st == c->st_main) slot = 0;
  else if (st == c->gen_st) slot = 1;
  else if (st == c->enc_st) slot = 2 + c->P;
  else
    for (int q = 0; q < c->P; ++q)
      if (q != c->rank && st == c->comm_st[q]) slot = 2 + q;
  if (slot < 0) return;
  ++g_dbg_launch;
  const char* name = nullptr;
  if (cudaFuncGetName(&name, kern) != cudaSuccess) { name = "?"; cudaGetLastError(); }
  std::fprintf(stderr, "[bm r%d] launch %u stream %d %s\n", c->rank, g_dbg_launch, slot, name ? name : "?");
  drv().write32((CUstream)st, (CUdeviceptr)(c->progress + 16 * slot + 1), g_dbg_launch, 0);
}

static cudaEvent_t next_event(bm_ctx& c) {
  cudaEvent_t e = c.evpool[c.evnext];
  c.evnext = (c.evnext + 1) % c.evpool.size();
  return e;
}
// trace events (timing-enabled, pooled; bm_ctx_set_trace)
static cudaEvent_t trace_event(bm_ctx& c) {
  if (c.trace_used == c.trace_pool.size()) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c.trace_pool.push_back(e);
  }
  return c.trace_pool[c.trace_used++];
}
static int stream_slot(const bm_ctx& c, cudaStream_t st) {
  if (st == c.st_main) return 0;
  if (st == c.gen_st) return 1;
  if (st == c.enc_st) return 2 + c.P;
  for (int q = 0; q < c.P; ++q)
    if (q != c.rank && st == c.comm_st[q]) return 2 + q;
  return 0;
}
static cudaEvent_t trace_mark(bm_ctx& c, cudaStream_t st) {
  cudaEvent_t e = trace_event(c);
  if (e) cudaEventRecord(e, st);
  return e;
}

// generator row shard of rank r: equal shards over the ranks not in
// bm_model_cfg.gen_exclude (in rank order), empty on the excluded ranks
static void shard_rows(const bm_ctx& c, int m, int r, int* lo, int* hi) {
  const int n = c.n_gen[m];
  if (c.gen_last) { *lo = 0; *hi = n; return; }
  const uint32_t ex = (uint32_t)c.mc.gen_exclude;
  int k = 0, nk = 0;   // r's index among the included ranks, their count
  for (int q = 0; q < c.P; ++q)
    if (!((ex >> q) & 1u)) {
      if (q < r) ++k;
      ++nk;
    }
  if ((ex >> r) & 1u) {
    *lo = *hi = (int)(((int64_t)k * n) / nk);
    return;
  }
  *lo = (int)(((int64_t)k * n) / nk);
  *hi = (int)(((int64_t)(k + 1) * n) / nk);
}

// head shard r of microbatch m (head_dp): absolute rows of the text range [n_mod, S)
static void head_rows_of(const bm_ctx& c, int m, int r, int* lo, int* hi) {
  if (!c.head_dp) { *lo = *hi = 0; return; }
  const int n_mod = c.n_mod[m], n_text = c.mc.S - n_mod;
  *lo = n_mod + (int)(((int64_t)r * n_text) / c.P);
  *hi = n_mod + (int)(((int64_t)(r + 1) * n_text) / c.P);
}

static bm_status wait_flag(bm_ctx& c, cudaStream_t on, char* flag, uint32_t v, const char* what);
// ------------------------------------------------------------------ FSDP one-sided pull
// barrier of the pipeline group on stream `on` (all-gather baseline): every rank must
// reach the same bucket before any proceeds -- FSDP's synchronisation point
static bm_status fsdp_barrier(bm_ctx& c, int k, cudaStream_t on) {
  PullChain& ch = c.chain[k];
  const uint32_t v = ++ch.bar;
  for (int q = 0; q < c.P; ++q) {
    char* f = c.peer[q] + c.sum_off[q] + SUMBLK_FSDP + (int64_t)(k * BM_MAX_SUM_PEERS + c.rank) * 64;
    CUresult r = drv().write32((CUstream)on, (CUdeviceptr)f, v, 0);
    if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 (fsdp barrier) failed"); return BM_E_CUDA; }
  }
  for (int q = 0; q < c.P; ++q)
    if (q != c.rank)
      BM_TRY(wait_flag(c, on, c.comm + c.sum_off[c.rank] + SUMBLK_FSDP + (int64_t)(k * BM_MAX_SUM_PEERS + q) * 64, v,
                       "fsdp all-gather"));
  return BM_OK;
}
// materialise block seq[j] of chain k into slot j % 2: the shard of every owner q is
// read from q's weight buffer (own shard locally) -- no participation of the owners
static bm_status fsdp_issue(bm_ctx& c, int k, int j, cudaStream_t op_st) {
  PullChain& ch = c.chain[k];
  const int s = j & 1;
  cudaStream_t st = c.fsdp == BM_FSDP_ALLGATHER ? op_st : ch.st;
  if (ch.freed_pending[s]) {   // the op that read this slot last has finished with it
    if (st != op_st) BM_CUDA_TRY(cudaStreamWaitEvent(st, ch.freed[s], 0));
    ch.freed_pending[s] = false;
  }
  if (c.fsdp == BM_FSDP_ALLGATHER) BM_TRY(fsdp_barrier(c, k, st));
  const auto bl = ch.blocks[ch.seq[j]];
  for (int q = 0; q < c.P; ++q) {
    int64_t qlo, qhi;
    chunk_of(c.dp_elems, c.P, q, &qlo, &qhi);
    const int64_t a = std::max(bl.first, qlo), e = std::min(bl.second, qhi);
    if (e <= a) continue;
    const char* src = (q == c.rank ? c.W : c.peer_w[q]) + (a - qlo) * c.es;
    BM_CUDA_TRY(cudaMemcpyAsync(ch.slot[s] + (a - bl.first) * c.es, src, (size_t)(e - a) * c.es,
                                cudaMemcpyDeviceToDevice, st));
    if (q != c.rank) c.pull_bytes += (e - a) * c.es;
  }
  BM_CUDA_TRY(cudaEventRecord(ch.ready[s], st));
  return BM_OK;
}
// an op starts using chain k with blocks `seq` in this order: prefetch the first two
static bm_status fsdp_begin(bm_ctx& c, int k, std::vector<int> seq, cudaStream_t op_st) {
  if (!c.fsdp) return BM_OK;
  PullChain& ch = c.chain[k];
  // (no wait on op_st: weights are constant within a step, so a pull may run ahead;
  // slot reuse is ordered by the freed events of the slot's last reader)
  ch.seq = std::move(seq);
  for (int j = 0; j < 2 && j < (int)ch.seq.size(); ++j) BM_TRY(fsdp_issue(c, k, j, op_st));
  return BM_OK;
}
// block seq[j] is needed now on op_st: wait for its pull; parameter lookups resolve into it
static bm_status fsdp_acquire(bm_ctx& c, int k, int j, cudaStream_t op_st) {
  if (!c.fsdp) return BM_OK;
  PullChain& ch = c.chain[k];
  if (c.fsdp != BM_FSDP_ALLGATHER) BM_CUDA_TRY(cudaStreamWaitEvent(op_st, ch.ready[j & 1], 0));
  ch.cur = ch.slot[j & 1];
  ch.cur_lo = ch.blocks[ch.seq[j]].first;
  ch.cur_hi = ch.blocks[ch.seq[j]].second;
  return BM_OK;
}
// block seq[j]'s kernels are enqueued: its slot is free once they ran; pull seq[j + 2]
static bm_status fsdp_release(bm_ctx& c, int k, int j, cudaStream_t op_st) {
  if (!c.fsdp) return BM_OK;
  PullChain& ch = c.chain[k];
  BM_CUDA_TRY(cudaEventRecord(ch.freed[j & 1], op_st));
  ch.freed_pending[j & 1] = true;
  ch.cur_lo = ch.cur_hi = 0;
  if (j + 2 < (int)ch.seq.size()) BM_TRY(fsdp_issue(c, k, j + 2, op_st));
  return BM_OK;
}
static std::vector<int> fsdp_order(int nblocks, bool reverse) {
  std::vector<int> v(nblocks);
  for (int i = 0; i < nblocks; ++i) v[i] = reverse ? nblocks - 1 - i : i;
  return v;
}

// ------------------------------------------------------------------ residual MLP blocks (encoder / generator)
// k: FSDP chain, j0: position of block 0 in the op's block sequence (forward order)
static bm_status mlp_blocks_fwd(bm_ctx& c, MlpSlot& sl, const char* prefix, int Lb, int n, int dm, int fm, int k = 0,
                                int j0 = 0) {
  char nm[64];
  for (int i = 0; i < Lb; ++i) {
    BM_TRY(fsdp_acquire(c, k, j0 + i, c.st));
    snprintf(nm, sizeof nm, "%s.blk%d.norm", prefix, i);
    BM_TRY(norm_fwd(c, n, dm, sl.E[i], P_(c, nm), sl.xn[i], sl.rstd[i]));
    snprintf(nm, sizeof nm, "%s.blk%d.fc1", prefix, i);
    BM_TRY(lin_fwd(c, n, dm, fm, sl.xn[i], dm, P_(c, nm), LD_(c, nm), sl.a[i]));
    BM_TRY(gelu_f(c, (int64_t)n * fm, sl.a[i], sl.z[i]));
    snprintf(nm, sizeof nm, "%s.blk%d.fc2", prefix, i);
    BM_TRY(lin_fwd(c, n, fm, dm, sl.z[i], fm, P_(c, nm), LD_(c, nm), sl.E[i + 1], BM_EPI_ADD, sl.E[i]));
    BM_TRY(fsdp_release(c, k, j0 + i, c.st));
  }
  return BM_OK;
}
// dE (n x dm) in/out, updated in place through the blocks in reverse
// blocks in reverse; block i is at position j0 + (Lb - 1 - i) of the op's sequence
static bm_status mlp_blocks_bwd(bm_ctx& c, MlpSlot& sl, const char* prefix, int Lb, int n, int dm, int fm, char* dE,
                                char* dz, char* da, char* dxn, int k = 0, int j0 = 0) {
  char nm[64];
  for (int i = Lb - 1; i >= 0; --i) {
    BM_TRY(fsdp_acquire(c, k, j0 + (Lb - 1 - i), c.st));
    snprintf(nm, sizeof nm, "%s.blk%d.fc2", prefix, i);
    BM_TRY(lin_wgrad(c, n, fm, dm, dE, sl.z[i], fm, G_(c, nm), LD_(c, nm)));
    BM_TRY(lin_dgrad(c, n, fm, dm, dE, P_(c, nm), LD_(c, nm), dz, fm));
    BM_TRY(gelu_b(c, (int64_t)n * fm, dz, sl.a[i], da));
    snprintf(nm, sizeof nm, "%s.blk%d.fc1", prefix, i);
    BM_TRY(lin_wgrad(c, n, dm, fm, da, sl.xn[i], dm, G_(c, nm), LD_(c, nm)));
    BM_TRY(lin_dgrad(c, n, dm, fm, da, P_(c, nm), LD_(c, nm), dxn, dm));
    snprintf(nm, sizeof nm, "%s.blk%d.norm", prefix, i);
    BM_TRY(norm_bwd(c, n, dm, dxn, sl.E[i], P_(c, nm), sl.rstd[i], dE, dE, G_(c, nm)));
    BM_TRY(fsdp_release(c, k, j0 + (Lb - 1 - i), c.st));
  }
  return BM_OK;
}

// ------------------------------------------------------------------ op handlers
static char* recv_slot(bm_ctx& c, int src, int pay, int seq) {
  const Chan& ch = c.chans[c.chan_idx.at(std::make_tuple(src, c.rank, pay))];
  return c.comm + ch.data_off + (int64_t)(seq % ch.K) * ch.slot_bytes;
}

struct RecvState {  // the Recv ops seen since the last compute op (consumer inputs)
  std::vector<const bm_op*> ops;
};

static bm_status op_enc_fwd(bm_ctx& c, const bm_op& o) {
  const auto& m = c.mc;
  const int mb = o.mb, n = c.n_mod[mb];
  const int es_slot = c.enc_next;
  c.enc_next = (c.enc_next + 1) % c.n_enc_slots;
  c.enc_slot_of[mb] = es_slot;
  MlpSlot& sl = c.enc[es_slot];
  const int nb = m.L_e + 2;   // FSDP buckets: patch, the L_e blocks, projector
  BM_TRY(fsdp_begin(c, 0, fsdp_order(nb, false), c.st));
  BM_TRY(fsdp_acquire(c, 0, 0, c.st));
  BM_TRY(lin_fwd(c, n, m.d_in, m.d_e, c.mb_patches[mb], c.ld_patch, P_(c, "enc.patch"), LD_(c, "enc.patch"), sl.E[0]));
  BM_TRY(fsdp_release(c, 0, 0, c.st));
  BM_TRY(mlp_blocks_fwd(c, sl, "enc", m.L_e, n, m.d_e, m.f_e, 0, 1));
  BM_TRY(fsdp_acquire(c, 0, nb - 1, c.st));
  BM_TRY(lin_fwd(c, n, m.d_e, m.d, sl.E[m.L_e], m.d_e, P_(c, "enc.proj1"), LD_(c, "enc.proj1"), sl.a1));
  BM_TRY(gelu_f(c, (int64_t)n * m.d, sl.a1, sl.p1));
  BM_TRY(lin_fwd(c, n, m.d, m.d, sl.p1, m.d, P_(c, "enc.proj2"), LD_(c, "enc.proj2"), sl.out));
  BM_TRY(fsdp_release(c, 0, nb - 1, c.st));
  c.last_src = sl.out;
  c.last_src_ring = -1;
  return BM_OK;
}

static bm_status op_enc_bwd(bm_ctx& c, const bm_op& o, const RecvState& rs) {
  const auto& m = c.mc;
  const int mb = o.mb, n = c.n_mod[mb];
  MlpSlot& sl = c.enc[c.enc_slot_of.at(mb)];
  c.enc_slot_of.erase(mb);
  const char* dout = c.rank == 0 ? c.emb_local : recv_slot(c, 0, BM_PAY_EMBGRAD, rs.ops.at(0)->seq);
  const int nb = m.L_e + 2;   // FSDP buckets in reverse: projector, blocks L_e-1..0, patch
  BM_TRY(fsdp_begin(c, 0, fsdp_order(nb, true), c.st));
  BM_TRY(fsdp_acquire(c, 0, 0, c.st));
  BM_TRY(lin_wgrad(c, n, m.d, m.d, dout, sl.p1, m.d, G_(c, "enc.proj2"), LD_(c, "enc.proj2")));
  BM_TRY(lin_dgrad(c, n, m.d, m.d, dout, P_(c, "enc.proj2"), LD_(c, "enc.proj2"), c.e_dp, m.d));
  BM_TRY(gelu_b(c, (int64_t)n * m.d, c.e_dp, sl.a1, c.e_da));
  BM_TRY(lin_wgrad(c, n, m.d_e, m.d, c.e_da, sl.E[m.L_e], m.d_e, G_(c, "enc.proj1"), LD_(c, "enc.proj1")));
  BM_TRY(lin_dgrad(c, n, m.d_e, m.d, c.e_da, P_(c, "enc.proj1"), LD_(c, "enc.proj1"), c.e_dE, m.d_e));
  BM_TRY(fsdp_release(c, 0, 0, c.st));
  BM_TRY(mlp_blocks_bwd(c, sl, "enc", m.L_e, n, m.d_e, m.f_e, c.e_dE, c.e_dz, c.e_da, c.e_dxn, 0, 1));
  BM_TRY(fsdp_acquire(c, 0, nb - 1, c.st));   // the patch embedding (weight gradient only)
  BM_TRY(lin_wgrad(c, n, m.d_in, m.d_e, c.e_dE, c.mb_patches[mb], c.ld_patch, G_(c, "enc.patch"), LD_(c, "enc.patch")));
  BM_TRY(fsdp_release(c, 0, nb - 1, c.st));
  return BM_OK;
}

static bm_status op_llm_fwd(bm_ctx& c, const bm_op& o, const RecvState& rs) {
  const auto& m = c.mc;
  const int mb = o.mb, ch = o.chunk, s = ch * c.P + c.rank;
  const int64_t S = m.S, d = m.d, es = c.es;
  if (c.llm_free.empty()) {
    set_error("no free LLM stash slot (schedule/peak mismatch)");
    return BM_E_STATE;
  }
  const int slot = c.llm_free.back();
  c.llm_free.pop_back();
  c.llm_live[{mb, ch}] = slot;
  LlmSlot& sl = c.llm[slot];
  // stage input (P:297 embed_preprocess at the entry stage)
  if (s == 0) {
    const int n_mod = c.n_mod[mb];
    const int owner = c.enc_entry ? 0 : sched::enc_owner(c.sc, mb);
    if (c.use_enc_stream && owner == 0)   // this rank's own encoder output (EncFwd on the encoder stream)
      BM_CUDA_TRY(cudaStreamWaitEvent(c.st, c.enc_fwd_ev[c.enc_slot_of.at(mb)], 0));
    const char* emb = owner == 0 ? c.enc[c.enc_slot_of.at(mb)].out : recv_slot(c, owner, BM_PAY_EMB, rs.ops.at(0)->seq);
    BM_TRY(TY(c, embed_fwd<bf16>(m.S, m.d, n_mod, c.ids + (int64_t)mb * S, (const bf16*)P_(c, "llm.embed"), (const bf16*)emb, (bf16*)sl.x[0], c.st),
              embed_fwd<float>(m.S, m.d, n_mod, c.ids + (int64_t)mb * S, (const float*)P_(c, "llm.embed"), (const float*)emb, (float*)sl.x[0], c.st)));
  } else if ((s - 1) % c.P == c.rank) {
    // a boundary inside layer l brings [x_l | h_l] into x[0] (h[0] follows x[0])
    const LlmSlot& pv = c.llm[c.llm_live.at({mb, ch - 1})];
    BM_TRY(d2d(c, sl.x[0], pv.sp.a_last ? pv.x[pv.nl - 1] : pv.x[pv.nl], boundary_bytes(c, s - 1)));
  } else {
    BM_TRY(d2d(c, sl.x[0], recv_slot(c, (s - 1) % c.P, BM_PAY_ACT, rs.ops.at(0)->seq), boundary_bytes(c, s - 1)));
  }
  const Span sp = stage_span(m, c.P * c.V, s);
  const int nl = sp.nl;
  sl.nl = nl;
  sl.sp = sp;
  char nm[64];
  for (int j = 0; j < nl; ++j) {
    const int l = sp.l0 + j;
    if (sp.has_a(j)) {   // A_l: RMSNorm -> gate_up GEMM with SwiGLU
      snprintf(nm, sizeof nm, "llm.layer%d.norm", l);
      BM_TRY(norm_fwd(c, m.S, m.d, sl.x[j], P_(c, nm), sl.xn[j], sl.rstd[j]));
      snprintf(nm, sizeof nm, "llm.layer%d.gate_up", l);
      BM_TRY(lin_gate_up(c, sl.xn[j], P_(c, nm), LD_(c, nm), sl.gu[j], sl.h[j]));
    }
    if (sp.has_b(j)) {   // B_l: down GEMM + residual
      snprintf(nm, sizeof nm, "llm.layer%d.down", l);
      BM_TRY(lin_fwd(c, m.S, m.f, m.d, sl.h[j], m.f, P_(c, nm), LD_(c, nm), sl.x[j + 1], BM_EPI_ADD, sl.x[j]));
    }
  }
  c.last_src = sp.a_last ? sl.x[nl - 1] : sl.x[nl];   // [x_l | h_l] when the stage ends inside layer l
  c.last_src_ring = -1;
  if (s == c.P * c.V - 1) {
    // last stage: final norm, LM head + CE (fwd and bwd through the head), generator inputs
    const int n_mod = c.n_mod[mb], n_text = m.S - n_mod;
    BM_TRY(norm_fwd(c, m.S, m.d, sl.x[nl], P_(c, "llm.final_norm"), sl.Hn, sl.rstd_f));
    // Hn is final: the generator (own shard on the generator stream, remote shards
    // through their genin sends) starts now, overlapping the LM head and CE below
    if (c.hn_ev) BM_CUDA_TRY(cudaEventRecord(c.hn_ev, c.st));
    BM_TRY(zero_bytes(sl.dHn, (int64_t)n_mod * d * es, c.st));
    if (n_text > 0 && !c.head_dp) {
      const char* hn_text = sl.Hn + (int64_t)n_mod * d * es;
      BM_TRY(lin_fwd(c, n_text, m.d, m.vocab, hn_text, m.d, P_(c, "llm.head"), LD_(c, "llm.head"), c.logits));
      const float sg = c.gscale / (float)n_text;
      BM_TRY(TY(c, ce_fwd_bwd<bf16>(n_text, m.vocab, (bf16*)c.logits, c.labels + (int64_t)mb * S + n_mod, sg, c.loss + mb, 1.f, 0, c.ce_scr, c.st),
                ce_fwd_bwd<float>(n_text, m.vocab, (float*)c.logits, c.labels + (int64_t)mb * S + n_mod, sg, c.loss + mb, 1.f, 0, c.ce_scr, c.st)));
      BM_TRY(lin_dgrad(c, n_text, m.d, m.vocab, c.logits, P_(c, "llm.head"), LD_(c, "llm.head"),
                       sl.dHn + (int64_t)n_mod * d * es, m.d));
      BM_TRY(lin_wgrad(c, n_text, m.d, m.vocab, c.logits, hn_text, m.d, G_(c, "llm.head"), LD_(c, "llm.head")));
    }
    const int n_gen = c.n_gen[mb];
    c.genin_src.assign(c.P, nullptr);
    c.headin_src.assign(c.P, nullptr);
    for (int q = 0; q < c.P; ++q) {
      int lo, hi;
      shard_rows(c, mb, q, &lo, &hi);
      c.genin_src[q] = sl.Hn + (int64_t)(m.S - n_gen + lo) * d * es;
      head_rows_of(c, mb, q, &lo, &hi);
      c.headin_src[q] = sl.Hn + (int64_t)lo * d * es;
    }
  }
  return BM_OK;
}

static bm_status op_llm_bwd(bm_ctx& c, const bm_op& o, const RecvState& rs) {
  const auto& m = c.mc;
  const int mb = o.mb, ch = o.chunk, s = ch * c.P + c.rank;
  const int64_t S = m.S, d = m.d, es = c.es;
  const int slot = c.llm_live.at({mb, ch});
  LlmSlot& sl = c.llm[slot];
  const char* cur;
  if (s == c.P * c.V - 1) {
    // add the generator input-gradient shards into dHn, then final-norm backward
    const int n_gen = c.n_gen[mb];
    auto og = c.own_gout.find(mb);
    if (c.head_dp) {
      // head shards' dHn (text rows, disjoint across shards) first, then the generator adds
      for (const bm_op* r : rs.ops) {
        int lo, hi;
        head_rows_of(c, mb, r->peer, &lo, &hi);
        BM_TRY(d2d(c, sl.dHn + (int64_t)lo * d * es, recv_slot(c, r->peer, BM_PAY_GENGRAD, r->seq), (int64_t)(hi - lo) * d * es));
      }
      if (og != c.own_gout.end()) {
        int lo, hi;
        head_rows_of(c, mb, c.rank, &lo, &hi);
        BM_TRY(d2d(c, sl.dHn + (int64_t)lo * d * es, c.gout[og->second], (int64_t)(hi - lo) * d * es));
      }
    }
    if (c.has_gen && !c.gen_last) {
      for (const bm_op* r : rs.ops) {
        int lo, hi, hlo, hhi;
        shard_rows(c, mb, r->peer, &lo, &hi);
        head_rows_of(c, mb, r->peer, &hlo, &hhi);
        char* dst = sl.dHn + (int64_t)(m.S - n_gen + lo) * d * es;
        const char* src = recv_slot(c, r->peer, BM_PAY_GENGRAD, r->seq) + (int64_t)(hhi - hlo) * d * es;
        BM_TRY(add_(c, (int64_t)(hi - lo) * d, dst, src, dst));
      }
    }
    if (og != c.own_gout.end()) {
      // this rank's own shard (the whole generator under BM_GEN_LAST_STAGE)
      int lo, hi, hlo, hhi;
      shard_rows(c, mb, c.rank, &lo, &hi);
      head_rows_of(c, mb, c.rank, &hlo, &hhi);
      char* dst = sl.dHn + (int64_t)(m.S - n_gen + lo) * d * es;
      BM_TRY(add_(c, (int64_t)(hi - lo) * d, dst, c.gout[og->second] + (int64_t)(hhi - hlo) * d * es, dst));
      // the generator stream must not overwrite this gout slot before the add ran
      BM_CUDA_TRY(cudaEventRecord(c.gout_ev[og->second], c.st));
      c.gout_pending[og->second] = true;
      c.own_gout.erase(og);
    }
    char* top = (c.zb && sl.nl > 0) ? sl.wdy[sl.nl - 1] : c.dwork[0];
    BM_TRY(norm_bwd(c, m.S, m.d, sl.dHn, sl.x[sl.nl], P_(c, "llm.final_norm"), sl.rstd_f, nullptr, top,
                    G_(c, "llm.final_norm")));
    cur = top;
  } else if ((s + 1) % c.P == c.rank) {
    cur = sl.gin;
  } else {
    cur = recv_slot(c, (s + 1) % c.P, BM_PAY_GRAD, rs.ops.at(0)->seq);
  }
  // output ring buffer (must not be overwritten before its previous send copy finished)
  const int b = c.bsel;
  c.bsel ^= 1;
  if (c.bout_pending[b]) {
    BM_CUDA_TRY(cudaStreamWaitEvent(c.st, c.bout_ev[b], 0));
    c.bout_pending[b] = false;
  }
  char nm[64];
  const Span sp = sl.sp;
  const int l0 = sp.l0, nl = sp.nl;
  // a stage ending inside layer l receives [dx_{l+1} | dh_l] (cur, cur + S d): only A_l's
  // backward runs here; one starting inside layer l sends [dx_{l+1} | dh_l] (R24)
  auto swiglu_bwd_of = [&](const char* dh, const char* gu, char* dgu) -> bm_status {
    return TY(c, swiglu_bwd<bf16>(m.S, m.f, (const bf16*)dh, (const bf16*)gu, (bf16*)dgu, c.st),
              swiglu_bwd<float>(m.S, m.f, (const float*)dh, (const float*)gu, (float*)dgu, c.st));
  };
  if (c.zb) {
    // ZB-H1 B: input gradient only; every layer's dY and dgu stay in the slot for W (R23)
    if (nl > 0 && sp.has_b(nl - 1) && cur != sl.wdy[nl - 1]) BM_TRY(d2d(c, sl.wdy[nl - 1], cur, S * d * es));
    for (int j = nl - 1; j >= 0; --j) {
      const int l = l0 + j;
      char* out = (j == 0) ? c.bout[b] : sl.wdy[j - 1];
      if (!sp.has_a(j)) {   // B_l only (j = 0): send [dx_{l+1} | dh_l]
        snprintf(nm, sizeof nm, "llm.layer%d.down", l);
        BM_TRY(lin_dgrad(c, m.S, m.f, m.d, sl.wdy[j], P_(c, nm), LD_(c, nm), out + S * d * es, m.f));
        BM_TRY(d2d(c, out, sl.wdy[j], S * d * es));
        continue;
      }
      const char* resid = sl.wdy[j];
      if (!sp.has_b(j)) {   // A_l only (j = nl - 1): dgu from the received dh
        BM_TRY(swiglu_bwd_of(cur + S * d * es, sl.gu[j], sl.wdgu[j]));
        resid = cur;
      } else {
        snprintf(nm, sizeof nm, "llm.layer%d.down", l);
        BM_TRY(lin_down_dgrad_swiglu(c, sl.wdy[j], P_(c, nm), LD_(c, nm), sl.gu[j], c.dh, sl.wdgu[j]));
      }
      snprintf(nm, sizeof nm, "llm.layer%d.gate_up", l);
      BM_TRY(lin_dgrad(c, m.S, m.d, 2 * m.f, sl.wdgu[j], P_(c, nm), LD_(c, nm), c.dxn, m.d));
      snprintf(nm, sizeof nm, "llm.layer%d.norm", l);
      BM_TRY(norm_bwd(c, m.S, m.d, c.dxn, sl.x[j], P_(c, nm), sl.rstd[j], resid, out, G_(c, nm)));
    }
  }
  for (int j = c.zb ? -1 : nl - 1; j >= 0; --j) {
    const int l = l0 + j;
    char* out = (j == 0) ? c.bout[b] : (cur == c.dwork[0] ? c.dwork[1] : c.dwork[0]);
    if (!sp.has_a(j)) {   // B_l only (j = 0): down wgrad, dh = dY W_down, send [dY | dh]
      snprintf(nm, sizeof nm, "llm.layer%d.down", l);
      BM_TRY(lin_wgrad(c, m.S, m.f, m.d, cur, sl.h[j], m.f, G_(c, nm), LD_(c, nm)));
      BM_TRY(lin_dgrad(c, m.S, m.f, m.d, cur, P_(c, nm), LD_(c, nm), out + S * d * es, m.f));
      BM_TRY(d2d(c, out, cur, S * d * es));
      cur = out;
      continue;
    }
    if (!sp.has_b(j)) {   // A_l only (j = nl - 1): dgu = SwiGLU backward of the received dh
      BM_TRY(swiglu_bwd_of(cur + S * d * es, sl.gu[j], c.dgu));
    } else {
      snprintf(nm, sizeof nm, "llm.layer%d.down", l);
      if (c.fuse_swiglu && c.dtype == BM_BF16 && m.f % 32 == 0) {
        // down wgrad + down dgrad with the SwiGLU backward in its epilogue: one grouped launch
        GemmSpec gs[2] = {spec_wgrad(m.S, m.f, m.d, cur, sl.h[j], m.f, G_(c, nm), LD_(c, nm)),
                          GemmSpec{(int)m.S, m.f, m.d, cur, m.d, 0, P_(c, nm), LD_(c, nm), 1, c.dgu, 2 * (int64_t)m.f,
                                   BM_BF16, BM_EPI_DSWIGLU, sl.gu[j], 2 * (int64_t)m.f, 1.f, m.f, nullptr, 0}};
        BM_TRY(timed_group(c, gs, 2));
      } else {
        BM_TRY(lin_wgrad(c, m.S, m.f, m.d, cur, sl.h[j], m.f, G_(c, nm), LD_(c, nm)));
        BM_TRY(lin_down_dgrad_swiglu(c, cur, P_(c, nm), LD_(c, nm), sl.gu[j], c.dh, c.dgu));
      }
    }
    snprintf(nm, sizeof nm, "llm.layer%d.gate_up", l);
    {
      // gate_up dgrad + gate_up wgrad: one grouped launch
      GemmSpec gs[2] = {spec_dgrad(c, m.S, m.d, 2 * m.f, c.dgu, P_(c, nm), LD_(c, nm), c.dxn, m.d),
                        spec_wgrad(m.S, m.d, 2 * m.f, c.dgu, sl.xn[j], m.d, G_(c, nm), LD_(c, nm))};
      BM_TRY(timed_group(c, gs, 2));
    }
    snprintf(nm, sizeof nm, "llm.layer%d.norm", l);
    BM_TRY(norm_bwd(c, m.S, m.d, c.dxn, sl.x[j], P_(c, nm), sl.rstd[j], cur, out, G_(c, nm)));
    cur = out;
  }
  c.last_src = c.bout[b];
  c.last_src_ring = 0;
  c.last_src_idx = b;
  if (s == 0) {
    const int n_mod = c.n_mod[mb];
    BM_TRY(TY(c, embed_bwd<bf16>(m.S, m.d, n_mod, c.ids + (int64_t)mb * S, (const bf16*)c.bout[b], G_(c, "llm.embed"), c.embscr, c.st),
              embed_bwd<float>(m.S, m.d, n_mod, c.ids + (int64_t)mb * S, (const float*)c.bout[b], G_(c, "llm.embed"), c.embscr, c.st)));
    if (c.enc_entry || sched::enc_owner(c.sc, mb) == 0) {
      if (c.emb_free_pending) {   // the previous EncBwd (encoder stream) has read emb_local
        BM_CUDA_TRY(cudaStreamWaitEvent(c.st, c.emb_free_ev, 0));
        c.emb_free_pending = false;
      }
      BM_TRY(d2d(c, c.emb_local, c.bout[b], (int64_t)n_mod * d * es));
      if (c.use_enc_stream) BM_CUDA_TRY(cudaEventRecord(c.emb_ready_ev, c.st));
    }
  } else if ((s - 1) % c.P == c.rank) {
    BM_TRY(d2d(c, c.llm[c.llm_live.at({mb, ch - 1})].gin, c.bout[b], boundary_bytes(c, s - 1)));
  }
  if (!c.zb) {   // under ZB-H1 the stash lives until W
    c.llm_live.erase({mb, ch});
    c.llm_free.push_back(slot);
  }
  return BM_OK;
}

// ZB-H1 W (R23): the two weight-gradient GEMMs of every layer, dW += dY^T X with the
// operands B left in the slot (down: dY, h; gate_up: dgu, xn); then the slot is free
static bm_status op_llm_w(bm_ctx& c, const bm_op& o) {
  const auto& m = c.mc;
  const int slot = c.llm_live.at({o.mb, o.chunk});
  LlmSlot& sl = c.llm[slot];
  const Span sp = sl.sp;
  char nd[64], ng[64];
  for (int j = sp.nl - 1; j >= 0; --j) {
    snprintf(nd, sizeof nd, "llm.layer%d.down", sp.l0 + j);
    snprintf(ng, sizeof ng, "llm.layer%d.gate_up", sp.l0 + j);
    GemmSpec gs[2];
    int n = 0;
    if (sp.has_b(j)) gs[n++] = spec_wgrad(m.S, m.f, m.d, sl.wdy[j], sl.h[j], m.f, G_(c, nd), LD_(c, nd));
    if (sp.has_a(j)) gs[n++] = spec_wgrad(m.S, m.d, 2 * m.f, sl.wdgu[j], sl.xn[j], m.d, G_(c, ng), LD_(c, ng));
    BM_TRY(timed_group(c, gs, n));
  }
  c.llm_live.erase({o.mb, o.chunk});
  c.llm_free.push_back(slot);
  return BM_OK;
}

static bm_status op_gen_fwd(bm_ctx& c, const bm_op& o, const RecvState& rs) {
  const auto& m = c.mc;
  const int mb = o.mb;
  const int64_t row = (int64_t)m.d * c.es;
  // this microbatch's gout slot ([dHn head rows | generator dX rows]); it must not be
  // overwritten before its previous send copy / own-shard add finished
  const int b = c.gsel;
  c.gsel ^= 1;
  c.gen_b = b;
  if (c.gout_pending[b]) {
    BM_CUDA_TRY(cudaStreamWaitEvent(c.st, c.gout_ev[b], 0));
    c.gout_pending[b] = false;
  }
  const bool own = c.rank == c.P - 1;
  const char* slot = own ? nullptr : recv_slot(c, c.P - 1, BM_PAY_GENIN, rs.ops.at(0)->seq);
  int hlo, hhi;
  head_rows_of(c, mb, c.rank, &hlo, &hhi);
  const int nh = hhi - hlo;
  if (nh > 0) {
    // LM head shard (head_dp): logits, CE fwd+bwd with the full-microbatch denominator
    // (R8), dHn rows into gout, head weight gradient (DP parameter)
    const char* Xh = own ? c.headin_src[c.rank] : slot;
    const int n_text = m.S - c.n_mod[mb];
    BM_TRY(lin_fwd(c, nh, m.d, m.vocab, Xh, m.d, P_(c, "llm.head"), LD_(c, "llm.head"), c.logits));
    const float sg = c.gscale / (float)n_text;
    const float sl_ = (float)nh / (float)n_text;
    BM_TRY(TY(c, ce_fwd_bwd<bf16>(nh, m.vocab, (bf16*)c.logits, c.labels + (int64_t)mb * m.S + hlo, sg, c.loss + mb, sl_, 1, c.ce_scr, c.st),
              ce_fwd_bwd<float>(nh, m.vocab, (float*)c.logits, c.labels + (int64_t)mb * m.S + hlo, sg, c.loss + mb, sl_, 1, c.ce_scr, c.st)));
    BM_TRY(lin_dgrad(c, nh, m.d, m.vocab, c.logits, P_(c, "llm.head"), LD_(c, "llm.head"), c.gout[b], m.d));
    BM_TRY(lin_wgrad(c, nh, m.d, m.vocab, c.logits, Xh, m.d, G_(c, "llm.head"), LD_(c, "llm.head")));
  }
  int lo, hi;
  shard_rows(c, mb, c.rank, &lo, &hi);
  const int n = hi - lo;
  if (n <= 0) return BM_OK;
  const char* X = own ? c.genin_src[c.rank] : slot + (int64_t)nh * row;
  MlpSlot& sl = c.gen;
  const int nb = m.L_g + 2;   // FSDP buckets: in-projection, the L_g blocks, out-projection
  BM_TRY(fsdp_begin(c, 1, fsdp_order(nb, false), c.st));
  BM_TRY(fsdp_acquire(c, 1, 0, c.st));
  BM_TRY(lin_fwd(c, n, m.d, m.d_g, X, m.d, P_(c, "gen.in"), LD_(c, "gen.in"), sl.E[0]));
  BM_TRY(fsdp_release(c, 1, 0, c.st));
  BM_TRY(mlp_blocks_fwd(c, sl, "gen", m.L_g, n, m.d_g, m.f_g, 1, 1));
  BM_TRY(fsdp_acquire(c, 1, nb - 1, c.st));
  BM_TRY(lin_fwd(c, n, m.d_g, m.d_t, sl.E[m.L_g], m.d_g, P_(c, "gen.out"), LD_(c, "gen.out"), sl.out));
  BM_TRY(fsdp_release(c, 1, nb - 1, c.st));
  const char* t = c.mb_targets[mb] + (int64_t)lo * m.d_t * c.es;
  const float denom = (float)c.n_gen[mb] * m.d_t;
  BM_TRY(TY(c, mse_fwd_bwd<bf16>(n, m.d_t, (const bf16*)sl.out, (const bf16*)t, denom, c.gscale, 1.f, c.loss + c.M + mb, (bf16*)sl.dout, c.st),
            mse_fwd_bwd<float>(n, m.d_t, (const float*)sl.out, (const float*)t, denom, c.gscale, 1.f, c.loss + c.M + mb, (float*)sl.dout, c.st)));
  return BM_OK;
}

static bm_status op_gen_bwd(bm_ctx& c, const bm_op& o, const char* X) {
  const auto& m = c.mc;
  const int mb = o.mb;
  int lo, hi, hlo, hhi;
  shard_rows(c, mb, c.rank, &lo, &hi);
  head_rows_of(c, mb, c.rank, &hlo, &hhi);
  const int n = hi - lo;
  MlpSlot& sl = c.gen;
  const int b = c.gen_b;   // chosen (and waited for) by GenFwd
  c.last_src = c.gout[b];
  c.last_src_ring = 1;
  c.last_src_idx = b;
  if (c.rank == c.P - 1) c.own_gout[mb] = b;
  if (n <= 0) return BM_OK;
  const int nb = m.L_g + 2;   // FSDP buckets in reverse
  BM_TRY(fsdp_begin(c, 1, fsdp_order(nb, true), c.st));
  BM_TRY(fsdp_acquire(c, 1, 0, c.st));
  BM_TRY(lin_wgrad(c, n, m.d_g, m.d_t, sl.dout, sl.E[m.L_g], m.d_g, G_(c, "gen.out"), LD_(c, "gen.out")));
  BM_TRY(lin_dgrad(c, n, m.d_g, m.d_t, sl.dout, P_(c, "gen.out"), LD_(c, "gen.out"), c.g_dG, m.d_g));
  BM_TRY(fsdp_release(c, 1, 0, c.st));
  BM_TRY(mlp_blocks_bwd(c, sl, "gen", m.L_g, n, m.d_g, m.f_g, c.g_dG, c.g_dz, c.g_da, c.g_dxn, 1, 1));
  BM_TRY(fsdp_acquire(c, 1, nb - 1, c.st));
  BM_TRY(lin_wgrad(c, n, m.d, m.d_g, c.g_dG, X, m.d, G_(c, "gen.in"), LD_(c, "gen.in")));
  // dX of this shard into the gout ring: sent to the last stage, or (own shard on
  // the last stage) added into dHn by B(mb, V-1) -- never written into dHn here,
  // where the LM-head dgrad of the same rows may still be running on the compute stream
  BM_TRY(lin_dgrad(c, n, m.d, m.d_g, c.g_dG, P_(c, "gen.in"), LD_(c, "gen.in"),
                   c.gout[b] + (int64_t)(hhi - hlo) * m.d * c.es, m.d));
  BM_TRY(fsdp_release(c, 1, nb - 1, c.st));
  return BM_OK;
}

// ------------------------------------------------------------------ comm ops
// bytes of a message this rank sends (src_rank_for_shard: the shard's rank for genin / gengrad)
static int64_t payload_bytes(const bm_ctx& c, const bm_op& o, int src_rank_for_shard) {
  const int64_t row = (int64_t)c.mc.d * c.es;
  switch (o.payload) {
    case BM_PAY_ACT: return boundary_bytes(c, o.chunk * c.P + c.rank);
    case BM_PAY_GRAD: return boundary_bytes(c, o.chunk * c.P + c.rank - 1);
    case BM_PAY_EMB:
    case BM_PAY_EMBGRAD: return c.n_mod[o.mb] * row;
    default: {   // genin / gengrad: [head rows | generator rows] of the shard's rank
      int lo, hi, hlo, hhi;
      shard_rows(c, o.mb, src_rank_for_shard, &lo, &hi);
      head_rows_of(c, o.mb, src_rank_for_shard, &hlo, &hhi);
      return (int64_t)(hi - lo + hhi - hlo) * row;
    }
  }
}

// NVLink write of one message into the peer's receive slot: a copy-engine copy on
// the comm stream (no SM time taken from the GEMMs; measured 138.3 vs 135.0
// samples/s for an SM copy kernel at C2, N = 4).  BM_PEER_COPY=sm selects the SM
// copy kernel (bm_k_copy) instead.
static bm_status peer_copy(bm_ctx& c, char* dst, const char* src, int64_t bytes, cudaStream_t cs) {
  if (c.peer_copy_ce) {
    BM_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, cs));
    return BM_OK;
  }
  return copy_bytes(dst, src, bytes, c.peer_copy_ctas, cs);
}

// stream-ordered wait until a local flag (written by a peer) reaches v
static bm_status wait_flag(bm_ctx& c, cudaStream_t on, char* flag, uint32_t v, const char* what) {
  if (c.spin_wait) return spin_wait((const uint32_t*)flag, v, on);
  CUresult r = drv().wait32((CUstream)on, (CUdeviceptr)flag, v, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    set_error(std::string("cuStreamWaitValue32 (") + what + ") failed " + std::to_string((int)r));
    return BM_E_CUDA;
  }
  return BM_OK;
}

static bm_status do_send(bm_ctx& c, const bm_op& o, int idx) {
  const Chan& ch = c.chans[c.chan_idx.at(std::make_tuple(c.rank, o.peer, o.payload))];
  cudaStream_t cs = c.comm_st[o.peer];
  if (o.payload == BM_PAY_GENIN && c.hn_ev) {
    BM_CUDA_TRY(cudaStreamWaitEvent(cs, c.hn_ev, 0));   // Hn rows exist (mid F(m, V-1))
  } else {
    if (!c.producer_ev) {
      c.producer_ev = next_event(c);
      BM_CUDA_TRY(cudaEventRecord(c.producer_ev, c.producer_st ? c.producer_st : c.st));
    }
    BM_CUDA_TRY(cudaStreamWaitEvent(cs, c.producer_ev, 0));
  }
  const uint32_t base = (uint32_t)(c.step * ch.nmsg);
  if (o.seq >= ch.K) {
    BM_TRY(wait_flag(c, cs, c.comm + ch.credit_off, base + (uint32_t)(o.seq - ch.K) + 1, "credit"));
  }
  // the message as (source, bytes) segments packed back to back into the slot:
  // genin = [head rows of Hn (head_dp) | generator rows of Hn]; others one segment
  const char* seg_src[2] = {nullptr, nullptr};
  int64_t seg_bytes[2] = {0, 0};
  if (o.payload == BM_PAY_GENIN) {
    int hlo, hhi;
    head_rows_of(c, o.mb, o.peer, &hlo, &hhi);
    seg_src[0] = c.headin_src.empty() ? nullptr : c.headin_src[o.peer];
    seg_bytes[0] = (int64_t)(hhi - hlo) * c.mc.d * c.es;
    seg_src[1] = c.genin_src[o.peer];
    seg_bytes[1] = payload_bytes(c, o, o.peer) - seg_bytes[0];
  } else {
    seg_src[0] = (const char*)c.last_src;
    seg_bytes[0] = payload_bytes(c, o, c.rank);
  }
  const int64_t bytes = seg_bytes[0] + seg_bytes[1];
  char* dst = c.peer[o.peer] + ch.data_off + (int64_t)(o.seq % ch.K) * ch.slot_bytes;
  auto copy_msg = [&]() -> bm_status {
    if (seg_bytes[0] > 0) BM_TRY(peer_copy(c, dst, seg_src[0], seg_bytes[0], cs));
    if (seg_bytes[1] > 0) BM_TRY(peer_copy(c, dst + seg_bytes[0], seg_src[1], seg_bytes[1], cs));
    return BM_OK;
  };
  cudaEvent_t tr_a = c.tracing ? trace_mark(c, cs) : nullptr;
  if (c.timing && bytes > 0) {
    const int pool = (int)(c.step & 1);
    auto& ev = c.cev[pool];
    const size_t k = c.cbytes[pool].size();
    while (ev.size() < 2 * (k + 1)) {
      cudaEvent_t e;
      BM_CUDA_TRY(cudaEventCreate(&e));
      ev.push_back(e);
    }
    BM_CUDA_TRY(cudaEventRecord(ev[2 * k], cs));
    BM_TRY(copy_msg());
    BM_CUDA_TRY(cudaEventRecord(ev[2 * k + 1], cs));
    c.cbytes[pool].push_back(bytes);
  } else if (bytes > 0) {
    BM_TRY(copy_msg());
  }
  CUresult r = drv().write32((CUstream)cs, (CUdeviceptr)(c.peer[o.peer] + ch.flag_off), base + (uint32_t)o.seq + 1, 0);
  if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 (data flag) failed " + std::to_string((int)r)); return BM_E_CUDA; }
  if (c.tracing) c.trace.push_back({idx, (int32_t)o.kind, 2 + o.peer, o.mb, tr_a, trace_mark(c, cs)});
  if (c.last_src_ring == 0 && o.payload != BM_PAY_GENIN) {
    BM_CUDA_TRY(cudaEventRecord(c.bout_ev[c.last_src_idx], cs));
    c.bout_pending[c.last_src_idx] = true;
  } else if (c.last_src_ring == 1 && o.payload == BM_PAY_GENGRAD) {
    BM_CUDA_TRY(cudaEventRecord(c.gout_ev[c.last_src_idx], cs));
    c.gout_pending[c.last_src_idx] = true;
  }
  return BM_OK;
}

static bm_status do_recv_wait(bm_ctx& c, const bm_op& o, cudaStream_t on) {
  const Chan& ch = c.chans[c.chan_idx.at(std::make_tuple(o.peer, c.rank, o.payload))];
  const uint32_t base = (uint32_t)(c.step * ch.nmsg);
  return wait_flag(c, on, c.comm + ch.flag_off, base + (uint32_t)o.seq + 1, "data");
}

static bm_status do_release(bm_ctx& c, const bm_op& o, cudaStream_t on) {
  const Chan& ch = c.chans[c.chan_idx.at(std::make_tuple(o.peer, c.rank, o.payload))];
  const uint32_t base = (uint32_t)(c.step * ch.nmsg);
  CUresult r = drv().write32((CUstream)on, (CUdeviceptr)(c.peer[o.peer] + ch.credit_off), base + (uint32_t)o.seq + 1, 0);
  if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 (credit) failed " + std::to_string((int)r)); return BM_E_CUDA; }
  return BM_OK;
}

// ------------------------------------------------------------------ step-end sums over peer memory
// barrier over all P D processes: write v into this process's flag slot at every
// process, then wait until every process has written >= v into ours
static bm_status psum_barrier(bm_ctx& c, uint32_t v) {
  const int world = (int)c.ps_comm.size(), me = c.replica * c.P + c.rank;
  for (int g = 0; g < world; ++g) {
    CUresult r = drv().write32((CUstream)c.st, (CUdeviceptr)(c.ps_comm[g] + 64 * me), v, 0);
    if (r != CUDA_SUCCESS) { set_error("cuStreamWriteValue32 (sum barrier) failed " + std::to_string((int)r)); return BM_E_CUDA; }
  }
  for (int g = 0; g < world; ++g)
    if (g != me) BM_TRY(wait_flag(c, c.st, c.ps_comm[me] + 64 * g, v, "sum barrier"));
  return BM_OK;
}

// reduce-scatter of [off, off + count) of the gradient buffers over `group`
// (process indices): this process sums chunk me_idx in group order, in place
static bm_status psum_reduce_scatter(bm_ctx& c, const std::vector<int>& group, int me_idx, int64_t off, int64_t count) {
  int64_t lo, hi;
  chunk_of(count, (int)group.size(), me_idx, &lo, &hi);
  if (hi <= lo) return BM_OK;
  PeerSrc s{};
  for (size_t q = 0; q < group.size(); ++q) s.p[q] = c.ps_grad[group[q]] + off + lo;
  return peer_sum(s, (int)group.size(), c.G + off + lo, hi - lo, c.st);
}
// all-gather: copy every other member's reduced chunk
static bm_status psum_all_gather(bm_ctx& c, const std::vector<int>& group, int me_idx, int64_t off, int64_t count) {
  for (size_t q = 0; q < group.size(); ++q) {
    if ((int)q == me_idx) continue;
    int64_t lo, hi;
    chunk_of(count, (int)group.size(), (int)q, &lo, &hi);
    if (hi > lo)
      BM_CUDA_TRY(cudaMemcpyAsync(c.G + off + lo, c.ps_grad[group[q]] + off + lo, (size_t)(hi - lo) * 4,
                                  cudaMemcpyDeviceToDevice, c.st));
  }
  return BM_OK;
}

// DP parameters over every process, the stage's LLM parameters over its D replicas,
// loss terms over the pipeline, the global-batch loss over everyone (A18)
static bm_status peer_finalize(bm_ctx& x) {
  const int world = x.P * x.D, me = x.replica * x.P + x.rank;
  const uint32_t base = (uint32_t)(x.step * 4);
  float* raw = (float*)(x.ps_comm[me] + SUMBLK_LOSS);
  BM_CUDA_TRY(cudaMemcpyAsync(raw, x.loss, (size_t)2 * x.M * 4, cudaMemcpyDeviceToDevice, x.st));
  BM_TRY(psum_barrier(x, base + 1));   // every gradient and loss term of the step is final
  std::vector<int> all(world), stage(x.D), pipe(x.P);
  for (int g = 0; g < world; ++g) all[g] = g;
  for (int k = 0; k < x.D; ++k) stage[k] = k * x.P + x.rank;
  for (int r = 0; r < x.P; ++r) pipe[r] = x.replica * x.P + r;
  BM_TRY(psum_reduce_scatter(x, all, me, 0, x.dp_elems));
  if (x.D > 1) BM_TRY(psum_reduce_scatter(x, stage, x.replica, x.dp_elems, x.total_elems - x.dp_elems));
  PeerSrc sp{}, sw{};
  for (int r = 0; r < x.P; ++r) sp.p[r] = (const float*)(x.ps_comm[pipe[r]] + SUMBLK_LOSS);
  for (int g = 0; g < world; ++g) sw.p[g] = (const float*)(x.ps_comm[g] + SUMBLK_LOSS);
  BM_TRY(peer_loss(sp, x.P, sw, world, x.M, 1.f / ((float)x.M * (float)x.D), x.loss, x.st));
  BM_TRY(psum_barrier(x, base + 2));   // every owned chunk is reduced
  // FSDP keeps only the own shard of the DP gradients (reduce-scatter; the chunks are
  // the weight shards, chunk_of over the pipeline group)
  if (!x.fsdp) BM_TRY(psum_all_gather(x, all, me, 0, x.dp_elems));
  if (x.D > 1) BM_TRY(psum_all_gather(x, stage, x.replica, x.dp_elems, x.total_elems - x.dp_elems));
  BM_TRY(psum_barrier(x, base + 3));   // nobody reads this step's buffers any more
  return BM_OK;
}

}  // namespace bm

// ================================================================ C ABI
extern "C" {

bm_status bm_param_count(const bm_model_cfg* mc, const bm_sched_cfg* sc, int32_t rank, int32_t* n,
                         int64_t* total_elems, int64_t* dp_elems) {
  BM_CHECK_ARG(mc && sc && n && total_elems && dp_elems, "null argument");
  BM_CHECK_ARG(rank >= 0 && rank < sc->stages, "rank out of range");
  BM_TRY(check_model(*mc, *sc));
  auto v = param_layout(*mc, *sc, rank, total_elems, dp_elems);
  *n = (int32_t)v.size();
  return BM_OK;
}

bm_status bm_param_info_get(const bm_model_cfg* mc, const bm_sched_cfg* sc, int32_t rank, int32_t idx,
                            bm_param_info* out) {
  BM_CHECK_ARG(mc && sc && out, "null argument");
  BM_CHECK_ARG(rank >= 0 && rank < sc->stages, "rank out of range");
  BM_TRY(check_model(*mc, *sc));
  int64_t t, dp;
  auto v = param_layout(*mc, *sc, rank, &t, &dp);
  BM_CHECK_ARG(idx >= 0 && idx < (int)v.size(), "param index out of range");
  std::memset(out, 0, sizeof(*out));
  std::strncpy(out->name, v[idx].name.c_str(), sizeof(out->name) - 1);
  out->rows = v[idx].rows;
  out->cols = v[idx].cols;
  out->offset = v[idx].off;
  out->kind = v[idx].kind;
  out->ld = v[idx].ld;
  return BM_OK;
}

bm_status bm_ctx_create(const bm_model_cfg* mc, const bm_schedule* s, int32_t rank, bm_ctx** out) {
  BM_CHECK_ARG(mc && s && out, "null argument");
  BM_CHECK_ARG(rank >= 0 && rank < s->cfg.stages, "rank out of range");
  BM_TRY(check_model(*mc, s->cfg));
  auto* c = new bm_ctx();
  c->mc = *mc;
  c->sc = s->cfg;
  c->s = s;
  c->rank = rank;
  c->P = s->cfg.stages;
  c->M = s->cfg.microbatches;
  c->gscale = 1.f / (float)c->M;
  c->V = s->cfg.vchunks;
  c->lps = max_stage_layers(*mc, c->P, c->V, rank);
  c->dtype = mc->dtype;
  c->es = mc->dtype == BM_BF16 ? 2 : 4;
  c->params = param_layout(*mc, s->cfg, rank, &c->total_elems, &c->dp_elems);
  for (size_t i = 0; i < c->params.size(); ++i) c->pidx[c->params[i].name] = (int)i;
  c->has_enc = s->cfg.enc_place != BM_ENC_NONE;
  c->has_gen = s->cfg.gen_place != BM_GEN_NONE;
  c->gen_last = s->cfg.gen_place == BM_GEN_LAST_STAGE;
  c->enc_entry = s->cfg.enc_place == BM_ENC_ENTRY_STAGE;
  if (!c->has_enc) {
    delete c;
    set_error("the executor requires an encoder placement (embed_preprocess consumes encoder outputs)");
    return BM_E_INVALID;
  }
  const bm_sched_stats& st = s->stats[rank];
  c->zb = s->cfg.llm_sched == BM_LLM_ZB_H1;
  for (int b = 0; b + 1 < c->P * c->V; ++b)
    if (stage_span(*mc, c->P * c->V, b).a_last) c->mid_cols = mc->f;
  c->n_llm_slots = std::max(st.peak_llm_inflight, 1);   // F..B (F..W under ZB-H1)
  c->n_enc_slots = std::max(st.peak_enc_units, 1);
  {
    int nk = 0;
    for (int q = 0; q < c->P; ++q) nk += !(((uint32_t)mc->gen_exclude >> q) & 1u);
    const bool ex = ((uint32_t)mc->gen_exclude >> rank) & 1u;
    c->gen_rows = c->gen_last ? (rank == c->P - 1 ? mc->max_n_gen : 0) : (ex ? 0 : (mc->max_n_gen + nk - 1) / nk);
    c->gen_rows_max = c->gen_last ? mc->max_n_gen : (mc->max_n_gen + nk - 1) / nk;
  }
  if (!c->has_gen) c->gen_rows = c->gen_rows_max = 0;
  c->head_dp = head_dp(*mc, s->cfg);
  c->head_rows = c->head_dp ? (mc->S + c->P - 1) / c->P : 0;
  c->fsdp = mc->fsdp;
  if (c->fsdp) {
    chunk_of(c->dp_elems, c->P, rank, &c->dp_lo, &c->dp_hi);
    // bucket chains: [patch] [blk0] .. [blk L_e-1] [proj1 proj2]; [gen.in] [blk0] .. [gen.out]
    auto range = [&](std::initializer_list<std::string> names) {
      int64_t lo = INT64_MAX, hi = 0;
      for (const auto& n : names) {
        const PEntry& e = c->params[c->pidx.at(n)];
        lo = std::min(lo, e.off);
        hi = std::max(hi, e.off + (int64_t)e.rows * e.ld);
      }
      return std::make_pair(lo, hi);
    };
    auto& ce = c->chain[0].blocks;
    ce.push_back(range({"enc.patch"}));
    for (int i = 0; i < mc->L_e; ++i) {
      const std::string p = "enc.blk" + std::to_string(i);
      ce.push_back(range({p + ".norm", p + ".fc1", p + ".fc2"}));
    }
    ce.push_back(range({"enc.proj1", "enc.proj2"}));
    auto& cg = c->chain[1].blocks;
    cg.push_back(range({"gen.in"}));
    for (int i = 0; i < mc->L_g; ++i) {
      const std::string p = "gen.blk" + std::to_string(i);
      cg.push_back(range({p + ".norm", p + ".fc1", p + ".fc2"}));
    }
    cg.push_back(range({"gen.out"}));
  } else {
    c->dp_lo = 0;
    c->dp_hi = c->dp_elems;
  }
  comm_layout(*c);
  work_layout(*c, nullptr);
  // release annotations: Recv at i is released after the compute op j (genin: the following GenBwd)
  const auto& ops = s->ranks[rank];
  c->release_of.assign(ops.size(), {});
  for (size_t i = 0; i < ops.size(); ++i) {
    if (ops[i].kind != BM_OP_RECV) continue;
    size_t j = i + 1;
    while (is_comm(ops[j].kind)) ++j;
    if (ops[i].payload == BM_PAY_GENIN)
      while (ops[j].kind != BM_OP_GEN_BWD) ++j;
    c->release_of[j].push_back((int)i);
  }
  c->consumer_kind.assign(ops.size(), -1);
  for (size_t i = 0; i < ops.size(); ++i) {
    size_t j = i;
    while (j < ops.size() && is_comm(ops[j].kind)) ++j;
    c->consumer_kind[i] = j < ops.size() ? ops[j].kind : -1;
  }
  // generator ops run on a high-priority stream whenever there is a generator: they
  // start when Hn (final norm) of F(m, V-1) exists and overlap the LM head / CE
  c->use_gen_stream = c->has_gen && !(getenv("BM_GEN_STREAM") && getenv("BM_GEN_STREAM")[0] == '0');
  // on by default at P = 1 (C2: 50.7 vs 48.6 samples/s with W = 2); at P > 1 the encoder
  // kernels would compete with LLM ops on other ranks' critical path (N = 2: 89.1 vs 90.6),
  // so BM_ENC_STREAM=1 / 0 forces it on / off
  // bm_model_cfg.enc_stream = 1 / 2 forces it on / off: with the encoder concentrated on the
  // lightest stage (bench.py at P > 1) its own stream overlaps it with that stage's LLM ops
  // (C2, N = 4: 189.1 vs 185.0 samples/s, profiles/r02/zb/ab_encstream.log)
  {
    const char* e = getenv("BM_ENC_STREAM");
    bool want = e ? e[0] == '1' : c->P == 1;
    if (mc->enc_stream == 1) want = true;
    if (mc->enc_stream == 2) want = false;
    c->use_enc_stream = c->has_enc && !c->enc_entry && want;
  }
  *out = c;
  return BM_OK;
}

bm_status bm_ctx_sizes_get(const bm_ctx* c, bm_ctx_sizes* out) {
  BM_CHECK_ARG(c && out, "null argument");
  // FSDP: this rank's shard of the DP parameters, then its LLM parameters
  out->weight_bytes = (c->total_elems - c->dp_elems + (c->dp_hi - c->dp_lo)) * (int64_t)c->es;
  out->grad_bytes = c->total_elems * 4;
  out->work_bytes = c->work_bytes;
  out->comm_bytes = c->comm_size[c->rank];
  return BM_OK;
}

bm_status bm_ctx_bind(bm_ctx* c, const bm_buffers* b) {
  BM_CHECK_ARG(c && b && b->weights && b->grads && b->work && b->comm, "null buffer");
  for (const void* p : {b->weights, b->grads, b->work, b->comm})
    BM_CHECK_ARG((reinterpret_cast<uintptr_t>(p) & 255) == 0, "buffers must be 256-byte aligned");
  {
    const int64_t need[4] = {(c->total_elems - c->dp_elems + (c->dp_hi - c->dp_lo)) * (int64_t)c->es,
                             c->total_elems * 4, c->work_bytes, c->comm_size[c->rank]};
    const int64_t have[4] = {b->weight_bytes, b->grad_bytes, b->work_bytes, b->comm_bytes};
    static const char* nm[4] = {"weights", "grads", "work", "comm"};
    for (int i = 0; i < 4; ++i)
      if (have[i] < need[i]) {
        set_error(std::string("buffer '") + nm[i] + "' is " + std::to_string(have[i]) + " bytes, the context needs " +
                  std::to_string(need[i]));
        return BM_E_OOM;
      }
  }
  // every kernel loaded before the first step (lazy loading stalls behind flag waits)
  BM_TRY(preload_kernels());
  c->W = (char*)b->weights;
  c->G = (float*)b->grads;
  c->work = (char*)b->work;
  c->comm = (char*)b->comm;
  work_layout(*c, c->work);
  if (c->debug_progress) {
    // progress words in mapped pinned memory: a dump must not need a CUDA call, which a
    // device-synchronising call blocked inside the step would hold up
    if (!c->progress_h) {
      void* h = nullptr;
      BM_CUDA_TRY(cudaHostAlloc(&h, (size_t)(2 + c->P) * 64, cudaHostAllocMapped));
      std::memset(h, 0, (size_t)(2 + c->P) * 64);
      c->progress_h = (volatile uint32_t*)h;
    }
    void* d = nullptr;
    BM_CUDA_TRY(cudaHostGetDevicePointer(&d, (void*)c->progress_h, 0));
    c->progress = (uint32_t*)d;
  }
  c->peer.assign(c->P, nullptr);
  c->peer[c->rank] = c->comm;
  if (c->comm_st.empty()) {
    c->comm_st.resize(c->P, nullptr);
    for (int r = 0; r < c->P; ++r)
      if (r != c->rank) BM_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_st[r], cudaStreamNonBlocking));
    c->evpool.resize(64);
    for (auto& e : c->evpool) BM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      BM_CUDA_TRY(cudaEventCreateWithFlags(&c->bout_ev[i], cudaEventDisableTiming));
      BM_CUDA_TRY(cudaEventCreateWithFlags(&c->gout_ev[i], cudaEventDisableTiming));
    }
    if (c->use_enc_stream) {
      BM_CUDA_TRY(cudaStreamCreateWithFlags(&c->enc_st, cudaStreamNonBlocking));
      c->enc_fwd_ev.assign(c->n_enc_slots, nullptr);
      for (auto& e : c->enc_fwd_ev) BM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      BM_CUDA_TRY(cudaEventCreateWithFlags(&c->emb_ready_ev, cudaEventDisableTiming));
      BM_CUDA_TRY(cudaEventCreateWithFlags(&c->emb_free_ev, cudaEventDisableTiming));
    }
    if (c->use_gen_stream) {
      int least = 0, greatest = 0;
      BM_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      BM_CUDA_TRY(cudaStreamCreateWithPriority(&c->gen_st, cudaStreamNonBlocking, greatest));
      BM_CUDA_TRY(cudaEventCreateWithFlags(&c->gen_done_ev, cudaEventDisableTiming));
    }
    if (c->has_gen) BM_CUDA_TRY(cudaEventCreateWithFlags(&c->hn_ev, cudaEventDisableTiming));
    BM_CUDA_TRY(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
    if (c->fsdp)
      for (auto& ch : c->chain) {
        BM_CUDA_TRY(cudaStreamCreateWithFlags(&ch.st, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
          BM_CUDA_TRY(cudaEventCreateWithFlags(&ch.ready[i], cudaEventDisableTiming));
          BM_CUDA_TRY(cudaEventCreateWithFlags(&ch.freed[i], cudaEventDisableTiming));
        }
      }
  }
  c->peer_w.assign(c->P, nullptr);
  c->peer_w[c->rank] = c->W;
  if (!drv().wait32 || !drv().write32) {
    set_error("cuStreamWaitValue32/cuStreamWriteValue32 unavailable");
    return BM_E_CUDA;
  }
  if (c->P > 1) {
    // every stream of the rank (compute, generator, encoder, P-1 comm, 2 FSDP pull, NCCL)
    // needs its own hardware queue: a comm stream parked on a credit wait must not
    // block an unrelated stream sharing its queue (a deadlock observed in round 1)
    const char* e = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    const int need = c->P + 6;
    if (!e || std::atoi(e) < need) {
      set_error("CUDA_DEVICE_MAX_CONNECTIONS must be >= " + std::to_string(need) +
                " (set before the CUDA context is created) for a multi-rank context");
      return BM_E_STATE;
    }
  }
  c->bound = true;
  return BM_OK;
}

bm_status bm_ipc_export(const void* dptr, uint8_t handle[64], int64_t* offset) {
  BM_CHECK_ARG(dptr && handle && offset, "null argument");
  CUdeviceptr base = 0;
  size_t sz = 0;
  if (!drv().addr_range || drv().addr_range(&base, &sz, (CUdeviceptr)dptr) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed");
    return BM_E_CUDA;
  }
  cudaIpcMemHandle_t h;
  BM_CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof(h) == 64, "ipc handle size");
  std::memcpy(handle, &h, 64);
  *offset = (int64_t)((CUdeviceptr)dptr - base);
  return BM_OK;
}

bm_status bm_ctx_open_peer(bm_ctx* c, int32_t peer, const uint8_t handle[64], int64_t offset) {
  BM_CHECK_ARG(c && handle && c->bound, "bind the context before opening peers");
  BM_CHECK_ARG(peer >= 0 && peer < c->P && peer != c->rank, "bad peer rank");
  BM_CHECK_ARG(!c->peer[peer], "peer already opened");
  void* p = nullptr;
  BM_TRY(ipc_open(handle, &p));
  c->ipc_bases.push_back(p);
  c->peer[peer] = (char*)p + offset;
  return BM_OK;
}

bm_status bm_ctx_init_fsdp(bm_ctx* c, const uint8_t* weight_handles, const int64_t* weight_offsets) {
  BM_CHECK_ARG(c && weight_handles && weight_offsets, "null argument");
  BM_CHECK_ARG(c->bound && c->fsdp, "bind an FSDP context (bm_model_cfg.fsdp) first");
  for (int q = 0; q < c->P; ++q) {
    if (q == c->rank || c->peer_w[q]) continue;
    void* p = nullptr;
    BM_TRY(ipc_open(weight_handles + 64 * (size_t)q, &p));
    c->ipc_bases.push_back(p);
    c->peer_w[q] = (char*)p + weight_offsets[q];
  }
  return BM_OK;
}

bm_status bm_ctx_dp_shard(const bm_ctx* c, int64_t* lo, int64_t* hi) {
  BM_CHECK_ARG(c && lo && hi, "null argument");
  *lo = c->dp_lo;
  *hi = c->dp_hi;
  return BM_OK;
}

bm_status bm_ctx_pull_bytes(const bm_ctx* c, int64_t* bytes) {
  BM_CHECK_ARG(c && bytes, "null argument");
  *bytes = c->pull_bytes;
  return BM_OK;
}

bm_status bm_ctx_init_peer_sum(bm_ctx* c, int32_t D, int32_t replica, const uint8_t* comm_handles,
                               const int64_t* comm_offsets, const uint8_t* grad_handles, const int64_t* grad_offsets) {
  BM_CHECK_ARG(c && comm_handles && comm_offsets && grad_handles && grad_offsets, "null argument");
  BM_CHECK_ARG(c->bound, "bind the context before bm_ctx_init_peer_sum");
  BM_CHECK_ARG(D >= 1 && replica >= 0 && replica < D, "replica out of range");
  BM_CHECK_ARG((int64_t)c->P * D <= BM_MAX_SUM_PEERS, "too many processes for the peer sum");
  BM_CHECK_ARG(!c->psum && !c->nc && !c->nc_world && !c->nc_stage, "step-end sums already initialised");
  BM_CHECK_ARG(!c->fsdp || D == 1, "FSDP shards over one pipeline's ranks (D = 1)");
  for (int r = 0; r < c->P; ++r)
    BM_CHECK_ARG(c->peer[r], "open the pipeline peers (bm_ctx_open_peer) before bm_ctx_init_peer_sum");
  const int world = c->P * D, me = replica * c->P + c->rank;
  c->ps_comm.assign(world, nullptr);
  c->ps_grad.assign(world, nullptr);
  for (int g = 0; g < world; ++g) {
    const int stage = g % c->P;
    if (g == me) {
      c->ps_comm[g] = c->comm + c->sum_off[stage];
      c->ps_grad[g] = c->G;
      continue;
    }
    if (g / c->P == replica) {
      c->ps_comm[g] = c->peer[stage] + c->sum_off[stage];
    } else {
      void* p = nullptr;
      BM_TRY(ipc_open(comm_handles + 64 * (size_t)g, &p));
      c->ipc_bases.push_back(p);
      c->ps_comm[g] = (char*)p + comm_offsets[g] + c->sum_off[stage];
    }
    void* p = nullptr;
    BM_TRY(ipc_open(grad_handles + 64 * (size_t)g, &p));
    c->ipc_bases.push_back(p);
    c->ps_grad[g] = (float*)((char*)p + grad_offsets[g]);
  }
  c->D = D;
  c->replica = replica;
  c->gscale = 1.f / ((float)c->M * (float)D);
  c->psum = true;
  return BM_OK;
}

bm_status bm_nccl_unique_id(uint8_t id[128]) {
  BM_CHECK_ARG(id, "null argument");
  if (!nccl().ok) {
    set_error("libnccl.so.2 not loadable");
    return BM_E_NCCL;
  }
  ncclUniqueId u;
  BM_NCCL_TRY(nccl().GetUniqueId(&u));
  static_assert(sizeof(u) == 128, "nccl id size");
  std::memcpy(id, &u, 128);
  return BM_OK;
}

bm_status bm_ctx_init_nccl(bm_ctx* c, const uint8_t id[128], int32_t nranks, int32_t rank) {
  BM_CHECK_ARG(c && id, "null argument");
  BM_CHECK_ARG(nranks == c->P && rank == c->rank, "NCCL group must be the pipeline group");
  if (!nccl().ok) {
    set_error("libnccl.so.2 not loadable");
    return BM_E_NCCL;
  }
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  BM_NCCL_TRY(nccl().CommInitRank(&c->nc, nranks, u, rank));
  return BM_OK;
}

bm_status bm_ctx_init_replicas(bm_ctx* c, int32_t D, int32_t replica, const uint8_t id_world[128],
                               const uint8_t id_stage[128]) {
  BM_CHECK_ARG(c && id_world && id_stage, "null argument");
  BM_CHECK_ARG(D >= 1 && replica >= 0 && replica < D, "replica out of range");
  BM_CHECK_ARG(!c->nc_world && !c->nc_stage, "replicas already initialised");
  BM_CHECK_ARG(!c->fsdp || D == 1, "FSDP shards over one pipeline's ranks (D = 1)");
  if (!nccl().ok) {
    set_error("libnccl.so.2 not loadable");
    return BM_E_NCCL;
  }
  c->D = D;
  c->replica = replica;
  c->gscale = 1.f / ((float)c->M * (float)D);
  if (D == 1) return BM_OK;
  ncclUniqueId u;
  std::memcpy(&u, id_world, 128);
  BM_NCCL_TRY(nccl().CommInitRank(&c->nc_world, c->P * D, u, replica * c->P + c->rank));
  std::memcpy(&u, id_stage, 128);
  BM_NCCL_TRY(nccl().CommInitRank(&c->nc_stage, D, u, replica));
  return BM_OK;
}

bm_status bm_step(bm_ctx* c, const bm_batch* b, void* stream) {
  BM_CHECK_ARG(c && b, "null argument");
  if (!c->bound) {
    set_error("bm_step before bm_ctx_bind");
    return BM_E_STATE;
  }
  BM_CHECK_ARG(b->M == c->M, "batch M does not match the schedule");
  for (int r = 0; r < c->P; ++r)
    if (!c->peer[r]) {
      set_error("peer " + std::to_string(r) + " not opened");
      return BM_E_STATE;
    }
  if (c->fsdp)
    for (int r = 0; r < c->P; ++r)
      if (!c->peer_w[r]) {
        set_error("FSDP: peer " + std::to_string(r) + "'s weight shard not opened (bm_ctx_init_fsdp)");
        return BM_E_STATE;
      }
  if (c->P > 1 && !c->nc && !c->psum) {
    set_error("step-end sums not initialised (bm_ctx_init_nccl or bm_ctx_init_peer_sum) for P > 1");
    return BM_E_STATE;
  }
  if (c->D > 1 && !c->psum && (!c->nc_world || !c->nc_stage)) {
    set_error("replica communicators not initialised (bm_ctx_init_replicas)");
    return BM_E_STATE;
  }
  bm_ctx& x = *c;
  const auto& m = x.mc;
  x.st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t launches0 = launch_count();
  if (x.timing) BM_TRY(harvest(x, (int)(x.step & 1)));   // pool of step-2, reused now
  // per-mb views of the batch
  x.n_mod.assign(b->n_mod, b->n_mod + x.M);
  x.n_gen.assign(b->n_gen, b->n_gen + x.M);
  int64_t tot_mod = 0, tot_gen = 0;
  for (int i = 0; i < x.M; ++i) {
    BM_CHECK_ARG(x.n_mod[i] >= 0 && x.n_mod[i] <= m.max_n_mod, "n_mod out of range");
    BM_CHECK_ARG(x.n_gen[i] >= 0 && x.n_gen[i] <= m.max_n_gen, "n_gen out of range");
    tot_mod += x.n_mod[i];
    tot_gen += x.n_gen[i];
  }
  BM_CHECK_ARG(b->ld_patch >= m.d_in && b->ld_patch % 8 == 0, "ld_patch must be >= d_in and a multiple of 8");
  const char *patches = (const char*)b->patches, *targets = (const char*)b->targets;
  x.ids = b->ids;
  x.labels = b->labels;
  x.ld_patch = b->ld_patch;
  if (b->on_host) {
    // end-to-end path: stage the host batch on the device inside the step
    BM_CHECK_ARG(tot_mod <= (int64_t)x.M * m.max_n_mod, "patch rows exceed staging");
    BM_CUDA_TRY(cudaMemcpy2DAsync(x.st_patches, (size_t)x.ld_patch_stage * x.es, patches, (size_t)b->ld_patch * x.es,
                                  (size_t)m.d_in * x.es, tot_mod, cudaMemcpyHostToDevice, x.st));
    BM_CUDA_TRY(cudaMemcpyAsync(x.st_ids, b->ids, (size_t)x.M * m.S * 4, cudaMemcpyHostToDevice, x.st));
    BM_CUDA_TRY(cudaMemcpyAsync(x.st_labels, b->labels, (size_t)x.M * m.S * 4, cudaMemcpyHostToDevice, x.st));
    BM_CUDA_TRY(cudaMemcpyAsync(x.st_targets, targets, (size_t)tot_gen * m.d_t * x.es, cudaMemcpyHostToDevice, x.st));
    patches = x.st_patches;
    targets = x.st_targets;
    x.ids = (const int32_t*)x.st_ids;
    x.labels = (const int32_t*)x.st_labels;
    x.ld_patch = x.ld_patch_stage;
  }
  x.mb_patches.resize(x.M);
  x.mb_targets.resize(x.M);
  int64_t pm = 0, pg = 0;
  for (int i = 0; i < x.M; ++i) {
    x.mb_patches[i] = patches + pm * x.ld_patch * x.es;
    x.mb_targets[i] = targets + pg * m.d_t * x.es;
    pm += x.n_mod[i];
    pg += x.n_gen[i];
  }
  // reset step state
  BM_TRY(zero_bytes(x.G, x.total_elems * 4, x.st));
  BM_TRY(zero_bytes(x.loss, (2 * (int64_t)x.M + 1) * 4, x.st));
  x.llm_free.clear();
  for (int i = x.n_llm_slots - 1; i >= 0; --i) x.llm_free.push_back(i);
  x.llm_live.clear();
  for (int i = 0; i < 2; ++i) { x.bout_pending[i] = false; x.gout_pending[i] = false; }
  // join: comm streams must see everything before this step (previous step's tail)
  {
    cudaEvent_t e = next_event(x);
    BM_CUDA_TRY(cudaEventRecord(e, x.st));
    for (int r = 0; r < x.P; ++r)
      if (r != x.rank) BM_CUDA_TRY(cudaStreamWaitEvent(x.comm_st[r], e, 0));
    if (x.use_gen_stream) BM_CUDA_TRY(cudaStreamWaitEvent(x.gen_st, e, 0));
    if (x.use_enc_stream) BM_CUDA_TRY(cudaStreamWaitEvent(x.enc_st, e, 0));
    x.emb_free_pending = false;
  }
  x.gen_done_pending = false;
  x.own_gout.clear();
  x.pull_bytes = 0;
  x.enc_slot_of.clear();
  x.enc_next = 0;
  cudaStream_t main_st = x.st;
  x.st_main = main_st;
  if (x.tracing) {
    x.trace.clear();
    x.trace_used = 0;
    x.trace_origin = trace_mark(x, main_st);
  }
  if (x.debug_progress) {
    g_dbg_ctx = c;
    g_launch_hook = dbg_launch_hook;
  }
  // ---- the opcode stream
  const auto& ops = x.s->ranks[x.rank];
  RecvState rs;
  const char* gen_x = nullptr;
  int64_t live_enc = 0, live_llm = 0, live_gen = 0;
  const int64_t enc_unit_bytes = (int64_t)m.max_n_mod * (m.d_e * (m.L_e + 1) + m.L_e * (m.d_e + 2 * m.f_e) + 3 * m.d) * x.es;
  const int64_t llm_unit_bytes = (int64_t)m.S * (x.lps * (2 * m.d + 3 * m.f + (x.zb ? m.d + 2 * m.f : 0)) + m.d) * x.es;
  const int64_t gen_unit_bytes = (int64_t)x.gen_rows * (m.d_g * (m.L_g + 1) + m.L_g * (m.d_g + 2 * m.f_g) + 2 * m.d_t) * x.es;
  for (int k = 0; k < 3; ++k) x.stash_peak[k] = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    const bm_op& o = ops[i];
    if (x.debug_progress) {
      std::fprintf(stderr, "[bm r%d s%lld] enqueue op %zu kind %d mb %d chunk %d peer %d pay %d seq %d\n", x.rank,
                   (long long)x.step, i, (int)o.kind, (int)o.mb, (int)o.chunk, (int)o.peer, (int)o.payload, (int)o.seq);
      std::fflush(stderr);
    }
    switch (o.kind) {
      case BM_OP_RECV: {
        const bool on_gen = x.use_gen_stream && x.consumer_kind[i] == BM_OP_GEN_FWD;
        const bool on_enc = x.use_enc_stream && x.consumer_kind[i] == BM_OP_ENC_BWD;
        cudaStream_t wst = on_gen ? x.gen_st : (on_enc ? x.enc_st : main_st);
        BM_TRY(do_recv_wait(x, o, wst));
        if (x.debug_progress && !on_enc)
          drv().write32((CUstream)wst, (CUdeviceptr)(x.progress + 16 * (on_gen ? 1 : 0)), (uint32_t)i + 1, 0);
        if (x.tracing) {
          cudaEvent_t e = trace_mark(x, wst);
          x.trace.push_back({(int32_t)i, (int32_t)o.kind, stream_slot(x, wst), o.mb, e, e});
        }
        rs.ops.push_back(&o);
        continue;
      }
      case BM_OP_SEND:
        BM_TRY(do_send(x, o, (int)i));
        if (x.debug_progress)
          drv().write32((CUstream)x.comm_st[o.peer], (CUdeviceptr)(x.progress + 16 * (2 + o.peer)), (uint32_t)i + 1, 0);
        continue;
      default:
        break;
    }
    x.producer_ev = nullptr;
    const bool gen_op = o.kind == BM_OP_GEN_FWD || o.kind == BM_OP_GEN_BWD;
    const bool enc_op = o.kind == BM_OP_ENC_FWD || o.kind == BM_OP_ENC_BWD;
    cudaStream_t op_st = (gen_op && x.use_gen_stream) ? x.gen_st : ((enc_op && x.use_enc_stream) ? x.enc_st : main_st);
    if (!gen_op && x.gen_done_pending && o.kind == BM_OP_LLM_BWD && o.chunk == x.V - 1 && x.rank == x.P - 1) {
      // the last stage's backward consumes the generator-input gradients (own shard added in place)
      BM_CUDA_TRY(cudaStreamWaitEvent(main_st, x.gen_done_ev, 0));
      x.gen_done_pending = false;
    }
    if (gen_op && x.use_gen_stream && o.kind == BM_OP_GEN_FWD && x.rank == x.P - 1)
      BM_CUDA_TRY(cudaStreamWaitEvent(x.gen_st, x.hn_ev, 0));   // Hn of F(m, V-1)
    x.st = op_st;
    x.producer_st = op_st;
    float* part_main = x.part;
    if (op_st == x.gen_st && op_st != main_st) x.part = x.part_gen;
    if (op_st == x.enc_st && op_st != main_st) x.part = x.part_enc;
    x.cur_ws = op_st == main_st ? x.ws : (op_st == x.gen_st ? x.ws_gen : x.ws_enc);
    set_sm_reserve((op_st == main_st && x.use_gen_stream && x.rank != x.P - 1) ? x.gen_reserve_sms : 0);
    cudaEvent_t tr_a = x.tracing ? trace_mark(x, op_st) : nullptr;
    switch (o.kind) {
      case BM_OP_ENC_FWD:
        BM_TRY(op_enc_fwd(x, o));
        if (x.use_enc_stream) BM_CUDA_TRY(cudaEventRecord(x.enc_fwd_ev[x.enc_slot_of.at(o.mb)], x.enc_st));
        live_enc += enc_unit_bytes;
        break;
      case BM_OP_ENC_BWD:
        if (x.use_enc_stream && x.rank == 0) BM_CUDA_TRY(cudaStreamWaitEvent(x.enc_st, x.emb_ready_ev, 0));
        BM_TRY(op_enc_bwd(x, o, rs));
        if (x.use_enc_stream && x.rank == 0) {   // emb_local read: B's next copy may overwrite it
          BM_CUDA_TRY(cudaEventRecord(x.emb_free_ev, x.enc_st));
          x.emb_free_pending = true;
        }
        live_enc -= enc_unit_bytes;
        break;
      case BM_OP_LLM_FWD:
        BM_TRY(op_llm_fwd(x, o, rs));
        live_llm += llm_unit_bytes;
        break;
      case BM_OP_LLM_BWD:
        BM_TRY(op_llm_bwd(x, o, rs));
        if (!x.zb) live_llm -= llm_unit_bytes;
        break;
      case BM_OP_LLM_W: BM_TRY(op_llm_w(x, o)); live_llm -= llm_unit_bytes; break;
      case BM_OP_GEN_FWD:
        gen_x = nullptr;
        if (x.rank != x.P - 1 && !rs.ops.empty()) {
          int hlo, hhi;   // the generator rows follow the head rows in the genin slot
          head_rows_of(x, o.mb, x.rank, &hlo, &hhi);
          gen_x = recv_slot(x, x.P - 1, BM_PAY_GENIN, rs.ops[0]->seq) + (int64_t)(hhi - hlo) * m.d * x.es;
        }
        BM_TRY(op_gen_fwd(x, o, rs));
        live_gen += gen_unit_bytes;
        break;
      case BM_OP_GEN_BWD: {
        const char* X = (x.rank == x.P - 1) ? x.genin_src[x.rank] : gen_x;
        BM_TRY(op_gen_bwd(x, o, X));
        live_gen -= gen_unit_bytes;
        if (x.use_gen_stream && x.rank == x.P - 1) {
          BM_CUDA_TRY(cudaEventRecord(x.gen_done_ev, x.gen_st));
          x.gen_done_pending = true;
        }
        break;
      }
      default:
        set_error("unknown op kind");
        return BM_E_INVALID;
    }
    x.stash_peak[0] = std::max(x.stash_peak[0], live_enc);
    x.stash_peak[1] = std::max(x.stash_peak[1], live_llm);
    x.stash_peak[2] = std::max(x.stash_peak[2], live_gen);
    rs.ops.clear();
    for (int ri : x.release_of[i]) BM_TRY(do_release(x, ops[ri], op_st));
    if (x.tracing) x.trace.push_back({(int32_t)i, (int32_t)o.kind, stream_slot(x, op_st), o.mb, tr_a, trace_mark(x, op_st)});
    if (x.debug_progress)
      drv().write32((CUstream)op_st, (CUdeviceptr)(x.progress + 16 * (op_st == main_st ? 0 : 1)), (uint32_t)i + 1, 0);
    x.st = main_st;
    x.part = part_main;
    set_sm_reserve(0);
  }
  if (x.use_gen_stream) {
    cudaEvent_t e = next_event(x);
    BM_CUDA_TRY(cudaEventRecord(e, x.gen_st));
    BM_CUDA_TRY(cudaStreamWaitEvent(main_st, e, 0));
  }
  if (x.use_enc_stream) {   // encoder gradients complete before the DP allreduce
    cudaEvent_t e = next_event(x);
    BM_CUDA_TRY(cudaEventRecord(e, x.enc_st));
    BM_CUDA_TRY(cudaStreamWaitEvent(main_st, e, 0));
  }
  x.producer_st = nullptr;
  // join the comm streams back into the compute stream
  for (int r = 0; r < x.P; ++r) {
    if (r == x.rank) continue;
    cudaEvent_t e = next_event(x);
    BM_CUDA_TRY(cudaEventRecord(e, x.comm_st[r]));
    BM_CUDA_TRY(cudaStreamWaitEvent(x.st, e, 0));
  }
  // finalize: DP gradient sum + loss terms
  cudaEvent_t tr_tail = x.tracing ? trace_mark(x, x.st) : nullptr;
  static const bool no_allreduce = getenv("BM_DEBUG_NO_ALLREDUCE") != nullptr;   // hang triage only
  if (x.psum && !no_allreduce) {
    BM_TRY(peer_finalize(x));
  } else if (!no_allreduce && (x.P > 1 || x.D > 1)) {
    // DP parameters over every process (the replica's pipeline group when D = 1),
    // this stage's LLM parameters over its D replicas, loss terms over the pipeline
    BM_NCCL_TRY(nccl().GroupStart());
    ncclComm_t dp_comm = x.D > 1 ? x.nc_world : x.nc;
    BM_NCCL_TRY(nccl().AllReduce(x.G, x.G, (size_t)x.dp_elems, ncclFloat32, ncclSum, dp_comm, x.st));
    if (x.D > 1 && x.total_elems > x.dp_elems)
      BM_NCCL_TRY(nccl().AllReduce(x.G + x.dp_elems, x.G + x.dp_elems, (size_t)(x.total_elems - x.dp_elems), ncclFloat32,
                                   ncclSum, x.nc_stage, x.st));
    if (x.P > 1) BM_NCCL_TRY(nccl().AllReduce(x.loss, x.loss, (size_t)(2 * x.M), ncclFloat32, ncclSum, x.nc, x.st));
    BM_NCCL_TRY(nccl().GroupEnd());
  }
  // L = (1/M) sum of the replica's terms; with replicas, the mean of the D replica losses
  if (!x.psum || no_allreduce) BM_TRY(loss_finalize(x.M, x.loss, 1.f / ((float)x.M * (float)x.D), x.st));
  if (x.D > 1 && !no_allreduce && !x.psum)
    BM_NCCL_TRY(nccl().AllReduce(x.loss + 2 * x.M, x.loss + 2 * x.M, 1, ncclFloat32, ncclSum, x.nc_stage, x.st));
  if (x.tracing) {
    x.trace_last = trace_mark(x, x.st);
    x.trace.push_back({-1, -1, 0, -1, tr_tail, x.trace_last});
  }
  BM_CUDA_TRY(cudaEventRecord(x.done_ev, x.st));
  x.step += 1;
  x.launches = launch_count() - launches0;
  return BM_OK;
}

// first unmet wait of this rank's step `stp` (op order), read from a host copy of its flags
static std::string blocked_op(const bm_ctx& c, int64_t stp, const std::vector<uint32_t>& fl) {
  static const char* PN[] = {"act", "grad", "emb", "embgrad", "genin", "gengrad"};
  static const char* KN[] = {"EncFwd", "EncBwd", "LlmFwd", "LlmBwd", "GenFwd", "GenBwd", "Send", "Recv", "LlmW"};
  const auto& ops = c.s->ranks[c.rank];
  for (size_t i = 0; i < ops.size(); ++i) {
    const bm_op& o = ops[i];
    if (o.kind != BM_OP_RECV && o.kind != BM_OP_SEND) continue;
    const bool recv = o.kind == BM_OP_RECV;
    const auto key = recv ? std::make_tuple((int)o.peer, c.rank, (int)o.payload) : std::make_tuple(c.rank, (int)o.peer, (int)o.payload);
    const Chan& ch = c.chans[c.chan_idx.at(key)];
    if (!recv && o.seq < ch.K) continue;   // a free slot: no credit wait
    const uint32_t base = (uint32_t)(stp * ch.nmsg);
    const uint32_t want = recv ? base + (uint32_t)o.seq + 1 : base + (uint32_t)(o.seq - ch.K) + 1;
    const uint32_t have = fl[(size_t)(recv ? ch.flag_off : ch.credit_off) / 4];
    if ((int32_t)(have - want) < 0)
      return "rank " + std::to_string(c.rank) + " blocked at op " + std::to_string(i) + " (" + KN[o.kind] + " " +
             PN[o.payload] + (recv ? " from " : " to ") + "rank " + std::to_string(o.peer) + ", mb " +
             std::to_string(o.mb) + ", seq " + std::to_string(o.seq) + "): " + (recv ? "data" : "credit") +
             " flag " + std::to_string(have) + " < " + std::to_string(want);
  }
  if (c.psum) {
    const int world = (int)c.ps_comm.size(), me = c.replica * c.P + c.rank;
    const uint32_t want = (uint32_t)(stp * 4 + 3);
    const size_t sb = (size_t)c.sum_off[c.rank] / 4;
    for (int g = 0; g < world; ++g)
      if (g != me && (int32_t)(fl[sb + 16 * g] - want) < 0)
        return "rank " + std::to_string(c.rank) + " blocked in the step-end sum barrier: process " + std::to_string(g) +
               " flag " + std::to_string(fl[sb + 16 * g]) + " < " + std::to_string(want);
  }
  return "rank " + std::to_string(c.rank) + ": every receive / credit / barrier flag is satisfied (blocked in a kernel "
         "or a collective)";
}

bm_status bm_step_wait(bm_ctx* c, int64_t timeout_ms) {
  BM_CHECK_ARG(c && c->bound, "bound context required");
  if (c->step == 0 || !c->done_ev) return BM_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaEventQuery(c->done_ev);
    if (e == cudaSuccess) return BM_OK;
    if (e != cudaErrorNotReady) BM_CUDA_TRY(e);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms > 0 && ms > (double)timeout_ms) break;
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  // diagnose from a host copy of this rank's flags (private stream, bounded wait)
  std::string why = "flags unreadable (the copy did not complete within 2 s)";
  const size_t bytes = (size_t)c->comm_size[c->rank];
  std::vector<uint32_t> fl(bytes / 4 + 1, 0);
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
    if (cudaMemcpyAsync(fl.data(), c->comm, bytes, cudaMemcpyDeviceToHost, s) == cudaSuccess) {
      const auto t1 = std::chrono::steady_clock::now();
      while (cudaStreamQuery(s) == cudaErrorNotReady &&
             std::chrono::steady_clock::now() - t1 < std::chrono::seconds(2))
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      if (cudaStreamQuery(s) == cudaSuccess) why = blocked_op(*c, c->step - 1, fl);
    }
    cudaStreamDestroy(s);   // released once its copy completes
  }
  set_error("step " + std::to_string(c->step - 1) + " did not finish within " + std::to_string(timeout_ms) + " ms: " + why);
  return BM_E_TIMEOUT;
}

bm_status bm_ctx_loss_ptr(const bm_ctx* c, const float** dptr) {
  BM_CHECK_ARG(c && dptr && c->bound, "bound context required");
  *dptr = c->loss;
  return BM_OK;
}

bm_status bm_ctx_launch_count(const bm_ctx* c, int64_t* n) {
  BM_CHECK_ARG(c && n, "null argument");
  *n = c->launches;
  return BM_OK;
}

bm_status bm_ctx_stash_peak(const bm_ctx* c, int64_t out[3]) {
  BM_CHECK_ARG(c && out, "null argument");
  for (int k = 0; k < 3; ++k) out[k] = c->stash_peak[k];
  return BM_OK;
}

bm_status bm_ctx_set_timing(bm_ctx* c, int32_t enable) {
  BM_CHECK_ARG(c, "null argument");
  if (c->timing && !enable) {
    BM_TRY(harvest(*c, 0));
    BM_TRY(harvest(*c, 1));
  }
  c->timing = enable != 0;
  c->gemm_flops = 0;
  c->gemm_ms = 0;
  c->gemm_count = 0;
  c->comm_ms = 0;
  c->comm_bytes = 0;
  c->comm_msgs = 0;
  return BM_OK;
}

bm_status bm_ctx_debug_dump(bm_ctx* c, char* buf, size_t cap) {
  BM_CHECK_ARG(c && buf && cap > 0 && c->bound, "bound context and buffer required");
  if (c->progress_h) {
    // host-mapped progress only: safe while the owning thread is blocked in the driver
    std::string out = "rank " + std::to_string(c->rank) + " step " + std::to_string(c->step) + " ops " +
                      std::to_string(c->s->ranks[c->rank].size()) + " progress main=" +
                      std::to_string(c->progress_h[0]) + " gen=" + std::to_string(c->progress_h[16]);
    for (int q = 0; q < c->P; ++q) out += " comm" + std::to_string(q) + "=" + std::to_string(c->progress_h[16 * (2 + q)]);
    out += "\n  last launch done: main=" + std::to_string(c->progress_h[1]) + " gen=" + std::to_string(c->progress_h[17]);
    for (int q = 0; q < c->P; ++q) out += " comm" + std::to_string(q) + "=" + std::to_string(c->progress_h[16 * (2 + q) + 1]);
    out += "\n";
    if (getenv("BM_DEBUG_DUMP_FLAGS") == nullptr) {
      std::strncpy(buf, out.c_str(), cap - 1);
      buf[cap - 1] = 0;
      return BM_OK;
    }
    std::strncpy(buf, out.c_str(), cap - 1);
    buf[cap - 1] = 0;
    const size_t used = std::strlen(buf);
    buf += used;
    cap -= used;
  }
  cudaStream_t s;
  BM_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int64_t fl = 0;
  for (auto& ch : c->chans) fl = std::max(fl, std::max(ch.flag_off, ch.credit_off) + 64);
  std::vector<uint32_t> flags((size_t)fl / 4 + 1, 0), prog((size_t)(2 + c->P) * 16, 0);
  if (fl > 0) BM_CUDA_TRY(cudaMemcpyAsync(flags.data(), c->comm, fl, cudaMemcpyDeviceToHost, s));
  BM_CUDA_TRY(cudaMemcpyAsync(prog.data(), c->progress, prog.size() * 4, cudaMemcpyDeviceToHost, s));
  BM_CUDA_TRY(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  std::string out = "rank " + std::to_string(c->rank) + " step " + std::to_string(c->step) + " ops " +
                    std::to_string(c->s->ranks[c->rank].size()) + " progress main=" + std::to_string(prog[0]) +
                    " gen=" + std::to_string(prog[16]);
  for (int q = 0; q < c->P; ++q) out += " comm" + std::to_string(q) + "=" + std::to_string(prog[16 * (2 + q)]);
  out += "\n";
  static const char* PN[] = {"act", "grad", "emb", "embgrad", "genin", "gengrad"};
  for (auto& ch : c->chans) {
    if (ch.dst == c->rank)
      out += "  recv " + std::to_string(ch.src) + "->" + std::to_string(ch.dst) + " " + PN[ch.pay] +
             " data_flag=" + std::to_string(flags[ch.flag_off / 4]) + " nmsg=" + std::to_string(ch.nmsg) +
             " K=" + std::to_string(ch.K) + "\n";
    if (ch.src == c->rank)
      out += "  send " + std::to_string(ch.src) + "->" + std::to_string(ch.dst) + " " + PN[ch.pay] +
             " credit=" + std::to_string(flags[ch.credit_off / 4]) + " nmsg=" + std::to_string(ch.nmsg) +
             " K=" + std::to_string(ch.K) + "\n";
  }
  std::strncpy(buf, out.c_str(), cap - 1);
  buf[cap - 1] = 0;
  return BM_OK;
}

bm_status bm_ctx_set_trace(bm_ctx* c, int32_t enable) {
  BM_CHECK_ARG(c, "null argument");
  c->tracing = enable != 0;
  if (!c->tracing) c->trace.clear();
  return BM_OK;
}

bm_status bm_ctx_trace_get(bm_ctx* c, bm_trace_rec* out, int64_t cap, int64_t* n, int64_t* total) {
  BM_CHECK_ARG(c && n && total && (cap == 0 || out), "null argument");
  *total = (int64_t)c->trace.size();
  *n = 0;
  if (c->trace.empty() || !c->trace_last || !c->trace_origin) return BM_OK;
  BM_CUDA_TRY(cudaEventSynchronize(c->trace_last));
  for (const auto& t : c->trace) {
    if (*n >= cap) break;
    if (!t.a || !t.b) continue;
    bm_trace_rec& r = out[(*n)++];
    r.op = t.op;
    r.kind = t.kind;
    r.stream = t.stream;
    r.mb = t.mb;
    BM_CUDA_TRY(cudaEventSynchronize(t.b));
    BM_CUDA_TRY(cudaEventElapsedTime(&r.t_start_ms, c->trace_origin, t.a));
    BM_CUDA_TRY(cudaEventElapsedTime(&r.t_end_ms, c->trace_origin, t.b));
  }
  return BM_OK;
}

bm_status bm_ctx_comm_stats(bm_ctx* c, int64_t* n_msgs, double* bytes, double* ms) {
  BM_CHECK_ARG(c && n_msgs && bytes && ms, "null argument");
  BM_TRY(harvest(*c, 0));
  BM_TRY(harvest(*c, 1));
  *n_msgs = c->comm_msgs;
  *bytes = c->comm_bytes;
  *ms = c->comm_ms;
  return BM_OK;
}

bm_status bm_ctx_gemm_stats(bm_ctx* c, int64_t* n_gemm, double* flops, double* ms) {
  BM_CHECK_ARG(c && n_gemm && flops && ms, "null argument");
  BM_TRY(harvest(*c, 0));
  BM_TRY(harvest(*c, 1));
  if (getenv("BM_GEMM_LOG")) {
    for (auto& kv : c->shape_ms) {
      const auto& k = kv.first;
      const double fl = 2.0 * k[0] * k[1] * k[2] * kv.second.first;
      fprintf(stderr, "GEMM M=%d N=%d K=%d epi=%d n=%lld ms=%.3f tflops=%.1f\n", k[0], k[1], k[2], k[3],
              (long long)kv.second.first, kv.second.second, fl / (kv.second.second / 1e3) / 1e12);
    }
    c->shape_ms.clear();
  }
  *n_gemm = c->gemm_count;
  *flops = c->gemm_flops;
  *ms = c->gemm_ms;
  return BM_OK;
}

void bm_ctx_destroy(bm_ctx* c) { delete c; }

}  // extern "C"
