// sched.cpp -- host schedule builder: BigMac's pipeline scheduler.
//
//   get_llm_schedule   Megatron-style 1F1B / interleaved 1F1B lists,
//                      or ZB-H1 zero-bubble lists with B/W split (R23)
//   columns            cut timeline = integer DES of the LLM lists with the
//                      cost_fwd:cost_bwd ratio (R1)
//   build_schedule     W warmup encoder units, then a sweep over LLM op starts
//                      and trigger events: GEN(m) at the end of F(m, V-1) on
//                      the last rank (llm_output_ready), ENC(u) at the
//                      end of G_u = B(uP+P-1, 0) on rank 0 (encoder_grad_ready,
//                      P:265) -> EncBwd(u) + EncFwd(next)
//   insert_comm_ops    Recv right before each consumer, Send right after each
//                      producer; act/grad, emb/embgrad gather and
//                      scatter, genin/gengrad
//   deadlock_check     happens-before graph (program order, per-peer send
//                      chains, data edges, credit edges of the receive rings)
//                      must be acyclic; rings sized minimal + slack
// Output is bit-identical to oracle/schedule.py (tests/test_sched_parity.py).
#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/bigmac.h"

namespace bm {
void set_error(const std::string& msg);
}

#include "sched_internal.h"

namespace bm {
namespace sched {

struct Fail {
  bm_status code;
  std::string msg;
};

enum { LF = 0, LB = 1, LW = 2 };  // F, B (input gradient under ZB-H1), W (weight gradient)
struct LOp {
  int k;
  int mb, chunk;
};
static const int LLM_OPK[3] = {BM_OP_LLM_FWD, BM_OP_LLM_BWD, BM_OP_LLM_W};

static int wgrad_cost(const bm_sched_cfg& c) { return c.cost_wgrad > 0 ? c.cost_wgrad : c.cost_bwd / 2; }

static bm_op mk(int kind, int mb = -1, int chunk = -1, int unit = -1, int peer = -1, int payload = -1) {
  bm_op o;
  o.kind = kind; o.mb = mb; o.chunk = chunk; o.unit = unit; o.peer = peer; o.payload = payload;
  o.slot = -1; o.seq = -1;
  return o;
}

static void validate(const bm_sched_cfg& c) {
  const int P = c.stages, M = c.microbatches, V = c.vchunks;
  if (P < 1 || M < 1 || V < 1 || c.warmup_units < 0) throw Fail{BM_E_INVALID, "P, M, V must be >= 1 and W >= 0"};
  if (c.cost_fwd < 1 || c.cost_bwd < 1 || c.ring_slack < 0)
    throw Fail{BM_E_INVALID, "costs must be >= 1 and ring_slack >= 0"};
  if (c.llm_sched == BM_LLM_1F1B && V != 1) throw Fail{BM_E_INVALID, "1F1B requires V == 1"};
  if (c.llm_sched == BM_LLM_INTERLEAVED && V < 2) throw Fail{BM_E_INVALID, "interleaved 1F1B requires V >= 2"};
  if (c.llm_sched != BM_LLM_1F1B && c.llm_sched != BM_LLM_INTERLEAVED && c.llm_sched != BM_LLM_ZB_H1)
    throw Fail{BM_E_INVALID, "unknown llm_sched"};
  if (c.cost_wgrad < 0) throw Fail{BM_E_INVALID, "cost_wgrad must be >= 0"};
  if (c.llm_sched == BM_LLM_ZB_H1) {
    if (V != 1) throw Fail{BM_E_INVALID, "ZB-H1 requires V == 1"};
    const int cw = wgrad_cost(c);
    if (cw < 1 || cw >= c.cost_bwd) throw Fail{BM_E_INVALID, "ZB-H1 needs 1 <= W cost < cost_bwd (B and W both >= 1)"};
  }
  if (c.enc_place != BM_ENC_NONE && c.enc_place != BM_ENC_DP_UNIT && c.enc_place != BM_ENC_ENTRY_STAGE)
    throw Fail{BM_E_INVALID, "unknown enc_place"};
  if (c.gen_place != BM_GEN_NONE && c.gen_place != BM_GEN_DP_SHARD && c.gen_place != BM_GEN_LAST_STAGE)
    throw Fail{BM_E_INVALID, "unknown gen_place"};
  for (int i = 0; i < 2; ++i)
    if (c.reserved[i] != 0) throw Fail{BM_E_INVALID, "reserved fields must be zero"};
  const int lcp = c.llm_cp > 0 ? c.llm_cp : 1, ecp = c.enc_cp > 0 ? c.enc_cp : 1;
  if (c.llm_cp < 0 || c.enc_cp < 0 || ecp > lcp || (P * lcp) % ecp)
    throw Fail{BM_E_INVALID, "need 1 <= enc_cp <= llm_cp and enc_cp dividing P * llm_cp"};
  const bool cp = lcp > 1 || ecp > 1;
  if (cp && (c.enc_place == BM_ENC_ENTRY_STAGE || c.gen_place == BM_GEN_DP_SHARD || c.enc_exclude))
    throw Fail{BM_E_INVALID, "decoupled CP: enc_place none / dp_unit, gen_place none / last_stage, no enc_exclude"};
  const int unit = P * lcp / ecp;
  if (M % unit != 0)
    throw Fail{BM_E_REMAINDER, "M=" + std::to_string(M) + " is not a multiple of the encoder unit " + std::to_string(unit)};
  if (c.enc_exclude) {
    const int64_t full = (P >= 31) ? -1 : (((int64_t)1 << P) - 1);
    if (c.enc_exclude < 0 || (P < 31 && ((int64_t)c.enc_exclude & ~full)) || (int64_t)c.enc_exclude == full)
      throw Fail{BM_E_INVALID, "enc_exclude: a mask of ranks < P leaving at least one rank"};
    if (c.enc_place != BM_ENC_DP_UNIT) throw Fail{BM_E_INVALID, "enc_exclude applies to the DP encoder units"};
  }
}

// rank running microbatch m's encoder: m % P (reading R3), or, if that rank is in
// enc_exclude, the nearest lower rank not in the mask, cyclically (reading R22)
int enc_owner(const bm_sched_cfg& c, int m) {
  const int P = c.stages;
  int r = m % P;
  while ((c.enc_exclude >> r) & 1) r = (r - 1 + P) % P;
  return r;
}

// ---------------------------------------------------------------- LLM base lists
static std::vector<std::vector<LOp>> base_lists(int P, int M, int V) {
  std::vector<std::vector<LOp>> out(P);
  for (int r = 0; r < P; ++r) {
    std::vector<LOp> fwd, bwd;
    int w;
    if (V == 1) {
      w = std::min(P - r - 1, M);
      for (int m = 0; m < M; ++m) { fwd.push_back({LF, m, 0}); bwd.push_back({LB, m, 0}); }
    } else {
      w = std::min(2 * (P - r - 1) + (V - 1) * P, M * V);
      for (int k = 0; k < M * V; ++k) {
        const int g = k / (P * V), j = k % (P * V);
        const int c = j / P, m = g * P + (j % P);
        fwd.push_back({LF, m, c});
        bwd.push_back({LB, m, V - 1 - c});
      }
    }
    const int total = (int)fwd.size();
    auto& ops = out[r];
    for (int k = 0; k < w; ++k) ops.push_back(fwd[k]);
    for (int i = 0; i < total - w; ++i) { ops.push_back(fwd[w + i]); ops.push_back(bwd[i]); }
    for (int i = total - w; i < total; ++i) ops.push_back(bwd[i]);
  }
  return out;
}

// ZB-H1 (R23): 1F1B order of F and B per rank, at most P microbatches
// held between F and W; ranks simulated in time order, a free rank preferring
// (1) the oldest pending W if its next op is an F and P are held, (2) its next
// F/B if the producer has finished, (3) the oldest pending W if it ends no later
// than the earliest start of that F/B (producer's end, or producer rank's free
// time + producer cost if unscheduled), (4) waiting one unit.
static std::vector<std::vector<LOp>> zb_h1_lists(int P, int M, int cf, int cb, int cw) {
  std::vector<std::vector<LOp>> fb(P), out(P);
  for (int r = 0; r < P; ++r) {
    const int w = std::min(P - r - 1, M);
    for (int m = 0; m < w; ++m) fb[r].push_back({LF, m, 0});
    for (int i = 0; i < M - w; ++i) { fb[r].push_back({LF, w + i, 0}); fb[r].push_back({LB, i, 0}); }
    for (int i = M - w; i < M; ++i) fb[r].push_back({LB, i, 0});
  }
  std::vector<int64_t> endF((size_t)P * M, -1), endB((size_t)P * M, -1), t(P, 0);
  std::vector<size_t> ptr(P, 0);
  std::vector<int> held(P, 0);
  std::vector<std::deque<int>> pending(P);
  std::vector<bool> active(P, true);
  int n_active = P;
  auto run_w = [&](int r) {
    const int m = pending[r].front();
    pending[r].pop_front();
    out[r].push_back({LW, m, 0});
    t[r] += cw;
    --held[r];
  };
  while (n_active) {
    int r = -1;
    for (int x = 0; x < P; ++x)
      if (active[x] && (r < 0 || t[x] < t[r])) r = x;
    if (ptr[r] == fb[r].size()) {
      if (!pending[r].empty()) run_w(r);
      else { active[r] = false; --n_active; }
      continue;
    }
    const LOp o = fb[r][ptr[r]];
    if (o.k == LF && held[r] >= P) { run_w(r); continue; }
    int64_t dep = 0;  // 0: no producer; -1: producer not scheduled yet
    int q = -1, qcost = 0;
    if (o.k == LF && r > 0) { q = r - 1; qcost = cf; dep = endF[(size_t)q * M + o.mb]; }
    if (o.k == LB && r < P - 1) { q = r + 1; qcost = cb; dep = endB[(size_t)q * M + o.mb]; }
    if (dep >= 0 && dep <= t[r]) {
      out[r].push_back(o);
      t[r] += (o.k == LF) ? cf : cb;
      if (o.k == LF) { endF[(size_t)r * M + o.mb] = t[r]; ++held[r]; }
      else { endB[(size_t)r * M + o.mb] = t[r]; pending[r].push_back(o.mb); }
      ++ptr[r];
    } else {
      const int64_t earliest = dep >= 0 ? dep : std::max(t[r], t[q]) + qcost;
      if (!pending[r].empty() && t[r] + cw <= earliest) run_w(r);
      else ++t[r];
    }
  }
  return out;
}

struct Times {
  int P, M, V;
  std::vector<int64_t> st, en;  // index(r, kind, m, c)
  size_t idx(int r, int k, int m, int c) const { return (((size_t)r * 3 + k) * M + m) * V + c; }
};

static Times des_llm(const std::vector<std::vector<LOp>>& base, int P, int M, int V, int cf, int cb, int cw) {
  Times T{P, M, V, {}, {}};
  T.st.assign((size_t)P * 3 * M * V, -1);
  T.en.assign((size_t)P * 3 * M * V, -1);
  std::vector<size_t> ptr(P, 0);
  std::vector<int64_t> freet(P, 0);
  size_t remaining = 0;
  for (auto& l : base) remaining += l.size();
  while (remaining) {
    bool prog = false;
    for (int r = 0; r < P; ++r) {
      while (ptr[r] < base[r].size()) {
        const LOp& o = base[r][ptr[r]];
        const int s = o.chunk * P + r;
        int64_t dep_end = 0;
        bool has = false;
        if (o.k == LF && s > 0) {
          const size_t d = T.idx((s - 1) % P, LF, o.mb, (s - 1) / P);
          if (T.en[d] < 0) break;
          dep_end = T.en[d]; has = true;
        }
        if (o.k == LB && s < P * V - 1) {
          const size_t d = T.idx((s + 1) % P, LB, o.mb, (s + 1) / P);
          if (T.en[d] < 0) break;
          dep_end = T.en[d]; has = true;
        }
        const int64_t start = std::max(freet[r], has ? dep_end : (int64_t)0);
        const int64_t end = start + (o.k == LF ? cf : o.k == LB ? cb : cw);
        const size_t me = T.idx(r, o.k, o.mb, o.chunk);
        T.st[me] = start; T.en[me] = end;
        freet[r] = end;
        ++ptr[r]; --remaining; prog = true;
      }
    }
    if (!prog) throw Fail{BM_E_DEPENDENCY, "LLM base schedule stalls"};
  }
  return T;
}

static int w_star(const std::vector<LOp>& base0, int P, int M) {
  std::map<std::tuple<int, int, int>, int> pos;
  for (int i = 0; i < (int)base0.size(); ++i) pos[{base0[i].k, base0[i].mb, base0[i].chunk}] = i;
  const int n_u = M / P;
  int best = 1;
  for (int i = 0; i < n_u; ++i) {
    const int g = pos[{LB, i * P + P - 1, 0}];
    int cnt = 0;
    for (int j = i; j < n_u; ++j)
      if (pos[{LF, j * P, 0}] < g) ++cnt;
    best = std::max(best, cnt);
  }
  return best;
}

// ---------------------------------------------------------------- nesting
static std::vector<std::vector<bm_op>> nest(const bm_sched_cfg& c, const std::vector<std::vector<LOp>>& base,
                                            const Times& T, int& W_out) {
  const int P = c.stages, M = c.microbatches, V = c.vchunks;
  const int n_u = M / P;
  const bool entry = c.enc_place == BM_ENC_ENTRY_STAGE;
  const int W = entry ? 0 : (c.warmup_units > 0 ? c.warmup_units : w_star(base[0], P, M));
  W_out = W;
  const bool enc = c.enc_place == BM_ENC_DP_UNIT;
  struct Ev {
    int64_t t;
    int cls, tb;
    int r, idx;  // LLM: rank, index in base[r]; GEN: m; ENC: u
  };
  std::vector<Ev> ev;
  for (int r = 0; r < P; ++r)
    for (int i = 0; i < (int)base[r].size(); ++i) {
      const LOp& o = base[r][i];
      ev.push_back({T.st[T.idx(r, o.k, o.mb, o.chunk)], 2, r, r, i});
    }
  if (c.gen_place != BM_GEN_NONE)
    for (int m = 0; m < M; ++m) ev.push_back({T.en[T.idx(P - 1, LF, m, V - 1)], 0, m, 0, m});
  if (enc)
    for (int u = 0; u < n_u; ++u) ev.push_back({T.en[T.idx(0, LB, u * P + P - 1, 0)], 1, u, 0, u});
  std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.cls != b.cls) return a.cls < b.cls;
    return a.tb < b.tb;
  });
  std::vector<std::vector<bm_op>> lists(P);
  int nxt = 0;
  // the unit's encoder microbatches on every rank, each rank in microbatch order
  auto unit_ops = [&](int kind, int u) {
    for (int r = 0; r < P; ++r)
      for (int m = u * P; m < u * P + P; ++m)
        if (enc_owner(c, m) == r) lists[r].push_back(mk(kind, m, -1, u));
  };
  if (enc) {
    for (int u = 0; u < std::min(W, n_u); ++u) unit_ops(BM_OP_ENC_FWD, u);
    nxt = std::min(W, n_u);
  }
  for (const Ev& e : ev) {
    if (e.cls == 2) {
      const LOp& o = base[e.r][e.idx];
      if (enc && o.k == LF && e.r == 0 && o.chunk == 0 && o.mb / P >= nxt)
        throw Fail{BM_E_WARMUP, "W=" + std::to_string(W) + " too small: F(" + std::to_string(o.mb) +
                                    ",0)@0 precedes EncFwd(" + std::to_string(o.mb / P) + ")"};
      // memory-efficient baseline: the encoder is the entry stage's first layers
      if (entry && o.k == LF && e.r == 0 && o.chunk == 0) lists[0].push_back(mk(BM_OP_ENC_FWD, o.mb, -1, o.mb));
      lists[e.r].push_back(mk(LLM_OPK[o.k], o.mb, o.chunk));
      if (entry && o.k == LB && e.r == 0 && o.chunk == 0) lists[0].push_back(mk(BM_OP_ENC_BWD, o.mb, -1, o.mb));
    } else if (e.cls == 0) {
      const int m = e.idx;
      if (c.gen_place == BM_GEN_DP_SHARD) {
        for (int r = 0; r < P; ++r) {
          lists[r].push_back(mk(BM_OP_GEN_FWD, m));
          lists[r].push_back(mk(BM_OP_GEN_BWD, m));
        }
      } else {
        lists[P - 1].push_back(mk(BM_OP_GEN_FWD, m));
        lists[P - 1].push_back(mk(BM_OP_GEN_BWD, m));
      }
    } else {
      const int u = e.idx;
      unit_ops(BM_OP_ENC_BWD, u);
      if (nxt < n_u) {
        unit_ops(BM_OP_ENC_FWD, nxt);
        ++nxt;
      }
    }
  }
  return lists;
}

// ---------------------------------------------------------------- comm insertion
static bool is_compute(int k) { return k <= BM_OP_GEN_BWD || k == BM_OP_LLM_W; }

static void recvs_before(const bm_sched_cfg& c, int r, const bm_op& o, std::vector<bm_op>& out) {
  const int P = c.stages, V = c.vchunks;
  if (o.kind == BM_OP_LLM_FWD) {
    const int s = o.chunk * P + r;
    if (s > 0 && (s - 1) % P != r) out.push_back(mk(BM_OP_RECV, o.mb, o.chunk, -1, (s - 1) % P, BM_PAY_ACT));
    if (s == 0 && c.enc_place == BM_ENC_DP_UNIT && enc_owner(c, o.mb) != 0)
      out.push_back(mk(BM_OP_RECV, o.mb, -1, o.mb / P, enc_owner(c, o.mb), BM_PAY_EMB));
  } else if (o.kind == BM_OP_LLM_BWD) {
    const int s = o.chunk * P + r;
    if (s < P * V - 1 && (s + 1) % P != r) out.push_back(mk(BM_OP_RECV, o.mb, o.chunk, -1, (s + 1) % P, BM_PAY_GRAD));
    if (s == P * V - 1 && c.gen_place == BM_GEN_DP_SHARD)
      for (int q = 0; q < P; ++q)
        if (q != r) out.push_back(mk(BM_OP_RECV, o.mb, -1, -1, q, BM_PAY_GENGRAD));
  } else if (o.kind == BM_OP_ENC_BWD && r != 0 && c.enc_place == BM_ENC_DP_UNIT) {
    out.push_back(mk(BM_OP_RECV, o.mb, -1, o.unit, 0, BM_PAY_EMBGRAD));
  } else if (o.kind == BM_OP_GEN_FWD && c.gen_place == BM_GEN_DP_SHARD && r != P - 1) {
    out.push_back(mk(BM_OP_RECV, o.mb, -1, -1, P - 1, BM_PAY_GENIN));
  }
}

static void sends_after(const bm_sched_cfg& c, int r, const bm_op& o, std::vector<bm_op>& out) {
  const int P = c.stages, V = c.vchunks;
  if (o.kind == BM_OP_LLM_FWD) {
    const int s = o.chunk * P + r;
    if (s < P * V - 1 && (s + 1) % P != r) out.push_back(mk(BM_OP_SEND, o.mb, o.chunk, -1, (s + 1) % P, BM_PAY_ACT));
    if (s == P * V - 1 && c.gen_place == BM_GEN_DP_SHARD)
      for (int q = 0; q < P; ++q)
        if (q != r) out.push_back(mk(BM_OP_SEND, o.mb, -1, -1, q, BM_PAY_GENIN));
  } else if (o.kind == BM_OP_LLM_BWD) {
    const int s = o.chunk * P + r;
    if (s > 0 && (s - 1) % P != r) out.push_back(mk(BM_OP_SEND, o.mb, o.chunk, -1, (s - 1) % P, BM_PAY_GRAD));
    if (s == 0 && c.enc_place == BM_ENC_DP_UNIT && enc_owner(c, o.mb) != 0)
      out.push_back(mk(BM_OP_SEND, o.mb, -1, o.mb / P, enc_owner(c, o.mb), BM_PAY_EMBGRAD));
  } else if (o.kind == BM_OP_ENC_FWD && r != 0 && c.enc_place == BM_ENC_DP_UNIT) {
    out.push_back(mk(BM_OP_SEND, o.mb, -1, o.unit, 0, BM_PAY_EMB));
  } else if (o.kind == BM_OP_GEN_BWD && c.gen_place == BM_GEN_DP_SHARD && r != P - 1) {
    out.push_back(mk(BM_OP_SEND, o.mb, -1, -1, P - 1, BM_PAY_GENGRAD));
  }
}

typedef std::tuple<int, int, int> Chan;  // src, dst, payload

// ---------------------------------------------------------------- deadlock graph
struct Graph {
  int n = 0;
  std::vector<int> rank_base;
  std::map<std::pair<Chan, int>, int> send_at, recv_at, release_at;  // -> node id
  std::vector<std::pair<int, int>> base_edges;
};

static Graph build_graph(const std::vector<std::vector<bm_op>>& L) {
  Graph g;
  const int P = (int)L.size();
  g.rank_base.resize(P);
  for (int r = 0; r < P; ++r) { g.rank_base[r] = g.n; g.n += (int)L[r].size(); }
  for (int r = 0; r < P; ++r) {
    const auto& ops = L[r];
    for (int i = 0; i < (int)ops.size(); ++i) {
      const bm_op& o = ops[i];
      if (o.kind == BM_OP_SEND) {
        g.send_at[{Chan{r, o.peer, o.payload}, o.seq}] = g.rank_base[r] + i;
      } else if (o.kind == BM_OP_RECV) {
        Chan ch{o.peer, r, o.payload};
        g.recv_at[{ch, o.seq}] = g.rank_base[r] + i;
        int j = i + 1;
        while (!is_compute(ops[j].kind)) ++j;
        if (o.payload == BM_PAY_GENIN)
          while (ops[j].kind != BM_OP_GEN_BWD) ++j;
        g.release_at[{ch, o.seq}] = g.rank_base[r] + j;
      }
    }
    int prev = -1;
    std::map<int, int> last_send;
    for (int i = 0; i < (int)ops.size(); ++i) {
      const int id = g.rank_base[r] + i;
      if (ops[i].kind == BM_OP_SEND) {
        if (prev >= 0) g.base_edges.push_back({g.rank_base[r] + prev, id});
        auto it = last_send.find(ops[i].peer);
        if (it != last_send.end()) g.base_edges.push_back({g.rank_base[r] + it->second, id});
        last_send[ops[i].peer] = i;
      } else {
        if (prev >= 0) g.base_edges.push_back({g.rank_base[r] + prev, id});
        prev = i;
      }
    }
  }
  for (auto& kv : g.send_at) g.base_edges.push_back({kv.second, g.recv_at.at(kv.first)});
  return g;
}

static void credit_edges(const Graph& g, const Chan& ch, int K, int nmsg, std::vector<std::pair<int, int>>& out) {
  for (int j = K; j < nmsg; ++j) out.push_back({g.release_at.at({ch, j - K}), g.send_at.at({ch, j})});
}

static bool acyclic(int n, const std::vector<std::pair<int, int>>& e1, const std::vector<std::pair<int, int>>& e2) {
  std::vector<int> indeg(n, 0), head(n, -1), nxt(e1.size() + e2.size()), to(e1.size() + e2.size());
  int k = 0;
  auto add = [&](const std::pair<int, int>& e) {
    to[k] = e.second; nxt[k] = head[e.first]; head[e.first] = k; ++indeg[e.second]; ++k;
  };
  for (auto& e : e1) add(e);
  for (auto& e : e2) add(e);
  std::vector<int> q;
  q.reserve(n);
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) q.push_back(i);
  size_t qi = 0;
  while (qi < q.size()) {
    const int x = q[qi++];
    for (int e = head[x]; e >= 0; e = nxt[e])
      if (--indeg[to[e]] == 0) q.push_back(to[e]);
  }
  return (int)q.size() == n;
}

// ---------------------------------------------------------------- verification
static void verify_deps(const bm_sched_cfg& c, const std::vector<std::vector<bm_op>>& lists) {
  const int P = c.stages, V = c.vchunks;
  std::map<std::tuple<int, int, int, int>, int> nid;  // (rank, kind, mb, chunk)
  auto key = [](int r, const bm_op& o) {
    const bool llm = o.kind == BM_OP_LLM_FWD || o.kind == BM_OP_LLM_BWD || o.kind == BM_OP_LLM_W;
    return std::make_tuple(r, o.kind, o.mb, llm ? o.chunk : -1);
  };
  int n = 0;
  for (int r = 0; r < P; ++r)
    for (auto& o : lists[r]) {
      auto k = key(r, o);
      if (nid.count(k)) throw Fail{BM_E_DEPENDENCY, "duplicate compute op"};
      nid[k] = n++;
    }
  std::vector<std::pair<int, int>> edges;
  auto dep = [&](int r, int kind, int mb, int chunk, int to) {
    auto it = nid.find(std::make_tuple(r, kind, mb, chunk));
    if (it == nid.end()) throw Fail{BM_E_DEPENDENCY, "missing producer"};
    edges.push_back({it->second, to});
  };
  for (int r = 0; r < P; ++r) {
    for (size_t i = 0; i < lists[r].size(); ++i) {
      const bm_op& o = lists[r][i];
      const int me = nid[key(r, o)];
      if (i) edges.push_back({nid[key(r, lists[r][i - 1])], me});
      if (o.kind == BM_OP_LLM_FWD) {
        const int s = o.chunk * P + r;
        if (s > 0) dep((s - 1) % P, BM_OP_LLM_FWD, o.mb, (s - 1) / P, me);
        else if (c.enc_place == BM_ENC_DP_UNIT) dep(enc_owner(c, o.mb), BM_OP_ENC_FWD, o.mb, -1, me);
        else if (c.enc_place == BM_ENC_ENTRY_STAGE) dep(0, BM_OP_ENC_FWD, o.mb, -1, me);
      } else if (o.kind == BM_OP_LLM_BWD) {
        const int s = o.chunk * P + r;
        dep(r, BM_OP_LLM_FWD, o.mb, o.chunk, me);
        if (s < P * V - 1) dep((s + 1) % P, BM_OP_LLM_BWD, o.mb, (s + 1) / P, me);
        else if (c.gen_place == BM_GEN_DP_SHARD) for (int q = 0; q < P; ++q) dep(q, BM_OP_GEN_BWD, o.mb, -1, me);
        else if (c.gen_place == BM_GEN_LAST_STAGE) dep(P - 1, BM_OP_GEN_BWD, o.mb, -1, me);
      } else if (o.kind == BM_OP_LLM_W) {
        dep(r, BM_OP_LLM_BWD, o.mb, o.chunk, me);
      } else if (o.kind == BM_OP_ENC_BWD) {
        dep(r, BM_OP_ENC_FWD, o.mb, -1, me);
        dep(0, BM_OP_LLM_BWD, o.mb, 0, me);
      } else if (o.kind == BM_OP_GEN_FWD) {
        dep(P - 1, BM_OP_LLM_FWD, o.mb, V - 1, me);
      } else if (o.kind == BM_OP_GEN_BWD) {
        dep(r, BM_OP_GEN_FWD, o.mb, -1, me);
      }
    }
  }
  if (!acyclic(n, edges, {})) throw Fail{BM_E_DEPENDENCY, "dependency cycle in the nested schedule"};
}

static int peak_window(const std::vector<bm_op>& ops, int open_k, int close_k) {
  int cur = 0, best = 0;
  for (auto& o : ops) {
    if (o.kind == open_k) best = std::max(best, ++cur);
    else if (o.kind == close_k) --cur;
  }
  return best;
}

// sequence numbers, ring sizing (P:317 deadlock_check), slots and statistics of a
// schedule with comm ops; R ranks, rank r running stage r % P's LLM list
static bm_schedule* finish_schedule(const bm_sched_cfg& c, const std::vector<std::vector<LOp>>& base, const Times& T,
                                    const std::vector<std::vector<bm_op>>& lists, std::vector<std::vector<bm_op>>& full,
                                    int W, int ws, bool zb, int cb, int cw, int R) {
  const int P = c.stages;
  std::map<Chan, int> scnt, rcnt;
  for (int r = 0; r < R; ++r)
    for (auto& o : full[r]) {
      if (o.kind == BM_OP_SEND) o.seq = scnt[Chan{r, o.peer, o.payload}]++;
      else if (o.kind == BM_OP_RECV) o.seq = rcnt[Chan{o.peer, r, o.payload}]++;
    }
  if (scnt != rcnt) throw Fail{BM_E_DEPENDENCY, "unmatched send/recv counts"};
  // ring sizing
  Graph g = build_graph(full);
  if (!acyclic(g.n, g.base_edges, {})) throw Fail{BM_E_DEADLOCK, "schedule deadlocks even with unbounded slots"};
  std::map<Chan, int> K;
  for (auto& kv : scnt) {
    const int nmsg = kv.second;
    int k = 1;
    while (k < nmsg) {
      std::vector<std::pair<int, int>> ce;
      credit_edges(g, kv.first, k, nmsg, ce);
      if (acyclic(g.n, g.base_edges, ce)) break;
      ++k;
    }
    K[kv.first] = std::min(k + c.ring_slack, nmsg);
  }
  for (;;) {
    std::vector<std::pair<int, int>> ce;
    for (auto& kv : scnt) credit_edges(g, kv.first, K[kv.first], kv.second, ce);
    if (acyclic(g.n, g.base_edges, ce)) break;
    bool grew = false;
    for (auto& kv : scnt)
      if (K[kv.first] < kv.second) { ++K[kv.first]; grew = true; }
    if (!grew) throw Fail{BM_E_DEADLOCK, "credit rings cannot be sized"};
  }
  for (int r = 0; r < R; ++r)
    for (auto& o : full[r]) {
      if (o.kind == BM_OP_SEND) o.slot = o.seq % K[Chan{r, o.peer, o.payload}];
      else if (o.kind == BM_OP_RECV) o.slot = o.seq % K[Chan{o.peer, r, o.payload}];
    }
  // stats
  auto* s = new bm_schedule();
  s->cfg = c;
  s->ranks = std::move(full);
  for (auto& kv : scnt) s->rings[kv.first] = {K[kv.first], kv.second};
  int64_t makespan = 0;
  for (auto e : T.en) makespan = std::max(makespan, e);
  const bool enc = c.enc_place == BM_ENC_DP_UNIT;
  for (int r = 0; r < R; ++r) {
    bm_sched_stats st;
    std::memset(&st, 0, sizeof(st));
    st.w_star = ws;
    st.warmup_units = enc ? W : 0;
    st.peak_enc_units = peak_window(lists[r], BM_OP_ENC_FWD, BM_OP_ENC_BWD);
    st.peak_gen_shards = peak_window(lists[r], BM_OP_GEN_FWD, BM_OP_GEN_BWD);
    // stage activations live from F until B (until W under ZB-H1)
    st.peak_llm_inflight = peak_window(lists[r], BM_OP_LLM_FWD, zb ? BM_OP_LLM_W : BM_OP_LLM_BWD);
    st.n_ops = (int)s->ranks[r].size();
    int64_t busy = 0;
    for (auto& o : base[r % P]) busy += o.k == LF ? c.cost_fwd : o.k == LB ? cb : cw;
    st.llm_idle_cost_units = makespan - busy;
    st.makespan_cost_units = makespan;
    for (auto& kv : s->rings)
      if (std::get<1>(kv.first) == r) {
        int p = std::get<2>(kv.first);
        st.ring_slots[p] = std::max(st.ring_slots[p], kv.second.first);
      }
    s->stats.push_back(st);
  }
  return s;
}

static bm_schedule* build_cp(const bm_sched_cfg& c);

// ---------------------------------------------------------------- driver
static bm_schedule* build(const bm_sched_cfg& c) {
  validate(c);
  if (c.llm_cp > 1 || c.enc_cp > 1) return build_cp(c);
  const int P = c.stages, M = c.microbatches, V = c.vchunks;
  const bool zb = c.llm_sched == BM_LLM_ZB_H1;
  const int cw = zb ? wgrad_cost(c) : 0, cb = c.cost_bwd - cw;
  auto base = zb ? zb_h1_lists(P, M, c.cost_fwd, cb, cw) : base_lists(P, M, V);
  Times T = des_llm(base, P, M, V, c.cost_fwd, cb, cw);
  int W = 0;
  auto lists = nest(c, base, T, W);
  verify_deps(c, lists);
  for (int r = 0; r < P; ++r) {  // LLM order preserved
    size_t k = 0;
    for (auto& o : lists[r]) {
      if (o.kind != BM_OP_LLM_FWD && o.kind != BM_OP_LLM_BWD && o.kind != BM_OP_LLM_W) continue;
      if (k >= base[r].size() || LLM_OPK[base[r][k].k] != o.kind || base[r][k].mb != o.mb ||
          base[r][k].chunk != o.chunk)
        throw Fail{BM_E_DEPENDENCY, "LLM order changed"};
      ++k;
    }
  }
  // comm insertion + sequence numbers
  std::vector<std::vector<bm_op>> full(P);
  for (int r = 0; r < P; ++r)
    for (auto& o : lists[r]) {
      recvs_before(c, r, o, full[r]);
      full[r].push_back(o);
      sends_after(c, r, o, full[r]);
    }
  return finish_schedule(c, base, T, lists, full, W, c.enc_place == BM_ENC_DP_UNIT ? w_star(base[0], P, M) : 0, zb,
                         cb, cw, P);
}

// ---------------------------------------------------------------- decoupled CP (R25)
// P llm_cp ranks, rank k = cp P + stage; encoder CP groups of enc_cp consecutive ranks,
// one microbatch each, units of U = P llm_cp / enc_cp microbatches; the
// CP-conversion all-to-all as emb / embgrad messages between the microbatch's encoder
// group and the stage-0 ranks.  Mirrors oracle/schedule.py build_cp.
static bm_schedule* build_cp(const bm_sched_cfg& c) {
  const int P = c.stages, M = c.microbatches, V = c.vchunks;
  const int lcp = c.llm_cp > 0 ? c.llm_cp : 1, ecp = c.enc_cp > 0 ? c.enc_cp : 1;
  const int R = P * lcp, U = R / ecp, n_u = M / U;
  const bool zb = c.llm_sched == BM_LLM_ZB_H1;
  const int cw = zb ? wgrad_cost(c) : 0, cb = c.cost_bwd - cw;
  auto base = zb ? zb_h1_lists(P, M, c.cost_fwd, cb, cw) : base_lists(P, M, V);
  Times T = des_llm(base, P, M, V, c.cost_fwd, cb, cw);
  const bool enc = c.enc_place == BM_ENC_DP_UNIT;
  const bool gen = c.gen_place != BM_GEN_NONE;
  const int W = enc ? (c.warmup_units > 0 ? c.warmup_units : w_star(base[0], U, M)) : 0;
  auto grp_lo = [&](int m) { return (m % U) * ecp; };   // encoder ranks [grp_lo, grp_lo + ecp)
  // ---- nesting
  struct Ev {
    int64_t t;
    int cls, tb, k, idx;
  };
  std::vector<Ev> ev;
  for (int k = 0; k < R; ++k)
    for (int i = 0; i < (int)base[k % P].size(); ++i) {
      const LOp& o = base[k % P][i];
      ev.push_back({T.st[T.idx(k % P, o.k, o.mb, o.chunk)], 2, k, k, i});
    }
  if (gen)
    for (int m = 0; m < M; ++m) ev.push_back({T.en[T.idx(P - 1, LF, m, V - 1)], 0, m, 0, m});
  if (enc)
    for (int u = 0; u < n_u; ++u) ev.push_back({T.en[T.idx(0, LB, u * U + U - 1, 0)], 1, u, 0, u});
  std::sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.cls != b.cls) return a.cls < b.cls;
    return a.tb < b.tb;
  });
  std::vector<std::vector<bm_op>> lists(R);
  auto unit_ops = [&](int kind, int u) {
    for (int k = 0; k < R; ++k)
      for (int m = u * U; m < u * U + U; ++m)
        if (k >= grp_lo(m) && k < grp_lo(m) + ecp) lists[k].push_back(mk(kind, m, -1, u));
  };
  int nxt = 0;
  if (enc) {
    for (int u = 0; u < std::min(W, n_u); ++u) unit_ops(BM_OP_ENC_FWD, u);
    nxt = std::min(W, n_u);
  }
  for (const Ev& e : ev) {
    if (e.cls == 2) {
      const LOp& o = base[e.k % P][e.idx];
      if (enc && o.k == LF && e.k % P == 0 && o.chunk == 0 && o.mb / U >= nxt)
        throw Fail{BM_E_WARMUP, "W=" + std::to_string(W) + " too small: F(" + std::to_string(o.mb) + ",0)@" +
                                    std::to_string(e.k) + " precedes EncFwd(" + std::to_string(o.mb / U) + ")"};
      lists[e.k].push_back(mk(LLM_OPK[o.k], o.mb, o.chunk));
    } else if (e.cls == 0) {
      for (int cc = 0; cc < lcp; ++cc) {
        lists[cc * P + P - 1].push_back(mk(BM_OP_GEN_FWD, e.idx));
        lists[cc * P + P - 1].push_back(mk(BM_OP_GEN_BWD, e.idx));
      }
    } else {
      unit_ops(BM_OP_ENC_BWD, e.idx);
      if (nxt < n_u) {
        unit_ops(BM_OP_ENC_FWD, nxt);
        ++nxt;
      }
    }
  }
  // ---- verification: program order + data dependencies (incl. the all-to-all) acyclic
  {
    std::map<std::tuple<int, int, int, int>, int> nid;
    auto key = [](int k, const bm_op& o) {
      const bool llm = o.kind == BM_OP_LLM_FWD || o.kind == BM_OP_LLM_BWD || o.kind == BM_OP_LLM_W;
      return std::make_tuple(k, o.kind, o.mb, llm ? o.chunk : -1);
    };
    int n = 0;
    for (int k = 0; k < R; ++k)
      for (auto& o : lists[k]) {
        auto kk = key(k, o);
        if (nid.count(kk)) throw Fail{BM_E_DEPENDENCY, "duplicate compute op"};
        nid[kk] = n++;
      }
    std::vector<std::pair<int, int>> edges;
    auto dep = [&](int k, int kind, int mb, int chunk, int to) {
      auto it = nid.find(std::make_tuple(k, kind, mb, chunk));
      if (it == nid.end()) throw Fail{BM_E_DEPENDENCY, "missing producer"};
      edges.push_back({it->second, to});
    };
    for (int k = 0; k < R; ++k) {
      const int cc = k / P, r = k % P;
      for (size_t i = 0; i < lists[k].size(); ++i) {
        const bm_op& o = lists[k][i];
        const int me = nid[key(k, o)];
        if (i) edges.push_back({nid[key(k, lists[k][i - 1])], me});
        const int s = o.chunk * P + r;
        if (o.kind == BM_OP_LLM_FWD) {
          if (s > 0) dep(cc * P + (s - 1) % P, BM_OP_LLM_FWD, o.mb, (s - 1) / P, me);
          else if (enc)
            for (int q = grp_lo(o.mb); q < grp_lo(o.mb) + ecp; ++q) dep(q, BM_OP_ENC_FWD, o.mb, -1, me);
        } else if (o.kind == BM_OP_LLM_BWD) {
          dep(k, BM_OP_LLM_FWD, o.mb, o.chunk, me);
          if (s < P * V - 1) dep(cc * P + (s + 1) % P, BM_OP_LLM_BWD, o.mb, (s + 1) / P, me);
          else if (c.gen_place == BM_GEN_LAST_STAGE) dep(k, BM_OP_GEN_BWD, o.mb, -1, me);
        } else if (o.kind == BM_OP_LLM_W) {
          dep(k, BM_OP_LLM_BWD, o.mb, o.chunk, me);
        } else if (o.kind == BM_OP_ENC_BWD) {
          dep(k, BM_OP_ENC_FWD, o.mb, -1, me);
          for (int c2 = 0; c2 < lcp; ++c2) dep(c2 * P, BM_OP_LLM_BWD, o.mb, 0, me);
        } else if (o.kind == BM_OP_GEN_FWD) {
          dep(k, BM_OP_LLM_FWD, o.mb, V - 1, me);
        } else if (o.kind == BM_OP_GEN_BWD) {
          dep(k, BM_OP_GEN_FWD, o.mb, -1, me);
        }
      }
    }
    if (!acyclic(n, edges, {})) throw Fail{BM_E_DEPENDENCY, "dependency cycle in the nested schedule"};
  }
  for (int k = 0; k < R; ++k) {  // LLM order preserved
    size_t i = 0;
    const auto& b = base[k % P];
    for (auto& o : lists[k]) {
      if (o.kind != BM_OP_LLM_FWD && o.kind != BM_OP_LLM_BWD && o.kind != BM_OP_LLM_W) continue;
      if (i >= b.size() || LLM_OPK[b[i].k] != o.kind || b[i].mb != o.mb || b[i].chunk != o.chunk)
        throw Fail{BM_E_DEPENDENCY, "LLM order changed"};
      ++i;
    }
  }
  // ---- comm insertion: act / grad within a CP index, CP conversion emb / embgrad
  std::vector<std::vector<bm_op>> full(R);
  for (int k = 0; k < R; ++k) {
    const int cc = k / P, r = k % P;
    for (auto& o : lists[k]) {
      std::vector<bm_op> before, after;
      const int s = o.chunk * P + r;
      if (o.kind == BM_OP_LLM_FWD) {
        if (s > 0 && (s - 1) % P != r) before.push_back(mk(BM_OP_RECV, o.mb, o.chunk, -1, cc * P + (s - 1) % P, BM_PAY_ACT));
        if (s == 0 && enc)
          for (int q = grp_lo(o.mb); q < grp_lo(o.mb) + ecp; ++q)
            if (q != k) before.push_back(mk(BM_OP_RECV, o.mb, -1, o.mb / U, q, BM_PAY_EMB));
        if (s < P * V - 1 && (s + 1) % P != r) after.push_back(mk(BM_OP_SEND, o.mb, o.chunk, -1, cc * P + (s + 1) % P, BM_PAY_ACT));
      } else if (o.kind == BM_OP_LLM_BWD) {
        if (s < P * V - 1 && (s + 1) % P != r) before.push_back(mk(BM_OP_RECV, o.mb, o.chunk, -1, cc * P + (s + 1) % P, BM_PAY_GRAD));
        if (s > 0 && (s - 1) % P != r) after.push_back(mk(BM_OP_SEND, o.mb, o.chunk, -1, cc * P + (s - 1) % P, BM_PAY_GRAD));
        if (s == 0 && enc)
          for (int q = grp_lo(o.mb); q < grp_lo(o.mb) + ecp; ++q)
            if (q != k) after.push_back(mk(BM_OP_SEND, o.mb, -1, o.mb / U, q, BM_PAY_EMBGRAD));
      } else if (o.kind == BM_OP_ENC_FWD && enc) {
        for (int c2 = 0; c2 < lcp; ++c2)
          if (c2 * P != k) after.push_back(mk(BM_OP_SEND, o.mb, -1, o.unit, c2 * P, BM_PAY_EMB));
      } else if (o.kind == BM_OP_ENC_BWD && enc) {
        for (int c2 = 0; c2 < lcp; ++c2)
          if (c2 * P != k) before.push_back(mk(BM_OP_RECV, o.mb, -1, o.unit, c2 * P, BM_PAY_EMBGRAD));
      }
      for (auto& x : before) full[k].push_back(x);
      full[k].push_back(o);
      for (auto& x : after) full[k].push_back(x);
    }
  }
  return finish_schedule(c, base, T, lists, full, W, enc ? w_star(base[0], U, M) : 0, zb, cb, cw, R);
}

}  // namespace sched
}  // namespace bm

// ================================================================ C ABI
static const char* KIND_NAMES[] = {"EncFwd", "EncBwd", "LlmFwd", "LlmBwd", "GenFwd", "GenBwd", "Send", "Recv", "LlmW"};
static const char* PAY_NAMES[] = {"act", "grad", "emb", "embgrad", "genin", "gengrad"};

extern "C" {

bm_status bm_build_schedule(const bm_sched_cfg* cfg, bm_schedule** out) {
  if (!cfg || !out) {
    bm::set_error("null argument");
    return BM_E_INVALID;
  }
  try {
    *out = bm::sched::build(*cfg);
    return BM_OK;
  } catch (const bm::sched::Fail& f) {
    bm::set_error(f.msg);
    *out = nullptr;
    return f.code;
  } catch (const std::exception& e) {
    bm::set_error(std::string("internal error: ") + e.what());
    *out = nullptr;
    return BM_E_DEPENDENCY;
  }
}

bm_status bm_schedule_rank_ops(const bm_schedule* s, int32_t rank, const bm_op** ops, int64_t* n) {
  if (!s || !ops || !n || rank < 0 || rank >= (int)s->ranks.size()) {
    bm::set_error("bad schedule/rank");
    return BM_E_INVALID;
  }
  *ops = s->ranks[rank].data();
  *n = (int64_t)s->ranks[rank].size();
  return BM_OK;
}

bm_status bm_schedule_stats(const bm_schedule* s, int32_t rank, bm_sched_stats* out) {
  if (!s || !out || rank < 0 || rank >= (int)s->stats.size()) {
    bm::set_error("bad schedule/rank");
    return BM_E_INVALID;
  }
  *out = s->stats[rank];
  return BM_OK;
}

bm_status bm_schedule_ring(const bm_schedule* s, int32_t src, int32_t dst, int32_t payload, int32_t* K,
                           int32_t* nmsg) {
  if (!s || !K || !nmsg) {
    bm::set_error("null argument");
    return BM_E_INVALID;
  }
  auto it = s->rings.find(std::make_tuple(src, dst, payload));
  *K = it == s->rings.end() ? 0 : it->second.first;
  *nmsg = it == s->rings.end() ? 0 : it->second.second;
  return BM_OK;
}

bm_status bm_schedule_serialize(const bm_schedule* s, char* buf, size_t cap, size_t* needed) {
  if (!s || !needed) {
    bm::set_error("null argument");
    return BM_E_INVALID;
  }
  std::string out;
  auto f = [&](int v) { out += (v < 0) ? std::string("-") : std::to_string(v); };
  for (size_t r = 0; r < s->ranks.size(); ++r)
    for (size_t i = 0; i < s->ranks[r].size(); ++i) {
      const bm_op& o = s->ranks[r][i];
      out += std::to_string(r); out += '\t';
      out += std::to_string(i); out += '\t';
      out += KIND_NAMES[o.kind]; out += '\t';
      f(o.mb); out += '\t';
      f(o.chunk); out += '\t';
      f(o.unit); out += '\t';
      f(o.peer); out += '\t';
      out += (o.payload < 0) ? "-" : PAY_NAMES[o.payload]; out += '\t';
      f(o.slot); out += '\t';
      f(o.seq); out += '\n';
    }
  *needed = out.size() + 1;
  if (cap == 0 || !buf) return BM_OK;
  if (cap < out.size() + 1) {
    bm::set_error("buffer too small");
    return BM_E_INVALID;
  }
  std::memcpy(buf, out.c_str(), out.size() + 1);
  return BM_OK;
}

void bm_schedule_free(bm_schedule* s) { delete s; }

}  // extern "C"
