// gemm_tc.cu -- bf16 GEMM on the 5th-gen tensor cores (sm_100a).
//
// C[m, n] = sum_k A(m, k) B(n, k) with fp32 accumulation in TMEM, for the
// dense block contractions of the synthetic MLLM (every Linear layer's
// forward, data-grad and weight-grad; PAPER P:290-304 gives the model
// functions, DESIGN.md "Kernels" the shapes).
//
// Design (sm_100a, one CTA per SM, persistent):
//   warp 0      TMA producer: cp.async.bulk.tensor 2D tiles, 128B swizzle,
//               STAGES-deep smem ring guarded by full/empty mbarriers
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (kind::f16, M=128, N=BN, K=16 per instruction); commits free
//               smem stages and publish finished accumulators
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused
//               epilogue (store / fp32 accumulate / residual add) -> global
//   TMEM holds two BN-column accumulators so the epilogue of tile i overlaps
//   the MMAs of tile i+1.
// A and B may each be K-major or MN-major; the UMMA smem descriptors and the
// instruction descriptor's major bits express the transpose, so forward,
// dgrad and wgrad need no transposed copies.
#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <unordered_set>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace bm {
int gemm_mode();
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;                  // 64 bf16 = 128 B = one swizzle row
constexpr int NUM_THREADS = 192;

// epilogue staging: per epilogue warp 2 slots of EPI_SLOT bytes (one 32x32
// output sub-tile per output tensor, 128B/64B-swizzled for the TMA store)
constexpr int EPI_WARPS = 4;
template <int BN> struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;          // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;             // double-buffered accumulators
  static constexpr int EPI_SLOT = 4096;
  static constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_SLOT;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct EpiArgs {
  int M, N, K;
  void* C;
  int64_t ldc;
  int c_f32;       // C is fp32
  int epi;         // bm_epilogue
  const void* R;
  int64_t ldr;
  float alpha;
  int f;           // SwiGLU width (BM_EPI_SWIGLU / BM_EPI_DSWIGLU)
  int tma;         // outputs written by TMA stores from swizzled smem staging
  int splits;      // split-K factor (1-CTA kernel); > 1: fp32 partials to the workspace map
  int kb_per;      // K blocks per split
  int mpad;        // workspace rows per split (M rounded up to the tile height)
  // stream-K (CTA-pair kernel, sk != 0): pair p runs the k-iterations
  // [p T / npairs, (p+1) T / npairs) of the T = tiles * nk (tile, k-block) sequence
  int sk;
  float* sk_ws;          // fp32 tail partials: [npairs][2 CTAs][128 rows][BN]
  uint32_t* sk_flags;    // [npairs][2 CTAs][8 epilogue warps], = sk_epoch when a partial is ready
  uint32_t sk_epoch;     // unique per launch on this flag set
  int group;             // raster group (m-tiles per n sweep) of the CTA-pair kernel
  // sk == 2 (DP + split remainder): the first dp_tiles tiles round-robin as whole
  // tiles; the other rem tiles are cut into ksplit k-ranges, pieces ordered
  // k-range-major (piece i: range i / rem of remainder tile i % rem) and dealt
  // round-robin, so concurrent pieces read the same k-range of A and B
  int dp_tiles, rem, ksplit;
  int mbar_cluster;      // 1: .acquire.cluster barrier waits (default); 0: BM_MBAR_SCOPE=cta
  int sk_tma;            // partials written by TMA stores through tmC2 (swizzled smem staging)
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with the default .acquire.cta semantics (as CUTLASS's barrier waits):
// the guarded data moves through the async proxy (TMA, tcgen05) whose completion
// the barrier itself tracks, so no cluster-scope acquire -- which the compiler
// implements as an L1 invalidation (CCTL.IVALL) on every poll -- is needed.
// cluster_scope = 1 (default) uses .acquire.cluster; BM_MBAR_SCOPE=cta selects the
// CTA-scope form (parity-tested, no measurable step difference: 47.8-48.0 both,
// profiles/r01/bench_n1_mbar_*.log).
__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity, int cluster_scope) {
  uint32_t ok;
  if (cluster_scope) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  }
  return ok != 0;
}
// Wait for the phase with `parity`; a protocol bug traps after ~20 s instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int cluster_scope = 0) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity, cluster_scope)) return;
  const long long t0 = clock64();
  while (!mbar_try(a, parity, cluster_scope)) {
    if (clock64() - t0 > 40000000000LL) __trap();
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// ---- TMA stores (epilogue)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load whose completion is signalled on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// commit: arrive on the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B, version 1 (sm_100).
//   K-major : LBO unused (1), SBO = 1024 B (8 rows x 128 B)
//   MN-major: LBO = byte stride between 64-element MN chunks, SBO = 1024 B
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (sm_100)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> fp32, M = 128, N = BN.
__host__ __device__ constexpr uint32_t make_idesc(int N, bool a_mn, bool b_mn, int M = BM) {
  return (1u << 4)                     // D format fp32
         | (1u << 7)                   // A bf16
         | (1u << 10)                  // B bf16
         | ((a_mn ? 1u : 0u) << 15)    // A major
         | ((b_mn ? 1u : 0u) << 16)    // B major
         | ((uint32_t)(N >> 3) << 17)  // N / 8
         | ((uint32_t)(M >> 4) << 24); // M / 16
}

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& mb, int& nb, int G = 8) {
  // grouped raster: G m-tiles share each n sweep for L2 reuse of B
  int per_group = G * tiles_n;
  int group = t / per_group;
  int first_m = group * G;
  int gm = min(G, tiles_m - first_m);
  int r = t % per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

// The (tile, k-block range) segments of one CTA pair: round-robin whole tiles,
// or (stream-K) the pair's contiguous share of the tile-major k-iteration
// sequence.  With tiles >= pairs a share spans >= nk iterations, so a tile is
// cut at most once: its head [0, kb1) ends the share of pair p and its tail
// [kb1, nk) starts the share of pair p + 1.
struct SegIter {
  int sk, nk, num_tiles, step, t;
  int64_t g, g1;
  int dp, rem, ks, piece;   // sk == 2
  int q = -1, tr = -1;      // sk == 2: k-range index and remainder tile of the last piece (-1: whole tile)
  __device__ SegIter(const EpiArgs& a, int pair, int npairs, int tiles, int nk_)
      : sk(a.sk), nk(nk_), num_tiles(tiles), step(npairs), t(pair), dp(a.dp_tiles), rem(a.rem), ks(a.ksplit),
        piece(pair) {
    const int64_t tot = (int64_t)tiles * nk_;
    g = tot * pair / npairs;
    g1 = tot * (pair + 1) / npairs;
  }
  __device__ bool next(int& tile, int& kb0, int& kb1) {
    if (sk == 2) {
      if (t < dp) {
        tile = t;
        kb0 = 0;
        kb1 = nk;
        t += step;
        q = tr = -1;
        return true;
      }
      if (piece >= rem * ks) return false;
      q = piece / rem;
      tr = piece % rem;
      tile = dp + tr;
      kb0 = (int)((int64_t)q * nk / ks);
      kb1 = (int)((int64_t)(q + 1) * nk / ks);
      piece += step;
      return true;
    }
    if (!sk) {
      if (t >= num_tiles) return false;
      tile = t;
      kb0 = 0;
      kb1 = nk;
      t += step;
      return true;
    }
    if (g >= g1) return false;
    tile = (int)(g / nk);
    kb0 = (int)(g % nk);
    kb1 = (int)min((int64_t)nk, (int64_t)kb0 + (g1 - g));
    g += kb1 - kb0;
    return true;
  }
};
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}


// ---------------------------------------------------------------- TMA epilogue
// One epilogue warp owns 32 rows of the tile.  For each 32-column chunk it
// writes its outputs into a swizzled 32x32 staging sub-tile (64B rows for bf16
// with SWIZZLE_64B, 128B rows for fp32 with SWIZZLE_128B) and one lane issues
// the TMA store (or, for fp32 weight gradients, a TMA reduce-add into global).
// Two staging slots per warp; a slot is reused only after its previous bulk
// group has been read (cp.async.bulk.wait_group.read 1).
__device__ __forceinline__ void stage_bf16(uint32_t buf, int lane, const float* w) {
  const uint32_t row = buf + lane * 64;
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t p[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(w[8 * j + 2 * q], w[8 * j + 2 * q + 1]);
      p[q] = *reinterpret_cast<uint32_t*>(&h2);
    }
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((j ^ sw) << 4)), "r"(p[0]), "r"(p[1]),
                 "r"(p[2]), "r"(p[3])
                 : "memory");
  }
}
__device__ __forceinline__ void stage_f32(uint32_t buf, int lane, const float* w) {
  const uint32_t row = buf + lane * 128;
  const int sw = lane & 7;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((j ^ sw) << 4)), "f"(w[4 * j]),
                 "f"(w[4 * j + 1]), "f"(w[4 * j + 2]), "f"(w[4 * j + 3])
                 : "memory");
}
// sigmoid(x) = 0.5 + 0.5 tanh(x / 2): one MUFU.TANH instead of ex2 + reciprocal
__device__ __forceinline__ float sigmoidf_(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * x));
  return fmaf(0.5f, t, 0.5f);
}

// outputs for one 32-column chunk of a plain / accumulate / residual / dswiglu epilogue
__device__ __forceinline__ void epi_chunk_tma(const EpiArgs& a, const CUtensorMap* tmC, uint32_t slot, int lane,
                                              int row0, int col0, const float* v) {
  const int row = row0 + lane;
  const bool rv = row < a.M;
  float w[32];
  if (a.epi == BM_EPI_DSWIGLU) {
    // v = dh; g, u from R = gu [.., 2f]; outputs dg -> cols [col0..], du -> cols [f + col0..]
    float wu[32];
    const bf16* gu = reinterpret_cast<const bf16*>(a.R) + (int64_t)row * a.ldr;
    const bool full = rv && col0 + 32 <= a.N;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      float g[8], u[8];
      if (full) {
        uint4 gv = *reinterpret_cast<const uint4*>(gu + col0 + j);
        uint4 uv = *reinterpret_cast<const uint4*>(gu + a.f + col0 + j);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          g[q] = __bfloat162float(reinterpret_cast<const bf16*>(&gv)[q]);
          u[q] = __bfloat162float(reinterpret_cast<const bf16*>(&uv)[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const bool ok = rv && col0 + j + q < a.N;
          g[q] = ok ? __bfloat162float(gu[col0 + j + q]) : 0.f;
          u[q] = ok ? __bfloat162float(gu[a.f + col0 + j + q]) : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float d = a.alpha * v[j + q], sg = sigmoidf_(g[q]);
        w[j + q] = d * u[q] * sg * (1.f + g[q] * (1.f - sg));
        wu[j + q] = d * g[q] * sg;
      }
    }
    stage_bf16(slot, lane, w);
    stage_bf16(slot + 2048, lane, wu);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(tmC, slot, col0, row0);
      tma_store_2d(tmC, slot + 2048, a.f + col0, row0);
      bulk_commit();
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) w[j] = a.alpha * v[j];
  if (a.epi == BM_EPI_ADD) {
    if (a.c_f32) {
      const float* r = reinterpret_cast<const float*>(a.R) + (int64_t)row * a.ldr + col0;
#pragma unroll
      for (int j = 0; j < 32; ++j) w[j] += (rv && col0 + j < a.N) ? r[j] : 0.f;
    } else {
      const bf16* r = reinterpret_cast<const bf16*>(a.R) + (int64_t)row * a.ldr + col0;
      if (rv && col0 + 32 <= a.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 q4 = *reinterpret_cast<const uint4*>(r + j);
#pragma unroll
          for (int q = 0; q < 8; ++q) w[j + q] += __bfloat162float(reinterpret_cast<const bf16*>(&q4)[q]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) w[j] += (rv && col0 + j < a.N) ? __bfloat162float(r[j]) : 0.f;
      }
    }
  }
  if (a.c_f32) stage_f32(slot, lane, w);
  else stage_bf16(slot, lane, w);
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (a.epi == BM_EPI_ACCUM) tma_reduce_add_2d(tmC, slot, col0, row0);
    else tma_store_2d(tmC, slot, col0, row0);
    bulk_commit();
  }
}

// gate/up pair chunk with fused SwiGLU: g -> gu[:, j0..], u -> gu[:, f + j0..], h -> h[:, j0..]
__device__ __forceinline__ void epi_swiglu_tma(const EpiArgs& a, const CUtensorMap* tmGU, const CUtensorMap* tmH,
                                               uint32_t slot, int lane, int row0, int j0, const float* vg,
                                               const float* vu) {
  float g[32], u[32], h[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float gr = __bfloat162float(__float2bfloat16_rn(a.alpha * vg[j]));
    const float ur = __bfloat162float(__float2bfloat16_rn(a.alpha * vu[j]));
    g[j] = gr;
    u[j] = ur;
    h[j] = gr * sigmoidf_(gr) * ur;
  }
  stage_bf16(slot, lane, g);
  stage_bf16(slot + 2048, lane, u);
  stage_bf16(slot + 4096, lane, h);
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmGU, slot, j0, row0);
    tma_store_2d(tmGU, slot + 2048, a.f + j0, row0);
    tma_store_2d(tmH, slot + 4096, j0, row0);
    bulk_commit();
  }
}

__device__ __forceinline__ void epilogue_row(const EpiArgs& a, int row, int col0, const float* v) {
  // one thread writes up to 32 consecutive columns of one row
  const int ncols = min(32, a.N - col0);
  if (ncols <= 0) return;
  const float alpha = a.alpha;
  if (a.epi == BM_EPI_DSWIGLU) {
    // v = dh[row, col0..]; gu = R [.., 2f]; write dgu = C [.., 2f]
    const bf16* gu = reinterpret_cast<const bf16*>(a.R) + (int64_t)row * a.ldr;
    bf16* dgu = reinterpret_cast<bf16*>(a.C) + (int64_t)row * a.ldc;
    if (ncols == 32) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 gv = *reinterpret_cast<const uint4*>(gu + col0 + j);
        uint4 uv = *reinterpret_cast<const uint4*>(gu + a.f + col0 + j);
        const bf16* gb = reinterpret_cast<const bf16*>(&gv);
        const bf16* ub = reinterpret_cast<const bf16*>(&uv);
        uint4 og, ou;
        bf16* ogb = reinterpret_cast<bf16*>(&og);
        bf16* oub = reinterpret_cast<bf16*>(&ou);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float g = __bfloat162float(gb[q]), u = __bfloat162float(ub[q]), d = alpha * v[j + q];
          const float sg = sigmoidf_(g);
          ogb[q] = __float2bfloat16_rn(d * u * sg * (1.f + g * (1.f - sg)));
          oub[q] = __float2bfloat16_rn(d * g * sg);
        }
        *reinterpret_cast<uint4*>(dgu + col0 + j) = og;
        *reinterpret_cast<uint4*>(dgu + a.f + col0 + j) = ou;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncols) {
          const float g = __bfloat162float(gu[col0 + j]), u = __bfloat162float(gu[a.f + col0 + j]), d = alpha * v[j];
          const float sg = sigmoidf_(g);
          dgu[col0 + j] = __float2bfloat16_rn(d * u * sg * (1.f + g * (1.f - sg)));
          dgu[a.f + col0 + j] = __float2bfloat16_rn(d * g * sg);
        }
      }
    }
    return;
  }
  if (a.c_f32) {
    float* c = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc + col0;
    const bool vec = (ncols == 32) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0);
    if (a.epi == BM_EPI_ACCUM) {
      if (vec) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = *reinterpret_cast<float4*>(c + j);
          o.x += alpha * v[j]; o.y += alpha * v[j + 1]; o.z += alpha * v[j + 2]; o.w += alpha * v[j + 3];
          *reinterpret_cast<float4*>(c + j) = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < ncols) c[j] += alpha * v[j];
      }
    } else {
      const float* r = (a.epi == BM_EPI_ADD) ? reinterpret_cast<const float*>(a.R) + (int64_t)row * a.ldr + col0 : nullptr;
      if (vec && (r == nullptr || (reinterpret_cast<uintptr_t>(r) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4 o = make_float4(alpha * v[j], alpha * v[j + 1], alpha * v[j + 2], alpha * v[j + 3]);
          if (r) {
            float4 q = *reinterpret_cast<const float4*>(r + j);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4*>(c + j) = o;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < ncols) c[j] = alpha * v[j] + (r ? r[j] : 0.f);
      }
    }
  } else {
    bf16* c = reinterpret_cast<bf16*>(a.C) + (int64_t)row * a.ldc + col0;
    const bf16* r = (a.epi == BM_EPI_ADD) ? reinterpret_cast<const bf16*>(a.R) + (int64_t)row * a.ldr + col0 : nullptr;
    const bool vec = (ncols == 32) && ((reinterpret_cast<uintptr_t>(c) & 15) == 0) &&
                     (r == nullptr || (reinterpret_cast<uintptr_t>(r) & 15) == 0);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = alpha * v[j + q];
        if (r) {
          uint4 rv = *reinterpret_cast<const uint4*>(r + j);
          const bf16* rb = reinterpret_cast<const bf16*>(&rv);
#pragma unroll
          for (int q = 0; q < 8; ++q) w[q] += __bfloat162float(rb[q]);
        }
        uint4 ov;
        bf16* ob = reinterpret_cast<bf16*>(&ov);
#pragma unroll
        for (int q = 0; q < 8; ++q) ob[q] = __float2bfloat16_rn(w[q]);
        *reinterpret_cast<uint4*>(c + j) = ov;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < ncols) {
          float w = alpha * v[j] + (r ? __bfloat162float(r[j]) : 0.f);
          c[j] = __float2bfloat16_rn(w);
        }
      }
    }
  }
}


// gate/up pair epilogue: g = v_g, u = v_u for features [j0, j0+32) of one row;
// writes gu[row, j0..] = g, gu[row, f + j0..] = u (C, ld 2f) and h = silu(g) u (R, ld f)
__device__ __forceinline__ void epilogue_swiglu(const EpiArgs& a, int row, int j0, const float* vg, const float* vu) {
  const int n = min(32, a.f - j0);
  if (n <= 0) return;
  bf16* gu = reinterpret_cast<bf16*>(a.C) + (int64_t)row * a.ldc;
  bf16* h = reinterpret_cast<bf16*>(const_cast<void*>(a.R)) + (int64_t)row * a.ldr;
  if (n == 32) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 og, ou, oh;
      bf16* ogb = reinterpret_cast<bf16*>(&og);
      bf16* oub = reinterpret_cast<bf16*>(&ou);
      bf16* ohb = reinterpret_cast<bf16*>(&oh);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float g = a.alpha * vg[j + q], u = a.alpha * vu[j + q];
        const bf16 gb = __float2bfloat16_rn(g), ub = __float2bfloat16_rn(u);
        ogb[q] = gb;
        oub[q] = ub;
        const float gr = __bfloat162float(gb), ur = __bfloat162float(ub);
        ohb[q] = __float2bfloat16_rn(gr * sigmoidf_(gr) * ur);
      }
      *reinterpret_cast<uint4*>(gu + j0 + j) = og;
      *reinterpret_cast<uint4*>(gu + a.f + j0 + j) = ou;
      *reinterpret_cast<uint4*>(h + j0 + j) = oh;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < n) {
        const bf16 gb = __float2bfloat16_rn(a.alpha * vg[j]), ub = __float2bfloat16_rn(a.alpha * vu[j]);
        gu[j0 + j] = gb;
        gu[a.f + j0 + j] = ub;
        const float gr = __bfloat162float(gb), ur = __bfloat162float(ub);
        h[j0 + j] = __float2bfloat16_rn(gr * sigmoidf_(gr) * ur);
      }
    }
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const __grid_constant__ CUtensorMap tmC, EpiArgs args) {
  using C = Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * C::A_BYTES;
  uint8_t* smE = smem + STAGES * C::STAGE_BYTES;  // epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(smE + C::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (args.M + BM - 1) / BM;
  const int tiles_n = (args.N + BN - 1) / BN;
  const int base_tiles = tiles_m * tiles_n;
  const int num_tiles = base_tiles * args.splits;   // (split, tile) work items
  const int nk_all = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();   // everything above is data independent (PDL overlap with the previous kernel)

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        const int sp = t / base_tiles;
        tile_coords(t - sp * base_tiles, tiles_m, tiles_n, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        const int kb_lo = sp * args.kb_per, kb_hi = min(nk_all, kb_lo + args.kb_per);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, args.mbar_cluster);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* a_dst = smA + stage * C::A_BYTES;
          uint8_t* b_dst = smB + stage * C::B_BYTES;
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(a_dst + j * (BK * 128), &tmA, &full[stage], m0 + 64 * j, k0);
          } else {
            tma_load_2d(a_dst, &tmA, &full[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(b_dst + j * (BK * 128), &tmB, &full[stage], n0 + 64 * j, k0);
          } else {
            tma_load_2d(b_dst, &tmB, &full[stage], k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = make_idesc(BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1, args.mbar_cluster);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        const int sp = t / base_tiles;
        const int kb_lo = sp * args.kb_per, kb_hi = min(nk_all, kb_lo + args.kb_per);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], phase, args.mbar_cluster);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(smB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t ad = A_MN ? make_desc(a_base + kk * 2048, BK * 128, 1024) : make_desc(a_base + kk * 32, 16, 1024);
            uint64_t bd = B_MN ? make_desc(b_base + kk * 2048, BK * 128, 1024) : make_desc(b_base + kk * 32, 16, 1024);
            umma_f16(tmem_d, ad, bd, idesc, (kb != kb_lo || kk != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 (TMEM lane quadrant = warp % 4)
    const int quad = warp & 3;
    const uint32_t ebase = smem_u32(smE) + (uint32_t)((warp - 2) * 2 * C::EPI_SLOT);
    int eiter = 0;
    int local = 0;
    // split-K partials: raw fp32 tiles stored at rows sp * mpad + row
    EpiArgs pa = args;
    pa.epi = BM_EPI_STORE;
    pa.c_f32 = 1;
    pa.alpha = 1.f;
    pa.M = args.splits * args.mpad;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      int mb, nb;
      const int sp = t / base_tiles;
      tile_coords(t - sp * base_tiles, tiles_m, tiles_n, mb, nb);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase, args.mbar_cluster);
      tc_fence_after();
      const int row0 = mb * BM + quad * 32;
      const int row = row0 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(taddr + c, v);
        if (args.tma) {
          if (nb * BN + c < args.N) {
            const uint32_t slot = ebase + (eiter & 1) * C::EPI_SLOT;
            if (eiter >= 2) {
              if (lane == 0) bulk_wait_read1();
              __syncwarp();
            }
            if (args.splits > 1) epi_chunk_tma(pa, &tmC, slot, lane, sp * args.mpad + row0, nb * BN + c, v);
            else epi_chunk_tma(args, &tmC, slot, lane, row0, nb * BN + c, v);
            ++eiter;
          }
        } else if (row < args.M) {
          epilogue_row(args, row, nb * BN + c, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)C::TMEM_COLS));
  }
}


// ============================================================================
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs computes a 256 x BN
// tile.  CTA r holds rows [128r, 128r+128) of the A tile and columns
// [r*BN/2, (r+1)*BN/2) of the B tile in its own shared memory; both CTAs' TMA
// loads complete on the leader's full barrier; the leader's single thread
// issues tcgen05.mma.cta_group::2 (M = 256, N = BN) which reads both CTAs'
// operands and writes rows 0-127 to CTA 0's TMEM and 128-255 to CTA 1's.
// Commits multicast to both CTAs' barriers; both epilogues report to the
// leader's tmem_empty barrier.  Per CTA and K-block this moves
// (128 + BN/2)*64*2 bytes instead of (128 + BN)*64*2.
// ============================================================================
constexpr int EPI_WARPS2 = 8;   // CTA-pair kernel: two epilogue warps per TMEM lane quadrant
constexpr int NUM_THREADS2 = 64 + 32 * EPI_WARPS2;
template <int BN, bool SWI = false> struct Cfg2 {
  static constexpr int A_BYTES = 128 * BK * 2;                 // 16 KB
  static constexpr int B_BYTES = (BN / 2) * BK * 2;            // 16 KB (BN = 256)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = SWI ? 5 : ((BN == 256) ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int EPI_SLOT = SWI ? 6144 : 4096;           // one staging slot per epilogue warp
  static constexpr int EPI_BYTES = EPI_WARPS2 * EPI_SLOT;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

template <int BN, bool A_MN, bool B_MN, bool SWIGLU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS2, 1)
gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2, EpiArgs args) {
  using C = Cfg2<BN, SWIGLU>;
  constexpr int STAGES = C::STAGES;
  constexpr int BNH = BN / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smA = smem;
  uint8_t* smB = smem + STAGES * C::A_BYTES;
  uint8_t* smE = smem + STAGES * C::STAGE_BYTES;  // epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(smE + C::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t cta = cluster_rank();
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int tiles_m = (args.M + 2 * BM - 1) / (2 * BM);
  const int tiles_n = SWIGLU ? (args.f + BNH - 1) / BNH : (args.N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nk = (args.K + BK - 1) / BK;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * EPI_WARPS2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      SegIter it(args, pair, npairs, num_tiles, nk);
      int t, kb0, kb1;
      while (it.next(t, kb0, kb1)) {
        int mb, nb;
        tile_coords(t, tiles_m, tiles_n, mb, nb, args.group);
        const int m0 = mb * 2 * BM + (int)cta * BM;
        // SwiGLU pairing: CTA 0 loads gate rows [nb*BNH, +BNH), CTA 1 the matching up rows
        const int n0 = SWIGLU ? (nb * BNH + (int)cta * args.f) : (nb * BN + (int)cta * BNH);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, args.mbar_cluster);
          if (cta == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const uint32_t lbar = mapa(smem_u32(&full[stage]), 0);
          uint8_t* a_dst = smA + stage * C::A_BYTES;
          uint8_t* b_dst = smB + stage * C::B_BYTES;
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(a_dst + j * (BK * 128), &tmA, lbar, m0 + 64 * j, k0);
          } else {
            tma_load_2d_pair(a_dst, &tmA, lbar, k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j) tma_load_2d_pair(b_dst + j * (BK * 128), &tmB, lbar, n0 + 64 * j, k0);
          } else {
            tma_load_2d_pair(b_dst, &tmB, lbar, k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (cta == 0 && lane == 0) {
      constexpr uint32_t idesc = make_idesc(BN, A_MN, B_MN, 2 * BM);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      SegIter it(args, pair, npairs, num_tiles, nk);
      int t, kb0, kb1;
      for (; it.next(t, kb0, kb1); ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1, args.mbar_cluster);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase, args.mbar_cluster);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(smB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t ad = A_MN ? make_desc(a_base + kk * 2048, BK * 128, 1024) : make_desc(a_base + kk * 32, 16, 1024);
            uint64_t bd = B_MN ? make_desc(b_base + kk * 2048, BK * 128, 1024) : make_desc(b_base + kk * 32, 16, 1024);
            umma_f16_pair(tmem_d, ad, bd, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
          }
          umma_commit_pair(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_pair(&tfull[acc]);
      }
    }
  } else {
    // epilogue warps 2..9: TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;
    const uint32_t slot = smem_u32(smE) + (uint32_t)((warp - 2) * C::EPI_SLOT);
    int eiter = 0;
    const uint32_t leader_tempty0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa(smem_u32(&tempty[1]), 0);
    int local = 0;
    SegIter it(args, pair, npairs, num_tiles, nk);
    int t, kb0, kb1;
    const int ew = warp - 2;   // epilogue warp: (quad, half) sub-block, the same in every pair
    for (; it.next(t, kb0, kb1); ++local) {
      int mb, nb;
      tile_coords(t, tiles_m, tiles_n, mb, nb, args.group);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase, args.mbar_cluster);
      tc_fence_after();
      const int row0 = mb * 2 * BM + (int)cta * BM + quad * 32;
      const int row = row0 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      // partial-sum producers: stream-K tails (slot = this pair) and split-remainder
      // pieces before the last k-range (slot = tr * (ksplit - 1) + q)
      const bool piece_part = args.sk == 2 && it.q >= 0 && it.q < args.ksplit - 1;
      if (!SWIGLU && ((args.sk == 1 && kb0 > 0) || piece_part)) {
        // this warp's 32 x BN/2 fp32 sub-block of the partial sum into the slot, then
        // publish it (the owner of the tile's last piece finishes the tile)
        const int64_t pslot = piece_part ? (int64_t)it.tr * (args.ksplit - 1) + it.q : pair;
        if (args.sk_tma) {
          // coalesced: swizzled 32 x 32 fp32 staging + TMA store into the workspace
          // viewed as [slots * 2 * 128 rows, BN] (the normal epilogue's path)
          const int prow = (int)((pslot * 2 + cta) * BM + quad * 32);
#pragma unroll 1
          for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            float v[32];
            tmem_ld32(taddr + c, v);
            if (eiter >= 1) {
              if (lane == 0) bulk_wait_read0();
              __syncwarp();
            }
            stage_f32(slot, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC2, slot, c, prow);
              bulk_commit();
            }
            ++eiter;
          }
          if (lane == 0) {   // stores performed, then visible to the owner's generic loads
            bulk_wait_all();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            __threadfence();
          }
          __syncwarp();
        } else {
          float* dst = args.sk_ws + (((pslot * 2 + cta) * BM + quad * 32 + lane) * BN);
#pragma unroll 1
          for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
            float v[32];
            tmem_ld32(taddr + c, v);
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              __stcg(reinterpret_cast<float4*>(dst + c + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
          }
          __threadfence();
          __syncwarp();
        }
        if (lane == 0) st_release_u32(args.sk_flags + (pslot * 2 + cta) * EPI_WARPS2 + ew, args.sk_epoch);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc ? leader_tempty1 : leader_tempty0);
        continue;
      }
      // consumers: a stream-K head adds pair + 1's tail; the last piece of a split
      // remainder tile adds the tile's ksplit - 1 partials in k-range order
      const bool sk_head = !SWIGLU && args.sk == 1 && kb1 < nk;
      const bool piece_last = !SWIGLU && args.sk == 2 && it.q == args.ksplit - 1;
      const int nparts = sk_head ? 1 : (piece_last ? args.ksplit - 1 : 0);
      const int64_t pslot0 = sk_head ? (int64_t)(pair + 1) : (int64_t)it.tr * (args.ksplit - 1);
      const float* part = nullptr;
      if (nparts > 0) {
        if (lane == 0) {
          for (int j = 0; j < nparts; ++j) {
            const uint32_t* fl = args.sk_flags + ((pslot0 + j) * 2 + cta) * EPI_WARPS2 + ew;
            const long long t0 = clock64();
            while (ld_acquire_u32(fl) != args.sk_epoch)
              if (clock64() - t0 > 40000000000LL) __trap();
          }
        }
        __syncwarp();
        part = args.sk_ws + (((pslot0 * 2 + cta) * BM + quad * 32 + lane) * BN);
      }
      if (SWIGLU) {
        constexpr int W = BNH / 2;   // features per warp
#pragma unroll 1
        for (int c = half * W; c < (half + 1) * W; c += 32) {
          float vg[32], vu[32];
          tmem_ld32(taddr + c, vg);
          tmem_ld32(taddr + BNH + c, vu);
          if (args.tma) {
            if (nb * BNH + c < args.f) {
              if (eiter >= 1) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              epi_swiglu_tma(args, &tmC, &tmC2, slot, lane, row0, nb * BNH + c, vg, vu);
              ++eiter;
            }
          } else if (row < args.M) {
            epilogue_swiglu(args, row, nb * BNH + c, vg, vu);
          }
        }
      } else {
        constexpr int W = BN / 2;    // columns per warp
#pragma unroll 1
        for (int c = half * W; c < (half + 1) * W; c += 32) {
          float v[32];
          tmem_ld32(taddr + c, v);
          for (int pj = 0; pj < nparts; ++pj) {   // fixed order: deterministic
            const float* pp = part + (int64_t)pj * 2 * BM * BN;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 q = __ldcg(reinterpret_cast<const float4*>(pp + c + j));
              v[j] += q.x; v[j + 1] += q.y; v[j + 2] += q.z; v[j + 3] += q.w;
            }
          }
          if (args.tma) {
            if (nb * BN + c < args.N) {
              if (eiter >= 1) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              epi_chunk_tma(args, &tmC, slot, lane, row0, nb * BN + c, v);
              ++eiter;
            }
          } else if (row < args.M) {
            epilogue_row(args, row, nb * BN + c, v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc ? leader_tempty1 : leader_tempty0);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)C::TMEM_COLS));
  }
}


// Deterministic split-K reduction: out = epilogue(sum_s ws[s]) in split order.
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(int M, int N, int splits, int mpad, const float* __restrict__ ws, EpiArgs a) {
  pdl_enter();
  const int64_t idx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int64_t total = (int64_t)M * N;
  if (idx >= total) return;
  const int row = (int)(idx / N), col = (int)(idx % N);   // N % 4 == 0
  float4 acc = *reinterpret_cast<const float4*>(ws + (int64_t)row * N + col);
  for (int sp = 1; sp < splits; ++sp) {
    const float4 p = *reinterpret_cast<const float4*>(ws + ((int64_t)sp * mpad + row) * N + col);
    acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
  }
  float w[4] = {a.alpha * acc.x, a.alpha * acc.y, a.alpha * acc.z, a.alpha * acc.w};
  if (a.c_f32) {
    float* c = reinterpret_cast<float*>(a.C) + (int64_t)row * a.ldc + col;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (a.epi == BM_EPI_ACCUM) c[q] += w[q];
      else if (a.epi == BM_EPI_ADD) c[q] = w[q] + reinterpret_cast<const float*>(a.R)[(int64_t)row * a.ldr + col + q];
      else c[q] = w[q];
    }
  } else {
    bf16* c = reinterpret_cast<bf16*>(a.C) + (int64_t)row * a.ldc + col;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v = w[q];
      if (a.epi == BM_EPI_ADD) v += __bfloat162float(reinterpret_cast<const bf16*>(a.R)[(int64_t)row * a.ldr + col + q]);
      c[q] = __float2bfloat16_rn(v);
    }
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* p;
  uint64_t inner, outer, stride;
  uint32_t box_outer;
  int kind;  // 0: bf16 operand (64 x box_outer, SW128); 1: bf16 output (32x32, SW64); 2: fp32 output (32x32, SW128)
  bool operator==(const MapKey& o) const {
    return p == o.p && inner == o.inner && outer == o.outer && stride == o.stride && box_outer == o.box_outer &&
           kind == o.kind;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.p);
    h = h * 1000003u ^ k.inner;
    h = h * 1000003u ^ k.outer;
    h = h * 1000003u ^ k.stride;
    h = h * 1000003u ^ k.box_outer;
    h = h * 1000003u ^ (size_t)k.kind;
    return h;
  }
};

static std::mutex g_map_mu;
static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2D tensor [outer][inner] with row stride `ld` elements.
//   kind 0: bf16 operand, box = 64 x box_outer, 128B swizzle (UMMA smem layout)
//   kind 1: bf16 epilogue output, box = 32 x 32, 64B swizzle (staging layout)
//   kind 2: fp32 epilogue output, box = 32 x 32, 128B swizzle
static bm_status make_map_k(const void* p, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_outer, int kind,
                            CUtensorMap* out) {
  MapKey key{p, inner, outer, ld, box_outer, kind};
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return BM_OK;
    }
  }
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BM_E_CUDA;
  }
  const uint64_t es = kind == 2 ? 4 : 2;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * es};
  cuuint32_t box[2] = {kind == 0 ? 64u : 32u, kind == 0 ? box_outer : 32u};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = kind == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUtensorMapSwizzle sw = kind == 1 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(out, dt, 2, const_cast<void*>(p), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") inner=" + std::to_string(inner) +
              " outer=" + std::to_string(outer) + " ld=" + std::to_string(ld) + " kind=" + std::to_string(kind));
    return BM_E_CUDA;
  }
  std::lock_guard<std::mutex> g(g_map_mu);
  if (g_maps.size() > 65536) g_maps.clear();
  g_maps.emplace(key, *out);
  return BM_OK;
}
static bm_status make_map(const void* p, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_outer,
                          CUtensorMap* out) {
  return make_map_k(p, inner, outer, ld, box_outer, 0, out);
}
// output map usable by the TMA epilogue? (16-byte aligned base and row stride)
static bool tma_out_ok(const void* p, int64_t ld, int es) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * es) % 16 == 0;
}

template <int BN, bool A_MN, bool B_MN>
static bm_status launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const EpiArgs& ea,
                        cudaStream_t st) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    BM_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<BN, A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int tiles = ceil_div(ea.M, BM) * ceil_div(ea.N, BN) * ea.splits;
  const int cap = gemm_sm_budget();
  const int grid = tiles < cap ? tiles : cap;
  BM_CUDA_TRY(launch_k(gemm_kernel<BN, A_MN, B_MN>, dim3(grid), dim3(NUM_THREADS), C::SMEM, st, ma, mb, mc, ea));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

template <int BN>
static bm_status dispatch_majors(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                                 const CUtensorMap& mc, const EpiArgs& ea, cudaStream_t st) {
  if (!a_mn && !b_mn) return launch<BN, false, false>(ma, mb, mc, ea, st);
  if (!a_mn && b_mn) return launch<BN, false, true>(ma, mb, mc, ea, st);
  if (a_mn && b_mn) return launch<BN, true, true>(ma, mb, mc, ea, st);
  return launch<BN, true, false>(ma, mb, mc, ea, st);
}


template <int BN, bool A_MN, bool B_MN, bool SWIGLU = false>
static bm_status launch2(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mc2,
                         const EpiArgs& ea, cudaStream_t st) {
  using C = Cfg2<BN, SWIGLU>;
  static bool attr_set = false;
  if (!attr_set) {
    BM_CUDA_TRY(cudaFuncSetAttribute(gemm2_kernel<BN, A_MN, B_MN, SWIGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     C::SMEM));
    attr_set = true;
  }
  const int tiles = ceil_div(ea.M, 2 * BM) * (SWIGLU ? ceil_div(ea.f, BN / 2) : ceil_div(ea.N, BN));
  const int pairs = gemm_sm_budget() / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);   // stream-K: tiles >= pairs, every pair busy
  BM_CUDA_TRY(launch_k(gemm2_kernel<BN, A_MN, B_MN, SWIGLU>, dim3(grid), dim3(NUM_THREADS2), C::SMEM, st, ma, mb, mc,
                       mc2, ea));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

template <int BN>
static bm_status dispatch_majors2(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                                  const CUtensorMap& mc, const EpiArgs& ea, cudaStream_t st,
                                  const CUtensorMap* mc2 = nullptr) {
  const CUtensorMap& m2 = mc2 ? *mc2 : mc;   // second map: the split-remainder partial workspace
  if (!a_mn && !b_mn) return launch2<BN, false, false>(ma, mb, mc, m2, ea, st);
  if (!a_mn && b_mn) return launch2<BN, false, true>(ma, mb, mc, m2, ea, st);
  if (a_mn && b_mn) return launch2<BN, true, true>(ma, mb, mc, m2, ea, st);
  return launch2<BN, true, false>(ma, mb, mc, m2, ea, st);
}

}  // namespace tc

// Workspace layout: [0, SK_FLAG_BYTES) stream-K ready flags (zeroed once per
// workspace, then only written with launch-unique epochs), then either split-K
// partial tiles (1-CTA kernel) or stream-K tail partials (CTA-pair kernel).
constexpr int64_t SK_FLAG_BYTES = 64 << 10;
static std::mutex g_sk_mu;
static std::unordered_set<const void*> g_sk_ready;   // workspaces whose flag region is zeroed
static uint32_t g_sk_epoch = 0;
static int g_raster_group = [] {   // BM_GEMM_GROUP: measurement override of the pair raster
  const char* e = getenv("BM_GEMM_GROUP");
  const int v = e ? atoi(e) : 8;
  return v >= 1 ? v : 8;
}();
static int g_mbar_cluster = [] {   // default: the fully validated .acquire.cluster waits
  const char* e = getenv("BM_MBAR_SCOPE");
  return e && std::string(e) == "cta" ? 0 : 1;
}();
static int g_sk_tma = [] {   // BM_SK_TMA=0: per-lane partial stores instead of TMA stores
  const char* e = getenv("BM_SK_TMA");
  return e ? (e[0] == '0' ? 0 : 1) : 1;
}();
static int g_split_rem = [] {   // BM_SPLIT_REM=1: DP + split-remainder schedule (opt-in: measured slower)
  const char* e = getenv("BM_SPLIT_REM");
  return e ? (e[0] == '1' ? 1 : 0) : 0;
}();
static int g_stream_k = [] {
  const char* e = getenv("BM_STREAM_K");
  return e ? (e[0] == '1' ? 1 : 0) : 0;   // opt-in: measured slower
}();

// 0 = auto (CTA pairs for large contractions), 1 = force 1-CTA, 2 = force CTA pairs
static int g_gemm_mode = [] {
  const char* e = getenv("BM_GEMM_MODE");
  return e ? (e[0] == '1' ? 1 : (e[0] == '2' ? 2 : 0)) : 0;
}();
int gemm_mode() { return g_gemm_mode; }
void set_gemm_mode(int m) { g_gemm_mode = m; }

bm_status gemm_bf16_tc(int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B, int64_t ldb,
                       int b_major, void* Cp, int64_t ldc, int c_dtype, int epi, const void* R, int64_t ldr,
                       float alpha, cudaStream_t st, int f, void* ws, int64_t ws_bytes) {
  using namespace tc;
  BM_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0, "lda/ldb must be multiples of 8 (16-byte TMA strides)");
  BM_CHECK_ARG((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
               "A/B must be 16-byte aligned");
  const bool amn = a_major != 0, bmn = b_major != 0;
  EpiArgs ea{M, N, K, Cp, ldc, c_dtype == BM_F32 ? 1 : 0, epi, R, ldr, alpha, f, 0, 1, 1 << 30, 0};
  ea.group = g_raster_group;
  ea.mbar_cluster = g_mbar_cluster;
  CUtensorMap ma, mb, mc, mc2;
  std::memset(&mc, 0, sizeof(mc));
  std::memset(&mc2, 0, sizeof(mc2));
  const int ces = c_dtype == BM_F32 ? 4 : 2;
  if (epi == BM_EPI_SWIGLU) {
    // gate/up GEMM with fused SwiGLU: always CTA pairs, BN = 256 (128 gate + 128 up features)
    BM_CHECK_ARG(b_major == 0 && c_dtype == BM_BF16 && N == 2 * f && f % 128 == 0, "SWIGLU epilogue: K-major B, bf16, N = 2f, f % 128 == 0");
    if (a_major == 0) BM_TRY(make_map(A, K, M, lda, BM, &ma));
    else BM_TRY(make_map(A, M, K, lda, BK, &ma));
    BM_TRY(make_map(B, K, N, ldb, 128, &mb));
    if (tma_out_ok(Cp, ldc, 2) && tma_out_ok(R, ldr, 2)) {
      BM_TRY(make_map_k(Cp, 2 * (uint64_t)f, M, ldc, 32, 1, &mc));
      BM_TRY(make_map_k(R, (uint64_t)f, M, ldr, 32, 1, &mc2));
      ea.tma = 1;
    }
    if (a_major == 0) return launch2<256, false, false, true>(ma, mb, mc, mc2, ea, st);
    return launch2<256, true, false, true>(ma, mb, mc, mc2, ea, st);
  }
  if (epi == BM_EPI_DSWIGLU) {
    BM_CHECK_ARG(c_dtype == BM_BF16 && N == f && ldc >= 2 * f && ldr >= 2 * f, "DSWIGLU epilogue: bf16, N = f, C/R are [M, 2f]");
    if (tma_out_ok(Cp, ldc, 2)) {
      BM_TRY(make_map_k(Cp, 2 * (uint64_t)f, M, ldc, 32, 1, &mc));
      ea.tma = 1;
    }
  } else if (tma_out_ok(Cp, ldc, ces)) {
    BM_TRY(make_map_k(Cp, (uint64_t)N, M, ldc, 32, c_dtype == BM_F32 ? 2 : 1, &mc));
    ea.tma = 1;
  }
  // CTA pairs for the large contractions (enough 256-row tiles to fill the
  // machine), 1-CTA tiles otherwise
  const int mode = gemm_mode();
  const int64_t pair_tiles = (int64_t)ceil_div(M, 2 * BM) * ceil_div(N, 256);
  const bool pair = mode == 2 || (mode == 0 && M >= 256 && N >= 256 && K >= 256 && pair_tiles >= num_sms() / 2);
  if (pair) {
    const int BN2 = (N >= 256) ? 256 : 128;
    if (a_major == 0) BM_TRY(make_map(A, K, M, lda, BM, &ma));
    else BM_TRY(make_map(A, M, K, lda, BK, &ma));
    if (b_major == 0) BM_TRY(make_map(B, K, N, ldb, BN2 / 2, &mb));
    else BM_TRY(make_map(B, N, K, ldb, BK, &mb));
    // stream-K when whole-tile waves would leave > 5 % of the pairs idle (e.g. the
    // C2 d = 2048 contractions: 128 tiles on 74 pairs = 1.73 waves -> 2)
    const int pairs = gemm_sm_budget() / 2;
    const int64_t tiles2 = (int64_t)ceil_div(M, 2 * BM) * ceil_div(N, BN2);
    const int64_t waves = (tiles2 + pairs - 1) / pairs;
    const int64_t sk_need = SK_FLAG_BYTES + (int64_t)pairs * 2 * BM * BN2 * 4;
    CUtensorMap mws2;
    bool have_mws2 = false;
    // DP + split remainder (opt-in): whole-tile waves, then the remainder tiles cut
    // into s k-ranges with s minimising ceil(rem s / pairs) / s (ties: smaller s)
    const int nkb = ceil_div(K, BK);
    const int64_t dp_t = tiles2 / pairs * pairs, rem_t = tiles2 - dp_t;
    int best_s = 1;
    double best = 1.0;
    for (int sp = 2; sp <= 4 && sp <= nkb && rem_t > 0; ++sp) {   // s <= 4 bounds the partial traffic
      const double r = (double)((rem_t * sp + pairs - 1) / pairs) / sp;
      if (r < best - 1e-9) { best = r; best_s = sp; }
    }
    const int64_t hy_need = SK_FLAG_BYTES + rem_t * (best_s - 1) * 2 * BM * BN2 * 4;
    const bool hybrid = g_split_rem && g_stream_k == 0 && ws && BN2 == 256 && tiles2 >= pairs && rem_t > 0 &&
                        best <= 0.9 && best_s <= nkb && ws_bytes >= hy_need &&
                        rem_t * (best_s - 1) * 2 * EPI_WARPS2 * 4 <= SK_FLAG_BYTES;
    if (hybrid) {
      {
        std::lock_guard<std::mutex> lk(g_sk_mu);
        if (!g_sk_ready.count(ws)) {
          BM_CUDA_TRY(cudaMemsetAsync(ws, 0, SK_FLAG_BYTES, st));
          g_sk_ready.insert(ws);
        }
        ea.sk_epoch = ++g_sk_epoch;
      }
      ea.sk = 2;
      ea.dp_tiles = (int)dp_t;
      ea.rem = (int)rem_t;
      ea.ksplit = best_s;
      ea.sk_flags = reinterpret_cast<uint32_t*>(ws);
      ea.sk_ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + SK_FLAG_BYTES);
      if (g_sk_tma) {
        BM_TRY(make_map_k(ea.sk_ws, (uint64_t)BN2, (uint64_t)rem_t * (best_s - 1) * 2 * BM, BN2, 32, 2, &mws2));
        ea.sk_tma = 1;
        have_mws2 = true;
      }
    } else if (g_stream_k && ws && ws_bytes >= sk_need && BN2 == 256 && tiles2 >= pairs && tiles2 % pairs != 0 &&
        (double)tiles2 / (double)(waves * pairs) < 0.95 && (int64_t)ceil_div(K, BK) >= 2) {
      {
        std::lock_guard<std::mutex> lk(g_sk_mu);
        if (!g_sk_ready.count(ws)) {
          BM_CUDA_TRY(cudaMemsetAsync(ws, 0, SK_FLAG_BYTES, st));
          g_sk_ready.insert(ws);
        }
        ea.sk_epoch = ++g_sk_epoch;
      }
      ea.sk = 1;
      ea.sk_flags = reinterpret_cast<uint32_t*>(ws);
      ea.sk_ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + SK_FLAG_BYTES);
    }
    if (BN2 == 256) return dispatch_majors2<256>(amn, bmn, ma, mb, mc, ea, st, have_mws2 ? &mws2 : nullptr);
    return dispatch_majors2<128>(amn, bmn, ma, mb, mc, ea, st);
  }
  // 1-CTA tiles: the largest BN that still gives ~a full wave of CTAs (small
  // encoder / generator contractions have only a few 128-row tiles)
  int BN = (N <= 64) ? 64 : (N <= 128 ? 128 : 256);
  const int tm = ceil_div(M, BM);
  while (BN > 64 && (int64_t)tm * ceil_div(N, BN) < (3 * num_sms()) / 4) BN /= 2;
  if (a_major == 0) BM_TRY(make_map(A, K, M, lda, BM, &ma));
  else BM_TRY(make_map(A, M, K, lda, BK, &ma));
  if (b_major == 0) BM_TRY(make_map(B, K, N, ldb, BN, &mb));
  else BM_TRY(make_map(B, N, K, ldb, BK, &mb));
  // split-K when a full wave of tiles is not available (deterministic: fp32
  // partial tiles in the caller's workspace, summed in split order)
  const int tiles = tm * ceil_div(N, BN);
  const int nk = ceil_div(K, BK);
  if (ws && ws_bytes > SK_FLAG_BYTES && tiles < num_sms() / 2 && nk >= 4 && N % 4 == 0 &&
      (epi == BM_EPI_STORE || epi == BM_EPI_ADD || epi == BM_EPI_ACCUM)) {
    int splits = std::min(8, std::min(num_sms() / tiles, nk / 2));
    const int mpad = tm * BM;
    ws = reinterpret_cast<char*>(ws) + SK_FLAG_BYTES;   // keep the stream-K flag region intact
    ws_bytes -= SK_FLAG_BYTES;
    while (splits > 1 && (int64_t)splits * mpad * N * 4 > ws_bytes) --splits;
    if (splits > 1) {
      const int kb_per = ceil_div(nk, splits);
      splits = ceil_div(nk, kb_per);
      EpiArgs pe = ea;
      pe.splits = splits;
      pe.kb_per = kb_per;
      pe.mpad = mpad;
      pe.tma = 1;
      CUtensorMap mws;
      BM_TRY(make_map_k(ws, (uint64_t)N, (uint64_t)splits * mpad, N, 32, 2, &mws));
      bm_status r;
      if (BN == 64) r = dispatch_majors<64>(amn, bmn, ma, mb, mws, pe, st);
      else if (BN == 128) r = dispatch_majors<128>(amn, bmn, ma, mb, mws, pe, st);
      else r = dispatch_majors<256>(amn, bmn, ma, mb, mws, pe, st);
      BM_TRY(r);
      const int64_t total = (int64_t)M * N / 4;
      BM_CUDA_TRY(launch_k(splitk_reduce_kernel, dim3((int)((total + 255) / 256)), dim3(256), 0, st, M, N, splits, mpad,
                           (const float*)ws, ea));
      count_launch();
      BM_CUDA_TRY(cudaGetLastError());
      return BM_OK;
    }
  }
  if (BN == 64) return dispatch_majors<64>(amn, bmn, ma, mb, mc, ea, st);
  if (BN == 128) return dispatch_majors<128>(amn, bmn, ma, mb, mc, ea, st);
  return dispatch_majors<256>(amn, bmn, ma, mb, mc, ea, st);
}

// every tcgen05 GEMM instantiation the dispatcher can launch (bm::preload_kernels)
template <int BN>
static void preload_bn(std::vector<const void*>& v) {
  using namespace tc;
  for (const void* f : {(const void*)gemm_kernel<BN, false, false>, (const void*)gemm_kernel<BN, false, true>,
                        (const void*)gemm_kernel<BN, true, true>, (const void*)gemm_kernel<BN, true, false>})
    v.push_back(f);
}
template <int BN>
static void preload_bn2(std::vector<const void*>& v) {
  using namespace tc;
  for (const void* f : {(const void*)gemm2_kernel<BN, false, false, false>, (const void*)gemm2_kernel<BN, false, true, false>,
                        (const void*)gemm2_kernel<BN, true, true, false>, (const void*)gemm2_kernel<BN, true, false, false>})
    v.push_back(f);
}
void preload_tc(std::vector<const void*>& v) {
  preload_bn<64>(v);
  preload_bn<128>(v);
  preload_bn<256>(v);
  preload_bn2<128>(v);
  preload_bn2<256>(v);
  v.push_back((const void*)tc::gemm2_kernel<256, false, false, true>);
  v.push_back((const void*)tc::gemm2_kernel<256, true, false, true>);
  v.push_back((const void*)tc::splitk_reduce_kernel);
}

}  // namespace bm
