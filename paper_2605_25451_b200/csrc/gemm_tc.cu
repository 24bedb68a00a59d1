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
#include "kernels.h"

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
  int group;       // raster group (m-tiles per n sweep) of the CTA-pair kernel
  int mbar_cluster;  // 1: .acquire.cluster barrier waits (default); 0: BM_MBAR_SCOPE=cta
  int prefetch = 1;  // pair epilogue: L2-prefetch the tile's g / u rows (BM_EPI_PREFETCH=0: off)
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
// remote arrive on the pair leader's barrier (default .release.cta semantics, as
// CUTLASS's ClusterBarrier::arrive: the TMEM reads it publishes are ordered by
// tcgen05.wait::ld + tcgen05.fence::before_thread_sync, not by the barrier's scope)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
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

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
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

// the same with a 4 KB staging slot: [g | u] first, then h once the TMA engine has read them
__device__ __forceinline__ void epi_swiglu_tma_4k(const EpiArgs& a, const CUtensorMap* tmGU, const CUtensorMap* tmH,
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
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmGU, slot, j0, row0);
    tma_store_2d(tmGU, slot + 2048, a.f + j0, row0);
    bulk_commit();
    bulk_wait_read0();
  }
  __syncwarp();
  stage_bf16(slot, lane, h);
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmH, slot, j0, row0);
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
// BN = 512 (pair tile 256 x 512, each CTA 128 x 512): a quarter less L2 -> SMEM
// traffic per FLOP than 256 x 256 (cuBLAS's tile on these shapes), at the price of a
// single TMEM accumulator (512 columns): the MMA waits for the epilogue between tiles
// BKP = 128: 128-deep K blocks (two 64-wide swizzle sub-tiles per operand, 64 KB stages,
// 3 stages) -- twice the MMAs per barrier round trip, same bytes per FLOP.
template <int BN, bool SWI = false, int BKP = 64> struct Cfg2 {
  static constexpr int A_BYTES = 128 * BKP * 2;                // 16 KB (BKP = 64)
  static constexpr int B_BYTES = (BN / 2) * BKP * 2;           // 16 KB (BN = 256), 32 KB (BN = 512)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // staging slots per epilogue warp: with 2, a chunk's TMA stores read one while the
  // next chunk is staged in the other (wait_group.read 1); with 1, read 0
  // (measured: 2 slots with 5 stages gains 1.5 % on the SwiGLU-backward dgrad and
  // loses 3-4 % on the fp32 wgrads, so the non-SwiGLU kernels keep 1 slot, 6 stages)
  static constexpr int NSLOT = 1;
  static constexpr int STAGES = SWI ? (BKP == 128 ? 3 : 5) : (BKP == 128 ? 3 : (BN == 512 ? 4 : ((BN == 256) ? 6 : 8)));
  static constexpr int NACC = BN == 512 ? 1 : 2;               // TMEM accumulator buffers
  static constexpr int TMEM_COLS = NACC * BN;
  static constexpr int EPI_SLOT = (SWI && BKP == 64) ? 6144 : 4096;   // staging slot of one epilogue warp
  static constexpr int EPI_BYTES = EPI_WARPS2 * NSLOT * EPI_SLOT;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

// One problem of a (grouped) CTA-pair launch: operand / output maps, epilogue,
// operand majors and tile grid.  Several independent contractions (a Linear's
// data- and weight-gradient) can share one persistent launch.
struct alignas(64) PairProblem {
  CUtensorMap tmA, tmB, tmC, tmC2;   // tmC2: SwiGLU h output
  EpiArgs ea;
  int a_mn, b_mn;
  int tiles_m, tiles_n, nk;
};
constexpr int MAX_PAIR_PROBLEMS = 2;
struct alignas(64) PairGroup {
  PairProblem prob[MAX_PAIR_PROBLEMS];
  int nprob;
  int tiles0;           // tiles of problem 0 (round-robin item t < tiles0: problem 0)
  int total_tiles;
  const int* work;      // optional static schedule: items of pair p = work[work_off[p] .. work_off[p+1])
  const int* work_off;  //   item = (problem << 24) | tile
};

// The work items of one CTA pair: round-robin over the concatenated tile lists,
// or the host-computed schedule (longest-processing-time list scheduling).
struct PairIter {
  const PairGroup& g;
  int pos, end, step;
  __device__ PairIter(const PairGroup& g_, int pair, int npairs) : g(g_) {
    if (g.work) {
      pos = g.work_off[pair];
      end = g.work_off[pair + 1];
      step = 1;
    } else {
      pos = pair;
      end = g.total_tiles;
      step = npairs;
    }
  }
  __device__ bool next(int& prob, int& tile) {
    if (pos >= end) return false;
    if (g.work) {
      const int it = g.work[pos];
      prob = it >> 24;
      tile = it & 0xFFFFFF;
    } else {
      prob = pos >= g.tiles0 ? 1 : 0;
      tile = pos - (prob ? g.tiles0 : 0);
    }
    pos += step;
    return true;
  }
};

// 32 g and 32 u values (bf16) of one row for the fused SwiGLU-backward epilogue,
// loaded ahead of the accumulator (they do not depend on the MMA result)
struct GU32 {
  uint4 g[4], u[4];
};
__device__ __forceinline__ void load_gu(const EpiArgs& a, int row, int col0, GU32& x) {
  if (row < a.M && col0 < a.N) {
    const bf16* gu = reinterpret_cast<const bf16*>(a.R) + (int64_t)row * a.ldr + col0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x.g[j] = __ldg(reinterpret_cast<const uint4*>(gu + 8 * j));
      x.u[j] = __ldg(reinterpret_cast<const uint4*>(gu + a.f + 8 * j));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) x.g[j] = x.u[j] = make_uint4(0, 0, 0, 0);
  }
}
// dg = dh u s (1 + g (1 - s)) -> w, du = dh g s -> v (in place of dh), s = sigmoid(g)
// packed fp32 pairs (sm_100 FFMA2 / FMUL2): the SwiGLU-backward epilogue is issue-bound
// (≈ 11 FP32 operations per element against the mainloop's length), so it runs its
// arithmetic two elements per instruction
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2(float lo, float hi) {
  return ((f32x2)__float_as_uint(hi) << 32) | (f32x2)__float_as_uint(lo);
}
__device__ __forceinline__ float f2lo(f32x2 x) { return __uint_as_float((uint32_t)x); }
__device__ __forceinline__ float f2hi(f32x2 x) { return __uint_as_float((uint32_t)(x >> 32)); }
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// two bf16 of one 32-bit word -> fp32 pair (element 2i in lo, 2i + 1 in hi)
__device__ __forceinline__ f32x2 bf2_to_f2(uint32_t w) {
  return f2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}
// dg = dh u s (1 + g (1 - s)) -> w, du = dh g s -> v (in place of dh), s = sigmoid(g)
__device__ __forceinline__ void dswiglu_math(float alpha, float* v, float* w, const GU32& x) {
  const f32x2 al = f2(alpha, alpha), half = f2(0.5f, 0.5f), one = f2(1.f, 1.f), mone = f2(-1.f, -1.f);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t* gw = reinterpret_cast<const uint32_t*>(&x.g[j]);
    const uint32_t* uw = reinterpret_cast<const uint32_t*>(&x.u[j]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = 8 * j + 2 * q;
      const f32x2 g = bf2_to_f2(gw[q]), u = bf2_to_f2(uw[q]);
      const f32x2 d = mul2(al, f2(v[e], v[e + 1]));
      const f32x2 gh = mul2(half, g);
      float t0, t1;
      asm("tanh.approx.f32 %0, %1;" : "=f"(t0) : "f"(f2lo(gh)));
      asm("tanh.approx.f32 %0, %1;" : "=f"(t1) : "f"(f2hi(gh)));
      const f32x2 sg = fma2(half, f2(t0, t1), half);       // sigmoid(g) = (1 + tanh(g / 2)) / 2
      const f32x2 b = fma2(g, fma2(mone, sg, one), one);   // 1 + g (1 - s)
      const f32x2 ds = mul2(d, sg);
      const f32x2 wg = mul2(mul2(ds, u), b);
      const f32x2 wu = mul2(ds, g);
      w[e] = f2lo(wg);
      w[e + 1] = f2hi(wg);
      v[e] = f2lo(wu);
      v[e + 1] = f2hi(wu);
    }
  }
}
// TMA stores of a full 32-column chunk: dg -> cols [col0, +32), du -> cols [f + col0, +32)
__device__ __forceinline__ void store_dswiglu_tma(const EpiArgs& a, const CUtensorMap* tmC, uint32_t slot, int lane,
                                                  int row0, int col0, const float* dg, const float* du) {
  stage_bf16(slot, lane, dg);
  stage_bf16(slot + 2048, lane, du);
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmC, slot, col0, row0);
    tma_store_2d(tmC, slot + 2048, a.f + col0, row0);
    bulk_commit();
  }
}

// AM / BM_: operand majors fixed at compile time (0 K-major, 1 MN-major) for
// single-problem launches, or -1: read per problem at run time (grouped launches)
// (Clusters of two pairs sharing A by TMA multicast were built, parity-tested and
// measured 8-12 % slower -- DESIGN.md §7 -- and removed.)
template <int BN, bool SWIGLU, int AM = -1, int BMJ = -1, int BKP = 64>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS2, 1)
gemm2_kernel(const __grid_constant__ PairGroup g) {
  static_assert(BKP == 64 || BN == 256, "BKP = 128: 256 x 256 pair tiles");
  constexpr int NSUB = BKP / 64;   // 64-wide swizzle sub-tiles per K block
  using C = Cfg2<BN, SWIGLU, BKP>;
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

  const uint32_t cta = cluster_rank();     // CTA within the pair
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int mbc = g.prob[0].ea.mbar_cluster;

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
    for (int p = 0; p < g.nprob; ++p) {
      tma_prefetch(&g.prob[p].tmA);
      tma_prefetch(&g.prob[p].tmB);
    }
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
      PairIter it(g, pair, npairs);
      int pi, t;
      while (it.next(pi, t)) {
        // per-tile scalars into registers: the barrier waits below invalidate L1
        // (acquire.cluster), so re-reading parameters inside the k-loop would go to L2
        const PairProblem& pr = g.prob[pi];
        const CUtensorMap* mA = &pr.tmA;
        const CUtensorMap* mB = &pr.tmB;
        const int nk = pr.nk;
        const bool amn = AM >= 0 ? AM != 0 : pr.a_mn != 0, bmn = BMJ >= 0 ? BMJ != 0 : pr.b_mn != 0;
        int mb, nb;
        tile_coords(t, pr.tiles_m, pr.tiles_n, mb, nb, pr.ea.group);
        const int m0 = mb * 2 * BM + (int)cta * BM;
        // SwiGLU pairing: CTA 0 loads gate rows [nb*BNH, +BNH), CTA 1 the matching up rows
        const int n0 = SWIGLU ? (nb * BNH + (int)cta * pr.ea.f) : (nb * BN + (int)cta * BNH);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1, mbc);
          if (cta == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const uint32_t lbar = mapa(smem_u32(&full[stage]), 0);
          uint8_t* a_dst = smA + stage * C::A_BYTES;
          uint8_t* b_dst = smB + stage * C::B_BYTES;
          const int k0 = kb * BKP;
          if (amn) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(a_dst + j * (BKP * 128), mA, lbar, m0 + 64 * j, k0);
          } else {
#pragma unroll
            for (int q = 0; q < NSUB; ++q) tma_load_2d_pair(a_dst + q * (BM * 128), mA, lbar, k0 + 64 * q, m0);
          }
          if (BN == 512) {
            // two 128-row halves, half h = global columns [nb*512 + h*256, +256) of the pair
            // (CTA c holds rows [c*128, +128) of each half), so TMEM columns map contiguously
            const int nh = nb * BN + (int)cta * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (bmn) {
#pragma unroll
                for (int j = 0; j < 2; ++j)
                  tma_load_2d_pair(b_dst + h * 16384 + j * (BK * 128), mB, lbar, nh + h * 256 + 64 * j, k0);
              } else {
                tma_load_2d_pair(b_dst + h * 16384, mB, lbar, k0, nh + h * 256);
              }
            }
          } else if (bmn) {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j) tma_load_2d_pair(b_dst + j * (BKP * 128), mB, lbar, n0 + 64 * j, k0);
          } else {
#pragma unroll
            for (int q = 0; q < NSUB; ++q) tma_load_2d_pair(b_dst + q * (BNH * 128), mB, lbar, k0 + 64 * q, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (cta == 0 && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      PairIter it(g, pair, npairs);
      int pi, t;
      for (; it.next(pi, t); ++local) {
        const PairProblem& pr = g.prob[pi];
        const bool amn = AM >= 0 ? AM != 0 : pr.a_mn != 0, bmn = BMJ >= 0 ? BMJ != 0 : pr.b_mn != 0;
        const int nk = pr.nk;
        const uint32_t idesc = make_idesc(BN == 512 ? 256 : BN, amn, bmn, 2 * BM);
        const int acc = C::NACC == 2 ? (local & 1) : 0;
        const uint32_t acc_phase = C::NACC == 2 ? ((local >> 1) & 1) : (local & 1);
        mbar_wait(&tempty[acc], acc_phase ^ 1, mbc);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase, mbc);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smA + stage * C::A_BYTES);
          const uint32_t b_base = smem_u32(smB + stage * C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKP / 16; ++kk) {
            const int q = kk / 4, w = kk % 4;   // K-major: sub-tile q, 16-deep step w within it
            uint64_t ad = amn ? make_desc(a_base + kk * 2048, BKP * 128, 1024)
                              : make_desc(a_base + q * (BM * 128) + w * 32, 16, 1024);
#pragma unroll
            for (int h = 0; h < (BN == 512 ? 2 : 1); ++h) {   // BN = 512: two N = 256 MMAs sharing A
              const uint32_t bh = b_base + h * 16384;
              uint64_t bd = bmn ? make_desc(bh + kk * 2048, BKP * 128, 1024)
                                : make_desc(bh + q * (BNH * 128) + w * 32, 16, 1024);
              umma_f16_pair(tmem_d + h * 256, ad, bd, idesc, (kb != 0 || kk != 0) ? 1u : 0u);
            }
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
    const uint32_t slot0 = smem_u32(smE) + (uint32_t)((warp - 2) * C::NSLOT * C::EPI_SLOT);
    uint32_t slot = slot0;
    int eiter = 0;
    const uint32_t leader_tempty0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t leader_tempty1 = mapa(smem_u32(&tempty[1]), 0);
    int local = 0;
    PairIter it(g, pair, npairs);
    int pi, t;
    for (; it.next(pi, t); ++local) {
      const PairProblem& pr = g.prob[pi];
      const EpiArgs ea = pr.ea;   // into registers (see the producer)
      const CUtensorMap* mC = &pr.tmC;
      const CUtensorMap* mC2 = &pr.tmC2;
      int mb, nb;
      tile_coords(t, pr.tiles_m, pr.tiles_n, mb, nb, ea.group);
      const int acc = C::NACC == 2 ? (local & 1) : 0;
      const uint32_t acc_phase = C::NACC == 2 ? ((local >> 1) & 1) : (local & 1);
      const int row0 = mb * 2 * BM + (int)cta * BM + quad * 32;
      const int row = row0 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      if (SWIGLU) {
        mbar_wait(&tfull[acc], acc_phase, mbc);
        tc_fence_after();
        constexpr int W = BNH / 2;   // features per warp
#pragma unroll 1
        for (int c = half * W; c < (half + 1) * W; c += 32) {
          float vg[32], vu[32];
          tmem_ld32(taddr + c, vg);
          tmem_ld32(taddr + BNH + c, vu);
          if (ea.tma) {
            if (nb * BNH + c < ea.f) {
              if (eiter >= 1) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
              }
              if (C::EPI_SLOT == 4096) epi_swiglu_tma_4k(ea, mC, mC2, slot, lane, row0, nb * BNH + c, vg, vu);
              else epi_swiglu_tma(ea, mC, mC2, slot, lane, row0, nb * BNH + c, vg, vu);
              ++eiter;
            }
          } else if (row < ea.M) {
            epilogue_swiglu(ea, row, nb * BNH + c, vg, vu);
          }
        }
      } else {
        constexpr int W = BN / 2;    // columns per warp
        const int cbeg = half * W, cend = (half + 1) * W;
        const bool dsw = ea.epi == BM_EPI_DSWIGLU && ea.tma;
        // the epilogue's global reads (g / u of the SwiGLU backward) for the whole tile into
        // L2 while the MMAs still run: the chunk loads then hit L2 instead of waiting on HBM
        // with one chunk in flight per warp
        // (SwiGLU backward only: standalone +1.5 % at C2, +5 % at C4 shapes; the residual
        // add's R lost 2 %; profiles/r02/bn512/pf_gemm.log)
        if (ea.prefetch && dsw && row < ea.M) {
          const int col0 = nb * BN + cbeg;
          const char* r = reinterpret_cast<const char*>(ea.R) + ((int64_t)row * ea.ldr + col0) * 2;
          const int nbytes = min(cend - cbeg, ea.N - col0) * 2;
          for (int o = 0; o < nbytes; o += 128) {
            prefetch_l2(r + o);
            prefetch_l2(r + (int64_t)ea.f * 2 + o);
          }
        }
        GU32 gu;
        if (dsw) load_gu(ea, row, nb * BN + cbeg, gu);   // ahead of the accumulator
        mbar_wait(&tfull[acc], acc_phase, mbc);
        tc_fence_after();
#pragma unroll 1
        for (int c = cbeg; c < cend; c += 32) {
          float v[32];
          tmem_ld32(taddr + c, v);
          if (dsw) {
            float w[32];
            dswiglu_math(ea.alpha, v, w, gu);
            if (c + 32 < cend) load_gu(ea, row, nb * BN + c + 32, gu);   // next chunk, in flight during the stores
            if (nb * BN + c < ea.N) {
              slot = slot0 + (uint32_t)((eiter % C::NSLOT) * C::EPI_SLOT);
              if (eiter >= C::NSLOT) {
                if (lane == 0) {
                  if (C::NSLOT == 2) bulk_wait_read1();
                  else bulk_wait_read0();
                }
                __syncwarp();
              }
              store_dswiglu_tma(ea, mC, slot, lane, row0, nb * BN + c, w, v);
              ++eiter;
            }
          } else if (ea.tma) {
            if (nb * BN + c < ea.N) {
              slot = slot0 + (uint32_t)((eiter % C::NSLOT) * C::EPI_SLOT);
              if (eiter >= C::NSLOT) {
                if (lane == 0) {
                  if (C::NSLOT == 2) bulk_wait_read1();
                  else bulk_wait_read0();
                }
                __syncwarp();
              }
              epi_chunk_tma(ea, mC, slot, lane, row0, nb * BN + c, v);
              ++eiter;
            }
          } else if (row < ea.M) {
            epilogue_row(ea, row, nb * BN + c, v);
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


template <int BN, bool SWIGLU = false, int AM = -1, int BMJ = -1, int BKP = 64>
static bm_status launch2(const PairGroup& g, int tiles, cudaStream_t st) {
  using C = Cfg2<BN, SWIGLU, BKP>;
  static bool attr_set = false;
  if (!attr_set) {
    BM_CUDA_TRY(cudaFuncSetAttribute(gemm2_kernel<BN, SWIGLU, AM, BMJ, BKP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const int pairs = gemm_sm_budget() / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  BM_CUDA_TRY(launch_k(gemm2_kernel<BN, SWIGLU, AM, BMJ, BKP>, dim3(grid), dim3(NUM_THREADS2), C::SMEM, st, g));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
// single-problem launch with the operand majors as template constants
template <int BN, int BKP = 64>
static bm_status launch2_static(const PairGroup& g, int tiles, cudaStream_t st) {
  const int a = g.prob[0].a_mn, b = g.prob[0].b_mn;
  if (!a && !b) return launch2<BN, false, 0, 0, BKP>(g, tiles, st);
  if (!a && b) return launch2<BN, false, 0, 1, BKP>(g, tiles, st);
  if (a && b) return launch2<BN, false, 1, 1, BKP>(g, tiles, st);
  return launch2<BN, false, 1, 0, BKP>(g, tiles, st);
}

}  // namespace tc

static int g_raster_group = [] {   // BM_GEMM_GROUP: measurement override of the pair raster
  const char* e = getenv("BM_GEMM_GROUP");
  const int v = e ? atoi(e) : 8;
  return v >= 1 ? v : 8;
}();
static int g_epi_prefetch = [] {
  const char* e = getenv("BM_EPI_PREFETCH");
  return e && e[0] == '0' ? 0 : 1;
}();
// barrier polls at CTA scope by default (as CUTLASS's waits: every barrier a thread
// polls lives in its own CTA and guards async-proxy data -- TMA bytes, tcgen05 commits,
// TMEM ordered by tcgen05 fences -- so no cluster-scope acquire is needed, and each
// .acquire.cluster poll costs an L1 invalidation, CCTL.IVALL: 27 % of the warp samples
// of the SwiGLU-backward GEMM, profiles/r02/bn512/ncu_dswiglu_stalls.txt).  Standalone
// +0.5..+2.5 %, C2 step 52.40 -> 52.55 samples/s (mbar_*.log); BM_MBAR_SCOPE=cluster
// restores the .acquire.cluster form
static int g_mbar_cluster = [] {
  const char* e = getenv("BM_MBAR_SCOPE");
  return e && std::string(e) == "cluster" ? 1 : 0;
}();
// 0 = auto (CTA pairs for large contractions), 1 = force 1-CTA, 2 = force CTA pairs
static int g_gemm_mode = [] {
  const char* e = getenv("BM_GEMM_MODE");
  return e ? (e[0] == '1' ? 1 : (e[0] == '2' ? 2 : 0)) : 0;
}();
int gemm_mode() { return g_gemm_mode; }
// split-K of the small 1-CTA GEMMs only when a tile has at least this many k-blocks
// (BM_SPLITK_MIN_NK; 0 disables split-K; each split launch adds a reduce kernel)
static int g_splitk_min_nk = [] {
  const char* e = getenv("BM_SPLITK_MIN_NK");
  return e ? atoi(e) : 4;
}();
// BM_GEMM_GROUP_INTERLEAVE=0: keep each pair's grouped tiles problem by problem (measurement)
static int g_group_interleave = [] {
  const char* e = getenv("BM_GEMM_GROUP_INTERLEAVE");
  return e && e[0] == '0' ? 0 : 1;
}();
// BM_GEMM_GROUP_RR=1: grouped pair launches deal tiles round-robin instead of the LPT schedule (measurement)
static int g_group_rr = [] {
  const char* e = getenv("BM_GEMM_GROUP_RR");
  return e && e[0] == '1' ? 1 : 0;
}();
void set_gemm_mode(int m) { g_gemm_mode = m; }
// 128-deep K blocks for 256 x 256 pair tiles (default; BM_GEMM_BK128=0: 64-deep, 6 stages).
// Twice the MMAs per full-barrier round trip at the same bytes per FLOP: standalone
// +3..+14 % on the 256-wide C2 / C4 contractions (C4 head wgrad -8 %), C2 step 50.5 ->
// 51.6 samples/s, in-step GEMM 0.84 -> 0.86 (profiles/r02/bn512/bk128_*.log).  The
// SwiGLU-forward kernel keeps 64-deep blocks (its 48 KB epilogue staging leaves room
// for two 64 KB stages only, so it stages [g | u] and h through 4 KB, see below).
static int g_bk128 = [] {
  const char* e = getenv("BM_GEMM_BK128");
  return e ? atoi(e) : 1;
}();
void set_gemm_bk128(int m) { g_bk128 = m; }
// 256 x 512 pair tiles (BM_GEMM_BN512: 0 = never, 1 = every pair GEMM with N >= 512,
// default 2 = by a wave-quantised cost model).  A 256 x 512 tile moves a quarter less
// L2 -> SMEM data per FLOP (its k-blocks run ~1.1x faster than two 256 x 256 ones) but
// has one TMEM accumulator, so its epilogue (~4096 clocks; fp32 reduce-add 6144) is not
// overlapped, and it halves the tile count (coarser last wave).  Model, per pair:
//   t256 = ceil(T256 / pairs) * nk * 512,  t512 = ceil(T512 / pairs) * (nk * 1024 / 1.1 + E)
// 512 when t512 < 0.98 t256.  It reproduces the measured gains within ~4 points
// (profiles/r02/bn512/bn512_knob.log: C2 down fwd +5 %, gate_up dgrad +10.5 %, head
// dgrad +16 %, 8192^3 +6 %; C4 down fwd -9 % and gate_up dgrad -7 % from the last
// wave).  The SwiGLU-backward epilogue (gu loads, two outputs) loses 20-27 % with the
// un-overlapped epilogue and always takes 256 x 256.
static int g_bn512 = [] {
  const char* e = getenv("BM_GEMM_BN512");
  return e ? atoi(e) : 2;
}();
void set_gemm_bn512(int m) { g_bn512 = m; }


// ... for the SwiGLU-forward kernel too (default; three 64 KB stages, 4 KB epilogue
// staging per warp, [g | u] and h stored one after the other): standalone +5.9 % (C2) /
// +5.6 % (C4), C2 step 51.1 -> 51.6 samples/s (profiles/r02/bn512/swbk_*.log);
// BM_GEMM_SWIGLU_BK128=0: 64-deep blocks, five stages, 6 KB staging
static int g_swiglu_bk128 = [] {
  const char* e = getenv("BM_GEMM_SWIGLU_BK128");
  return e ? atoi(e) : 1;
}();
void set_gemm_swiglu_bk128(int m) { g_swiglu_bk128 = m; }
static bool use_bn512(int M, int N, int K, int c_dtype, int epi) {
  if (N < 512 || g_bn512 == 0 || epi == BM_EPI_SWIGLU) return false;
  if (g_bn512 == 1) return true;   // forced (tests, A/B), the SwiGLU-backward epilogue included
  if (epi == BM_EPI_DSWIGLU) return false;
  const int64_t pairs = std::max(1, gemm_sm_budget() / 2);
  const int64_t tm = (M + 255) / 256, nk = (K + 63) / 64;
  const int64_t t256 = tm * ((N + 255) / 256), t512 = tm * ((N + 511) / 512);
  const double c256 = (double)((t256 + pairs - 1) / pairs) * nk * 512.0;
  // per-FLOP k-block speed of 256 x 512 over 256 x 256 tiles: 1.1 against 64-deep K blocks,
  // 1.03 against the 128-deep ones (most of the gain was the halved barrier round trips
  // per FLOP, which 128-deep blocks also get; profiles/r02/bn512/bn512_v2_knob.log)
  const double g = g_bk128 ? 1.03 : 1.1;
  const double c512 = (double)((t512 + pairs - 1) / pairs) * (nk * 1024.0 / g + (c_dtype == BM_F32 ? 6144.0 : 4096.0));
  return c512 < 0.98 * c256;
}

// fills the epilogue arguments and the output map of one contraction
static bm_status prepare_out(int M, int N, int K, void* Cp, int64_t ldc, int c_dtype, int epi, const void* R,
                             int64_t ldr, float alpha, int f, tc::EpiArgs* ea, CUtensorMap* mc) {
  using namespace tc;
  *ea = EpiArgs{M, N, K, Cp, ldc, c_dtype == BM_F32 ? 1 : 0, epi, R, ldr, alpha, f, 0, 1, 1 << 30, 0, 8, 1};
  ea->group = g_raster_group;
  ea->mbar_cluster = g_mbar_cluster;
  ea->prefetch = g_epi_prefetch;
  std::memset(mc, 0, sizeof(*mc));
  const int ces = c_dtype == BM_F32 ? 4 : 2;
  if (epi == BM_EPI_DSWIGLU) {
    BM_CHECK_ARG(c_dtype == BM_BF16 && N == f && f % 32 == 0 && ldc >= 2 * f && ldr >= 2 * f &&
                     (reinterpret_cast<uintptr_t>(R) & 15) == 0 && ldr % 8 == 0,
                 "DSWIGLU epilogue: bf16, N = f, f % 32 == 0, C/R are [M, 2f], 16-byte aligned");
    if (tma_out_ok(Cp, ldc, 2)) {
      BM_TRY(make_map_k(Cp, 2 * (uint64_t)f, M, ldc, 32, 1, mc));
      ea->tma = 1;
    }
  } else if (tma_out_ok(Cp, ldc, ces)) {
    BM_TRY(make_map_k(Cp, (uint64_t)N, M, ldc, 32, c_dtype == BM_F32 ? 2 : 1, mc));
    ea->tma = 1;
  }
  return BM_OK;
}

// one CTA-pair problem (256 x BN2 tiles) of a (grouped) pair launch
static bm_status pair_problem(int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B,
                              int64_t ldb, int b_major, void* Cp, int64_t ldc, int c_dtype, int epi, const void* R,
                              int64_t ldr, float alpha, int f, int BN2, tc::PairProblem* pr) {
  using namespace tc;
  std::memset(pr, 0, sizeof(*pr));
  BM_TRY(prepare_out(M, N, K, Cp, ldc, c_dtype, epi, R, ldr, alpha, f, &pr->ea, &pr->tmC));
  pr->tmC2 = pr->tmC;
  if (a_major == 0) BM_TRY(make_map(A, K, M, lda, BM, &pr->tmA));
  else BM_TRY(make_map(A, M, K, lda, BK, &pr->tmA));
  if (b_major == 0) BM_TRY(make_map(B, K, N, ldb, BN2 == 512 ? 128 : BN2 / 2, &pr->tmB));
  else BM_TRY(make_map(B, N, K, ldb, BK, &pr->tmB));
  pr->a_mn = a_major != 0;
  pr->b_mn = b_major != 0;
  pr->tiles_m = ceil_div(M, 2 * BM);
  pr->tiles_n = ceil_div(N, BN2);
  pr->nk = ceil_div(K, BK);
  return BM_OK;
}

bm_status gemm_bf16_tc(int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B, int64_t ldb,
                       int b_major, void* Cp, int64_t ldc, int c_dtype, int epi, const void* R, int64_t ldr,
                       float alpha, cudaStream_t st, int f, void* ws, int64_t ws_bytes) {
  using namespace tc;
  BM_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0, "lda/ldb must be multiples of 8 (16-byte TMA strides)");
  BM_CHECK_ARG((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
               "A/B must be 16-byte aligned");
  const bool amn = a_major != 0, bmn = b_major != 0;
  if (epi == BM_EPI_SWIGLU) {
    // gate/up GEMM with fused SwiGLU: always CTA pairs, BN = 256 (128 gate + 128 up features)
    BM_CHECK_ARG(b_major == 0 && c_dtype == BM_BF16 && N == 2 * f && f % 128 == 0, "SWIGLU epilogue: K-major B, bf16, N = 2f, f % 128 == 0");
    PairGroup g;
    std::memset(&g, 0, sizeof(g));
    PairProblem& pr = g.prob[0];
    pr.ea = EpiArgs{M, N, K, Cp, ldc, 0, epi, R, ldr, alpha, f, 0, 1, 1 << 30, 0, g_raster_group, g_mbar_cluster};
    const bool bk128 = g_bk128 != 0 && g_swiglu_bk128 != 0;
    if (a_major == 0) BM_TRY(make_map(A, K, M, lda, BM, &pr.tmA));
    else BM_TRY(make_map(A, M, K, lda, bk128 ? 128 : BK, &pr.tmA));
    BM_TRY(make_map(B, K, N, ldb, 128, &pr.tmB));
    if (tma_out_ok(Cp, ldc, 2) && tma_out_ok(R, ldr, 2)) {
      BM_TRY(make_map_k(Cp, 2 * (uint64_t)f, M, ldc, 32, 1, &pr.tmC));
      BM_TRY(make_map_k(R, (uint64_t)f, M, ldr, 32, 1, &pr.tmC2));
      pr.ea.tma = 1;
    }
    pr.a_mn = a_major != 0;
    pr.b_mn = 0;
    pr.tiles_m = ceil_div(M, 2 * BM);
    pr.tiles_n = ceil_div(f, 128);
    pr.nk = ceil_div(K, bk128 ? 128 : BK);
    g.nprob = 1;
    g.tiles0 = g.total_tiles = pr.tiles_m * pr.tiles_n;
    if (bk128) {
      if (a_major == 0) return launch2<256, true, 0, 0, 128>(g, g.total_tiles, st);
      return launch2<256, true, 1, 0, 128>(g, g.total_tiles, st);
    }
    if (a_major == 0) return launch2<256, true, 0, 0>(g, g.total_tiles, st);
    return launch2<256, true, 1, 0>(g, g.total_tiles, st);
  }
  // CTA pairs for the large contractions (enough 256-row tiles to fill the
  // machine), 1-CTA tiles otherwise
  const int mode = gemm_mode();
  const int64_t pair_tiles = (int64_t)ceil_div(M, 2 * BM) * ceil_div(N, 256);
  const bool pair = mode == 2 || (mode == 0 && M >= 256 && N >= 256 && K >= 256 && pair_tiles >= num_sms() / 2);
  if (pair) {
    const int BN2 = (N >= 256) ? (use_bn512(M, N, K, c_dtype, epi) ? 512 : 256) : 128;
    PairGroup g;
    std::memset(&g, 0, sizeof(g));
    BM_TRY(pair_problem(M, N, K, A, lda, a_major, B, ldb, b_major, Cp, ldc, c_dtype, epi, R, ldr, alpha, f, BN2,
                        &g.prob[0]));
    g.nprob = 1;
    const bool bk128 = g_bk128 != 0 && BN2 == 256;
    if (bk128) {   // MN-major operands as 64 x 128 boxes; 128-deep K blocks
      PairProblem& pr = g.prob[0];
      if (a_major != 0) BM_TRY(make_map(A, M, K, lda, 128, &pr.tmA));
      if (b_major != 0) BM_TRY(make_map(B, N, K, ldb, 128, &pr.tmB));
      pr.nk = ceil_div(K, 128);
    }
    g.tiles0 = g.total_tiles = g.prob[0].tiles_m * g.prob[0].tiles_n;
    if (bk128) return launch2_static<256, 128>(g, g.total_tiles, st);
    if (BN2 == 512) return launch2_static<512>(g, g.total_tiles, st);
    if (BN2 == 256) return launch2_static<256>(g, g.total_tiles, st);
    return launch2_static<128>(g, g.total_tiles, st);
  }
  EpiArgs ea;
  CUtensorMap ma, mb, mc;
  BM_TRY(prepare_out(M, N, K, Cp, ldc, c_dtype, epi, R, ldr, alpha, f, &ea, &mc));
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
  if (g_splitk_min_nk > 0 && ws && ws_bytes > 0 && tiles < num_sms() / 2 && nk >= g_splitk_min_nk && N % 4 == 0 &&
      (epi == BM_EPI_STORE || epi == BM_EPI_ADD || epi == BM_EPI_ACCUM)) {
    int splits = std::min(8, std::min(num_sms() / tiles, nk / 2));
    const int mpad = tm * BM;
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

// ---------------------------------------------------------------- grouped pair launches
// Static schedule of several independent contractions on the CTA pairs:
// longest-processing-time list scheduling with a tile's cost = its k-blocks
// (every 256 x 256 tile of a problem costs the same), problems with longer
// tiles first, each problem's tiles in raster order.  Cached per shape set.
struct WorkKey {
  std::vector<int> k;
  bool operator==(const WorkKey& o) const { return k == o.k; }
};
struct WorkKeyHash {
  size_t operator()(const WorkKey& w) const {
    size_t h = 0;
    for (int v : w.k) h = h * 1000003u ^ (size_t)v;
    return h;
  }
};
static std::mutex g_work_mu;
static std::unordered_map<WorkKey, std::pair<int*, int*>, WorkKeyHash> g_work;

static bm_status pair_schedule(const tc::PairGroup& g, int pairs, const int** work, const int** work_off) {
  WorkKey key;
  key.k.push_back(pairs);
  for (int p = 0; p < g.nprob; ++p) {
    key.k.push_back(g.prob[p].tiles_m);
    key.k.push_back(g.prob[p].tiles_n);
    key.k.push_back(g.prob[p].nk);
  }
  std::lock_guard<std::mutex> lk(g_work_mu);
  auto it = g_work.find(key);
  if (it == g_work.end()) {
    std::vector<int> order(g.nprob);
    for (int p = 0; p < g.nprob; ++p) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return g.prob[a].nk > g.prob[b].nk; });
    std::vector<std::vector<int>> per(pairs);
    std::vector<int64_t> load(pairs, 0);
    for (int p : order) {
      const int tiles = g.prob[p].tiles_m * g.prob[p].tiles_n;
      for (int t = 0; t < tiles; ++t) {
        int best = 0;
        for (int q = 1; q < pairs; ++q)
          if (load[q] < load[best]) best = q;   // ties: lowest pair (deterministic)
        per[best].push_back((p << 24) | t);
        load[best] += g.prob[p].nk;
      }
    }
    // alternate the problems within each pair's list (same set of tiles, same load):
    // a tile with a heavy epilogue (fused SwiGLU backward, fp32 reduce-add) then runs
    // its epilogue under the next tile's mainloop of the other problem
    if (g_group_interleave && g.nprob == 2) {
      for (auto& lst : per) {
        std::vector<int> a, b, m;
        for (int it : lst) ((it >> 24) == order[0] ? a : b).push_back(it);
        size_t i = 0, j = 0;
        while (i < a.size() || j < b.size()) {
          if (i < a.size()) m.push_back(a[i++]);
          if (j < b.size()) m.push_back(b[j++]);
        }
        lst.swap(m);
      }
    }
    std::vector<int> flat, off(pairs + 1, 0);
    for (int q = 0; q < pairs; ++q) {
      off[q] = (int)flat.size();
      flat.insert(flat.end(), per[q].begin(), per[q].end());
    }
    off[pairs] = (int)flat.size();
    int *dw = nullptr, *doff = nullptr;
    BM_CUDA_TRY(cudaMalloc(&dw, std::max<size_t>(flat.size(), 1) * sizeof(int)));
    BM_CUDA_TRY(cudaMalloc(&doff, off.size() * sizeof(int)));
    BM_CUDA_TRY(cudaMemcpy(dw, flat.data(), flat.size() * sizeof(int), cudaMemcpyHostToDevice));
    BM_CUDA_TRY(cudaMemcpy(doff, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice));
    it = g_work.emplace(key, std::make_pair(dw, doff)).first;
  }
  *work = it->second.first;
  *work_off = it->second.second;
  return BM_OK;
}

bm_status gemm_bf16_tc_group(const GemmSpec* sp, int n, cudaStream_t st) {
  using namespace tc;
  BM_CHECK_ARG(n >= 1 && n <= MAX_PAIR_PROBLEMS, "group of 1..2 contractions");
  const int mode = gemm_mode();
  bool ok = mode != 1;
  int64_t ptiles = 0;
  for (int i = 0; i < n; ++i) {
    const GemmSpec& s = sp[i];
    BM_CHECK_ARG(s.M > 0 && s.N > 0 && s.K > 0, "grouped GEMM: empty contraction");
    ok = ok && s.epi != BM_EPI_SWIGLU && s.N >= 256 && s.M >= 256 && s.K >= 64 && s.lda % 8 == 0 &&
         s.ldb % 8 == 0 && (reinterpret_cast<uintptr_t>(s.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(s.B) & 15) == 0;
    ptiles += (int64_t)ceil_div(s.M, 2 * BM) * ceil_div(s.N, 256);
  }
  // auto mode: like single launches, CTA pairs only when the group fills the machine
  ok = ok && (mode == 2 || ptiles >= num_sms() / 2);
  if (!ok || n == 1) {   // not pair-shaped: one launch per contraction
    for (int i = 0; i < n; ++i) {
      const GemmSpec& s = sp[i];
      BM_TRY(gemm_bf16_tc(s.M, s.N, s.K, s.A, s.lda, s.a_major, s.B, s.ldb, s.b_major, s.C, s.ldc, s.c_dtype, s.epi,
                          s.R, s.ldr, s.alpha, st, s.f, s.ws, s.ws_bytes));
    }
    return BM_OK;
  }
  PairGroup g;
  std::memset(&g, 0, sizeof(g));
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    const GemmSpec& s = sp[i];
    BM_TRY(pair_problem(s.M, s.N, s.K, s.A, s.lda, s.a_major, s.B, s.ldb, s.b_major, s.C, s.ldc, s.c_dtype, s.epi, s.R,
                        s.ldr, s.alpha, s.f, 256, &g.prob[i]));
    tiles += g.prob[i].tiles_m * g.prob[i].tiles_n;
  }
  g.nprob = n;
  g.tiles0 = g.prob[0].tiles_m * g.prob[0].tiles_n;
  g.total_tiles = tiles;
  const int pairs = std::min(gemm_sm_budget() / 2, tiles);
  if (!g_group_rr) BM_TRY(pair_schedule(g, pairs, &g.work, &g.work_off));
  bool b_all_mn = true;
  for (int i = 0; i < n; ++i) b_all_mn = b_all_mn && g.prob[i].b_mn;
  if (b_all_mn) return launch2<256, false, -1, 1>(g, tiles, st);   // a Linear's dgrad + wgrad: B MN-major
  return launch2<256>(g, tiles, st);
}

// every tcgen05 GEMM instantiation the dispatcher can launch (bm::preload_kernels)
template <int BN>
static void preload_bn(std::vector<const void*>& v) {
  using namespace tc;
  for (const void* f : {(const void*)gemm_kernel<BN, false, false>, (const void*)gemm_kernel<BN, false, true>,
                        (const void*)gemm_kernel<BN, true, true>, (const void*)gemm_kernel<BN, true, false>})
    v.push_back(f);
}
void preload_tc(std::vector<const void*>& v) {
  preload_bn<64>(v);
  preload_bn<128>(v);
  preload_bn<256>(v);
  v.push_back((const void*)tc::gemm2_kernel<256, false>);   // grouped (run-time majors)
  v.push_back((const void*)tc::gemm2_kernel<256, false, -1, 1>);
  for (const void* f : {(const void*)tc::gemm2_kernel<128, false, 0, 0>, (const void*)tc::gemm2_kernel<128, false, 0, 1>,
                        (const void*)tc::gemm2_kernel<128, false, 1, 1>, (const void*)tc::gemm2_kernel<128, false, 1, 0>,
                        (const void*)tc::gemm2_kernel<256, false, 0, 0>, (const void*)tc::gemm2_kernel<256, false, 0, 1>,
                        (const void*)tc::gemm2_kernel<256, false, 1, 1>, (const void*)tc::gemm2_kernel<256, false, 1, 0>,
                        (const void*)tc::gemm2_kernel<256, true, 0, 0>, (const void*)tc::gemm2_kernel<256, true, 1, 0>})
    v.push_back(f);
  v.push_back((const void*)tc::splitk_reduce_kernel);
}

}  // namespace bm
