// elementwise.cu -- HBM-bound kernels of the step: RMSNorm fwd/bwd, SwiGLU,
// GELU, embed_preprocess fwd/bwd, cross-entropy and MSE losses.
//
// All kernels move 16-byte vectors (8 bf16 / 4 fp32 per access), keep
// reductions in fp32 with fixed (deterministic) shuffle/shared-memory trees,
// and accumulate weight-like gradients (RMSNorm gains, text table) through
// deterministic two-pass reductions so reruns are bitwise identical.
#include <algorithm>
#include <cfloat>

#include <vector>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include "common.cuh"

namespace bm {

// ------------------------------------------------------------------ vectors
template <typename T> struct V16;
template <> struct V16<bf16> {
  static constexpr int N = 8;
  uint4 raw;
  __device__ __forceinline__ float get(int i) const { return __bfloat162float(reinterpret_cast<const bf16*>(&raw)[i]); }
  __device__ __forceinline__ void set(int i, float v) { reinterpret_cast<bf16*>(&raw)[i] = __float2bfloat16_rn(v); }
};
template <> struct V16<float> {
  static constexpr int N = 4;
  float4 raw;
  __device__ __forceinline__ float get(int i) const { return reinterpret_cast<const float*>(&raw)[i]; }
  __device__ __forceinline__ void set(int i, float v) { reinterpret_cast<float*>(&raw)[i] = v; }
};
template <typename T> __device__ __forceinline__ V16<T> vload(const T* p) {
  V16<T> v;
  v.raw = *reinterpret_cast<const decltype(v.raw)*>(p);
  return v;
}
template <typename T> __device__ __forceinline__ void vstore(T* p, const V16<T>& v) {
  *reinterpret_cast<decltype(v.raw)*>(p) = v.raw;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// deterministic block reduction (blockDim.x multiple of 32, <= 1024)
__device__ __forceinline__ float block_sum(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x / 32;
  float r = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.f;
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}
__device__ __forceinline__ float block_max(float v, float* sh) {
  v = warp_max(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x / 32;
  float r = (threadIdx.x < nw) ? sh[threadIdx.x] : -FLT_MAX;
  if (w == 0) r = warp_max(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

constexpr float RMS_EPS = 1e-5f;
constexpr float GELU_C = 0.7978845608028654f;  // sqrt(2/pi)

__device__ __forceinline__ float gelu_f(float a) {
  return 0.5f * a * (1.f + tanhf(GELU_C * (a + 0.044715f * a * a * a)));
}
__device__ __forceinline__ float gelu_grad(float a) {
  const float t = tanhf(GELU_C * (a + 0.044715f * a * a * a));
  return 0.5f * (1.f + t) + 0.5f * a * (1.f - t * t) * GELU_C * (1.f + 3.f * 0.044715f * a * a);
}

// ------------------------------------------------------------------ RMSNorm
// BM_RMS_WIDE=0: the per-warp-row fused backward for wide rows too (measurement only;
// a register-resident forward was measured and dropped: 16.3 vs 12.4 us at 4096 x 2048)
static int g_rms_wide = [] {   // BM_RMS_WIDE=0: the per-warp-row fused kernel for wide rows too (measurement)
  const char* e = getenv("BM_RMS_WIDE");
  return e && e[0] == '0' ? 0 : 1;
}();
template <typename T>
__global__ void rmsnorm_fwd_kernel(int rows, int cols, const T* __restrict__ x, const T* __restrict__ g,
                                   T* __restrict__ y, float* __restrict__ rstd) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const T* xr = x + (int64_t)row * cols;
  float ss = 0.f;
  for (int c = lane * N; c < cols; c += 32 * N) {
    V16<T> v = vload(xr + c);
#pragma unroll
    for (int i = 0; i < N; ++i) { float f = v.get(i); ss += f * f; }
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / cols + RMS_EPS);
  if (lane == 0) rstd[row] = r;
  T* yr = y + (int64_t)row * cols;
  for (int c = lane * N; c < cols; c += 32 * N) {
    V16<T> v = vload(xr + c), gv = vload(g + c), o;
#pragma unroll
    for (int i = 0; i < N; ++i) o.set(i, v.get(i) * r * gv.get(i));
    vstore(yr + c, o);
  }
}

template <typename T>
__global__ void rmsnorm_bwd_kernel(int rows, int cols, const T* __restrict__ dy, const T* __restrict__ x,
                                   const T* __restrict__ g, const float* __restrict__ rstd, const T* dres, T* dx) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const int64_t off = (int64_t)row * cols;
  const float r = rstd[row];
  float dot = 0.f;
  for (int c = lane * N; c < cols; c += 32 * N) {
    V16<T> dv = vload(dy + off + c), xv = vload(x + off + c), gv = vload(g + c);
#pragma unroll
    for (int i = 0; i < N; ++i) dot += dv.get(i) * gv.get(i) * xv.get(i) * r;
  }
  dot = warp_sum(dot) / cols;
  for (int c = lane * N; c < cols; c += 32 * N) {
    V16<T> dv = vload(dy + off + c), xv = vload(x + off + c), gv = vload(g + c), o;
    V16<T> rv;
    if (dres) rv = vload(dres + off + c);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      float v = r * (dv.get(i) * gv.get(i) - xv.get(i) * r * dot);
      if (dres) v += rv.get(i);
      o.set(i, v);
    }
    vstore(dx + off + c, o);
  }
}

// partial[chunk][col] = sum_{rows in chunk} dy * x * rstd
template <typename T>
__global__ void rmsnorm_dg_partial_kernel(int rows, int cols, int nchunk, const T* __restrict__ dy,
                                          const T* __restrict__ x, const float* __restrict__ rstd,
                                          float* __restrict__ partial) {
  pdl_enter();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (col >= cols) return;
  const int per = (rows + nchunk - 1) / nchunk;
  const int r0 = chunk * per, r1 = min(rows, r0 + per);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r) {
    const int64_t o = (int64_t)r * cols + col;
    acc += to_f(dy[o]) * to_f(x[o]) * rstd[r];
  }
  partial[(int64_t)chunk * cols + col] = acc;
}
// out[col] += sum_k partial[k][col]; 32 columns per block, 8 row groups per
// column summed in a fixed order (deterministic)
__global__ void __launch_bounds__(256)
colsum2_accum_kernel(int nchunk, int cols, const float* __restrict__ partial, float* __restrict__ out) {
  pdl_enter();
  __shared__ float sh[8][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int g = threadIdx.x >> 5;
  float acc = 0.f;
  if (c < cols)
    for (int k = g; k < nchunk; k += 8) acc += partial[(int64_t)k * cols + c];
  sh[g][threadIdx.x & 31] = acc;
  __syncthreads();
  if (g == 0 && c < cols) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[q][threadIdx.x];
    out[c] += s;
  }
}
// 32 columns x 32 row groups per block (1024 threads): the wide backward's many
// partial rows summed with 4x the memory parallelism of colsum2; fixed order
__global__ void __launch_bounds__(1024)
colsum32_accum_kernel(int nchunk, int cols, const float* __restrict__ partial, float* __restrict__ out) {
  pdl_enter();
  __shared__ float sh[32][33];
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  const int g = threadIdx.x >> 5;
  float acc = 0.f;
  if (c < cols)
    for (int k = g; k < nchunk; k += 32) acc += partial[(int64_t)k * cols + c];
  sh[g][threadIdx.x & 31] = acc;
  __syncthreads();
  if (g == 0 && c < cols) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 32; ++q) s += sh[q][threadIdx.x];
    out[c] += s;
  }
}
__global__ void colsum_accum_kernel(int nchunk, int cols, const float* __restrict__ partial, float* __restrict__ out) {
  pdl_enter();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= cols) return;
  float acc = 0.f;
  for (int k = 0; k < nchunk; ++k) acc += partial[(int64_t)k * cols + col];
  out[col] += acc;
}

static int dg_chunks(int rows) { return rows < 64 ? (rows > 0 ? rows : 1) : 64; }

// ------------------------------------------------------------------ SwiGLU / GELU
template <typename T>
__global__ void __launch_bounds__(256)
swiglu_fwd_kernel(int rows, int f, const T* __restrict__ gu, T* __restrict__ h) {
  pdl_enter();
  // 2-D grid: blockIdx.y = row, x over 16-byte vectors of the row (no division)
  constexpr int N = V16<T>::N;
  const int64_t i = blockIdx.y;
  const T* row = gu + i * 2 * (int64_t)f;
  T* out = h + i * (int64_t)f;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) * N; j < f; j += gridDim.x * blockDim.x * N) {
    V16<T> gv = vload(row + j), uv = vload(row + f + j), o;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float gg = gv.get(q);
      o.set(q, gg * uv.get(q) / (1.f + __expf(-gg)));
    }
    vstore(out + j, o);
  }
}
template <typename T>
__global__ void __launch_bounds__(256)
swiglu_bwd_kernel(int rows, int f, const T* __restrict__ dh, const T* __restrict__ gu, T* __restrict__ dgu) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int64_t i = blockIdx.y;
  const T* row = gu + i * 2 * (int64_t)f;
  const T* drow = dh + i * (int64_t)f;
  T* orow = dgu + i * 2 * (int64_t)f;
  for (int j = (blockIdx.x * blockDim.x + threadIdx.x) * N; j < f; j += gridDim.x * blockDim.x * N) {
    V16<T> gv = vload(row + j), uv = vload(row + f + j), dv = vload(drow + j), og, ou;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float gg = gv.get(q), uu = uv.get(q), d = dv.get(q);
      const float s = 1.f / (1.f + __expf(-gg));
      og.set(q, d * uu * s * (1.f + gg * (1.f - s)));
      ou.set(q, d * gg * s);
    }
    vstore(orow + j, og);
    vstore(orow + f + j, ou);
  }
}
template <typename T>
__global__ void gelu_fwd_kernel(int64_t n, const T* __restrict__ a, T* __restrict__ z) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int64_t nv = n / N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    V16<T> av = vload(a + v * N), o;
#pragma unroll
    for (int q = 0; q < N; ++q) o.set(q, gelu_f(av.get(q)));
    vstore(z + v * N, o);
  }
  for (int64_t e = nv * N + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    z[e] = from_f<T>(gelu_f(to_f(a[e])));
}
template <typename T>
__global__ void gelu_bwd_kernel(int64_t n, const T* __restrict__ dz, const T* __restrict__ a, T* __restrict__ da) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int64_t nv = n / N;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
    V16<T> av = vload(a + v * N), dv = vload(dz + v * N), o;
#pragma unroll
    for (int q = 0; q < N; ++q) o.set(q, dv.get(q) * gelu_grad(av.get(q)));
    vstore(da + v * N, o);
  }
  for (int64_t e = nv * N + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    da[e] = from_f<T>(to_f(dz[e]) * gelu_grad(to_f(a[e])));
}
template <typename T>
__global__ void add_kernel(int64_t n, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    o[e] = from_f<T>(to_f(a[e]) + to_f(b[e]));
}
template <typename S, typename D>
__global__ void cast_kernel(int64_t n, const S* __restrict__ a, D* __restrict__ o) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    o[e] = from_f<D>(to_f(a[e]));
}

// ------------------------------------------------------------------ copies / fills on SMs
// Every byte move inside the step runs as a kernel on the issuing stream's own
// compute channel: a copy-engine copy can queue in a copy channel behind another
// stream's copy that is parked on a peer credit wait ("copy
// channels"), turning an acyclic schedule into a device deadlock.  dst may be a
// peer GPU's IPC-mapped buffer (NVLink stores).
__global__ void copy16_kernel(int64_t n16, const uint4* __restrict__ src, uint4* __restrict__ dst) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; e + 3 * stride < n16; e += 4 * stride) {
    const uint4 a = __ldg(src + e), b = __ldg(src + e + stride), c = __ldg(src + e + 2 * stride),
                d = __ldg(src + e + 3 * stride);
    dst[e] = a;
    dst[e + stride] = b;
    dst[e + 2 * stride] = c;
    dst[e + 3 * stride] = d;
  }
  for (; e < n16; e += stride) dst[e] = __ldg(src + e);
}
__global__ void copy1_kernel(int64_t n, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}
__global__ void zero16_kernel(int64_t n16, uint4* __restrict__ dst) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n16; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = make_uint4(0, 0, 0, 0);
}
__global__ void zero1_kernel(int64_t n, uint8_t* __restrict__ dst) {
  pdl_enter();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) dst[e] = 0;
}

// ------------------------------------------------------------------ flag wait on an SM
// One thread polls a 32-bit flag (written by a peer GPU over NVLink or by another
// stream) until it reaches v (unsigned, >=).  Used instead of a stream wait-value
// operation when BM_WAIT=spin.  Traps after 60 s so a lost message becomes an error.
__global__ void spin_wait_kernel(const uint32_t* flag, uint32_t v) {
  if (threadIdx.x != 0) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    if ((int32_t)(x - v) >= 0) break;
    __nanosleep(200);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) {
      printf("bigmac: spin wait timeout flag=%p have=%u want=%u\n", flag, x, v);
      __trap();
    }
  }
}

// ------------------------------------------------------------------ embed_preprocess
template <typename T>
__global__ void embed_fwd_kernel(int S, int d, int n_mod, const int32_t* __restrict__ ids, const T* __restrict__ table,
                                 const T* __restrict__ emb, T* __restrict__ X) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  const int warps = blockDim.x / 32;
  const int row = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= S) return;
  const T* src = (row < n_mod) ? emb + (int64_t)row * d : table + (int64_t)ids[row] * d;
  T* dst = X + (int64_t)row * d;
  for (int c = lane * N; c < d; c += 32 * N) vstore(dst + c, vload(src + c));
}

// Sort (id, position) for positions [n_mod, S) in one CTA (bitonic, smem),
// emit positions in sorted order and segment starts.
// scratch layout (int32): [0] nseg | order[S] | seg_start[S+1]
__global__ void embed_sort_kernel(int S, int n_mod, const int32_t* __restrict__ ids, int32_t* __restrict__ scratch) {
  pdl_enter();
  extern __shared__ unsigned long long keys[];
  __shared__ int wsum[32];
  const int cnt = S - n_mod;
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int i = threadIdx.x; i < n2; i += blockDim.x)
    keys[i] = (i < cnt) ? (((unsigned long long)(unsigned)ids[n_mod + i] << 32) | (unsigned)(n_mod + i)) : ~0ull;
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const bool up = (i & k) == 0;
          unsigned long long a = keys[i], b = keys[ixj];
          if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
  int32_t* order = scratch + 1;
  int32_t* seg = scratch + 1 + S;
  // heads + exclusive scan (each thread owns a contiguous span)
  const int per = (cnt + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per, b1 = min(cnt, b0 + per);
  int local = 0;
  for (int i = b0; i < b1; ++i) {
    order[i] = (int32_t)(keys[i] & 0xffffffffu);
    if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ++local;
  }
  // block exclusive scan of `local`
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  int v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    int s = (lane < (int)(blockDim.x / 32)) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += t;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  int base = v - local + (w > 0 ? wsum[w - 1] : 0);
  for (int i = b0; i < b1; ++i) {
    if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) seg[base++] = i;
  }
  if (threadIdx.x == blockDim.x - 1) {
    const int total = v + (w > 0 ? wsum[w - 1] : 0);
    scratch[0] = total;
    seg[total] = cnt;
  }
}

// Same output as embed_sort_kernel (order = text positions sorted by id, equal
// ids in position order; seg = segment starts; scratch[0] = #segments) with a
// stable CUB block radix sort of (id, position) pairs: ITEMS * 1024 >= S - n_mod.
template <int ITEMS>
__global__ void __launch_bounds__(1024) embed_radix_sort_kernel(int S, int n_mod, const int32_t* __restrict__ ids,
                                                                int32_t* __restrict__ scratch) {
  pdl_enter();
  using Sort = cub::BlockRadixSort<unsigned, 1024, ITEMS, int>;
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ unsigned last_key[1024];
  const int cnt = S - n_mod;
  unsigned key[ITEMS];
  int pos[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {   // blocked arrangement: thread t holds items [t ITEMS, (t+1) ITEMS)
    const int i = threadIdx.x * ITEMS + k;
    key[k] = i < cnt ? (unsigned)ids[n_mod + i] : 0xffffffffu;
    pos[k] = n_mod + i;
  }
  Sort(tmp.sort).Sort(key, pos);   // stable: equal ids stay in position order
  last_key[threadIdx.x] = key[ITEMS - 1];
  __syncthreads();
  int32_t* order = scratch + 1;
  int32_t* seg = scratch + 1 + S;
  bool head[ITEMS];
  int local = 0;
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int i = threadIdx.x * ITEMS + k;
    const unsigned prev = k > 0 ? key[k - 1] : (threadIdx.x > 0 ? last_key[threadIdx.x - 1] : 0u);
    head[k] = i < cnt && (i == 0 || key[k] != prev);
    local += head[k] ? 1 : 0;
    if (i < cnt) order[i] = pos[k];
  }
  int base = 0, total = 0;
  __syncthreads();   // tmp.sort -> tmp.scan
  Scan(tmp.scan).ExclusiveSum(local, base, total);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k)
    if (head[k]) seg[base++] = threadIdx.x * ITEMS + k;
  if (threadIdx.x == 0) {
    scratch[0] = total;
    seg[total] = cnt;
  }
}

template <typename T>
__global__ void embed_segsum_kernel(int S, int d, const int32_t* __restrict__ ids, const T* __restrict__ dX,
                                    const int32_t* __restrict__ scratch, float* __restrict__ dT) {
  pdl_enter();
  const int nseg = scratch[0];
  const int32_t* order = scratch + 1;
  const int32_t* seg = scratch + 1 + S;
  const int warps = blockDim.x / 32;
  const int lane = threadIdx.x % 32;
  constexpr int N = V16<T>::N;   // d % N == 0 (embed_bwd checks)
  for (int s = blockIdx.x * warps + threadIdx.x / 32; s < nseg; s += gridDim.x * warps) {
    const int i0 = seg[s], i1 = seg[s + 1];
    const int id = ids[order[i0]];
    float* dst = dT + (int64_t)id * d;
    for (int c = lane * N; c < d; c += 32 * N) {
      float acc[N];
#pragma unroll
      for (int j = 0; j < N; ++j) acc[j] = 0.f;
      for (int i = i0; i < i1; ++i) {   // segment members in position order (deterministic)
        const V16<T> v = vload(dX + (int64_t)order[i] * d + c);
#pragma unroll
        for (int j = 0; j < N; ++j) acc[j] += v.get(j);
      }
#pragma unroll
      for (int j = 0; j < N; j += 4) {
        float4 o = *reinterpret_cast<float4*>(dst + c + j);
        o.x += acc[j]; o.y += acc[j + 1]; o.z += acc[j + 2]; o.w += acc[j + 3];
        *reinterpret_cast<float4*>(dst + c + j) = o;
      }
    }
  }
}

// ------------------------------------------------------------------ losses
template <typename T>
__global__ void ce_row_kernel(int V, T* __restrict__ logits, const int32_t* __restrict__ labels, float scale_grad,
                              float* __restrict__ row_loss) {
  pdl_enter();
  __shared__ float sh[32];
  const int row = blockIdx.x;
  T* z = logits + (int64_t)row * V;
  float mx = -FLT_MAX;
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, to_f(z[j]));
  mx = block_max(mx, sh);
  float s = 0.f;
  for (int j = threadIdx.x; j < V; j += blockDim.x) s += __expf(to_f(z[j]) - mx);
  s = block_sum(s, sh);
  const float lse = mx + __logf(s);
  const int lab = labels[row];
  const float zl = to_f(z[lab]);
  __syncthreads();
  if (threadIdx.x == 0) row_loss[row] = lse - zl;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const float p = __expf(to_f(z[j]) - lse);
    z[j] = from_f<T>((p - (j == lab ? 1.f : 0.f)) * scale_grad);
  }
}
__global__ void sum_scale_kernel(int n, const float* __restrict__ v, float scale, int accumulate, float* out) {
  pdl_enter();
  __shared__ float sh[32];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[0] = (accumulate ? out[0] : 0.f) + s * scale;
}
template <typename T>
__global__ void mse_kernel(int64_t n, const T* __restrict__ out, const T* __restrict__ t, float inv_denom,
                           float scale_grad, float scale_loss, float* loss, T* __restrict__ dout) {
  pdl_enter();
  __shared__ float sh[32];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const float df = to_f(out[i]) - to_f(t[i]);
    s += df * df;
    dout[i] = from_f<T>(2.f * df * inv_denom * scale_grad);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) loss[0] += s * inv_denom * scale_loss;
}


// Fused RMSNorm backward: one pass computes dx (+ dres) for RB rows per block
// and this block's deterministic partial of dg (per-warp register partials,
// reduced across the block's warps in a fixed order through shared memory).
// partial[block][col]; a second tiny kernel sums the blocks in order.
template <typename T, int CH>
__global__ void __launch_bounds__(256)
rmsnorm_bwd_fused_kernel(int rows, int cols, int rows_per_block, const T* __restrict__ dy, const T* __restrict__ x,
                         const T* __restrict__ g, const float* __restrict__ rstd, const T* dres, T* dx,
                         float* __restrict__ partial) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  extern __shared__ float sdg[];  // [8 warps][cols]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float acc[CH][N];
#pragma unroll
  for (int k = 0; k < CH; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) acc[k][i] = 0.f;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  for (int row = r0 + warp; row < r1; row += 8) {
    const int64_t off = (int64_t)row * cols;
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int c = (k * 32 + lane) * N;
      if (c < cols) {
        V16<T> dv = vload(dy + off + c), xv = vload(x + off + c), gv = vload(g + c);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const float xh = xv.get(i) * r;
          dot += dv.get(i) * gv.get(i) * xh;
          acc[k][i] += dv.get(i) * xh;
        }
      }
    }
    dot = warp_sum(dot) / cols;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int c = (k * 32 + lane) * N;
      if (c < cols) {
        V16<T> dv = vload(dy + off + c), xv = vload(x + off + c), gv = vload(g + c), o, rv;
        if (dres) rv = vload(dres + off + c);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float v = r * (dv.get(i) * gv.get(i) - xv.get(i) * r * dot);
          if (dres) v += rv.get(i);
          o.set(i, v);
        }
        vstore(dx + off + c, o);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * 32 + lane) * N;
    if (c < cols) {
#pragma unroll
      for (int i = 0; i < N; ++i) sdg[warp * cols + c + i] = acc[k][i];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += sdg[w * cols + c];
    partial[(int64_t)blockIdx.x * cols + c] = s;
  }
}

// Cross-entropy, vectorized: pass 1 online max/sum over 16-byte vectors, pass 2
// writes dz = (softmax - onehot) * scale in place.
template <typename T>
__global__ void __launch_bounds__(256)
ce_row_vec_kernel(int V, T* __restrict__ logits, const int32_t* __restrict__ labels, float scale_grad,
                  float* __restrict__ row_loss) {
  pdl_enter();
  constexpr int N = V16<T>::N;
  __shared__ float shm[32], shs[32];
  const int row = blockIdx.x;
  T* z = logits + (int64_t)row * V;
  const int nv = V / N;
  float m = -FLT_MAX, sum = 0.f;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    V16<T> a = vload(z + (int64_t)v * N);
    float vm = a.get(0);
#pragma unroll
    for (int i = 1; i < N; ++i) vm = fmaxf(vm, a.get(i));
    if (vm > m) { sum *= __expf(m - vm); m = vm; }
#pragma unroll
    for (int i = 0; i < N; ++i) sum += __expf(a.get(i) - m);
  }
  for (int j = nv * N + threadIdx.x; j < V; j += blockDim.x) {
    const float a = to_f(z[j]);
    if (a > m) { sum *= __expf(m - a); m = a; }
    sum += __expf(a - m);
  }
  // combine (m, sum) across the block deterministically
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
    const float mm = fmaxf(m, m2);
    sum = sum * __expf(m - mm) + s2 * __expf(m2 - mm);
    m = mm;
  }
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) { shm[w] = m; shs[w] = sum; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x / 32;
    m = l < nw ? shm[l] : -FLT_MAX;
    sum = l < nw ? shs[l] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float mm = fmaxf(m, m2);
      sum = (sum == 0.f ? 0.f : sum * __expf(m - mm)) + (s2 == 0.f ? 0.f : s2 * __expf(m2 - mm));
      m = mm;
    }
    if (l == 0) { shm[0] = m; shs[0] = sum; }
  }
  __syncthreads();
  const float lse = shm[0] + __logf(shs[0]);
  const int lab = labels[row];
  if (threadIdx.x == 0) row_loss[row] = lse - to_f(z[lab]);
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    V16<T> a = vload(z + (int64_t)v * N), o;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int j = v * N + i;
      o.set(i, (__expf(a.get(i) - lse) - (j == lab ? 1.f : 0.f)) * scale_grad);
    }
    vstore(z + (int64_t)v * N, o);
  }
  for (int j = nv * N + threadIdx.x; j < V; j += blockDim.x)
    z[j] = from_f<T>((__expf(to_f(z[j]) - lse) - (j == lab ? 1.f : 0.f)) * scale_grad);
}

// ================================================================== launchers
static int ew_grid(int64_t work_items) {
  int64_t g = (work_items + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

template <typename T>
bm_status rmsnorm_fwd(int rows, int cols, const T* x, const T* g, T* y, float* rstd, cudaStream_t st) {
  if (rows <= 0) return BM_OK;
  BM_CHECK_ARG(cols % V16<T>::N == 0, "rmsnorm cols must be a multiple of the vector width");
  BM_CUDA_TRY(launch_k(rmsnorm_fwd_kernel<T>, dim3(ceil_div(rows, 8)), dim3(256), 0, st, rows, cols, x, g, y, rstd));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
// rows per block of the fused backward: ~2 waves of blocks over the 148 SMs
// Wide rows (cols >= 256 vectors): the block's 256 threads split a row's columns
// (CH 16-byte vectors per thread), so each thread keeps only CH x N gain-gradient
// accumulators and a group of 4 rows' dy / x in registers between the two passes
// (no re-read): pass 1 forms the 4 row dot products (warp sums -> smem -> fixed-order
// block sums), pass 2 writes dx.  High occupancy instead of 64 accumulators per lane.
template <typename T, int CH>
__global__ void __launch_bounds__(256)
rmsnorm_bwd_wide_kernel(int rows, int cols, int rows_per_block, const T* __restrict__ dy, const T* __restrict__ x,
                        const T* __restrict__ g, const float* __restrict__ rstd, const T* dres, T* dx,
                        float* __restrict__ partial) {
  pdl_enter();
  constexpr int N = V16<T>::N, RG = 4;
  __shared__ float red[2][RG][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float acc[CH][N];
  V16<T> gv[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * 256 + threadIdx.x) * N;
    if (c < cols) gv[k] = vload(g + c);
#pragma unroll
    for (int i = 0; i < N; ++i) acc[k][i] = 0.f;
  }
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  int par = 0;
  for (int rb = r0; rb < r1; rb += RG, par ^= 1) {
    V16<T> dv[RG][CH], xv[RG][CH];
    float rs[RG];
#pragma unroll
    for (int j = 0; j < RG; ++j) {
      const int row = rb + j;
      rs[j] = row < r1 ? rstd[row] : 0.f;
      float dot = 0.f;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = (k * 256 + threadIdx.x) * N;
        if (row < r1 && c < cols) {
          const int64_t off = (int64_t)row * cols + c;
          dv[j][k] = vload(dy + off);
          xv[j][k] = vload(x + off);
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const float xh = xv[j][k].get(i) * rs[j];
            dot += dv[j][k].get(i) * gv[k].get(i) * xh;
            acc[k][i] += dv[j][k].get(i) * xh;
          }
        }
      }
      dot = warp_sum(dot);
      if (lane == 0) red[par][j][warp] = dot;
    }
    __syncthreads();   // red[par] complete; red[par ^ 1] is free for the next group
#pragma unroll
    for (int j = 0; j < RG; ++j) {
      const int row = rb + j;
      if (row >= r1) continue;
      float dot = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) dot += red[par][j][w];   // fixed order: deterministic
      dot /= cols;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = (k * 256 + threadIdx.x) * N;
        if (c < cols) {
          const int64_t off = (int64_t)row * cols + c;
          V16<T> o, rv;
          if (dres) rv = vload(dres + off);
#pragma unroll
          for (int i = 0; i < N; ++i) {
            float v = rs[j] * (dv[j][k].get(i) * gv[k].get(i) - xv[j][k].get(i) * rs[j] * dot);
            if (dres) v += rv.get(i);
            o.set(i, v);
          }
          vstore(dx + off, o);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const int c = (k * 256 + threadIdx.x) * N;
    if (c < cols) {
#pragma unroll
      for (int i = 0; i < N; ++i) partial[(int64_t)blockIdx.x * cols + c + i] = acc[k][i];
    }
  }
}
template <typename T, int CH>
static bm_status launch_rms_bwd_wide(int rows, int cols, const T* dy, const T* x, const T* g, const float* rstd,
                                     const T* dres, T* dx, float* dg, float* partial, cudaStream_t st) {
  // ~4 blocks per SM, rows per block a multiple of the 4-row group
  int rb = ceil_div(rows, 4 * num_sms());
  rb = rb < 4 ? 4 : (rb + 3) / 4 * 4;
  const int nb = ceil_div(rows, rb);
  BM_CUDA_TRY(launch_k(rmsnorm_bwd_wide_kernel<T, CH>, dim3(nb), dim3(256), 0, st, rows, cols, rb, dy, x, g, rstd, dres,
                       dx, partial));
  BM_CUDA_TRY(launch_k(colsum32_accum_kernel, dim3(ceil_div(cols, 32)), dim3(1024), 0, st, nb, cols, partial, dg));
  count_launch(2);
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}


static int rb_rows(int rows) {
  int rb = ceil_div(rows, 2 * num_sms());
  rb = (rb + 7) / 8 * 8;
  return rb < 8 ? 8 : rb;
}
template <typename T, int CH>
static bm_status launch_rms_bwd_fused(int rows, int cols, const T* dy, const T* x, const T* g, const float* rstd,
                                      const T* dres, T* dx, float* dg, float* partial, cudaStream_t st) {
  const int rb = rb_rows(rows);
  const int nb = ceil_div(rows, rb);
  const int smem = 8 * cols * 4;
  static bool attr = false;
  if (!attr) {
    BM_CUDA_TRY(cudaFuncSetAttribute(rmsnorm_bwd_fused_kernel<T, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  BM_CUDA_TRY(launch_k(rmsnorm_bwd_fused_kernel<T, CH>, dim3(nb), dim3(256), smem, st, rows, cols, rb, dy, x, g, rstd, dres, dx, partial));
  BM_CUDA_TRY(launch_k(colsum2_accum_kernel, dim3(ceil_div(cols, 32)), dim3(256), 0, st, nb, cols, partial, dg));
  count_launch(2);
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

template <typename T>
bm_status rmsnorm_bwd(int rows, int cols, const T* dy, const T* x, const T* g, const float* rstd, const T* dres,
                      T* dx, float* dg, float* partial, cudaStream_t st) {
  if (rows <= 0) return BM_OK;
  constexpr int N = V16<T>::N;
  BM_CHECK_ARG(cols % N == 0, "rmsnorm cols must be a multiple of the vector width");
  const int ch = ceil_div(cols, 32 * N);  // vector chunks per lane
  const int wide = ceil_div(cols, 256 * N);   // vector chunks per thread of a 256-thread row split
  if (g_rms_wide && cols >= 256 * N && wide <= 4 && cols % (256 * N) == 0) {
    if (wide == 1) return launch_rms_bwd_wide<T, 1>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    if (wide == 2) return launch_rms_bwd_wide<T, 2>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    return launch_rms_bwd_wide<T, 4>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
  }
  if (ch <= 16 && cols <= 6144) {
    if (ch <= 1) return launch_rms_bwd_fused<T, 1>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    if (ch <= 2) return launch_rms_bwd_fused<T, 2>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    if (ch <= 4) return launch_rms_bwd_fused<T, 4>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    if (ch <= 8) return launch_rms_bwd_fused<T, 8>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
    return launch_rms_bwd_fused<T, 16>(rows, cols, dy, x, g, rstd, dres, dx, dg, partial, st);
  }
  // wide rows: separate gain-gradient pass
  const int nch = dg_chunks(rows);
  BM_CUDA_TRY(launch_k(rmsnorm_dg_partial_kernel<T>, dim3(dim3(ceil_div(cols, 256), nch)), dim3(256), 0, st, rows, cols, nch, dy, x, rstd, partial));
  BM_CUDA_TRY(launch_k(colsum_accum_kernel, dim3(ceil_div(cols, 256)), dim3(256), 0, st, nch, cols, partial, dg));
  BM_CUDA_TRY(launch_k(rmsnorm_bwd_kernel<T>, dim3(ceil_div(rows, 8)), dim3(256), 0, st, rows, cols, dy, x, g, rstd, dres, dx));
  count_launch(3);
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status swiglu_fwd(int rows, int f, const T* gu, T* h, cudaStream_t st) {
  const int64_t total = (int64_t)rows * f;
  if (total == 0) return BM_OK;
  BM_CHECK_ARG(f % V16<T>::N == 0, "swiglu f must be a multiple of the vector width");
  const int vx = ceil_div(f / V16<T>::N, 256);
  BM_CUDA_TRY(launch_k(swiglu_fwd_kernel<T>, dim3(dim3(vx > 4 ? 4 : vx, rows)), dim3(256), 0, st, rows, f, gu, h));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status swiglu_bwd(int rows, int f, const T* dh, const T* gu, T* dgu, cudaStream_t st) {
  const int64_t total = (int64_t)rows * f;
  if (total == 0) return BM_OK;
  BM_CHECK_ARG(f % V16<T>::N == 0, "swiglu f must be a multiple of the vector width");
  const int vx = ceil_div(f / V16<T>::N, 256);
  BM_CUDA_TRY(launch_k(swiglu_bwd_kernel<T>, dim3(dim3(vx > 4 ? 4 : vx, rows)), dim3(256), 0, st, rows, f, dh, gu, dgu));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status gelu_fwd(int64_t n, const T* a, T* z, cudaStream_t st) {
  if (n == 0) return BM_OK;
  BM_CUDA_TRY(launch_k(gelu_fwd_kernel<T>, dim3(ew_grid(n / V16<T>::N + 1)), dim3(256), 0, st, n, a, z));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status gelu_bwd(int64_t n, const T* dz, const T* a, T* da, cudaStream_t st) {
  if (n == 0) return BM_OK;
  BM_CUDA_TRY(launch_k(gelu_bwd_kernel<T>, dim3(ew_grid(n / V16<T>::N + 1)), dim3(256), 0, st, n, dz, a, da));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status embed_fwd(int S, int d, int n_mod, const int32_t* ids, const T* table, const T* emb, T* X, cudaStream_t st) {
  BM_CHECK_ARG(d % V16<T>::N == 0, "embed width must be a multiple of the vector width");
  BM_CUDA_TRY(launch_k(embed_fwd_kernel<T>, dim3(ceil_div(S, 8)), dim3(256), 0, st, S, d, n_mod, ids, table, emb, X));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
int64_t embed_bwd_scratch_bytes(int S) { return (int64_t)(2 * S + 2) * 4; }

template <typename T>
bm_status embed_bwd(int S, int d, int n_mod, const int32_t* ids, const T* dX, float* dT, void* scratch, cudaStream_t st) {
  const int cnt = S - n_mod;
  if (cnt <= 0) return BM_OK;
  BM_CHECK_ARG(S <= 16384, "embed_bwd supports S <= 16384");
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  const int smem = n2 * 8;
  static bool attr = false;
  if (!attr) {
    BM_CUDA_TRY(cudaFuncSetAttribute(embed_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 8));
    attr = true;
  }
  BM_CHECK_ARG(d % V16<T>::N == 0, "embed width must be a multiple of the vector width");
  int32_t* sc = reinterpret_cast<int32_t*>(scratch);
  if (cnt <= 4096) BM_CUDA_TRY(launch_k(embed_radix_sort_kernel<4>, dim3(1), dim3(1024), 0, st, S, n_mod, ids, sc));
  else if (cnt <= 8192) BM_CUDA_TRY(launch_k(embed_radix_sort_kernel<8>, dim3(1), dim3(1024), 0, st, S, n_mod, ids, sc));
  else BM_CUDA_TRY(launch_k(embed_sort_kernel, dim3(1), dim3(1024), smem, st, S, n_mod, ids, sc));
  BM_CUDA_TRY(launch_k(embed_segsum_kernel<T>, dim3(ceil_div(cnt, 8)), dim3(256), 0, st, S, d, ids, dX, reinterpret_cast<int32_t*>(scratch), dT));
  count_launch(2);
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status ce_fwd_bwd(int n, int V, T* logits, const int32_t* labels, float scale_grad, float* loss_out,
                     float scale_loss, int accumulate, float* scratch, cudaStream_t st) {
  if (n <= 0) return BM_OK;
  if (V % V16<T>::N == 0)
    BM_CUDA_TRY(launch_k(ce_row_vec_kernel<T>, dim3(n), dim3(256), 0, st, V, logits, labels, scale_grad, scratch));
  else
    BM_CUDA_TRY(launch_k(ce_row_kernel<T>, dim3(n), dim3(256), 0, st, V, logits, labels, scale_grad, scratch));
  BM_CUDA_TRY(launch_k(sum_scale_kernel, dim3(1), dim3(1024), 0, st, n, scratch, scale_loss / n, accumulate, loss_out));
  count_launch(2);
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status mse_fwd_bwd(int n, int dt, const T* out, const T* t, float denom, float scale_grad, float scale_loss,
                      float* loss_out, T* dout, cudaStream_t st) {
  if (n <= 0) return BM_OK;
  BM_CUDA_TRY(launch_k(mse_kernel<T>, dim3(1), dim3(1024), 0, st, (int64_t)n * dt, out, t, 1.f / denom, scale_grad, scale_loss, loss_out, dout));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
template <typename T>
bm_status add(int64_t n, const T* a, const T* b, T* o, cudaStream_t st) {
  if (n == 0) return BM_OK;
  BM_CUDA_TRY(launch_k(add_kernel<T>, dim3(ew_grid(n)), dim3(256), 0, st, n, a, b, o));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
bm_status copy_bytes(void* dst, const void* src, int64_t bytes, int max_ctas, cudaStream_t st) {
  if (bytes <= 0) return BM_OK;
  const bool v = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | (uintptr_t)bytes) & 15) == 0;
  const int64_t items = v ? bytes / 16 : bytes;
  int grid = ew_grid(v ? items / 4 + 1 : items);
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  if (v) BM_CUDA_TRY(launch_k(copy16_kernel, dim3(grid), dim3(256), 0, st, items, (const uint4*)src, (uint4*)dst));
  else BM_CUDA_TRY(launch_k(copy1_kernel, dim3(grid), dim3(256), 0, st, items, (const uint8_t*)src, (uint8_t*)dst));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
bm_status spin_wait(const uint32_t* flag, uint32_t v, cudaStream_t st) {
  spin_wait_kernel<<<1, 32, 0, st>>>(flag, v);
  if (g_launch_hook) g_launch_hook(st, (const void*)spin_wait_kernel);
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
bm_status zero_bytes(void* dst, int64_t bytes, cudaStream_t st) {
  if (bytes <= 0) return BM_OK;
  const bool v = ((reinterpret_cast<uintptr_t>(dst) | (uintptr_t)bytes) & 15) == 0;
  const int64_t items = v ? bytes / 16 : bytes;
  if (v) BM_CUDA_TRY(launch_k(zero16_kernel, dim3(ew_grid(items)), dim3(256), 0, st, items, (uint4*)dst));
  else BM_CUDA_TRY(launch_k(zero1_kernel, dim3(ew_grid(items)), dim3(256), 0, st, items, (uint8_t*)dst));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}
bm_status cast(int sd, int dd, int64_t n, const void* s, void* d, cudaStream_t st) {
  if (n == 0) return BM_OK;
  if (sd == BM_F32 && dd == BM_BF16) BM_CUDA_TRY(launch_k(cast_kernel<float, bf16>, dim3(ew_grid(n)), dim3(256), 0, st, n, (const float*)s, (bf16*)d));
  else if (sd == BM_BF16 && dd == BM_F32) BM_CUDA_TRY(launch_k(cast_kernel<bf16, float>, dim3(ew_grid(n)), dim3(256), 0, st, n, (const bf16*)s, (float*)d));
  else if (sd == BM_F32 && dd == BM_F32) BM_CUDA_TRY(launch_k(cast_kernel<float, float>, dim3(ew_grid(n)), dim3(256), 0, st, n, (const float*)s, (float*)d));
  else BM_CUDA_TRY(launch_k(cast_kernel<bf16, bf16>, dim3(ew_grid(n)), dim3(256), 0, st, n, (const bf16*)s, (bf16*)d));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

#define BM_INST(T)                                                                                              \
  template bm_status rmsnorm_fwd<T>(int, int, const T*, const T*, T*, float*, cudaStream_t);                    \
  template bm_status rmsnorm_bwd<T>(int, int, const T*, const T*, const T*, const float*, const T*, T*, float*, \
                                    float*, cudaStream_t);                                                      \
  template bm_status swiglu_fwd<T>(int, int, const T*, T*, cudaStream_t);                                       \
  template bm_status swiglu_bwd<T>(int, int, const T*, const T*, T*, cudaStream_t);                             \
  template bm_status gelu_fwd<T>(int64_t, const T*, T*, cudaStream_t);                                          \
  template bm_status gelu_bwd<T>(int64_t, const T*, const T*, T*, cudaStream_t);                                \
  template bm_status embed_fwd<T>(int, int, int, const int32_t*, const T*, const T*, T*, cudaStream_t);         \
  template bm_status embed_bwd<T>(int, int, int, const int32_t*, const T*, float*, void*, cudaStream_t);        \
  template bm_status ce_fwd_bwd<T>(int, int, T*, const int32_t*, float, float*, float, int, float*, cudaStream_t); \
  template bm_status mse_fwd_bwd<T>(int, int, const T*, const T*, float, float, float, float*, T*, cudaStream_t); \
  template bm_status add<T>(int64_t, const T*, const T*, T*, cudaStream_t);
BM_INST(bf16)
BM_INST(float)

int64_t rmsnorm_bwd_scratch_floats(int rows, int cols) {
  const int64_t fused = (int64_t)std::max(ceil_div(rows, 8), ceil_div(rows, 4)) * cols;
  const int64_t split = (int64_t)dg_chunks(rows) * cols;
  return fused > split ? fused : split;
}

// step loss L = (1/M) sum_m (CE_m + MSE_m) from loss[0:2M] into loss[2M]
bm_status loss_finalize(int M, float* loss, float scale, cudaStream_t st) {
  BM_CUDA_TRY(launch_k(sum_scale_kernel, dim3(1), dim3(1024), 0, st, 2 * M, loss, scale, 0, loss + 2 * M));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

// every kernel of this file (bm::preload_kernels)
template <typename T>
static void preload_t(std::vector<const void*>& v) {
  for (const void* f : {(const void*)rmsnorm_fwd_kernel<T>, (const void*)rmsnorm_bwd_kernel<T>,
                        (const void*)rmsnorm_dg_partial_kernel<T>, (const void*)rmsnorm_bwd_fused_kernel<T, 1>,
                        (const void*)rmsnorm_bwd_fused_kernel<T, 2>, (const void*)rmsnorm_bwd_fused_kernel<T, 4>,
                        (const void*)rmsnorm_bwd_fused_kernel<T, 8>, (const void*)rmsnorm_bwd_fused_kernel<T, 16>,
                        (const void*)rmsnorm_bwd_wide_kernel<T, 1>, (const void*)rmsnorm_bwd_wide_kernel<T, 2>,
                        (const void*)rmsnorm_bwd_wide_kernel<T, 4>,
                        (const void*)swiglu_fwd_kernel<T>, (const void*)swiglu_bwd_kernel<T>,
                        (const void*)gelu_fwd_kernel<T>, (const void*)gelu_bwd_kernel<T>, (const void*)add_kernel<T>,
                        (const void*)embed_fwd_kernel<T>, (const void*)embed_segsum_kernel<T>,
                        (const void*)ce_row_kernel<T>, (const void*)ce_row_vec_kernel<T>, (const void*)mse_kernel<T>})
    v.push_back(f);
}
void preload_elementwise(std::vector<const void*>& v) {
  preload_t<bf16>(v);
  preload_t<float>(v);
  for (const void* f : {(const void*)cast_kernel<float, bf16>, (const void*)cast_kernel<bf16, float>,
                        (const void*)cast_kernel<float, float>, (const void*)cast_kernel<bf16, bf16>,
                        (const void*)colsum_accum_kernel, (const void*)colsum2_accum_kernel,
                        (const void*)colsum32_accum_kernel, (const void*)copy16_kernel,
                        (const void*)copy1_kernel, (const void*)zero16_kernel, (const void*)zero1_kernel,
                        (const void*)spin_wait_kernel, (const void*)embed_sort_kernel, (const void*)sum_scale_kernel,
                        (const void*)embed_radix_sort_kernel<4>, (const void*)embed_radix_sort_kernel<8>})
    v.push_back(f);
}

}  // namespace bm
