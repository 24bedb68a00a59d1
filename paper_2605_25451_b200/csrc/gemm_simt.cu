// gemm_simt.cu -- exact fp32 GEMM (FFMA, no TF32) for the fp32 parity mode.
//
// The 1e-4 fp32 tolerance (BASELINE.json north_star) rules out TF32 tensor
// cores (rel. err ~1e-3); C1-sized parity runs use this 64x64-tile FFMA
// kernel with the same operand conventions and epilogues as gemm_tc.cu.
#include <vector>
#include "common.cuh"

namespace bm {

namespace {
constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256)
gemm_f32_kernel(int M, int N, int K, const float* __restrict__ A, int64_t lda, int a_mn,
                const float* __restrict__ B, int64_t ldb, int b_mn, float* __restrict__ C, int64_t ldc,
                int epi, const float* __restrict__ R, int64_t ldr, float alpha) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  pdl_enter();
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      int mm, kk;
      if (!a_mn) { mm = i / TK; kk = i % TK; } else { kk = i / TM; mm = i % TM; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) v = a_mn ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < TN * TK; i += 256) {
      int nn, kk;
      if (!b_mn) { nn = i / TK; kk = i % TK; } else { kk = i / TN; nn = i % TN; }
      const int gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < K) v = b_mn ? B[(int64_t)gk * ldb + gn] : B[(int64_t)gn * ldb + gk];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float* c = C + (int64_t)gm * ldc + gn;
      const float v = alpha * acc[i][j];
      if (epi == BM_EPI_ACCUM) *c += v;
      else if (epi == BM_EPI_ADD) *c = v + R[(int64_t)gm * ldr + gn];
      else *c = v;
    }
  }
}
}  // namespace

bm_status gemm_f32_simt(int M, int N, int K, const float* A, int64_t lda, int a_major, const float* B, int64_t ldb,
                        int b_major, float* C, int64_t ldc, int epi, const float* R, int64_t ldr, float alpha,
                        cudaStream_t st) {
  dim3 grid(ceil_div(N, TN), ceil_div(M, TM));
  BM_CUDA_TRY(launch_k(gemm_f32_kernel, grid, dim3(256), 0, st, M, N, K, A, lda, a_major, B, ldb, b_major, C, ldc, epi, R,
                       ldr, alpha));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

void preload_simt(std::vector<const void*>& v) { v.push_back((const void*)gemm_f32_kernel); }

}  // namespace bm
