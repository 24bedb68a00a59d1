// kernels.h -- internal launcher declarations (C++), shared by the C-ABI
// wrappers and the executor.
#pragma once

#include "common.cuh"

namespace bm {

bm_status gemm_bf16_tc(int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B, int64_t ldb,
                       int b_major, void* C, int64_t ldc, int c_dtype, int epi, const void* R, int64_t ldr,
                       float alpha, cudaStream_t st, int f = 0, void* ws = nullptr, int64_t ws_bytes = 0);
bm_status gemm_f32_simt(int M, int N, int K, const float* A, int64_t lda, int a_major, const float* B, int64_t ldb,
                        int b_major, float* C, int64_t ldc, int epi, const float* R, int64_t ldr, float alpha,
                        cudaStream_t st);
// one contraction C = epilogue(alpha A B^T) (gemm_bf16_tc's arguments)
struct GemmSpec {
  int M, N, K;
  const void* A;
  int64_t lda;
  int a_major;
  const void* B;
  int64_t ldb;
  int b_major;
  void* C;
  int64_t ldc;
  int c_dtype, epi;
  const void* R;
  int64_t ldr;
  float alpha;
  int f;
  void* ws;
  int64_t ws_bytes;
};
// independent bf16 contractions (n <= 2, e.g. a Linear's data and weight gradient) in
// ONE persistent CTA-pair launch on a longest-processing-time tile schedule; shapes
// that do not fit the pair kernel fall back to one gemm_bf16_tc launch each
bm_status gemm_bf16_tc_group(const GemmSpec* specs, int n, cudaStream_t st);
// dtype-dispatching GEMM (bf16 -> tcgen05, fp32 -> exact FFMA)
bm_status gemm(int dtype, int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B, int64_t ldb,
               int b_major, void* C, int64_t ldc, int c_dtype, int epi, const void* R, int64_t ldr, float alpha,
               cudaStream_t st, int f = 0, void* ws = nullptr, int64_t ws_bytes = 0);

template <typename T>
bm_status rmsnorm_fwd(int rows, int cols, const T* x, const T* g, T* y, float* rstd, cudaStream_t st);
template <typename T>
bm_status rmsnorm_bwd(int rows, int cols, const T* dy, const T* x, const T* g, const float* rstd, const T* dres,
                      T* dx, float* dg, float* partial, cudaStream_t st);
int64_t rmsnorm_bwd_scratch_floats(int rows, int cols);
template <typename T> bm_status swiglu_fwd(int rows, int f, const T* gu, T* h, cudaStream_t st);
template <typename T> bm_status swiglu_bwd(int rows, int f, const T* dh, const T* gu, T* dgu, cudaStream_t st);
template <typename T> bm_status gelu_fwd(int64_t n, const T* a, T* z, cudaStream_t st);
template <typename T> bm_status gelu_bwd(int64_t n, const T* dz, const T* a, T* da, cudaStream_t st);
template <typename T>
bm_status embed_fwd(int S, int d, int n_mod, const int32_t* ids, const T* table, const T* emb, T* X, cudaStream_t st);
template <typename T>
bm_status embed_bwd(int S, int d, int n_mod, const int32_t* ids, const T* dX, float* dT, void* scratch, cudaStream_t st);
int64_t embed_bwd_scratch_bytes(int S);
template <typename T>
bm_status ce_fwd_bwd(int n, int V, T* logits, const int32_t* labels, float scale_grad, float* loss_out,
                     float scale_loss, int accumulate, float* scratch, cudaStream_t st);
template <typename T>
bm_status mse_fwd_bwd(int n, int dt, const T* out, const T* t, float denom, float scale_grad, float scale_loss,
                      float* loss_out, T* dout, cudaStream_t st);
template <typename T> bm_status add(int64_t n, const T* a, const T* b, T* o, cudaStream_t st);
bm_status cast(int sd, int dd, int64_t n, const void* s, void* d, cudaStream_t st);
// load every library kernel onto the current device (defeats lazy loading; see kernels_capi.cu)
bm_status preload_kernels();
// SM copy / zero fill (16-byte vectors when aligned); max_ctas <= 0: full elementwise grid
bm_status copy_bytes(void* dst, const void* src, int64_t bytes, int max_ctas, cudaStream_t st);
bm_status zero_bytes(void* dst, int64_t bytes, cudaStream_t st);
// one-thread kernel polling *flag until (int32)(*flag - v) >= 0 (BM_WAIT=spin)
bm_status spin_wait(const uint32_t* flag, uint32_t v, cudaStream_t st);
// loss[2M] = scale * sum(loss[0 .. 2M))
bm_status loss_finalize(int M, float* loss, float scale, cudaStream_t st);

// step-end sums over CUDA-IPC peer memory (peer_sum.cu)
#define BM_MAX_SUM_PEERS 64
struct PeerSrc {
  const float* p[BM_MAX_SUM_PEERS];
};
// dst[0:count) = sum_{q<n} s.p[q][0:count) in q order (dst may alias a source)
bm_status peer_sum(const PeerSrc& s, int n, float* dst, int64_t count, cudaStream_t st);
// loss[0:2M) = sum over the np pipeline sources; loss[2M] = scale * sum of all nw sources' terms
bm_status peer_loss(const PeerSrc& pipe, int np, const PeerSrc& world, int nw, int M, float scale, float* loss,
                    cudaStream_t st);

}  // namespace bm
