// kernels_capi.cu -- extern "C" entry points of include/bigmac_kernels.h and
// the library-wide helpers (error string, SM count, launch census).
#include <atomic>
#include <mutex>

#include <vector>
#include "common.cuh"
#include "kernels.h"

namespace bm {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    n = v;
  }
  return n;
}

// SMs left free by the persistent GEMM grids (set by the executor around compute
// ops that share the GPU with a high-priority generator stream)
static int g_sm_reserve = 0;
void set_sm_reserve(int n) { g_sm_reserve = n < 0 ? 0 : n; }
int gemm_sm_budget() {
  const int b = num_sms() - g_sm_reserve;
  return b < 2 ? 2 : b;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("BM_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static std::atomic<int64_t> g_launches{0};
void (*g_launch_hook)(cudaStream_t, const void*) = nullptr;
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

bm_status gemm(int dtype, int M, int N, int K, const void* A, int64_t lda, int a_major, const void* B, int64_t ldb,
               int b_major, void* C, int64_t ldc, int c_dtype, int epi, const void* R, int64_t ldr, float alpha,
               cudaStream_t st, int f, void* ws, int64_t ws_bytes) {
  if (M <= 0 || N <= 0) return BM_OK;
  if (epi == BM_EPI_SWIGLU || epi == BM_EPI_DSWIGLU) {
    BM_CHECK_ARG(dtype == BM_BF16 && K > 0, "fused SwiGLU epilogues are bf16 tensor-core only");
    return gemm_bf16_tc(M, N, K, A, lda, a_major, B, ldb, b_major, C, ldc, c_dtype, epi, R, ldr, alpha, st, f);
  }
  BM_CHECK_ARG(epi != BM_EPI_ACCUM || c_dtype == BM_F32, "ACCUM epilogue requires an fp32 C");
  if (K <= 0) {
    // empty contraction: C = 0 (STORE) / C = R (ADD) / unchanged (ACCUM)
    if (epi == BM_EPI_ACCUM) return BM_OK;
    const size_t es = c_dtype == BM_F32 ? 4 : 2;
    if (epi == BM_EPI_STORE) {
      BM_CUDA_TRY(cudaMemset2DAsync(C, ldc * es, 0, (size_t)N * es, M, st));
    } else {
      BM_CUDA_TRY(cudaMemcpy2DAsync(C, ldc * es, R, ldr * es, (size_t)N * es, M, cudaMemcpyDeviceToDevice, st));
    }
    return BM_OK;
  }
  if (dtype == BM_BF16) {
    return gemm_bf16_tc(M, N, K, A, lda, a_major, B, ldb, b_major, C, ldc, c_dtype, epi, R, ldr, alpha, st, f, ws,
                        ws_bytes);
  }
  BM_CHECK_ARG(c_dtype == BM_F32, "fp32 GEMM writes fp32 C");
  return gemm_f32_simt(M, N, K, (const float*)A, lda, a_major, (const float*)B, ldb, b_major, (float*)C, ldc, epi,
                       (const float*)R, ldr, alpha, st);
}

void preload_elementwise(std::vector<const void*>& v);
void preload_simt(std::vector<const void*>& v);
void preload_tc(std::vector<const void*>& v);
void preload_peer_sum(std::vector<const void*>& v);
// Load every kernel of the library onto the current device now.  Under CUDA lazy
// module loading (the default) a kernel is loaded at its first launch, and that
// load blocks while another stream of the context is parked on a cross-GPU flag
// wait: measured as a device-wide stall of the compute-efficient schedule at
// P = 4 (the first SwiGLU launch behind a send waiting for a credit).
bm_status preload_kernels() {
  std::vector<const void*> v;
  preload_elementwise(v);
  preload_simt(v);
  preload_tc(v);
  preload_peer_sum(v);
  for (const void* f : v) {
    cudaFuncAttributes a;
    BM_CUDA_TRY(cudaFuncGetAttributes(&a, f));
  }
  return BM_OK;
}
}  // namespace bm

using namespace bm;

#define ST(s) reinterpret_cast<cudaStream_t>(s)
#define DISPATCH(dtype, call_bf16, call_f32)                  \
  do {                                                        \
    if ((dtype) == BM_BF16) return call_bf16;                 \
    if ((dtype) == BM_F32) return call_f32;                   \
    set_error("unknown dtype");                               \
    return BM_E_INVALID;                                      \
  } while (0)

namespace bm { void set_gemm_mode(int m); void set_gemm_bn512(int m); void set_gemm_bk128(int m); void set_gemm_swiglu_bk128(int m); }

extern "C" {

const char* bm_last_error(void) { return get_error(); }

bm_status bm_k_gemm_mode(int32_t mode) {
  BM_CHECK_ARG(mode >= 0 && mode <= 2, "mode must be 0 (auto), 1 (1-CTA) or 2 (CTA pair)");
  bm::set_gemm_mode(mode);
  return BM_OK;
}

bm_status bm_k_gemm_bn512(int32_t mode) {
  BM_CHECK_ARG(mode >= 0 && mode <= 2, "mode must be 0 (never), 1 (always) or 2 (auto)");
  bm::set_gemm_bn512(mode);
  return BM_OK;
}

bm_status bm_k_gemm_bk128(int32_t on) {
  BM_CHECK_ARG(on == 0 || on == 1, "on must be 0 or 1");
  bm::set_gemm_bk128(on);
  return BM_OK;
}

bm_status bm_k_gemm_swiglu_bk128(int32_t on) {
  BM_CHECK_ARG(on == 0 || on == 1, "on must be 0 or 1");
  bm::set_gemm_swiglu_bk128(on);
  return BM_OK;
}

bm_status bm_k_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_major,
                    const void* B, int64_t ldb, int32_t b_major, void* C, int64_t ldc, int32_t c_dtype,
                    int32_t epilogue, const void* R, int64_t ldr, float alpha, void* stream) {
  BM_CHECK_ARG(epilogue >= BM_EPI_STORE && epilogue <= BM_EPI_ADD, "use bm_k_gemm_swiglu for fused SwiGLU epilogues");
  // standalone calls get a library-owned split-K workspace (the executor passes its own, per stream)
  static void* ws = nullptr;
  static const int64_t ws_bytes = 64ll << 20;
  if (!ws && dtype == BM_BF16) {
    if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) { ws = nullptr; cudaGetLastError(); }
  }
  return gemm(dtype, M, N, K, A, lda, a_major, B, ldb, b_major, C, ldc, c_dtype, epilogue, R, ldr, alpha, ST(stream),
              0, ws, ws ? ws_bytes : 0);
}

bm_status bm_k_gemm_swiglu(int32_t M, int32_t f, int32_t K, const void* X, int64_t ldx, const void* W, int64_t ldw,
                           void* gu, void* h, void* stream) {
  return gemm(BM_BF16, M, 2 * f, K, X, ldx, 0, W, ldw, 0, gu, 2 * (int64_t)f, BM_BF16, BM_EPI_SWIGLU, h, f, 1.f,
              ST(stream), f);
}

bm_status bm_k_gemm_group(const bm_gemm_desc* d, int32_t n, void* stream) {
  BM_CHECK_ARG(d && n >= 1 && n <= 2, "1..2 descriptors");
  GemmSpec sp[2];
  for (int i = 0; i < n; ++i)
    sp[i] = GemmSpec{d[i].M, d[i].N, d[i].K, d[i].A, d[i].lda, d[i].a_major, d[i].B, d[i].ldb, d[i].b_major, d[i].C,
                     d[i].ldc, d[i].c_dtype, d[i].epilogue, d[i].R, d[i].ldr, d[i].alpha, d[i].f, nullptr, 0};
  return gemm_bf16_tc_group(sp, n, ST(stream));
}

bm_status bm_k_gemm_dswiglu(int32_t M, int32_t f, int32_t K, const void* dY, int64_t lddy, const void* W, int64_t ldw,
                            const void* gu, void* dgu, void* stream) {
  return gemm(BM_BF16, M, f, K, dY, lddy, 0, W, ldw, 1, dgu, 2 * (int64_t)f, BM_BF16, BM_EPI_DSWIGLU, gu,
              2 * (int64_t)f, 1.f, ST(stream), f);
}

bm_status bm_k_rmsnorm_fwd(int32_t dtype, int32_t rows, int32_t cols, const void* x, const void* g, void* y,
                           float* rstd, void* stream) {
  DISPATCH(dtype, rmsnorm_fwd<bf16>(rows, cols, (const bf16*)x, (const bf16*)g, (bf16*)y, rstd, ST(stream)),
           rmsnorm_fwd<float>(rows, cols, (const float*)x, (const float*)g, (float*)y, rstd, ST(stream)));
}
bm_status bm_k_rmsnorm_bwd(int32_t dtype, int32_t rows, int32_t cols, const void* dy, const void* x, const void* g,
                           const float* rstd, const void* dres, void* dx, float* dg, float* partial, void* stream) {
  DISPATCH(dtype,
           rmsnorm_bwd<bf16>(rows, cols, (const bf16*)dy, (const bf16*)x, (const bf16*)g, rstd, (const bf16*)dres,
                             (bf16*)dx, dg, partial, ST(stream)),
           rmsnorm_bwd<float>(rows, cols, (const float*)dy, (const float*)x, (const float*)g, rstd,
                              (const float*)dres, (float*)dx, dg, partial, ST(stream)));
}
int64_t bm_k_rmsnorm_bwd_scratch(int32_t rows, int32_t cols) { return rmsnorm_bwd_scratch_floats(rows, cols); }

bm_status bm_k_swiglu_fwd(int32_t dtype, int32_t rows, int32_t f, const void* gu, void* h, void* stream) {
  DISPATCH(dtype, swiglu_fwd<bf16>(rows, f, (const bf16*)gu, (bf16*)h, ST(stream)),
           swiglu_fwd<float>(rows, f, (const float*)gu, (float*)h, ST(stream)));
}
bm_status bm_k_swiglu_bwd(int32_t dtype, int32_t rows, int32_t f, const void* dh, const void* gu, void* dgu,
                          void* stream) {
  DISPATCH(dtype, swiglu_bwd<bf16>(rows, f, (const bf16*)dh, (const bf16*)gu, (bf16*)dgu, ST(stream)),
           swiglu_bwd<float>(rows, f, (const float*)dh, (const float*)gu, (float*)dgu, ST(stream)));
}
bm_status bm_k_gelu_fwd(int32_t dtype, int64_t n, const void* a, void* z, void* stream) {
  DISPATCH(dtype, gelu_fwd<bf16>(n, (const bf16*)a, (bf16*)z, ST(stream)),
           gelu_fwd<float>(n, (const float*)a, (float*)z, ST(stream)));
}
bm_status bm_k_gelu_bwd(int32_t dtype, int64_t n, const void* dz, const void* a, void* da, void* stream) {
  DISPATCH(dtype, gelu_bwd<bf16>(n, (const bf16*)dz, (const bf16*)a, (bf16*)da, ST(stream)),
           gelu_bwd<float>(n, (const float*)dz, (const float*)a, (float*)da, ST(stream)));
}
bm_status bm_k_embed_fwd(int32_t dtype, int32_t S, int32_t d, int32_t n_mod, const int32_t* ids, const void* table,
                         const void* emb, void* X, void* stream) {
  DISPATCH(dtype, embed_fwd<bf16>(S, d, n_mod, ids, (const bf16*)table, (const bf16*)emb, (bf16*)X, ST(stream)),
           embed_fwd<float>(S, d, n_mod, ids, (const float*)table, (const float*)emb, (float*)X, ST(stream)));
}
bm_status bm_k_embed_bwd(int32_t dtype, int32_t S, int32_t d, int32_t n_mod, const int32_t* ids, const void* dX,
                         float* dT, void* scratch, void* stream) {
  DISPATCH(dtype, embed_bwd<bf16>(S, d, n_mod, ids, (const bf16*)dX, dT, scratch, ST(stream)),
           embed_bwd<float>(S, d, n_mod, ids, (const float*)dX, dT, scratch, ST(stream)));
}
int64_t bm_k_embed_bwd_scratch(int32_t S) { return embed_bwd_scratch_bytes(S); }

bm_status bm_k_ce_fwd_bwd(int32_t dtype, int32_t n, int32_t V, void* logits, const int32_t* labels, float scale_grad,
                          float* loss_out, float scale_loss, int32_t accumulate, float* scratch, void* stream) {
  DISPATCH(dtype,
           ce_fwd_bwd<bf16>(n, V, (bf16*)logits, labels, scale_grad, loss_out, scale_loss, accumulate, scratch,
                            ST(stream)),
           ce_fwd_bwd<float>(n, V, (float*)logits, labels, scale_grad, loss_out, scale_loss, accumulate, scratch,
                             ST(stream)));
}
bm_status bm_k_mse_fwd_bwd(int32_t dtype, int32_t n, int32_t dt, const void* out, const void* t, float denom,
                           float scale_grad, float scale_loss, float* loss_out, void* dout, void* stream) {
  DISPATCH(dtype,
           mse_fwd_bwd<bf16>(n, dt, (const bf16*)out, (const bf16*)t, denom, scale_grad, scale_loss, loss_out,
                             (bf16*)dout, ST(stream)),
           mse_fwd_bwd<float>(n, dt, (const float*)out, (const float*)t, denom, scale_grad, scale_loss, loss_out,
                              (float*)dout, ST(stream)));
}
bm_status bm_k_add(int32_t dtype, int64_t n, const void* a, const void* b, void* out, void* stream) {
  DISPATCH(dtype, add<bf16>(n, (const bf16*)a, (const bf16*)b, (bf16*)out, ST(stream)),
           add<float>(n, (const float*)a, (const float*)b, (float*)out, ST(stream)));
}
bm_status bm_k_cast(int32_t src_dtype, int32_t dst_dtype, int64_t n, const void* src, void* dst, void* stream) {
  return cast(src_dtype, dst_dtype, n, src, dst, ST(stream));
}

bm_status bm_k_copy(void* dst, const void* src, int64_t bytes, int32_t max_ctas, void* stream) {
  BM_CHECK_ARG(bytes >= 0 && (bytes == 0 || (dst && src)), "invalid copy");
  return copy_bytes(dst, src, bytes, max_ctas, ST(stream));
}
bm_status bm_k_zero(void* dst, int64_t bytes, void* stream) {
  BM_CHECK_ARG(bytes >= 0 && (bytes == 0 || dst), "invalid fill");
  return zero_bytes(dst, bytes, ST(stream));
}
bm_status bm_k_preload(void) { return preload_kernels(); }

}  // extern "C"
