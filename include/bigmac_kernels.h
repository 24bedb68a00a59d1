/*
 * bigmac_kernels.h -- C ABI of the individual sm_100a kernels the executor
 * uses for the model's compute (one entry point per device op on the hot path).
 * They exist so parity tests can check each kernel against the oracle; the
 * executor calls the same launchers internally.
 *
 * All pointers are device pointers unless noted; `stream` is a cudaStream_t
 * (0 = legacy default).  dtype is bm_dtype (0 bf16, 1 fp32).  Errors are
 * reported as bm_status with bm_last_error() (bigmac.h).  Launches are
 * asynchronous; argument errors are detected on the host before launch.
 */
#ifndef BIGMAC_KERNELS_H
#define BIGMAC_KERNELS_H

#include "bigmac.h"

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM epilogues */
typedef enum {
  BM_EPI_STORE = 0,   /* C = alpha*acc            (C dtype = c_dtype)           */
  BM_EPI_ACCUM = 1,   /* C += alpha*acc           (C must be fp32; wgrad, β = 1) */
  BM_EPI_ADD = 2,     /* C = alpha*acc + R        (R has c_dtype; residual add)  */
  BM_EPI_SWIGLU = 3,  /* internal: gate/up GEMM + SwiGLU (bm_k_gemm_swiglu)      */
  BM_EPI_DSWIGLU = 4  /* internal: down dgrad + SwiGLU backward (bm_k_gemm_dswiglu) */
} bm_epilogue;

/* C[m, n] = sum_k A(m, k) * B(n, k), fp32 accumulation.
 *   A(m, k) = A[m*lda + k] if a_major == 0 (K-major) else A[k*lda + m] (MN-major)
 *   B(n, k) = B[n*ldb + k] if b_major == 0 (K-major) else B[k*ldb + n] (MN-major)
 *   C[m*ldc + n], R[m*ldr + n].
 * dtype of A/B: BM_BF16 -> tcgen05.mma kind::f16 tiles fed by TMA (TMEM
 * accumulators); BM_F32 -> exact fp32 FFMA kernel (no TF32; parity mode).
 * Requirements (bf16): lda, ldb multiples of 8 elements, A/B 16-byte aligned.
 * The dense block contractions of the model (Linear layers of the
 * encoder, LLM and generator) are all instances: forward X W^T (A, B K-major),
 * data-grad dY W (B MN-major), weight-grad dY^T X (A, B MN-major, ACCUM). */
bm_status bm_k_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K,
                    const void* A, int64_t lda, int32_t a_major,
                    const void* B, int64_t ldb, int32_t b_major,
                    void* C, int64_t ldc, int32_t c_dtype, int32_t epilogue,
                    const void* R, int64_t ldr, float alpha, void* stream);

/* LLM gate/up projection with the SwiGLU activation fused into the epilogue
 * (bf16, tensor cores, CTA pairs):  [g | u] = X W^T with W = [W_gate; W_up]
 * ([2f, K] row-major, ldw), X [M, K] (ldx);  writes gu [M, 2f] (both halves,
 * kept for the backward) and h = silu(g) * u [M, f].  f % 128 == 0. */
bm_status bm_k_gemm_swiglu(int32_t M, int32_t f, int32_t K, const void* X, int64_t ldx,
                           const void* W, int64_t ldw, void* gu, void* h, void* stream);
/* LLM down-projection data gradient with the SwiGLU backward fused into the
 * epilogue:  dh = dY W_down ([M, K] x [K, f], W_down [K, f] row-major, ldw),
 * then dgu = [dh*u*s*(1 + g(1-s)), dh*g*s] with s = sigmoid(g), g|u from gu
 * [M, 2f];  writes dgu [M, 2f] (dh is never stored).  f % 32 == 0 (32-column
 * output chunks; BM_E_INVALID otherwise -- the executor then runs the GEMM and
 * bm_k_swiglu_bwd separately). */
bm_status bm_k_gemm_dswiglu(int32_t M, int32_t f, int32_t K, const void* dY, int64_t lddy,
                            const void* W, int64_t ldw, const void* gu, void* dgu, void* stream);

/* One bf16 contraction of a grouped launch, arguments as bm_k_gemm (epilogue
 * BM_EPI_DSWIGLU: the fused SwiGLU backward of bm_k_gemm_dswiglu, with N = f,
 * C = dgu [M, 2f], R = gu [M, 2f]; f is ignored otherwise). */
typedef struct {
  int32_t M, N, K;
  const void* A;
  int64_t lda;
  int32_t a_major;
  const void* B;
  int64_t ldb;
  int32_t b_major;
  void* C;
  int64_t ldc;
  int32_t c_dtype, epilogue;
  const void* R;
  int64_t ldr;
  float alpha;
  int32_t f;
} bm_gemm_desc;
/* n (1..2) independent bf16 contractions -- a Linear's data and weight gradient --
 * in ONE persistent CTA-pair tcgen05 launch: every pair processes whole 256 x 256
 * tiles of either problem on a host-computed longest-processing-time schedule (a
 * tile's cost = its K / 64 blocks), so neither problem's last wave leaves pairs
 * idle.  Shapes that do not fit the pair kernel (M or N < 256, misaligned
 * operands, or too few tiles in auto mode) run as separate bm_k_gemm launches.
 * Outputs must not overlap.  Errors: BM_E_INVALID, BM_E_CUDA. */
bm_status bm_k_gemm_group(const bm_gemm_desc* descs, int32_t n, void* stream);

/* Tuning / testing knob for the bf16 GEMM tile scheme: 0 = auto (CTA-pair
 * cta_group::2 256xBN tiles when M >= 512, N >= 256, K >= 256; 128xBN 1-CTA
 * tiles otherwise), 1 = always 1-CTA, 2 = always CTA pairs.  Process-wide. */
bm_status bm_k_gemm_mode(int32_t mode);
/* Pair-tile width of the CTA-pair GEMM: 0 = 256 x 256 tiles (two TMEM accumulators,
 * the epilogue of one tile overlaps the next tile's MMAs), 1 = 256 x 512 tiles
 * whenever N >= 512 (one 512-column accumulator; a quarter less L2 -> SMEM traffic
 * per FLOP), 2 = auto (default: a wave-quantised cost model picks 256 x 512 where
 * its per-FLOP gain beats the un-overlapped epilogue and the coarser last wave,
 * never for the SwiGLU-backward epilogue; gemm_tc.cu use_bn512).  Process-wide. */
bm_status bm_k_gemm_bn512(int32_t mode);
/* 1 (default): 256 x 256 CTA-pair GEMMs step K in 128-deep blocks (two 64-wide
 * swizzled sub-tiles per operand, three 64 KB stages); 0: 64-deep blocks, six
 * stages.  Process-wide. */
bm_status bm_k_gemm_bk128(int32_t on);
/* 1: the gate/up GEMM with the fused SwiGLU epilogue also steps K in 128-deep blocks
 * (three 64 KB stages; 4 KB epilogue staging per warp, [g | u] stored before h;
 * default); 0: 64-deep blocks, five stages.  Takes effect with bm_k_gemm_bk128(1). */
bm_status bm_k_gemm_swiglu_bk128(int32_t on);

/* RMSNorm y = x * rstd * g, rstd = 1/sqrt(mean(x^2) + 1e-5); rstd saved (fp32 [rows]). */
bm_status bm_k_rmsnorm_fwd(int32_t dtype, int32_t rows, int32_t cols, const void* x,
                           const void* g, void* y, float* rstd, void* stream);
/* dx = rstd*(dy*g - xhat*mean(dy*g*xhat)) [+ dres];  dg += sum_rows dy*xhat (fp32).
 * dres may be NULL; dx may alias dres.  `partial` is fp32 scratch of
 * bm_k_rmsnorm_bwd_scratch(rows, cols) floats. */
bm_status bm_k_rmsnorm_bwd(int32_t dtype, int32_t rows, int32_t cols, const void* dy,
                           const void* x, const void* g, const float* rstd, const void* dres,
                           void* dx, float* dg, float* partial, void* stream);
int64_t bm_k_rmsnorm_bwd_scratch(int32_t rows, int32_t cols);

/* h[i, j] = silu(gu[i, j]) * gu[i, f + j]   (gu: [rows, 2f], h: [rows, f]) */
bm_status bm_k_swiglu_fwd(int32_t dtype, int32_t rows, int32_t f, const void* gu, void* h, void* stream);
/* dgu = [dh*u*s*(1 + g(1-s)), dh*g*s],  s = sigmoid(g) */
bm_status bm_k_swiglu_bwd(int32_t dtype, int32_t rows, int32_t f, const void* dh, const void* gu,
                          void* dgu, void* stream);
/* z = gelu_tanh(a);  da = dz * gelu_tanh'(a)  (n elements) */
bm_status bm_k_gelu_fwd(int32_t dtype, int64_t n, const void* a, void* z, void* stream);
bm_status bm_k_gelu_bwd(int32_t dtype, int64_t n, const void* dz, const void* a, void* da, void* stream);

/* embed_preprocess: X[i] = emb[i] for i < n_mod, else table[ids[i]] */
bm_status bm_k_embed_fwd(int32_t dtype, int32_t S, int32_t d, int32_t n_mod, const int32_t* ids,
                         const void* table, const void* emb, void* X, void* stream);
/* text-table gradient: dT[ids[i]] += dX[i] for i in [n_mod, S), deterministic
 * (sorted segmented sum).  dT fp32.  scratch: bm_k_embed_bwd_scratch(S) bytes. */
bm_status bm_k_embed_bwd(int32_t dtype, int32_t S, int32_t d, int32_t n_mod, const int32_t* ids,
                         const void* dX, float* dT, void* scratch, void* stream);
int64_t bm_k_embed_bwd_scratch(int32_t S);

/* Cross-entropy over rows of logits [n, V]: loss_out[0] (+)= scale_loss * mean_i
 * (lse_i - z[i, label_i]); logits overwritten with dz = (softmax - onehot) * scale_grad.
 * accumulate != 0 adds into *loss_out.  scratch: n floats. */
bm_status bm_k_ce_fwd_bwd(int32_t dtype, int32_t n, int32_t V, void* logits, const int32_t* labels,
                          float scale_grad, float* loss_out, float scale_loss, int32_t accumulate,
                          float* scratch, void* stream);
/* MSE shard: loss_out[0] += sum((out - t)^2) / denom * scale_loss;
 * dout = 2 (out - t) / denom * scale_grad  (out, t, dout: [n, dt]) */
bm_status bm_k_mse_fwd_bwd(int32_t dtype, int32_t n, int32_t dt, const void* out, const void* t,
                           float denom, float scale_grad, float scale_loss, float* loss_out,
                           void* dout, void* stream);

/* Elementwise helpers used by the executor. */
bm_status bm_k_add(int32_t dtype, int64_t n, const void* a, const void* b, void* out, void* stream);
bm_status bm_k_cast(int32_t src_dtype, int32_t dst_dtype, int64_t n, const void* src, void* dst, void* stream);
/* Byte copy / zero fill on SMs (16-byte vectors when dst, src and bytes are 16-byte
 * aligned).  dst may be a peer GPU's IPC-mapped buffer (NVLink stores).  The
 * executor's stage-boundary sends use a copy-engine cudaMemcpyAsync by default
 * (no SM time taken from the GEMMs); BM_PEER_COPY=sm selects this kernel
 * instead.  max_ctas <= 0: the elementwise grid (8 CTAs per SM). */
bm_status bm_k_copy(void* dst, const void* src, int64_t bytes, int32_t max_ctas, void* stream);
bm_status bm_k_zero(void* dst, int64_t bytes, void* stream);

/* Load every kernel of the library onto the current device now (synchronous,
 * idempotent).  Under CUDA lazy module loading a kernel is otherwise loaded at its
 * first launch, and that load blocks while any stream of the context is parked on
 * a cross-GPU flag wait -- a device-wide stall of the pipelined step (measured:
 * compute-efficient schedule, P = 4).  bm_ctx_create calls it. */
bm_status bm_k_preload(void);

#ifdef __cplusplus
}
#endif
#endif /* BIGMAC_KERNELS_H */
