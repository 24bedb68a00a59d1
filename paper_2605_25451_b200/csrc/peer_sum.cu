// peer_sum.cu -- the step-end gradient / loss sums
// computed by the library itself over CUDA-IPC peer memory.
//
// Used when the P·D processes of a run cannot form an NCCL communicator (NCCL
// refuses two ranks on one device: the single-GPU multi-rank parity fixture),
// or when forced (bm_ctx_init_peer_sum).  Every process reads its peers'
// fp32 gradient buffers directly (NVLink or, on one device, plain HBM):
//   reduce-scatter  process i sums chunk i of the range over the group, in
//                   group order 0..n-1 (deterministic), in place;
//   all-gather      process i copies chunk q from process q for every q != i.
// Ordering between processes is carried by monotonic 32-bit flags written with
// cuStreamWriteValue32 (memory-barrier semantics) and waited on with
// cuStreamWaitValue32 (executor.cu), exactly like the stage-boundary rings.
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bm {

namespace {

// dst[i] = sum_{q < n} src[q][i] in q order; dst may alias one of the sources
// (each element is read and written by the same thread only)
__global__ void __launch_bounds__(256) peer_sum_f4_kernel(PeerSrc s, int n, float4* dst, int64_t n4) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = reinterpret_cast<const float4*>(s.p[0])[i];
    for (int q = 1; q < n; ++q) {
      const float4 b = reinterpret_cast<const float4*>(s.p[q])[i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    dst[i] = a;
  }
}

__global__ void __launch_bounds__(256) peer_sum_f1_kernel(PeerSrc s, int n, float* dst, int64_t count) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    float a = s.p[0][i];
    for (int q = 1; q < n; ++q) a += s.p[q][i];
    dst[i] = a;
  }
}

// loss[m] = sum over the pipeline's raw terms (m < 2M);
// loss[2M] = scale * sum over every process's raw terms (the global-batch loss)
__global__ void __launch_bounds__(256) peer_loss_kernel(PeerSrc pipe, int np, PeerSrc world, int nw, int two_m,
                                                        float scale, float* loss) {
  pdl_enter();
  __shared__ float red[256];
  for (int m = threadIdx.x; m < two_m; m += blockDim.x) {
    float a = pipe.p[0][m];
    for (int q = 1; q < np; ++q) a += pipe.p[q][m];
    loss[m] = a;
  }
  float t = 0.f;
  for (int q = 0; q < nw; ++q)
    for (int m = threadIdx.x; m < two_m; m += blockDim.x) t += world.p[q][m];
  red[threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[two_m] = scale * red[0];
}

int sum_grid(int64_t items) {
  const int64_t per = 256 * 4;
  int64_t g = (items + per - 1) / per;
  const int64_t cap = (int64_t)num_sms() * 8;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

bm_status peer_sum(const PeerSrc& s, int n, float* dst, int64_t count, cudaStream_t st) {
  if (count <= 0) return BM_OK;
  BM_CHECK_ARG(n >= 1 && n <= BM_MAX_SUM_PEERS, "peer count out of range");
  uintptr_t bits = reinterpret_cast<uintptr_t>(dst) | (uintptr_t)(count * 4);
  for (int q = 0; q < n; ++q) bits |= reinterpret_cast<uintptr_t>(s.p[q]);
  if ((bits & 15) == 0)
    BM_CUDA_TRY(launch_k(peer_sum_f4_kernel, dim3(sum_grid(count / 4)), dim3(256), 0, st, s, n, (float4*)dst, count / 4));
  else
    BM_CUDA_TRY(launch_k(peer_sum_f1_kernel, dim3(sum_grid(count)), dim3(256), 0, st, s, n, dst, count));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

bm_status peer_loss(const PeerSrc& pipe, int np, const PeerSrc& world, int nw, int M, float scale, float* loss,
                    cudaStream_t st) {
  BM_CHECK_ARG(np >= 1 && nw >= 1 && np <= BM_MAX_SUM_PEERS && nw <= BM_MAX_SUM_PEERS, "peer count out of range");
  BM_CUDA_TRY(launch_k(peer_loss_kernel, dim3(1), dim3(256), 0, st, pipe, np, world, nw, 2 * M, scale, loss));
  count_launch();
  BM_CUDA_TRY(cudaGetLastError());
  return BM_OK;
}

void preload_peer_sum(std::vector<const void*>& v) {
  v.push_back((const void*)peer_sum_f4_kernel);
  v.push_back((const void*)peer_sum_f1_kernel);
  v.push_back((const void*)peer_loss_kernel);
}

}  // namespace bm
