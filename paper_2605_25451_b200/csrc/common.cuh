// common.cuh -- shared helpers for the sm_100a kernels and the executor.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <utility>

#include "../../include/bigmac.h"
#include "../../include/bigmac_kernels.h"

namespace bm {

// thread-local error message (bm_last_error)
void set_error(const std::string& msg);
const char* get_error();

struct Err {
  bm_status code;
  std::string msg;
};

#define BM_CUDA_TRY(expr)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::bm::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" +  \
                      __FILE__ + ":" + std::to_string(__LINE__));                  \
      return BM_E_CUDA;                                                            \
    }                                                                              \
  } while (0)

#define BM_TRY(expr)                 \
  do {                               \
    bm_status _s = (expr);           \
    if (_s != BM_OK) return _s;      \
  } while (0)

#define BM_CHECK_ARG(cond, msg)                      \
  do {                                               \
    if (!(cond)) {                                   \
      ::bm::set_error(std::string("invalid argument: ") + (msg)); \
      return BM_E_INVALID;                           \
    }                                                \
  } while (0)

typedef __nv_bfloat16 bf16;

template <typename T> struct DT;
template <> struct DT<bf16> { static constexpr int id = BM_BF16; };
template <> struct DT<float> { static constexpr int id = BM_F32; };

__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();
// persistent-GEMM grid budget: num_sms() minus the SMs reserved by set_sm_reserve
int gemm_sm_budget();
void set_sm_reserve(int n);

// ---------------------------------------------------------------- PDL
// Every library kernel is launched with programmatic stream serialization
// (Programmatic Dependent Launch) unless BM_PDL=0: the next kernel's launch and
// its data-independent prologue overlap the tail of the previous kernel.  Each
// kernel executes griddepcontrol.wait before touching global memory and then
// griddepcontrol.launch_dependents.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// debug hook (BM_DEBUG_PROGRESS): called after every library kernel launch
extern void (*g_launch_hook)(cudaStream_t, const void*);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (g_launch_hook) g_launch_hook(st, (const void*)kern);
  return e;
}

// launch census (kernels launched through the library)
void count_launch(int n = 1);
int64_t launch_count();

}  // namespace bm
