// Shared internals of libsoakit_b200: error state, device/stream registry,
// dtype helpers and the PTX wrappers (mbarrier + bulk async copies) the
// kernels use.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdarg>

#include "soakit_b200.h"

namespace sk {

int set_error(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
void clear_error();

#define SK_TRY(call)                                              \
  do {                                                            \
    cudaError_t sk_e_ = (call);                                   \
    if (sk_e_ != cudaSuccess) return ::sk::cuda_fail(sk_e_, #call); \
  } while (0)

// Per-device state owned by the library (one non-blocking stream, helper
// streams for the transfer pipeline, the SM count).
struct DeviceState {
  bool init = false;
  int sm_count = 0;
  int max_smem_optin = 0;
  cudaStream_t stream = nullptr;   // default work stream
  cudaStream_t copy_in = nullptr;  // H2D stream of the transfer pipeline
  cudaStream_t copy_out = nullptr; // D2H stream of the transfer pipeline
  void* staging = nullptr;         // device staging for host<->device conversions
  size_t staging_bytes = 0;
};

int device_state(int device, DeviceState** out);
// resolves stream 0 to the device's library stream
cudaStream_t resolve_stream(int device, uintptr_t s);

inline int dtype_size(int t) {
  switch (t) {
    case SK_BOOL: case SK_U8: return 1;
    case SK_U16: return 2;
    case SK_U32: case SK_I32: case SK_F32: return 4;
    case SK_U64: case SK_I64: case SK_F64: return 8;
    default: return 0;
  }
}

// ---- PTX wrappers -------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// global -> shared bulk copy (TMA engine, non-tensor); completes tx on `bar`.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// shared -> global bulk copy, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// generic-proxy smem writes -> visible to the async proxy (bulk store source)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 0.0;" : "=l"(p));
  return p;
}

}  // namespace sk
