// Host-side internals of libsoakit_b200: error state, device/stream registry,
// dtype helpers. Device helpers (x86-exact float ops, PTX wrappers) live in
// sk_device.cuh.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdarg>

#include "soakit_b200.h"
#include "sk_device.cuh"

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
  int l2_bytes = 0;
  cudaStream_t stream = nullptr;   // default work stream
  cudaStream_t copy_in = nullptr;  // H2D stream of the transfer pipeline
  cudaStream_t copy_out = nullptr; // D2H stream of the transfer pipeline
  void* staging = nullptr;         // device staging for host<->device conversions
  size_t staging_bytes = 0;
  cudaEvent_t pipe_events[9] = {};  // the transfer pipeline's events, created once
};

// Captured graphs bake in device addresses, the pipeline's staging buffer
// included. While any graph is alive, a staging buffer that has to grow is
// retired (kept allocated) instead of freed; the last sk_graph_destroy frees
// the retired buffers.
void retire_or_free_staging(int device, void* p);
void graph_created();
void graph_destroyed();

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

}  // namespace sk
