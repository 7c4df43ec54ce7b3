// Memory-context plumbing of libsoakit_b200: allocation, copies, memset,
// memmove, streams/events, peer access, IPC. Replaces the mock device and the
// default copier of the reference (memctx.py:115-143, 304-360).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "sk_internal.cuh"

namespace sk {

static thread_local std::string g_last_error;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

void clear_error() { g_last_error.clear(); }

int cuda_fail(cudaError_t e, const char* what) {
  int code = SK_ERR_CUDA;
  if (e == cudaErrorMemoryAllocation) code = SK_ERR_ALLOC;
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) code = SK_ERR_NO_DEVICE;
  cudaGetLastError();  // clear sticky-free error state
  return set_error(code, "%s failed: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

static std::mutex g_dev_mu;
static DeviceState g_dev[64];

int device_state(int device, DeviceState** out) {
  if (device < 0 || device >= 64) return set_error(SK_ERR_INVALID, "device id %d out of range", device);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  DeviceState& d = g_dev[device];
  if (!d.init) {
    int count = 0;
    SK_TRY(cudaGetDeviceCount(&count));
    if (device >= count) return set_error(SK_ERR_NO_DEVICE, "device %d not present (%d devices)", device, count);
    SK_TRY(cudaSetDevice(device));
    SK_TRY(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, device));
    SK_TRY(cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    SK_TRY(cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, device));
    SK_TRY(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    SK_TRY(cudaStreamCreateWithFlags(&d.copy_in, cudaStreamNonBlocking));
    SK_TRY(cudaStreamCreateWithFlags(&d.copy_out, cudaStreamNonBlocking));
    // keep freed pool memory cached: layout growth reallocates often
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
    d.init = true;
  } else {
    SK_TRY(cudaSetDevice(device));
  }
  *out = &d;
  return SK_OK;
}

cudaStream_t resolve_stream(int device, uintptr_t s) {
  if (s) return reinterpret_cast<cudaStream_t>(s);
  DeviceState* d = nullptr;
  if (device_state(device, &d) != SK_OK) return nullptr;
  return d->stream;
}

static int stream_device(cudaStream_t s, int* device) {
  // the library's streams know their device; foreign streams use the current one
  for (int i = 0; i < 64; ++i) {
    if (g_dev[i].init && (g_dev[i].stream == s || g_dev[i].copy_in == s || g_dev[i].copy_out == s)) {
      *device = i;
      return SK_OK;
    }
  }
  SK_TRY(cudaGetDevice(device));
  return SK_OK;
}

static int stream_of(uintptr_t s, cudaStream_t* out) {
  if (s) {
    *out = reinterpret_cast<cudaStream_t>(s);
    int dev = 0;
    int rc = stream_device(*out, &dev);
    if (rc) return rc;
    SK_TRY(cudaSetDevice(dev));
    return SK_OK;
  }
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* d = nullptr;
  int rc = device_state(dev, &d);
  if (rc) return rc;
  *out = d->stream;
  return SK_OK;
}

}  // namespace sk

using namespace sk;

extern "C" {

const char* sk_last_error(void) { return g_last_error.c_str(); }

int sk_version(void) { return 0x000100; }

int sk_device_count(int* count) {
  if (!count) return set_error(SK_ERR_INVALID, "null count");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return SK_OK;
}

int sk_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem) {
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  cudaDeviceProp prop;
  SK_TRY(cudaGetDeviceProperties(&prop, device));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (total_mem) *total_mem = prop.totalGlobalMem;
  return SK_OK;
}

int sk_malloc(int device, size_t nbytes, void** out) {
  if (!out) return set_error(SK_ERR_INVALID, "null out pointer");
  *out = nullptr;
  if (nbytes == 0) return SK_OK;
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  // round up so vectorised tails never leave the allocation
  size_t padded = (nbytes + 255) & ~size_t(255);
  cudaError_t e = cudaMallocAsync(out, padded, d->stream);
  if (e != cudaSuccess) {
    *out = nullptr;
    return cuda_fail(e, "cudaMallocAsync");
  }
  return SK_OK;
}

int sk_free(int device, void* ptr) {
  if (!ptr) return SK_OK;
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  SK_TRY(cudaFreeAsync(ptr, d->stream));
  return SK_OK;
}

int sk_host_alloc_pinned(size_t nbytes, void** out) {
  if (!out) return set_error(SK_ERR_INVALID, "null out pointer");
  *out = nullptr;
  if (nbytes == 0) return SK_OK;
  cudaError_t e = cudaHostAlloc(out, nbytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    *out = nullptr;
    return cuda_fail(e, "cudaHostAlloc");
  }
  return SK_OK;
}

int sk_host_free_pinned(void* ptr) {
  if (!ptr) return SK_OK;
  SK_TRY(cudaFreeHost(ptr));
  return SK_OK;
}

int sk_host_register(void* ptr, size_t nbytes) {
  if (!ptr || !nbytes) return SK_OK;
  SK_TRY(cudaHostRegister(ptr, nbytes, cudaHostRegisterPortable));
  return SK_OK;
}

int sk_host_unregister(void* ptr) {
  if (!ptr) return SK_OK;
  SK_TRY(cudaHostUnregister(ptr));
  return SK_OK;
}

int sk_stream_default(int device, uintptr_t* stream) {
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  *stream = reinterpret_cast<uintptr_t>(d->stream);
  return SK_OK;
}

int sk_stream_sync(uintptr_t stream) {
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  SK_TRY(cudaStreamSynchronize(s));
  return SK_OK;
}

int sk_device_sync(int device) {
  SK_TRY(cudaSetDevice(device));
  SK_TRY(cudaDeviceSynchronize());
  return SK_OK;
}

int sk_event_create(uintptr_t* event) {
  cudaEvent_t e;
  SK_TRY(cudaEventCreate(&e));
  *event = reinterpret_cast<uintptr_t>(e);
  return SK_OK;
}

int sk_event_destroy(uintptr_t event) {
  SK_TRY(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(event)));
  return SK_OK;
}

int sk_event_record(uintptr_t event, uintptr_t stream) {
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  SK_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(event), s));
  return SK_OK;
}

int sk_event_elapsed_ms(uintptr_t start, uintptr_t stop, float* ms) {
  SK_TRY(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(stop)));
  SK_TRY(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(start), reinterpret_cast<cudaEvent_t>(stop)));
  return SK_OK;
}

int sk_memset_async(void* dst, int byte, size_t nbytes, uintptr_t stream) {
  if (nbytes == 0) return SK_OK;
  if (byte < 0 || byte > 255) return set_error(SK_ERR_INVALID, "memset byte %d outside [0, 255]", byte);
  cudaPointerAttributes a;
  SK_TRY(cudaPointerGetAttributes(&a, dst));
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
    memset(dst, byte, nbytes);  // host-resident buffer
    return SK_OK;
  }
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  SK_TRY(cudaMemsetAsync(dst, byte, nbytes, s));
  return SK_OK;
}

int sk_memcpy_async(void* dst, const void* src, size_t nbytes, uintptr_t stream) {
  if (nbytes == 0) return SK_OK;
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  SK_TRY(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, s));
  return SK_OK;
}

int sk_memmove_async(void* dst, const void* src, size_t nbytes, uintptr_t stream) {
  if (nbytes == 0 || dst == src) return SK_OK;
  const char* d = static_cast<const char*>(dst);
  const char* sp = static_cast<const char*>(src);
  bool overlap = (d < sp + nbytes) && (sp < d + nbytes);
  if (!overlap) return sk_memcpy_async(dst, src, nbytes, stream);
  cudaPointerAttributes a;
  SK_TRY(cudaPointerGetAttributes(&a, dst));
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) {
    memmove(dst, src, nbytes);
    return SK_OK;
  }
  // device overlap: go through a stream-ordered temporary (copy-via-temp is the
  // exact memmove contract, memctx.py:356-357)
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  void* tmp = nullptr;
  SK_TRY(cudaMallocAsync(&tmp, nbytes, s));
  SK_TRY(cudaMemcpyAsync(tmp, src, nbytes, cudaMemcpyDeviceToDevice, s));
  SK_TRY(cudaMemcpyAsync(dst, tmp, nbytes, cudaMemcpyDeviceToDevice, s));
  SK_TRY(cudaFreeAsync(tmp, s));
  return SK_OK;
}

int sk_peer_enable(int device, int peer) {
  if (device == peer) return SK_OK;
  int can = 0;
  SK_TRY(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return set_error(SK_ERR_UNSUPPORTED, "device %d cannot access peer %d", device, peer);
  SK_TRY(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SK_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return SK_OK;
}

int sk_malloc_shareable(int device, size_t nbytes, void** out) {
  if (!out) return set_error(SK_ERR_INVALID, "null out pointer");
  *out = nullptr;
  if (nbytes == 0) return SK_OK;
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  SK_TRY(cudaStreamSynchronize(d->stream));
  cudaError_t e = cudaMalloc(out, (nbytes + 255) & ~size_t(255));
  if (e != cudaSuccess) {
    *out = nullptr;
    return cuda_fail(e, "cudaMalloc");
  }
  return SK_OK;
}

int sk_free_shareable(int device, void* ptr) {
  if (!ptr) return SK_OK;
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  SK_TRY(cudaStreamSynchronize(d->stream));
  SK_TRY(cudaFree(ptr));
  return SK_OK;
}

int sk_ipc_handle_size(size_t* nbytes) {
  *nbytes = sizeof(cudaIpcMemHandle_t);
  return SK_OK;
}

int sk_ipc_get_handle(void* dev_ptr, void* handle_out) {
  cudaIpcMemHandle_t h;
  SK_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
  memcpy(handle_out, &h, sizeof(h));
  return SK_OK;
}

int sk_ipc_open_handle(int device, const void* handle, void** dev_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SK_TRY(cudaSetDevice(device));
  SK_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

int sk_ipc_close_handle(int device, void* dev_ptr) {
  SK_TRY(cudaSetDevice(device));
  SK_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return SK_OK;
}

}  // extern "C"

// ---- synthetic inputs -----------------------------------------------------------------

namespace sk {

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_random_kernel(uint8_t* dst, size_t nbytes, uint64_t seed, uint64_t first) {
  const size_t nw = nbytes / 8;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nw; i += stride)
    reinterpret_cast<uint64_t*>(dst)[i] = splitmix64(seed, first + i);
  const size_t tail = nbytes - nw * 8;
  if (blockIdx.x == 0 && threadIdx.x < tail)
    dst[nw * 8 + threadIdx.x] = static_cast<uint8_t>(splitmix64(seed, first + nw) >> (8 * threadIdx.x));
}

// ---- batched row moves of a layout splice (insert / erase / grow of every stream at once) ----
// Pass 1 stages every move's source in one temporary (so a move may overlap itself and a zero fill may
// cover another move's source), pass 2 writes the staged bytes to their destinations and applies the
// zero fills. Work is cut into 64 KB chunks over all ops; 16-byte vectors when the addresses allow.
constexpr int kMoveOps = 128;
constexpr uint64_t kMoveChunk = 64 << 10;

struct MoveBatch {
  int count;
  int pass;                 // 1: sources -> tmp; 2: tmp -> destinations, zero fills
  uint8_t* tmp;
  uint64_t chunk0[kMoveOps + 1];  // first chunk of op i (prefix over the ops active in this pass)
  uint64_t tmp_off[kMoveOps];
  sk_move op[kMoveOps];
};

__device__ __forceinline__ void copy_span(uint8_t* d, const uint8_t* s, uint64_t n) {
  const int t = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s) | n) & 15) == 0) {
    for (uint64_t i = t; i < n / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
  } else {
    for (uint64_t i = t; i < n; i += blockDim.x) d[i] = s[i];
  }
}

__device__ __forceinline__ void zero_span(uint8_t* d, uint64_t n) {
  const int t = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(d) | n) & 15) == 0) {
    for (uint64_t i = t; i < n / 16; i += blockDim.x) reinterpret_cast<uint4*>(d)[i] = make_uint4(0, 0, 0, 0);
  } else {
    for (uint64_t i = t; i < n; i += blockDim.x) d[i] = 0;
  }
}

__global__ void __launch_bounds__(256) move_batch_kernel(const __grid_constant__ MoveBatch B) {
  const uint64_t total = B.chunk0[B.count];
  for (uint64_t c = blockIdx.x; c < total; c += gridDim.x) {
    int i = 0;
    while (B.chunk0[i + 1] <= c) ++i;  // <= 128 ops: a short scan
    const sk_move& m = B.op[i];
    const uint64_t off = (c - B.chunk0[i]) * kMoveChunk;
    const uint64_t n = min(kMoveChunk, m.bytes - off);
    if (B.pass == 1) {
      copy_span(B.tmp + B.tmp_off[i] + off, static_cast<const uint8_t*>(m.src) + off, n);
    } else if (m.src) {
      copy_span(static_cast<uint8_t*>(m.dst) + off, B.tmp + B.tmp_off[i] + off, n);
    } else {
      zero_span(static_cast<uint8_t*>(m.dst) + off, n);
    }
  }
}

// mismatching bytes of a vs b (verification of full-size round trips on the
// device: a 32 GB identity check must not cross PCIe)
__global__ void compare_kernel(const uint8_t* a, const uint8_t* b, size_t n, unsigned long long* count) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const size_t tid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long bad = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
  size_t done = 0;
  if (vec) {
    const size_t nv = n / 16;
    const uint4* va = reinterpret_cast<const uint4*>(a);
    const uint4* vb = reinterpret_cast<const uint4*>(b);
    for (size_t i = tid; i < nv; i += stride) {
      const uint4 x = va[i], y = vb[i];
      const uint32_t d[4] = {x.x ^ y.x, x.y ^ y.y, x.z ^ y.z, x.w ^ y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)  // count bytes, not words
        bad += __popc(((d[k] | (d[k] >> 1) | (d[k] >> 2) | (d[k] >> 3) | (d[k] >> 4) | (d[k] >> 5) |
                        (d[k] >> 6) | (d[k] >> 7)) & 0x01010101u));
    }
    done = nv * 16;
  }
  for (size_t i = done + tid; i < n; i += stride) bad += a[i] != b[i];
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

}  // namespace sk

extern "C" int sk_move_batch_async(const sk_move* ops, int count, uintptr_t stream) {
  if (count < 0 || (count && !ops)) return set_error(SK_ERR_INVALID, "bad op list");
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* d = nullptr;
  rc = device_state(dev, &d);
  if (rc) return rc;
  for (int base = 0; base < count; base += sk::kMoveOps) {
    const int m = std::min(count - base, sk::kMoveOps);
    sk::MoveBatch B;
    memset(&B, 0, sizeof(B));
    uint64_t staged = 0;
    for (int i = 0; i < m; ++i) {
      B.op[i] = ops[base + i];
      if (B.op[i].src) {
        B.tmp_off[i] = staged;
        staged += (B.op[i].bytes + 255) & ~uint64_t(255);
      }
    }
    if (staged) SK_TRY(cudaMallocAsync(reinterpret_cast<void**>(&B.tmp), staged, s));
    for (int pass = staged ? 1 : 2; pass <= 2; ++pass) {
      // the ops of this pass: moves in pass 1, everything in pass 2
      sk::MoveBatch P = B;
      P.pass = pass;
      P.count = 0;
      uint64_t chunks = 0;
      for (int i = 0; i < m; ++i) {
        if (pass == 1 && !B.op[i].src) continue;
        if (!B.op[i].bytes) continue;
        P.op[P.count] = B.op[i];
        P.tmp_off[P.count] = B.tmp_off[i];
        P.chunk0[P.count] = chunks;
        chunks += (B.op[i].bytes + sk::kMoveChunk - 1) / sk::kMoveChunk;
        ++P.count;
      }
      P.chunk0[P.count] = chunks;
      if (!chunks) continue;
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(chunks, static_cast<uint64_t>(d->sm_count) * 8));
      sk::move_batch_kernel<<<grid, 256, 0, s>>>(P);
      SK_TRY(cudaGetLastError());
    }
    if (staged) SK_TRY(cudaFreeAsync(B.tmp, s));
  }
  return SK_OK;
}

extern "C" int sk_compare_bytes(const void* a, const void* b, size_t nbytes, unsigned long long* mismatches,
                                uintptr_t stream) {
  if (!mismatches) return set_error(SK_ERR_INVALID, "mismatch counter must be a device pointer");
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  SK_TRY(cudaMemsetAsync(mismatches, 0, sizeof(unsigned long long), s));
  if (nbytes == 0) return SK_OK;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* d = nullptr;
  rc = device_state(dev, &d);
  if (rc) return rc;
  sk::compare_kernel<<<d->sm_count * 8, 256, 0, s>>>(static_cast<const uint8_t*>(a), static_cast<const uint8_t*>(b),
                                                     nbytes, mismatches);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

extern "C" int sk_fill_random(void* dst, size_t nbytes, uint64_t seed, uint64_t first_word, uintptr_t stream) {
  if (nbytes == 0) return SK_OK;
  if (reinterpret_cast<uintptr_t>(dst) & 7) return set_error(SK_ERR_INVALID, "fill target must be 8-byte aligned");
  cudaStream_t s;
  int rc = stream_of(stream, &s);
  if (rc) return rc;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* d = nullptr;
  rc = device_state(dev, &d);
  if (rc) return rc;
  sk::fill_random_kernel<<<d->sm_count * 8, 256, 0, s>>>(static_cast<uint8_t*>(dst), nbytes, seed, first_word);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

// ---- CUDA graphs: capture the library stream, replay with one launch -------------------

extern "C" {

}  // extern "C"

namespace sk {

static std::mutex g_graph_mu;
static int g_graphs_alive = 0;
static std::vector<std::pair<int, void*>> g_retired;

void retire_or_free_staging(int device, void* p) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (g_graphs_alive > 0) g_retired.push_back({device, p});
  else cudaFree(p);
}

void graph_created() {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  ++g_graphs_alive;
}

void graph_destroyed() {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (--g_graphs_alive > 0) return;
  g_graphs_alive = 0;
  int cur = 0;
  cudaGetDevice(&cur);
  for (const auto& r : g_retired) {
    cudaSetDevice(r.first);
    cudaFree(r.second);
  }
  g_retired.clear();
  cudaSetDevice(cur);
}

}  // namespace sk

extern "C" {

int sk_capture_begin(int device) {
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  SK_TRY(cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeThreadLocal));
  return SK_OK;
}

int sk_capture_end(int device, void** graph_exec) {
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(d->stream, &g);
  if (e != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return cuda_fail(e, "cudaStreamEndCapture (an operation in the region cannot be captured)");
  }
  cudaGraphExec_t x = nullptr;
  e = cudaGraphInstantiate(&x, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  *graph_exec = x;
  graph_created();
  return SK_OK;
}

int sk_graph_launch(void* graph_exec, int device) {
  DeviceState* d = nullptr;
  int rc = device_state(device, &d);
  if (rc) return rc;
  SK_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec), d->stream));
  return SK_OK;
}

int sk_graph_destroy(void* graph_exec) {
  if (!graph_exec) return SK_OK;
  const cudaError_t e = cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec));
  graph_destroyed();
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphExecDestroy");
  return SK_OK;
}

}  // extern "C"
