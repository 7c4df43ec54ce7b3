// Case-study per-object kernel (K5) on per_field planes.
//
// Reference: calibrate_collection / noise_for_collection
// (detector/schemas.py:29-41):
//   energy = A * counts.astype(f32) + B          (two f32 roundings, no FMA)
//   noise  = nA * sqrt(max(energy, 0)) + nB;  noise *= 2 where noisy
// numpy evaluates each operator separately, so every product and sum is rounded
// on its own (__fmul_rn / __fadd_rn keep ptxas from contracting into FFMA).
#include <algorithm>

#include "sk_internal.cuh"

namespace sk {
namespace sensor {

constexpr int NT = 256;
constexpr int VEC = 4;

__device__ __forceinline__ float calib(uint64_t c, float a, float b) { return sensor_energy(c, a, b); }

__device__ __forceinline__ float noise_of(float e, float na, float nb, bool noisy) {
  return sensor_noise(e, na, nb, noisy);
}

// Both kernels stream their planes with 16-byte accesses, U vector groups per
// thread per step with every load issued before any arithmetic, so each warp
// keeps U * (bytes per group) in flight (a grid-stride loop that loads one
// group at a time left noise at 0.85 of the copy peak with half the warps idle).
constexpr int U = 4;

__global__ void __launch_bounds__(NT) calibrate_kernel(int64_t n, const uint64_t* __restrict__ counts,
                                                       const float* __restrict__ a, const float* __restrict__ b,
                                                       float* __restrict__ energy, bool vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  int64_t tail = 0;
  if (vec) {
    const int64_t nv = n / VEC;
    for (int64_t i0 = t; i0 < nv; i0 += U * stride) {
      float4 av[U], bv[U];
      ulonglong2 c0[U], c1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = min(i0 + u * stride, nv - 1);  // clamped: in range, dropped at the store
        av[u] = __ldcs(reinterpret_cast<const float4*>(a) + i);
        bv[u] = __ldcs(reinterpret_cast<const float4*>(b) + i);
        c0[u] = __ldcs(reinterpret_cast<const ulonglong2*>(counts) + 2 * i);
        c1[u] = __ldcs(reinterpret_cast<const ulonglong2*>(counts) + 2 * i + 1);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= nv) break;
        float4 e;
        e.x = calib(c0[u].x, av[u].x, bv[u].x);
        e.y = calib(c0[u].y, av[u].y, bv[u].y);
        e.z = calib(c1[u].x, av[u].z, bv[u].z);
        e.w = calib(c1[u].y, av[u].w, bv[u].w);
        reinterpret_cast<float4*>(energy)[i] = e;
      }
    }
    tail = nv * VEC;
  }
  for (int64_t i = tail + t; i < n; i += stride) energy[i] = calib(counts[i], a[i], b[i]);
}

__global__ void __launch_bounds__(NT) noise_kernel(int64_t n, const float* __restrict__ energy,
                                                   const float* __restrict__ na, const float* __restrict__ nb,
                                                   const uint8_t* __restrict__ noisy, float* __restrict__ noise,
                                                   bool vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  int64_t tail = 0;
  if (vec) {
    const int64_t nv = n / VEC;
    for (int64_t i0 = t; i0 < nv; i0 += U * stride) {
      float4 e[U], av[U], bv[U];
      uint32_t q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = min(i0 + u * stride, nv - 1);
        e[u] = __ldcs(reinterpret_cast<const float4*>(energy) + i);
        av[u] = __ldcs(reinterpret_cast<const float4*>(na) + i);
        bv[u] = __ldcs(reinterpret_cast<const float4*>(nb) + i);
        q[u] = __ldcs(reinterpret_cast<const unsigned int*>(noisy) + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * stride;
        if (i >= nv) break;
        float4 o;
        o.x = noise_of(e[u].x, av[u].x, bv[u].x, q[u] & 0xff);
        o.y = noise_of(e[u].y, av[u].y, bv[u].y, (q[u] >> 8) & 0xff);
        o.z = noise_of(e[u].z, av[u].z, bv[u].z, (q[u] >> 16) & 0xff);
        o.w = noise_of(e[u].w, av[u].w, bv[u].w, q[u] >> 24);
        reinterpret_cast<float4*>(noise)[i] = o;
      }
    }
    tail = nv * VEC;
  }
  for (int64_t i = tail + t; i < n; i += stride) noise[i] = noise_of(energy[i], na[i], nb[i], noisy[i] != 0);
}

// ---- on-device event generation (detector/events.py:37-133) --------------------------

__device__ __forceinline__ uint64_t mix(uint64_t seed, uint64_t k) {  // output k of the stream (events.py:37-44)
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit53(uint64_t o) { return static_cast<double>(o >> 11) * 0x1p-53; }

struct GenArgs {
  int64_t w, h, n_dep;
  int nevents;
  double foot[25];
  uint8_t* type;
  uint64_t* counts;
  uint8_t* noisy;
  float *a, *b, *na, *nb, *energy;
};

constexpr int MAX_EVENTS_PER_LAUNCH = 256;
struct Seeds {
  uint64_t s[MAX_EVENTS_PER_LAUNCH];
};

// per-type calibration parameters, computed in double then rounded once to
// f32 exactly as numpy does for np.float32(0.3 + 0.7 * u) (events.py:89-95)
__device__ __forceinline__ void type_params(uint64_t seed, int t, float* pa, float* pb, float* pna, float* pnb) {
  *pa = __double2float_rn(__dadd_rn(0.3, __dmul_rn(0.7, unit53(mix(seed, 4 * t + 0)))));
  *pb = __double2float_rn(__dmul_rn(2.0, unit53(mix(seed, 4 * t + 1))));
  *pna = __double2float_rn(__dadd_rn(1.0, __dmul_rn(1.0, unit53(mix(seed, 4 * t + 2)))));
  *pnb = __double2float_rn(__dadd_rn(0.5, __dmul_rn(1.5, unit53(mix(seed, 4 * t + 3)))));
}

__global__ void __launch_bounds__(NT) gen_cells_kernel(const __grid_constant__ GenArgs G,
                                                       const __grid_constant__ Seeds S, int ev0) {
  const int e = ev0 + blockIdx.y;
  const uint64_t seed = S.s[blockIdx.y];
  __shared__ float pa[4], pb[4], pna[4], pnb[4];
  if (threadIdx.x < 4) type_params(seed, threadIdx.x, &pa[threadIdx.x], &pb[threadIdx.x], &pna[threadIdx.x],
                                   &pnb[threadIdx.x]);
  __syncthreads();
  const int64_t n = G.w * G.h;
  const int64_t base = static_cast<int64_t>(e) * n;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * NT) {
    const uint64_t k = 16 + 3 * static_cast<uint64_t>(i);
    const int t = static_cast<int>(mix(seed, k) & 3);
    const int64_t o = base + i;
    G.type[o] = static_cast<uint8_t>(t);
    G.counts[o] = mix(seed, k + 1) & 15;
    G.noisy[o] = (mix(seed, k + 2) % 50) == 0;
    G.a[o] = pa[t];
    G.b[o] = pb[t];
    G.na[o] = pna[t];
    G.nb[o] = pnb[t];
    G.energy[o] = 0.0f;
  }
}

// deposits: 5x5 truncated footprint added to counts (events.py:109-122);
// integer adds commute, so concurrent deposits use 64-bit atomics
__global__ void __launch_bounds__(NT) gen_deposits_kernel(const __grid_constant__ GenArgs G,
                                                          const __grid_constant__ Seeds S, int ev0) {
  const int e = ev0 + blockIdx.y;
  const uint64_t seed = S.s[blockIdx.y];
  const int64_t n = G.w * G.h;
  const int64_t d = static_cast<int64_t>(blockIdx.x) * (NT / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (d >= G.n_dep || lane >= 25) return;
  const uint64_t k = 16 + 3 * static_cast<uint64_t>(n) + 3 * static_cast<uint64_t>(d);
  const int64_t cx = static_cast<int64_t>(mix(seed, k) % static_cast<uint64_t>(G.w));
  const int64_t cy = static_cast<int64_t>(mix(seed, k + 1) % static_cast<uint64_t>(G.h));
  const int64_t amp = 500 + static_cast<int64_t>(mix(seed, k + 2) % 1500ull);
  const int dy = lane / 5 - 2, dx = lane % 5 - 2;
  const int64_t y = cy + dy, x = cx + dx;
  if (y < 0 || y >= G.h || x < 0 || x >= G.w) return;
  const uint64_t add = static_cast<uint64_t>(static_cast<int64_t>(__dmul_rn(static_cast<double>(amp), G.foot[lane])));
  atomicAdd(reinterpret_cast<unsigned long long*>(&G.counts[static_cast<int64_t>(e) * n + y * G.w + x]),
            static_cast<unsigned long long>(add));
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// one resident wave: every CTA streams its share with U groups in flight per thread
template <typename K>
static int grid_for(K kernel, int64_t n, int* grid) {
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* ds = nullptr;
  int rc = device_state(dev, &ds);
  if (rc) return rc;
  static int occ[64] = {0};
  int& o = occ[dev & 63];
  if (!o) {
    SK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, NT, 0));
    o = std::max(o, 1);
  }
  const int64_t want = (n / VEC + static_cast<int64_t>(NT) * U - 1) / (static_cast<int64_t>(NT) * U);
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(ds->sm_count) * o)));
  return SK_OK;
}

}  // namespace sensor
}  // namespace sk

using namespace sk;

extern "C" {

int sk_sensor_calibrate(int64_t n, const uint64_t* counts, const float* a, const float* b, float* energy,
                        uintptr_t stream) {
  if (n < 0) return set_error(SK_ERR_INVALID, "negative count");
  if (n == 0) return SK_OK;
  int grid = 1, dev = 0;
  int rc = sensor::grid_for(sensor::calibrate_kernel, n, &grid);
  if (rc) return rc;
  SK_TRY(cudaGetDevice(&dev));
  const bool vec = sensor::al16(counts) && sensor::al16(a) && sensor::al16(b) && sensor::al16(energy);
  sensor::calibrate_kernel<<<grid, sensor::NT, 0, resolve_stream(dev, stream)>>>(n, counts, a, b, energy, vec);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

int sk_sensor_noise(int64_t n, const float* energy, const float* na, const float* nb, const uint8_t* noisy,
                    float* noise, uintptr_t stream) {
  if (n < 0) return set_error(SK_ERR_INVALID, "negative count");
  if (n == 0) return SK_OK;
  int grid = 1, dev = 0;
  int rc = sensor::grid_for(sensor::noise_kernel, n, &grid);
  if (rc) return rc;
  SK_TRY(cudaGetDevice(&dev));
  const bool vec = sensor::al16(energy) && sensor::al16(na) && sensor::al16(nb) &&
                   (reinterpret_cast<uintptr_t>(noisy) & 3) == 0 && sensor::al16(noise);
  sensor::noise_kernel<<<grid, sensor::NT, 0, resolve_stream(dev, stream)>>>(n, energy, na, nb, noisy, noise, vec);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

int sk_sensor_generate(int64_t w, int64_t h, const uint64_t* seeds, int nevents, int64_t n_dep,
                       const double* footprint25, uint8_t* type, uint64_t* counts, uint8_t* noisy, float* a, float* b,
                       float* na, float* nb, float* energy, uintptr_t stream) {
  if (w < 1 || h < 1 || nevents < 0 || n_dep < 0) return set_error(SK_ERR_INVALID, "bad event geometry");
  if (nevents == 0) return SK_OK;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* ds = nullptr;
  int rc = device_state(dev, &ds);
  if (rc) return rc;
  cudaStream_t s = resolve_stream(dev, stream);
  sensor::GenArgs G;
  G.w = w;
  G.h = h;
  G.n_dep = n_dep;
  G.nevents = nevents;
  for (int i = 0; i < 25; ++i) G.foot[i] = footprint25[i];
  G.type = type;
  G.counts = counts;
  G.noisy = noisy;
  G.a = a;
  G.b = b;
  G.na = na;
  G.nb = nb;
  G.energy = energy;
  const int64_t n = w * h;
  for (int ev0 = 0; ev0 < nevents; ev0 += sensor::MAX_EVENTS_PER_LAUNCH) {
    const int cnt = std::min(nevents - ev0, sensor::MAX_EVENTS_PER_LAUNCH);
    sensor::Seeds S;
    for (int i = 0; i < cnt; ++i) S.s[i] = seeds[ev0 + i];
    const int64_t bx = std::min<int64_t>((n + sensor::NT - 1) / sensor::NT, std::max(1, ds->sm_count * 8 / cnt));
    sensor::gen_cells_kernel<<<dim3(static_cast<unsigned>(std::max<int64_t>(bx, 1)), cnt), sensor::NT, 0, s>>>(
        G, S, ev0);
    SK_TRY(cudaGetLastError());
    if (n_dep) {
      const int64_t dx = (n_dep + sensor::NT / 32 - 1) / (sensor::NT / 32);
      sensor::gen_deposits_kernel<<<dim3(static_cast<unsigned>(dx), cnt), sensor::NT, 0, s>>>(G, S, ev0);
      SK_TRY(cudaGetLastError());
    }
  }
  return SK_OK;
}

}  // extern "C"
