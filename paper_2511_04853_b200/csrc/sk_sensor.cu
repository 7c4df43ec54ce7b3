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

__global__ void __launch_bounds__(NT) calibrate_kernel(int64_t n, const uint64_t* __restrict__ counts,
                                                       const float* __restrict__ a, const float* __restrict__ b,
                                                       float* __restrict__ energy, bool vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  if (vec) {
    const int64_t nv = n / VEC;
    for (; i < nv; i += stride) {
      const float4 av = reinterpret_cast<const float4*>(a)[i];
      const float4 bv = reinterpret_cast<const float4*>(b)[i];
      const ulonglong2 c0 = reinterpret_cast<const ulonglong2*>(counts)[2 * i];
      const ulonglong2 c1 = reinterpret_cast<const ulonglong2*>(counts)[2 * i + 1];
      float4 e;
      e.x = calib(c0.x, av.x, bv.x);
      e.y = calib(c0.y, av.y, bv.y);
      e.z = calib(c1.x, av.z, bv.z);
      e.w = calib(c1.y, av.w, bv.w);
      reinterpret_cast<float4*>(energy)[i] = e;
    }
    i = nv * VEC + (static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x);
  }
  for (; i < n; i += stride) energy[i] = calib(counts[i], a[i], b[i]);
}

__global__ void __launch_bounds__(NT) noise_kernel(int64_t n, const float* __restrict__ energy,
                                                   const float* __restrict__ na, const float* __restrict__ nb,
                                                   const uint8_t* __restrict__ noisy, float* __restrict__ noise,
                                                   bool vec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x;
  if (vec) {
    const int64_t nv = n / VEC;
    for (; i < nv; i += stride) {
      const float4 e = reinterpret_cast<const float4*>(energy)[i];
      const float4 av = reinterpret_cast<const float4*>(na)[i];
      const float4 bv = reinterpret_cast<const float4*>(nb)[i];
      const uint32_t q = reinterpret_cast<const uint32_t*>(noisy)[i];
      float4 o;
      o.x = noise_of(e.x, av.x, bv.x, q & 0xff);
      o.y = noise_of(e.y, av.y, bv.y, (q >> 8) & 0xff);
      o.z = noise_of(e.z, av.z, bv.z, (q >> 16) & 0xff);
      o.w = noise_of(e.w, av.w, bv.w, q >> 24);
      reinterpret_cast<float4*>(noise)[i] = o;
    }
    i = nv * VEC + (static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x);
  }
  for (; i < n; i += stride) noise[i] = noise_of(energy[i], na[i], nb[i], noisy[i] != 0);
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int grid_for(int64_t n, int* grid) {
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* ds = nullptr;
  int rc = device_state(dev, &ds);
  if (rc) return rc;
  const int64_t want = (n / VEC + NT - 1) / NT;
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(ds->sm_count) * 8)));
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
  int rc = sensor::grid_for(n, &grid);
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
  int rc = sensor::grid_for(n, &grid);
  if (rc) return rc;
  SK_TRY(cudaGetDevice(&dev));
  const bool vec = sensor::al16(energy) && sensor::al16(na) && sensor::al16(nb) &&
                   (reinterpret_cast<uintptr_t>(noisy) & 3) == 0 && sensor::al16(noise);
  sensor::noise_kernel<<<grid, sensor::NT, 0, resolve_stream(dev, stream)>>>(n, energy, na, nb, noisy, noise, vec);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

}  // extern "C"
