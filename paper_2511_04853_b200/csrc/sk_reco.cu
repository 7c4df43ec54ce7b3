// Particle reconstruction on the B200.
//
// Reference: reconstruct_arrays (detector/reconstruct.py:53-136) walks seeds
// (ratio > 5) in descending energy / ascending index; an unconsumed seed takes
// the unconsumed ratio > 2 cells of its grid-clipped 5x5 window. The walk is
// sequential, but two seeds interact only when their windows overlap
// (Chebyshev distance <= 4). Round-synchronous parallel greedy reproduces it
// exactly: in a round, a pending seed is READY when no pending seed of higher
// priority lies within distance 4; ready seeds have pairwise disjoint windows
// and every seed that could have affected them is already decided, so they are
// processed concurrently with the same outcome as the sequential walk. A seed
// consumed by another is decided (skipped) at once. Per-particle sums run in
// one thread in the reference's order (f64, row-major contributors), so the
// attributes are bit-identical; particles are finally ordered by priority.
// The one approximation: the reference squares deviations with Python's
// `x ** 2` (glibc pow) and this kernel with x * x; they differ by <= 1 ulp of
// a double in ~0.1% of cases, which reaches the float32 variance only when the
// double lies within 1e-16 of an f32 rounding boundary.
#include <algorithm>
#include <vector>

#include "sk_internal.cuh"

namespace sk {
namespace reco {

constexpr int NT = 256;
constexpr int MAXC = 25;  // contributors per particle (5x5 window)

enum : uint8_t { NONE = 0, PENDING = 1, DECIDED = 2 };

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

struct Slot {  // one reconstructed particle, before ordering
  float energy, x, y, xvar, yvar;
  float sig[4], ec[4];
  uint8_t nc[4];
  int32_t nsens;
  int32_t event;
  int64_t origin;  // seed flat index inside its event
  float key_e;     // priority: energy desc, then origin asc
};

struct Args {
  int64_t w, h, n;  // n = cells per event
  int nevents;
  const float* energy;
  const float* noise;
  const uint8_t* type;
  const uint8_t* noisy;
  float* ratio;
  uint8_t* state;
  uint8_t* consumed;
  int64_t* cand;
  unsigned long long* counters;  // [0] ncand [1] nready [2] pending [3] nparticles
  int64_t* ready;
  Slot* slots;
  uint64_t* contrib;  // MAXC per slot
  unsigned long long* event_count;
};

// appends: one atomic per warp instead of one per lane (a single counter shared
// by the whole grid serialises in L2 otherwise); returns this lane's slot if `take`
__device__ __forceinline__ unsigned long long warp_append(unsigned long long* ctr, bool take) {
  const unsigned m = __ballot_sync(__activemask(), take);
  if (!m) return 0;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(__activemask(), base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ bool higher(const Args& A, int64_t q, int64_t c) {
  const float eq = A.energy[q], ec = A.energy[c];
  return eq > ec || (eq == ec && q < c);  // argsort(-energy, stable) over ascending candidates
}

__global__ void init_kernel(Args A) {
  const int64_t total = A.n * A.nevents;
  // whole warps iterate together (the candidate append is warp-aggregated)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * NT + (threadIdx.x & ~31); i0 < total; i0 += stride) {
    const int64_t i = i0 + (threadIdx.x & 31);
    bool seed = false;
    if (i < total) {
      const float r = __fdiv_rn(A.energy[i], A.noise[i]);  // numpy f32 division (IEEE)
      A.ratio[i] = r;
      A.consumed[i] = 0;
      seed = r > 5.0f;
      A.state[i] = seed ? PENDING : NONE;
    }
    const unsigned long long slot = warp_append(&A.counters[0], seed);
    if (seed) A.cand[slot] = i;
  }
}

// phase 1 of a round: which pending seeds are ready
__global__ void ready_kernel(Args A) {
  const int64_t ncand = static_cast<int64_t>(A.counters[0]);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t k0 = static_cast<int64_t>(blockIdx.x) * NT + (threadIdx.x & ~31); k0 < ncand; k0 += stride) {
    const int64_t k = k0 + (threadIdx.x & 31);
    const int64_t c = k < ncand ? A.cand[k] : 0;
    const bool pend = k < ncand && A.state[c] == PENDING;
    bool ok = pend;
    if (pend) {
      const int64_t base = (c / A.n) * A.n, loc = c - base;
      const int64_t cy = loc / A.w, cx = loc - cy * A.w;
      for (int64_t y = imax64(0, cy - 4); ok && y <= imin64(A.h - 1, cy + 4); ++y)
        for (int64_t x = imax64(0, cx - 4); x <= imin64(A.w - 1, cx + 4); ++x) {
          const int64_t q = base + y * A.w + x;
          if (q != c && A.state[q] == PENDING && higher(A, q, c)) {
            ok = false;
            break;
          }
        }
    }
    warp_append(&A.counters[2], pend);
    const unsigned long long slot = warp_append(&A.counters[1], ok);
    if (ok) A.ready[slot] = c;
  }
}

// phase 2 of a round: process the ready seeds (pairwise disjoint windows)
__global__ void process_kernel(Args A) {
  const int64_t nready = static_cast<int64_t>(A.counters[1]);
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; k < nready;
       k += static_cast<int64_t>(gridDim.x) * NT) {
    const int64_t s = A.ready[k];
    if (A.consumed[s]) {  // taken by an earlier particle: the reference skips it
      A.state[s] = DECIDED;
      continue;
    }
    const int64_t ev = s / A.n, base = ev * A.n, loc = s - base;
    const int64_t sy = loc / A.w, sx = loc - sy * A.w;
    int64_t con[MAXC];
    int nc = 0;
    for (int64_t y = imax64(0, sy - 2); y <= imin64(A.h - 1, sy + 2); ++y)
      for (int64_t x = imax64(0, sx - 2); x <= imin64(A.w - 1, sx + 2); ++x) {
        const int64_t f = base + y * A.w + x;
        if (!A.consumed[f] && A.ratio[f] > 2.0f) {
          A.consumed[f] = 1;
          if (A.state[f] == PENDING && f != s) A.state[f] = DECIDED;  // a consumed seed is always skipped
          con[nc++] = f;
        }
      }
    // reconstruct.py:84-117, same operation order (no FMA: -fmad=false)
    double e64[4] = {0, 0, 0, 0}, sig64[4] = {0, 0, 0, 0};
    int cnt[4] = {0, 0, 0, 0};
    double sw = 0, swx = 0, swy = 0;
    for (int i = 0; i < nc; ++i) {
      const int64_t f = con[i], lf = f - base;
      const double e = static_cast<double>(A.energy[f]);
      const int t = A.type[f] & 3;
      e64[t] = __dadd_rn(e64[t], e);
      sig64[t] = __dadd_rn(sig64[t], static_cast<double>(A.ratio[f]));
      if (A.noisy[f]) ++cnt[t];
      sw = __dadd_rn(sw, e);
      swx = __dadd_rn(swx, __dmul_rn(e, static_cast<double>(lf % A.w)));
      swy = __dadd_rn(swy, __dmul_rn(e, static_cast<double>(lf / A.w)));
    }
    const double xbar = __ddiv_rn(swx, sw), ybar = __ddiv_rn(swy, sw);
    double vx = 0, vy = 0;
    for (int i = 0; i < nc; ++i) {
      const int64_t lf = con[i] - base;
      const double e = static_cast<double>(A.energy[con[i]]);
      const double dx = __dsub_rn(static_cast<double>(lf % A.w), xbar);
      const double dy = __dsub_rn(static_cast<double>(lf / A.w), ybar);
      vx = __dadd_rn(vx, __dmul_rn(e, __dmul_rn(dx, dx)));
      vy = __dadd_rn(vy, __dmul_rn(e, __dmul_rn(dy, dy)));
    }
    const unsigned long long p = atomicAdd(&A.counters[3], 1ull);
    Slot& S = A.slots[p];
    float e32[4];
    for (int t = 0; t < 4; ++t) {
      e32[t] = __double2float_rn(e64[t]);
      S.ec[t] = e32[t];
      S.sig[t] = __double2float_rn(sig64[t]);
      S.nc[t] = static_cast<uint8_t>(cnt[t]);
    }
    S.energy = __double2float_rn(__dadd_rn(__dadd_rn(__dadd_rn(static_cast<double>(e32[0]), static_cast<double>(e32[1])),
                                                      static_cast<double>(e32[2])),
                                            static_cast<double>(e32[3])));
    S.x = __double2float_rn(xbar);
    S.y = __double2float_rn(ybar);
    S.xvar = __double2float_rn(__ddiv_rn(vx, sw));
    S.yvar = __double2float_rn(__ddiv_rn(vy, sw));
    S.nsens = nc;
    S.event = static_cast<int32_t>(ev);
    S.origin = loc;
    S.key_e = A.energy[s];
    for (int i = 0; i < nc; ++i) A.contrib[p * MAXC + i] = static_cast<uint64_t>(con[i] - base);
    atomicAdd(&A.event_count[ev], 1ull);
    A.state[s] = DECIDED;
  }
}

// order: bucket particles by event, then rank by priority inside the event
__global__ void bucket_kernel(const Slot* slots, int64_t np, const int64_t* event_off,
                              unsigned long long* cursor, int64_t* order) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; p < np;
       p += static_cast<int64_t>(gridDim.x) * NT) {
    const int e = slots[p].event;
    order[event_off[e] + static_cast<int64_t>(atomicAdd(&cursor[e], 1ull))] = p;
  }
}

struct OutArgs {
  float *energy, *x, *y, *xvar, *yvar;
  uint64_t* origin;
  float* sig[4];
  float* ec[4];
  uint8_t* nc[4];
  int32_t* lens;
  int64_t* offsets;
};

constexpr int RANK_SMEM = 4096;  // particles of one event ranked out of shared memory

// one CTA per event: the event's priority keys go to smem (broadcast reads),
// each particle's rank = how many keys outrank it; events with more particles
// than RANK_SMEM read the keys from global memory instead
__global__ void __launch_bounds__(NT) write_kernel(const Slot* slots, const int64_t* event_off,
                                                   const int64_t* event_cnt, const int64_t* order, OutArgs O) {
  __shared__ float ke[RANK_SMEM];
  __shared__ int64_t ko[RANK_SMEM];
  const int64_t ev = blockIdx.x;
  const int64_t b = event_off[ev], m = event_cnt[ev];
  const bool in_smem = m <= RANK_SMEM;
  if (in_smem)
    for (int64_t j = threadIdx.x; j < m; j += NT) {
      const Slot& Q = slots[order[b + j]];
      ke[j] = Q.key_e;
      ko[j] = Q.origin;
    }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < m; i += NT) {
    const int64_t p = order[b + i];
    const Slot& S = slots[p];
    const float se = S.key_e;
    const int64_t so = S.origin;
    int64_t rank = 0;
    if (in_smem) {
      for (int64_t j = 0; j < m; ++j) rank += (ke[j] > se) || (ke[j] == se && ko[j] < so);
    } else {
      for (int64_t j = 0; j < m; ++j) {
        const Slot& Q = slots[order[b + j]];
        rank += (Q.key_e > se) || (Q.key_e == se && Q.origin < so);
      }
    }
    const int64_t o = b + rank;
    O.energy[o] = S.energy;
    O.x[o] = S.x;
    O.y[o] = S.y;
    O.xvar[o] = S.xvar;
    O.yvar[o] = S.yvar;
    O.origin[o] = static_cast<uint64_t>(S.origin);
    for (int t = 0; t < 4; ++t) {
      O.sig[t][o] = S.sig[t];
      O.ec[t][o] = S.ec[t];
      O.nc[t][o] = S.nc[t];
    }
    O.lens[o] = S.nsens;
    O.offsets[o] = p * MAXC;
  }
}

struct Handle {
  int device = 0;
  int64_t w = 0, h = 0, n = 0;
  int nevents = 0;
  int64_t np = 0;
  void* ws = nullptr;
  Args A;
  std::vector<int64_t> counts;
};

}  // namespace reco
}  // namespace sk

using namespace sk;

extern "C" {

int sk_reco_run(int64_t w, int64_t h, int nevents, const float* energy, const float* noise, const uint8_t* type,
                const uint8_t* noisy, int device, uintptr_t stream, void** handle, int64_t* nparticles,
                int* rounds) {
  if (!handle || w < 1 || h < 1 || nevents < 0) return set_error(SK_ERR_INVALID, "bad reconstruction arguments");
  DeviceState* ds = nullptr;
  int rc = device_state(device, &ds);
  if (rc) return rc;
  cudaStream_t s = resolve_stream(device, stream);
  auto* H = new reco::Handle();
  H->device = device;
  H->w = w;
  H->h = h;
  H->n = w * h;
  H->nevents = nevents;
  const int64_t total = H->n * nevents;
  // workspace: ratio f32 | state u8 | consumed u8 | cand i64 | ready i64 | counters | event counts
  const size_t sz_ratio = static_cast<size_t>(total) * 4, sz_u8 = static_cast<size_t>(total);
  const size_t sz_idx = static_cast<size_t>(total) * 8, sz_cnt = 64, sz_ev = static_cast<size_t>(nevents + 1) * 8;
  auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
  const size_t ws = al(sz_ratio) + 2 * al(sz_u8) + 2 * al(sz_idx) + al(sz_cnt) + al(sz_ev);
  cudaError_t e = cudaMallocAsync(&H->ws, ws, s);
  if (e != cudaSuccess) {
    delete H;
    return cuda_fail(e, "cudaMallocAsync(reconstruction workspace)");
  }
  uint8_t* p = static_cast<uint8_t*>(H->ws);
  reco::Args& A = H->A;
  memset(&A, 0, sizeof(A));
  A.w = w; A.h = h; A.n = H->n; A.nevents = nevents;
  A.energy = energy; A.noise = noise; A.type = type; A.noisy = noisy;
  A.ratio = reinterpret_cast<float*>(p); p += al(sz_ratio);
  A.state = p; p += al(sz_u8);
  A.consumed = p; p += al(sz_u8);
  A.cand = reinterpret_cast<int64_t*>(p); p += al(sz_idx);
  A.ready = reinterpret_cast<int64_t*>(p); p += al(sz_idx);
  A.counters = reinterpret_cast<unsigned long long*>(p); p += al(sz_cnt);
  A.event_count = reinterpret_cast<unsigned long long*>(p);
  SK_TRY(cudaMemsetAsync(A.counters, 0, sz_cnt, s));
  SK_TRY(cudaMemsetAsync(A.event_count, 0, sz_ev, s));
  const int grid = std::max(1, std::min<int>(ds->sm_count * 8, static_cast<int>((total + reco::NT - 1) / reco::NT)));
  if (total) reco::init_kernel<<<grid, reco::NT, 0, s>>>(A);
  SK_TRY(cudaGetLastError());
  unsigned long long ncand = 0;
  SK_TRY(cudaMemcpyAsync(&ncand, &A.counters[0], 8, cudaMemcpyDeviceToHost, s));
  SK_TRY(cudaStreamSynchronize(s));
  // particle slots: at most one per seed
  e = cudaMallocAsync(reinterpret_cast<void**>(&A.slots), std::max<size_t>(1, ncand) * sizeof(reco::Slot), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(reinterpret_cast<void**>(&A.contrib), std::max<size_t>(1, ncand) * reco::MAXC * 8, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(particle slots)");
  const int cgrid = std::max(1, std::min<int>(ds->sm_count * 8, static_cast<int>((ncand + reco::NT - 1) / reco::NT)));
  int r = 0;
  unsigned long long pending = ncand;
  while (pending) {
    for (int k = 0; k < 4; ++k, ++r) {  // four rounds per host check
      SK_TRY(cudaMemsetAsync(&A.counters[1], 0, 16, s));  // nready, pending
      reco::ready_kernel<<<cgrid, reco::NT, 0, s>>>(A);
      reco::process_kernel<<<cgrid, reco::NT, 0, s>>>(A);
    }
    SK_TRY(cudaGetLastError());
    SK_TRY(cudaMemcpyAsync(&pending, &A.counters[2], 8, cudaMemcpyDeviceToHost, s));
    SK_TRY(cudaStreamSynchronize(s));
  }
  unsigned long long np = 0;
  SK_TRY(cudaMemcpyAsync(&np, &A.counters[3], 8, cudaMemcpyDeviceToHost, s));
  H->counts.assign(nevents, 0);
  std::vector<unsigned long long> ec(nevents > 0 ? nevents : 1);
  if (nevents) SK_TRY(cudaMemcpyAsync(ec.data(), A.event_count, nevents * 8, cudaMemcpyDeviceToHost, s));
  SK_TRY(cudaStreamSynchronize(s));
  for (int i = 0; i < nevents; ++i) H->counts[i] = static_cast<int64_t>(ec[i]);
  H->np = static_cast<int64_t>(np);
  *nparticles = H->np;
  if (rounds) *rounds = r;
  *handle = H;
  return SK_OK;
}

int sk_reco_event_counts(void* handle, int64_t* counts) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H) return set_error(SK_ERR_INVALID, "null handle");
  for (int i = 0; i < H->nevents; ++i) counts[i] = H->counts[i];
  return SK_OK;
}

int sk_reco_write(void* handle, float* energy, float* x, float* y, uint64_t* origin, float* x_variance,
                  float* y_variance, float* const* significance, float* const* e_contribution,
                  uint8_t* const* noisy_count, int32_t* sensor_lens, int64_t* sensor_offsets,
                  const uint64_t** sensor_pool, uintptr_t stream) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H) return set_error(SK_ERR_INVALID, "null handle");
  DeviceState* ds = nullptr;
  int rc = device_state(H->device, &ds);
  if (rc) return rc;
  cudaStream_t s = resolve_stream(H->device, stream);
  if (sensor_pool) *sensor_pool = H->A.contrib;
  if (H->np == 0) return SK_OK;
  std::vector<int64_t> off(H->nevents + 1, 0);
  for (int i = 0; i < H->nevents; ++i) off[i + 1] = off[i] + H->counts[i];
  int64_t *d_off = nullptr, *d_cnt = nullptr, *order = nullptr;
  unsigned long long* cursor = nullptr;
  const size_t ev_bytes = static_cast<size_t>(H->nevents + 1) * 8;
  SK_TRY(cudaMallocAsync(&d_off, ev_bytes, s));
  SK_TRY(cudaMallocAsync(&d_cnt, ev_bytes, s));
  SK_TRY(cudaMallocAsync(&cursor, ev_bytes, s));
  SK_TRY(cudaMallocAsync(&order, static_cast<size_t>(H->np) * 8, s));
  SK_TRY(cudaMemcpyAsync(d_off, off.data(), ev_bytes, cudaMemcpyHostToDevice, s));
  SK_TRY(cudaMemcpyAsync(d_cnt, H->counts.data(), H->nevents * 8, cudaMemcpyHostToDevice, s));
  SK_TRY(cudaMemsetAsync(cursor, 0, ev_bytes, s));
  const int grid = std::max(1, std::min<int>(ds->sm_count * 8, static_cast<int>((H->np + reco::NT - 1) / reco::NT)));
  reco::bucket_kernel<<<grid, reco::NT, 0, s>>>(H->A.slots, H->np, d_off, cursor, order);
  reco::OutArgs O;
  O.energy = energy; O.x = x; O.y = y; O.xvar = x_variance; O.yvar = y_variance; O.origin = origin;
  for (int t = 0; t < 4; ++t) {
    O.sig[t] = significance[t];
    O.ec[t] = e_contribution[t];
    O.nc[t] = noisy_count[t];
  }
  O.lens = sensor_lens;
  O.offsets = sensor_offsets;
  if (H->nevents) reco::write_kernel<<<H->nevents, reco::NT, 0, s>>>(H->A.slots, d_off, d_cnt, order, O);
  SK_TRY(cudaGetLastError());
  cudaFreeAsync(d_off, s);
  cudaFreeAsync(d_cnt, s);
  cudaFreeAsync(cursor, s);
  cudaFreeAsync(order, s);
  return SK_OK;
}

int sk_reco_free(void* handle, uintptr_t stream) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H) return SK_OK;
  cudaStream_t s = resolve_stream(H->device, stream);
  if (H->A.slots) cudaFreeAsync(H->A.slots, s);
  if (H->A.contrib) cudaFreeAsync(H->A.contrib, s);
  if (H->ws) cudaFreeAsync(H->ws, s);
  delete H;
  return SK_OK;
}

}  // extern "C"
