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
#include <cstdio>
#include <cstdlib>
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
  // [0] ncand [1] nready (this round) [2] next pending list size [3] current pending list size
  // [4] this round's first slot [5] pending seeds seen this round [6] rounds
  unsigned long long* counters;
  int64_t* ready;
  int64_t* list[2];  // seeds (cell indices) still pending: this round's list and the next one's
  Slot* slots;
  uint64_t* contrib;  // MAXC per slot
  unsigned long long* event_count;
};

__device__ __forceinline__ bool higher(const Args& A, int64_t q, int64_t c) {
  const float eq = A.energy[q], ec = A.energy[c];
  return eq > ec || (eq == ec && q < c);  // argsort(-energy, stable) over ascending candidates
}

constexpr int SEED_CAP = 2048;  // seeds a CTA collects in smem before one global append

// ratio / state / consumed for every cell, and the seed (candidate) list. A CTA
// streams one contiguous range of cells (4 independent loads in flight per
// thread), collects its seeds in smem and appends them with ONE global atomic
// (a counter shared by the grid serialises at hundreds of thousands of atomics).
__global__ void __launch_bounds__(NT) init_kernel(Args A) {
  __shared__ int64_t seeds[SEED_CAP];
  __shared__ unsigned s_n;
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  const int64_t total = A.n * A.nevents;
  const int64_t chunk = ((total + gridDim.x - 1) / gridDim.x + 4 * NT - 1) / (4 * NT) * (4 * NT);
  const int64_t start = static_cast<int64_t>(blockIdx.x) * chunk, end = min(total, start + chunk);
  for (int64_t c0 = start; c0 < end; c0 += 4 * NT) {
    float e[4], nz[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = c0 + u * NT + threadIdx.x;
      e[u] = i < end ? A.energy[i] : 0.0f;
      nz[u] = i < end ? A.noise[i] : 1.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = c0 + u * NT + threadIdx.x;
      if (i < end) {
        const float r = __fdiv_rn(e[u], nz[u]);  // numpy f32 division (IEEE)
        A.ratio[i] = r;
        A.consumed[i] = 0;
        const bool seed = r > 5.0f;
        A.state[i] = seed ? PENDING : NONE;
        if (seed) {
          const unsigned pos = atomicAdd(&s_n, 1u);
          if (pos < SEED_CAP)
            seeds[pos] = i;
          else
            A.cand[atomicAdd(&A.counters[0], 1ull)] = i;  // an unusually dense range: straight to global
        }
      }
    }
  }
  __syncthreads();
  const unsigned m = min(s_n, static_cast<unsigned>(SEED_CAP));
  if (threadIdx.x == 0) s_base = m ? atomicAdd(&A.counters[0], static_cast<unsigned long long>(m)) : 0ull;
  __syncthreads();
  for (unsigned j = threadIdx.x; j < m; j += NT) A.cand[s_base + j] = seeds[j];
}

__device__ __forceinline__ unsigned long long ctr(const Args& A, int k) { return A.counters[k]; }

// phase 1 of a round, over the candidates still pending (a list that shrinks
// every round): a candidate consumed meanwhile drops out; one with a pending
// seed of higher priority within distance 4 goes to the next round's list;
// the rest are ready. Its 9x9 neighbourhood is scanned a row (9 independent
// loads) at a time; counts and appends are aggregated per warp. Every kernel
// of a round returns at once when nothing is pending any more, so the host
// queues rounds without checking in between.
__global__ void __launch_bounds__(NT) ready_kernel(Args A, int parity) {
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(ctr(A, 3));
  const int64_t* cur = A.list[parity];
  int64_t* nxt = A.list[parity ^ 1];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * NT + (threadIdx.x & ~31); i0 < m; i0 += stride) {
    const int64_t i = i0 + lane;
    const int64_t c = i < m ? cur[i] : 0;  // cells, not candidate indices: one dependent load less
    const bool pend = i < m && A.state[c] == PENDING;
    bool ok = pend;
    if (pend) {
      const int64_t base = (c / A.n) * A.n, loc = c - base;
      const int64_t cy = loc / A.w, cx = loc - cy * A.w;
      const int64_t x0 = imax64(0, cx - 4), x1 = imin64(A.w - 1, cx + 4);
      for (int64_t y = imax64(0, cy - 4); ok && y <= imin64(A.h - 1, cy + 4); ++y) {
        uint8_t st[9];
#pragma unroll
        for (int d = 0; d < 9; ++d) st[d] = x0 + d <= x1 ? A.state[base + y * A.w + x0 + d] : NONE;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
          const int64_t q = base + y * A.w + x0 + d;
          if (st[d] == PENDING && q != c && higher(A, q, c)) ok = false;
        }
      }
    }
    const bool wait = pend && !ok;
    const unsigned pm = __ballot_sync(0xffffffffu, pend), rm = __ballot_sync(0xffffffffu, ok);
    const unsigned wm = __ballot_sync(0xffffffffu, wait);
    unsigned long long rb = 0, wb = 0;
    if (lane == 0) {
      if (pm) atomicAdd(&A.counters[5], static_cast<unsigned long long>(__popc(pm)));
      if (rm) rb = atomicAdd(&A.counters[1], static_cast<unsigned long long>(__popc(rm)));
      if (wm) wb = atomicAdd(&A.counters[2], static_cast<unsigned long long>(__popc(wm)));
    }
    rb = __shfl_sync(0xffffffffu, rb, 0);
    wb = __shfl_sync(0xffffffffu, wb, 0);
    const unsigned below = (1u << lane) - 1u;
    if (ok) A.ready[rb + __popc(rm & below)] = c;
    if (wait) nxt[wb + __popc(wm & below)] = c;
  }
}

// phase 2 of a round: process the ready seeds (pairwise disjoint windows).
// A warp takes 32 ready seeds at a time in two steps:
//  1. for each of them in turn, lane l < 25 examines window cell
//     (l / 5 - 2, l % 5 - 2): every load in one round trip, the taken cells
//     marked consumed, the contributor list written, and the cell values kept
//     in shared memory;
//  2. lane j adds up seed j's contributors in the reference's row-major order
//     (reconstruct.py:84-117), f64 and no FMA, so every sum is bit-identical to
//     the sequential walk -- 32 particles' sums side by side instead of one
//     warp replaying one particle's serial sums.
constexpr int PNT = 128;             // process threads per CTA
constexpr int PW = PNT / 32;         // warps per CTA
constexpr unsigned SKIPPED = ~0u;    // window mask of a seed consumed before its turn

struct WinSmem {
  float e[32][25], r[32][25];
  uint8_t t[32][25], nz[32][25];
  unsigned mask[32];
};

__global__ void __launch_bounds__(PNT) process_kernel(Args A) {
  __shared__ WinSmem W[PW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WinSmem& S = W[wid];
  const int64_t nready = static_cast<int64_t>(ctr(A, 1));
  const unsigned long long slot0 = ctr(A, 4);
  // seeds per warp batch: spread over every warp of the grid (the window step is serial per warp)
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * PW;
  const int64_t per = max(static_cast<int64_t>(1), min(static_cast<int64_t>(32), (nready + nwarps - 1) / nwarps));
  const int64_t stride = nwarps * per;
  for (int64_t k0 = (static_cast<int64_t>(blockIdx.x) * PW + wid) * per; k0 < nready; k0 += stride) {
    const int nb = static_cast<int>(min(per, nready - k0));
    for (int j = 0; j < nb; ++j) {  // 1. windows, one seed at a time
      const int64_t s = A.ready[k0 + j];
      const unsigned long long p = slot0 + static_cast<unsigned long long>(k0 + j);
      const int64_t base = (s / A.n) * A.n, loc = s - base;
      const int64_t sy = loc / A.w, sx = loc - sy * A.w;
      const int64_t y = sy + lane / 5 - 2, x = sx + lane % 5 - 2;
      const bool inwin = lane < 25 && y >= 0 && y < A.h && x >= 0 && x < A.w;
      const int64_t f = inwin ? base + y * A.w + x : s;
      const uint8_t used = A.consumed[f];
      const float r32 = A.ratio[f], e32 = A.energy[f];
      const uint8_t t = A.type[f] & 3, nz = A.noisy[f] != 0;
      // lane 12 is the seed itself (window centre): consumed by an earlier particle -> skipped
      if (__shfl_sync(0xffffffffu, used, 12)) {
        if (lane == 0) {
          A.state[s] = DECIDED;
          A.slots[p].event = -1;
          S.mask[j] = SKIPPED;
        }
        continue;
      }
      const bool take = inwin && !used && r32 > 2.0f;
      __syncwarp();  // every lane has read `consumed` before any marks it
      if (take) {
        A.consumed[f] = 1;
        if (f != s && A.state[f] == PENDING) A.state[f] = DECIDED;  // a consumed seed is always skipped
      }
      const unsigned mask = __ballot_sync(0xffffffffu, take);
      if (take) {  // contributor list, row-major: rank of this lane among the taken ones
        A.contrib[p * MAXC + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint64_t>(f - base);
      }
      if (lane < 25) {
        S.e[j][lane] = e32;
        S.r[j][lane] = r32;
        S.t[j][lane] = t;
        S.nz[j][lane] = nz;
      }
      if (lane == 0) S.mask[j] = mask;
    }
    __syncwarp();
    // 2. sums, lane j for seed j
    if (lane < nb && S.mask[lane] != SKIPPED) {
      const int j = lane;
      const int64_t s = A.ready[k0 + j];
      const unsigned long long p = slot0 + static_cast<unsigned long long>(k0 + j);
      const int64_t ev = s / A.n, loc = s - ev * A.n;
      const int64_t sy = loc / A.w, sx = loc - sy * A.w;
      const unsigned mask = S.mask[j];
      double e64[4] = {0, 0, 0, 0}, sig64[4] = {0, 0, 0, 0};
      int cnt[4] = {0, 0, 0, 0};
      double sw = 0, swx = 0, swy = 0;
      for (unsigned m = mask; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const double e = static_cast<double>(S.e[j][i]);
        const double ri = static_cast<double>(S.r[j][i]);
        const int ti = S.t[j][i], ni = S.nz[j][i];
        const double xi = static_cast<double>(sx + i % 5 - 2), yi = static_cast<double>(sy + i / 5 - 2);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (ti == q) {
            e64[q] = __dadd_rn(e64[q], e);
            sig64[q] = __dadd_rn(sig64[q], ri);
            cnt[q] += ni;
          }
        }
        sw = __dadd_rn(sw, e);
        swx = __dadd_rn(swx, __dmul_rn(e, xi));
        swy = __dadd_rn(swy, __dmul_rn(e, yi));
      }
      const double xbar = __ddiv_rn(swx, sw), ybar = __ddiv_rn(swy, sw);
      double vx = 0, vy = 0;
      for (unsigned m = mask; m; m &= m - 1) {
        const int i = __ffs(m) - 1;
        const double e = static_cast<double>(S.e[j][i]);
        const double dx = __dsub_rn(static_cast<double>(sx + i % 5 - 2), xbar);
        const double dy = __dsub_rn(static_cast<double>(sy + i / 5 - 2), ybar);
        vx = __dadd_rn(vx, __dmul_rn(e, __dmul_rn(dx, dx)));
        vy = __dadd_rn(vy, __dmul_rn(e, __dmul_rn(dy, dy)));
      }
      Slot& P = A.slots[p];
      float c32[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        c32[q] = __double2float_rn(e64[q]);
        P.ec[q] = c32[q];
        P.sig[q] = __double2float_rn(sig64[q]);
        P.nc[q] = static_cast<uint8_t>(cnt[q]);
      }
      P.energy = __double2float_rn(__dadd_rn(
          __dadd_rn(__dadd_rn(static_cast<double>(c32[0]), static_cast<double>(c32[1])), static_cast<double>(c32[2])),
          static_cast<double>(c32[3])));
      P.x = __double2float_rn(xbar);
      P.y = __double2float_rn(ybar);
      P.xvar = __double2float_rn(__ddiv_rn(vx, sw));
      P.yvar = __double2float_rn(__ddiv_rn(vy, sw));
      P.nsens = __popc(mask);
      P.event = static_cast<int32_t>(ev);
      P.origin = loc;
      P.key_e = A.energy[s];
      atomicAdd(&A.event_count[ev], 1ull);
      A.state[s] = DECIDED;
    }
    __syncwarp();  // the window buffers are reused by the next batch
  }
}

// between rounds: the round's slots are taken, the next pending list becomes
// current, a round that still saw pending seeds is counted
__global__ void round_end_kernel(unsigned long long* counters) {
  counters[6] += counters[5] != 0;
  counters[4] += counters[1];
  counters[3] = counters[2];
  counters[1] = 0;
  counters[2] = 0;
  counters[5] = 0;
}

// the pending list starts as every candidate (their cells)
__global__ void __launch_bounds__(NT) list_init_kernel(unsigned long long* counters, const int64_t* cand,
                                                       int64_t* list) {
  const int64_t m = static_cast<int64_t>(counters[0]);
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; k < m; k += static_cast<int64_t>(gridDim.x) * NT)
    list[k] = cand[k];
  if (blockIdx.x == 0 && threadIdx.x == 0) counters[3] = counters[0];
}

// order: bucket particles by event, then rank by priority inside the event
__global__ void bucket_kernel(const Slot* slots, int64_t np, const int64_t* event_off,
                              unsigned long long* cursor, int64_t* order) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; p < np;
       p += static_cast<int64_t>(gridDim.x) * NT) {
    const int e = slots[p].event;
    if (e < 0) continue;  // a seed consumed before its turn
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
constexpr int RANK_SPLIT = 4;                 // threads per particle in the ranking
constexpr int RANK_PER_CTA = NT / RANK_SPLIT;  // particles ranked per CTA

__global__ void __launch_bounds__(NT) write_kernel(const Slot* slots, const int64_t* event_off,
                                                   const int64_t* event_cnt, const int64_t* order, OutArgs O) {
  __shared__ float ke[RANK_SMEM];
  __shared__ int64_t ko[RANK_SMEM];
  const int64_t ev = blockIdx.x;
  const int64_t b = event_off[ev], m = event_cnt[ev];
  const int64_t first = static_cast<int64_t>(blockIdx.y) * RANK_PER_CTA;  // particles [first, first + RANK_PER_CTA)
  if (first >= m) return;
  const bool in_smem = m <= RANK_SMEM;
  if (in_smem)
    for (int64_t j = threadIdx.x; j < m; j += NT) {
      const Slot& Q = slots[order[b + j]];
      ke[j] = Q.key_e;
      ko[j] = Q.origin;
    }
  __syncthreads();
  const int q = threadIdx.x % RANK_SPLIT;  // this thread counts keys j = q, q + RANK_SPLIT, ...
  for (int64_t i0 = first; i0 < m; i0 += static_cast<int64_t>(gridDim.y) * RANK_PER_CTA) {
    const int64_t i = i0 + threadIdx.x / RANK_SPLIT;
    const bool have = i < m;
    const int64_t p = have ? order[b + i] : 0;
    const Slot& S = slots[p];
    const float se = have ? S.key_e : 0.0f;
    const int64_t so = have ? S.origin : 0;
    int64_t rank = 0;
    if (have) {
      if (in_smem) {
        for (int64_t j = q; j < m; j += RANK_SPLIT)
          rank += static_cast<int>(ke[j] > se) | (static_cast<int>(ke[j] == se) & static_cast<int>(ko[j] < so));
      } else {
        for (int64_t j = q; j < m; j += RANK_SPLIT) {
          const Slot& Q = slots[order[b + j]];
          rank += static_cast<int>(Q.key_e > se) | (static_cast<int>(Q.key_e == se) & static_cast<int>(Q.origin < so));
        }
      }
    }
#pragma unroll
    for (int o = 1; o < RANK_SPLIT; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (!have || q) continue;
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
  int64_t np = 0;      // particles
  int64_t nslots = 0;  // particle slots written, holes (skipped seeds) included
  void* ws = nullptr;
  int64_t* lists = nullptr;  // the two pending lists
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
  // particle slots (at most one per seed) and the two pending lists
  const size_t nc1 = std::max<size_t>(1, ncand);
  e = cudaMallocAsync(reinterpret_cast<void**>(&A.slots), nc1 * sizeof(reco::Slot), s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&A.contrib), nc1 * reco::MAXC * 8, s);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&H->lists), nc1 * 16, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(particle slots)");
  A.list[0] = H->lists;
  A.list[1] = A.list[0] + nc1;
  const int rgrid = std::max(1, std::min<int>(ds->sm_count * 8, static_cast<int>((ncand + reco::NT - 1) / reco::NT)));
  // process: one warp per 32 ready seeds
  const int cgrid = std::max(1, std::min<int>(ds->sm_count * 8,
                                              static_cast<int>((ncand + reco::PNT - 1) / reco::PNT)));
  reco::list_init_kernel<<<rgrid, reco::NT, 0, s>>>(A.counters, A.cand, A.list[0]);
  // rounds are queued without a host check in between (a round with nothing pending returns at once):
  // 8 (full events converge in ~6), then 4 more at a time until the pending list is empty
  int launched = 0;
  for (unsigned long long left = ncand; left;) {
    for (int k = 0; k < (launched ? 4 : 8); ++k, ++launched) {
      reco::ready_kernel<<<rgrid, reco::NT, 0, s>>>(A, launched & 1);
      reco::process_kernel<<<cgrid, reco::PNT, 0, s>>>(A);
      reco::round_end_kernel<<<1, 1, 0, s>>>(A.counters);
    }
    SK_TRY(cudaGetLastError());
    SK_TRY(cudaMemcpyAsync(&left, &A.counters[3], 8, cudaMemcpyDeviceToHost, s));
    SK_TRY(cudaStreamSynchronize(s));
  }
  unsigned long long cnt[8] = {0};
  SK_TRY(cudaMemcpyAsync(cnt, A.counters, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  H->counts.assign(nevents, 0);
  std::vector<unsigned long long> ec(nevents > 0 ? nevents : 1);
  if (nevents) SK_TRY(cudaMemcpyAsync(ec.data(), A.event_count, nevents * 8, cudaMemcpyDeviceToHost, s));
  SK_TRY(cudaStreamSynchronize(s));
  int64_t np = 0;
  for (int i = 0; i < nevents; ++i) {
    H->counts[i] = static_cast<int64_t>(ec[i]);
    np += H->counts[i];
  }
  H->np = np;
  H->nslots = static_cast<int64_t>(cnt[4] + cnt[1]);  // slots of every round, holes included
  *nparticles = H->np;
  if (rounds) *rounds = static_cast<int>(cnt[6]);
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
  const int bgrid =
      std::max(1, std::min<int>(ds->sm_count * 8, static_cast<int>((H->nslots + reco::NT - 1) / reco::NT)));
  reco::bucket_kernel<<<bgrid, reco::NT, 0, s>>>(H->A.slots, H->nslots, d_off, cursor, order);
  reco::OutArgs O;
  O.energy = energy; O.x = x; O.y = y; O.xvar = x_variance; O.yvar = y_variance; O.origin = origin;
  for (int t = 0; t < 4; ++t) {
    O.sig[t] = significance[t];
    O.ec[t] = e_contribution[t];
    O.nc[t] = noisy_count[t];
  }
  O.lens = sensor_lens;
  O.offsets = sensor_offsets;
  int64_t mmax = 0;
  for (int i = 0; i < H->nevents; ++i) mmax = std::max(mmax, H->counts[i]);
  const unsigned chunks =
      static_cast<unsigned>(std::min<int64_t>((mmax + reco::RANK_PER_CTA - 1) / reco::RANK_PER_CTA, 65535));
  if (H->nevents && chunks)
    reco::write_kernel<<<dim3(H->nevents, chunks), reco::NT, 0, s>>>(H->A.slots, d_off, d_cnt, order, O);
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
  if (H->lists) cudaFreeAsync(H->lists, s);
  delete H;
  return SK_OK;
}

}  // extern "C"
