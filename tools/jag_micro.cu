// Standalone microbenchmark for the jagged gather (config 3 shape: 1M
// records, lens ~ U[0,20], u64 members, shuffled source segments with slack).
// Not part of the product: it measures what simple gather structures and L2
// policies reach, to pick the design of pack_fused_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/jag_micro.cu -o build/jag_micro
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <numeric>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int POL>
__device__ __forceinline__ uint64_t ld8(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  if constexpr (POL == 1)
    asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  else if constexpr (POL == 2)
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  else
    v = *p;
  return v;
}
template <int SP>
__device__ __forceinline__ void st8(uint64_t* p, uint64_t v, uint64_t pol) {
  if constexpr (SP == 1)
    asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else if constexpr (SP == 2)
    asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
  else
    *p = v;
}

// warp per group of 32 records; known int64 prefix
template <int MAXK, int POL, int SP>
__global__ void __launch_bounds__(256) gather_k(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
                                                const int64_t* __restrict__ P, const uint64_t* __restrict__ pool,
                                                uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (n + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const uint64_t pl = pol_last(), pf = pol_first();
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); g < ngroups; g += nw) {
    const int64_t r = g * 32 + lane;
    const int len = r < n ? lens[r] : 0;
    const int64_t o = r < n ? off[r] : 0;
    const int64_t base = P[g * 32];
    int x = len;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(~0u, x, s);
      if (lane >= s) x += y;
    }
    const int T = __shfl_sync(~0u, x, 31);
    const int ex = x - len;
    const int64_t d = o - ex;
    uint64_t v[MAXK];
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int m = k * 32 + lane;
      if (k * 32 < T) {
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int e = __shfl_sync(~0u, ex, lo + s);
          if (e <= m) lo += s;
        }
        const int64_t dd = __shfl_sync(~0u, d, lo);
        if (m < T) v[k] = ld8<POL>(pool + dd + m, pl);
      }
    }
#pragma unroll
    for (int k = 0; k < MAXK; ++k) {
      const int m = k * 32 + lane;
      if (m < T) st8<SP>(out + base + m, v[k], pf);
    }
    for (int m0 = MAXK * 32; m0 < T; m0 += 32) {  // long groups
      const int m = m0 + lane;
      int lo = 0;
      for (int s = 16; s >= 1; s >>= 1) {
        const int e = __shfl_sync(~0u, ex, lo + s);
        if (e <= m) lo += s;
      }
      const int64_t dd = __shfl_sync(~0u, d, lo);
      if (m < T) out[base + m] = pool[dd + m];
    }
  }
}

// owner-fill gather: each lane writes its record's source base d into a per-warp smem map at its
// members' positions; every member slot is then one LDS.64 + add + LD
template <int K>
__global__ void __launch_bounds__(256) gather_o(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
                                                const int64_t* __restrict__ P, const uint64_t* __restrict__ pool,
                                                uint64_t* __restrict__ out) {
  __shared__ int64_t smap[8][K * 32];
  int64_t* map = smap[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (n + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); g < ngroups; g += nw) {
    const int64_t r = g * 32 + lane;
    const int len = r < n ? lens[r] : 0;
    const int64_t o = r < n ? off[r] : 0;
    const int64_t base = P[g * 32];
    int x = len;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(~0u, x, s);
      if (lane >= s) x += y;
    }
    const int T = __shfl_sync(~0u, x, 31);
    const int ex = x - len;
    const int64_t d = o - ex;
    for (int m0 = 0; m0 < T; m0 += 32 * K) {
      __syncwarp();
      const int a = max(ex, m0), b = min(ex + len, m0 + 32 * K);
      for (int m = a; m < b; ++m) map[m - m0] = d;
      __syncwarp();
      uint64_t v[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < T) v[q] = pool[map[q * 32 + lane] + m];
      }
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < T) st8<1>(out + base + m, v[q], 0);
      }
    }
  }
}

// memcpy-like ceiling: out[i] = pool[i] for the member count
__global__ void copy_k(int64_t m, const uint4* __restrict__ a, uint4* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

__global__ void flush_k(uint4* p, int64_t n, int v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, i, v, i);
}


constexpr uint64_t FLAG_A = 1ull << 62, FLAG_P = 2ull << 62, VAL_MASK = (1ull << 62) - 1;
__device__ __forceinline__ uint64_t ld_poll(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <int NT> __device__ __forceinline__ void bar1() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

// fused: ticketed tiles of 2048 records (8 warps x 8 groups x 32), decoupled look-back, register gather
template <int K, int MINB, int SP, int GPW, int DBG = 0, int NW = 8, int OWN = 0>
__global__ void __launch_bounds__(NW * 32, MINB) fused_k(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
    const uint64_t* __restrict__ pool, uint64_t* __restrict__ out, int* __restrict__ P, unsigned* ticket,
    uint64_t* status, int64_t* total) {
  constexpr int TR = NW * GPW * 32;
  __shared__ int64_t sd[TR];
  __shared__ int sex[TR];
  __shared__ int64_t sgb[NW * GPW + 1];
  __shared__ int64_t swt[NW];
  __shared__ int64_t sE;
  __shared__ unsigned st;
  __shared__ int64_t smap[OWN == 1 ? NW : 1][OWN == 1 ? K * 32 : 1];
  __shared__ int64_t sdc[NW][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) st = (DBG & 2) ? blockIdx.x : atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t t = st, r0 = t * TR, rw = r0 + warp * (GPW * 32);
  int len[GPW];
  int64_t o[GPW];
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    len[k] = r < n ? lens[r] : 0;
    o[k] = r < n ? off[r] : 0;
  }
  int64_t wsum = 0;
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    int x = len[k];
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(~0u, x, s);
      if (lane >= s) x += y;
    }
    const int T = __shfl_sync(~0u, x, 31);
    const int e = warp * GPW * 32 + k * 32 + lane;
    sex[e] = x - len[k];
    sd[e] = o[k] - (x - len[k]);
    if (lane == 0) sgb[warp * GPW + k] = wsum;
    wsum += T;
  }
  if (lane == 0) swt[warp] = wsum;
  __syncthreads();
  int64_t A = 0, Wo = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    Wo += w < warp ? swt[w] : 0;
    A += swt[w];
  }
  if (tid == 0) st_rel(&status[t], (t == 0 && !(DBG & 4) ? FLAG_P : FLAG_A) | (uint64_t(A) & VAL_MASK));
  bool haveE = false;
  int64_t E = 0;
  auto getE = [&]() {
    if (warp == 0) {
      int64_t acc = 0;
      if (t > 0 && (DBG & 4)) {
        // sum every predecessor's aggregate, 256 per round (no chain through inclusive prefixes)
        for (int64_t e0 = 0; e0 < t; e0 += 256) {
          uint64_t s[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int64_t j = e0 + q * 32 + lane;
            s[q] = j < t ? ld_poll(&status[j]) : FLAG_A;
          }
          bool miss = false;
#pragma unroll
          for (int q = 0; q < 8; ++q) miss |= (s[q] >> 62) == 0;
          while (__any_sync(~0u, miss)) {
            miss = false;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if ((s[q] >> 62) == 0) s[q] = ld_poll(&status[e0 + q * 32 + lane]);
              miss |= (s[q] >> 62) == 0;
            }
          }
          int64_t v = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) if (e0 + q * 32 + lane < t) v += int64_t(s[q] & VAL_MASK);
#pragma unroll
          for (int q = 16; q; q >>= 1) v += __shfl_xor_sync(~0u, v, q);
          acc += v;
        }
      } else if (t > 0 && !(DBG & 1)) {
        int64_t idx = t - 1;
        while (true) {
          const int64_t j = idx - lane;
          uint64_t s = j >= 0 ? ld_poll(&status[j]) : FLAG_P;
          while (__any_sync(~0u, (s >> 62) == 0)) {
            if ((s >> 62) == 0) s = ld_poll(&status[j]);
          }
          const unsigned pm = __ballot_sync(~0u, (s >> 62) == 2);
          const int pl = pm ? __ffs(pm) - 1 : 32;
          int64_t v = (lane <= pl && j >= 0) ? int64_t(s & VAL_MASK) : 0;
#pragma unroll
          for (int q = 16; q; q >>= 1) v += __shfl_xor_sync(~0u, v, q);
          acc += v;
          if (pm) break;
          idx -= 32;
        }
        if (lane == 0) st_rel(&status[t], FLAG_P | (uint64_t(acc + A) & VAL_MASK));
      }
      if (lane == 0) sE = acc;
    }
    bar1<NW * 32>();
    E = sE;
    haveE = true;
  };
  const uint64_t pf = 0;
#pragma unroll 1
  for (int k = 0; k < GPW; ++k) {
    const int g = warp * GPW + k;
    const int64_t gb = (k + 1 < GPW ? sgb[g + 1] : wsum) , g0 = sgb[g];
    const int T = int(gb - g0);
    const int e = g * 32 + lane;
    const int ex = sex[e];
    const int64_t d = sd[e];
    int cnt = 0;
#pragma unroll 1
    for (int m0 = 0; m0 < T; m0 += 32 * K) {
      uint64_t v[K];
      if constexpr (OWN == 2) {
        // mask/rank search: record starts of each 32-member window by REDUX.OR, rank by popc,
        // source base from the warp's compacted table of non-empty records
        const int lenl = (lane < 31 ? sex[e + 1] : T) - ex;
        const unsigned le = 0xffffffffu >> (31 - lane);
        if (m0 == 0) {
          const unsigned nz = __ballot_sync(~0u, lenl > 0);
          if (lenl > 0) sdc[warp][__popc(nz & (le >> 1))] = d;
          __syncwarp();
          cnt = 0;
        }
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int base = m0 + q * 32;
          if (base < T) {
            const unsigned sb = (lenl > 0 && ex >= base && ex < base + 32) ? 1u << (ex - base) : 0u;
            const unsigned mask = __reduce_or_sync(~0u, sb);
            const int k2 = cnt + __popc(mask & le) - 1;
            cnt += __popc(mask);
            if (base + lane < T) v[q] = pool[sdc[warp][k2] + base + lane];
          }
        }
      } else if constexpr (OWN == 1) {
        int64_t* map = smap[warp];
        __syncwarp();
        const int lenl = (lane < 31 ? sex[e + 1] : T) - ex;
        const int a = max(ex, m0), b = min(ex + lenl, m0 + 32 * K);
        for (int m = a; m < b; ++m) map[m - m0] = d;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int m = m0 + q * 32 + lane;
          if (m < T) v[q] = pool[map[q * 32 + lane] + m];
        }
      } else {
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m0 + q * 32 < T) {
          int lo = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const int ee = __shfl_sync(~0u, ex, lo + s);
            if (ee <= m) lo += s;
          }
          const int64_t dd = __shfl_sync(~0u, d, lo);
          if (m < T) v[q] = pool[dd + m];
        }
      }
      }
      if (!haveE) getE();
      uint64_t* ob = out + E + Wo + g0;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < T) st8<SP>(ob + m, v[q], pf);
      }
    }
  }
  if (!haveE) getE();
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    const int e = warp * GPW * 32 + k * 32 + lane;
    if (r < n) P[r] = int(E + Wo + sgb[warp * GPW + k] + sex[e]);
  }
  if (r0 + TR >= n && tid == 0) {
    P[n] = int(E + A);
    *total = E + A;
  }
}

__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// fused with cp.async landing: NS items (<= 32*K members each) in flight per warp
template <int K, int NS, int NW, int GPW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB) fused_cp(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
    const uint64_t* __restrict__ pool, uint64_t* __restrict__ out, int* __restrict__ P, unsigned* ticket,
    uint64_t* status, int64_t* total) {
  constexpr int TR = NW * GPW * 32;
  extern __shared__ __align__(16) uint64_t dsm[];
  uint64_t* stage = dsm + (threadIdx.x >> 5) * NS * K * 32;
  int64_t* sd = reinterpret_cast<int64_t*>(dsm + NW * NS * K * 32);
  int* sex = reinterpret_cast<int*>(sd + TR);
  __shared__ int64_t sgb[NW * GPW + 1];
  __shared__ int64_t swt[NW];
  __shared__ int64_t sE;
  __shared__ unsigned st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) st = atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t t = st, r0 = t * TR, rw = r0 + warp * (GPW * 32);
  int len[GPW];
  int64_t o[GPW];
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    len[k] = r < n ? lens[r] : 0;
    o[k] = r < n ? off[r] : 0;
  }
  int64_t wsum = 0;
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    int x = len[k];
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(~0u, x, s);
      if (lane >= s) x += y;
    }
    const int T = __shfl_sync(~0u, x, 31);
    const int e = warp * GPW * 32 + k * 32 + lane;
    sex[e] = x - len[k];
    sd[e] = o[k] - (x - len[k]);
    if (lane == 0) sgb[warp * GPW + k] = wsum;
    wsum += T;
  }
  if (lane == 0) swt[warp] = wsum;
  __syncthreads();
  int64_t A = 0, Wo = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    Wo += w < warp ? swt[w] : 0;
    A += swt[w];
  }
  if (tid == 0) st_rel(&status[t], (t == 0 ? FLAG_P : FLAG_A) | (uint64_t(A) & VAL_MASK));
  bool haveE = false;
  int64_t E = 0;
  auto getE = [&]() {
    if (warp == 0) {
      int64_t acc = 0;
      if (t > 0) {
        int64_t idx = t - 1;
        while (true) {
          const int64_t j = idx - lane;
          uint64_t s = j >= 0 ? ld_poll(&status[j]) : FLAG_P;
          while (__any_sync(~0u, (s >> 62) == 0)) {
            if ((s >> 62) == 0) s = ld_poll(&status[j]);
          }
          const unsigned pm = __ballot_sync(~0u, (s >> 62) == 2);
          const int pl = pm ? __ffs(pm) - 1 : 32;
          int64_t v = (lane <= pl && j >= 0) ? int64_t(s & VAL_MASK) : 0;
#pragma unroll
          for (int q = 16; q; q >>= 1) v += __shfl_xor_sync(~0u, v, q);
          acc += v;
          if (pm) break;
          idx -= 32;
        }
        if (lane == 0) st_rel(&status[t], FLAG_P | (uint64_t(acc + A) & VAL_MASK));
      }
      if (lane == 0) sE = acc;
    }
    bar1<NW * 32>();
    E = sE;
    haveE = true;
  };
  // items: (group k, chunk m0); pending ring of NS items: out base and count
  int64_t pbase[NS];
  int pcnt[NS];
  int issued = 0, drained = 0;
  auto drain_one = [&]() {
    const int slot = drained % NS;
    int64_t b = 0; int c = 0;
#pragma unroll
    for (int i = 0; i < NS; ++i) if (i == slot) { b = pbase[i]; c = pcnt[i]; }
    if (!haveE) getE();
    const uint64_t* s = stage + slot * K * 32;
    uint64_t* ob = out + E + b;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const int m = q * 32 + lane;
      if (m < c) st8<1>(ob + m, s[m], 0);
    }
    ++drained;
  };
#pragma unroll 1
  for (int k = 0; k < GPW; ++k) {
    const int g = warp * GPW + k;
    const int64_t g0 = sgb[g];
    const int T = int((k + 1 < GPW ? sgb[g + 1] : wsum) - g0);
    const int e = g * 32 + lane;
    const int ex = sex[e];
    const int64_t d = sd[e];
    int cnt = 0;
#pragma unroll 1
    for (int m0 = 0; m0 < T; m0 += 32 * K) {
      if (issued - drained == NS) {
        cpa_wait<NS - 1>();
        __syncwarp();
        drain_one();
        __syncwarp();
      }
      const int slot = issued % NS;
      uint64_t* s = stage + slot * K * 32;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m0 + q * 32 < T) {
          int lo = 0;
#pragma unroll
          for (int sh = 16; sh >= 1; sh >>= 1) {
            const int ee = __shfl_sync(~0u, ex, lo + sh);
            if (ee <= m) lo += sh;
          }
          const int64_t dd = __shfl_sync(~0u, d, lo);
          if (m < T) cpa8(s + q * 32 + lane, pool + dd + m);
        }
      }
      cpa_commit();
#pragma unroll
      for (int i = 0; i < NS; ++i) if (i == slot) { pbase[i] = Wo + g0 + m0; pcnt[i] = min(32 * K, T - m0); }
      ++issued;
    }
  }
  cpa_wait<0>();
  __syncwarp();
  while (drained < issued) drain_one();
  if (!haveE) getE();
#pragma unroll
  for (int k = 0; k < GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    const int e = warp * GPW * 32 + k * 32 + lane;
    if (r < n) P[r] = int(E + Wo + sgb[warp * GPW + k] + sex[e]);
  }
  if (r0 + TR >= n && tid == 0) {
    P[n] = int(E + A);
    *total = E + A;
  }
}

// warp-tiled persistent fused pack: each warp takes tiles of 32*GPW records by ticket, decoupled look-back per warp tile
template <int K, int GPW, int MINB, bool PF>
__global__ void __launch_bounds__(256, MINB) fused_w(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
    const uint64_t* __restrict__ pool, uint64_t* __restrict__ out, int* __restrict__ P, unsigned* ticket,
    uint64_t* status, int64_t* total) {
  const int lane = threadIdx.x & 31;
  const int64_t nwt = (n + 32 * GPW - 1) / (32 * GPW);
  unsigned tk = 0;
  if (lane == 0) tk = atomicAdd(ticket, 1u);
  int64_t t = __shfl_sync(~0u, tk, 0);
  int len[GPW];
  int64_t o[GPW];
  auto load_meta = [&](int64_t tt, int (&l)[GPW], int64_t (&oo)[GPW]) {
#pragma unroll
    for (int k = 0; k < GPW; ++k) {
      const int64_t r = tt * 32 * GPW + k * 32 + lane;
      l[k] = r < n ? lens[r] : 0;
      oo[k] = r < n ? off[r] : 0;
    }
  };
  if (t < nwt) load_meta(t, len, o);
  while (t < nwt) {
    if (lane == 0) tk = atomicAdd(ticket, 1u);
    int ex[GPW];
    int64_t gb[GPW + 1];
    gb[0] = 0;
#pragma unroll
    for (int k = 0; k < GPW; ++k) {
      int x = len[k];
#pragma unroll
      for (int s = 1; s < 32; s <<= 1) {
        const int y = __shfl_up_sync(~0u, x, s);
        if (lane >= s) x += y;
      }
      ex[k] = x - len[k];
      o[k] -= ex[k];  // o becomes d
      gb[k + 1] = gb[k] + __shfl_sync(~0u, x, 31);
    }
    const int64_t A = gb[GPW];
    if (lane == 0) st_rel(&status[t], (t == 0 ? FLAG_P : FLAG_A) | (uint64_t(A) & VAL_MASK));
    const int64_t tn = __shfl_sync(~0u, tk, 0);
    int nlen[GPW];
    int64_t no[GPW];
    if (PF && tn < nwt) load_meta(tn, nlen, no);
    bool haveE = false;
    int64_t E = 0;
    auto getE = [&]() {
      int64_t acc = 0;
      if (t > 0) {
        int64_t idx = t - 1;
        while (true) {
          const int64_t j = idx - lane;
          uint64_t s = j >= 0 ? ld_poll(&status[j]) : FLAG_P;
          while (__any_sync(~0u, (s >> 62) == 0)) {
            if ((s >> 62) == 0) s = ld_poll(&status[j]);
          }
          const unsigned pm = __ballot_sync(~0u, (s >> 62) == 2);
          const int pl = pm ? __ffs(pm) - 1 : 32;
          int64_t v = (lane <= pl && j >= 0) ? int64_t(s & VAL_MASK) : 0;
#pragma unroll
          for (int q = 16; q; q >>= 1) v += __shfl_xor_sync(~0u, v, q);
          acc += v;
          if (pm) break;
          idx -= 32;
        }
        if (lane == 0) st_rel(&status[t], FLAG_P | (uint64_t(acc + A) & VAL_MASK));
      }
      E = acc;
      haveE = true;
    };
#pragma unroll
    for (int k = 0; k < GPW; ++k) {
      const int T = int(gb[k + 1] - gb[k]);
#pragma unroll 1
      for (int m0 = 0; m0 < T; m0 += 32 * K) {
        uint64_t v[K];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int m = m0 + q * 32 + lane;
          if (m0 + q * 32 < T) {
            int lo = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
              const int ee = __shfl_sync(~0u, ex[k], lo + s);
              if (ee <= m) lo += s;
            }
            const int64_t dd = __shfl_sync(~0u, o[k], lo);
            if (m < T) v[q] = pool[dd + m];
          }
        }
        if (!haveE) getE();
        uint64_t* ob = out + E + gb[k];
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int m = m0 + q * 32 + lane;
          if (m < T) st8<1>(ob + m, v[q], 0);
        }
      }
    }
    if (!haveE) getE();
#pragma unroll
    for (int k = 0; k < GPW; ++k) {
      const int64_t r = t * 32 * GPW + k * 32 + lane;
      if (r < n) P[r] = int(E + gb[k] + ex[k]);
    }
    if ((t + 1) * 32 * GPW >= n && lane == 0) {
      P[n] = int(E + A);
      *total = E + A;
    }
    t = tn;
    if (PF) {
#pragma unroll
      for (int k = 0; k < GPW; ++k) { len[k] = nlen[k]; o[k] = no[k]; }
    } else if (t < nwt) {
      load_meta(t, len, o);
    }
  }
}

// static-block fused pack: blocks of br records by ticket; block totals summed by warp 0 (no chain),
// groups of 32 records claimed by warps, register gather
template <int K, int MINB, int RPT>
__global__ void __launch_bounds__(256, MINB) fused_b(int64_t n, const int* __restrict__ lens, const int64_t* __restrict__ off,
    const uint64_t* __restrict__ pool, uint64_t* __restrict__ out, int* __restrict__ P, unsigned* ticket,
    uint64_t* status, int64_t* total, int64_t br) {
  constexpr int MAXR = 256 * RPT;
  __shared__ int64_t sLx[MAXR + 1];
  __shared__ int64_t sD[MAXR];
  __shared__ int64_t swt[8];
  __shared__ volatile int64_t sE;
  __shared__ volatile int sEready;
  __shared__ int snext;
  __shared__ unsigned st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { st = atomicAdd(ticket, 1u); sEready = 0; snext = 0; }
  __syncthreads();
  const int64_t t = st, rec0 = t * br;
  const int cnt = int(min(br, n - rec0));
  int len[RPT];
  int64_t o[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int e = tid * RPT + i;
    len[i] = e < cnt ? lens[rec0 + e] : 0;
    o[i] = e < cnt ? off[rec0 + e] : 0;
  }
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) acc += len[i];
  int64_t x = acc;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int64_t y = __shfl_up_sync(~0u, x, s);
    if (lane >= s) x += y;
  }
  if (lane == 31) swt[warp] = x;
  __syncthreads();
  int64_t A = 0, woff = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) { woff += w < warp ? swt[w] : 0; A += swt[w]; }
  if (tid == 0) { st_rel(&status[t], FLAG_A | (uint64_t(A) & VAL_MASK)); __threadfence(); }
  int64_t run = woff + x - acc;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int e = tid * RPT + i;
    sLx[e] = run;
    sD[e] = o[i] - run;
    run += len[i];
  }
  if (tid == 255) sLx[MAXR] = run;
  __syncthreads();
  bool haveE = false;
  int64_t E = 0;
  auto getE = [&]() {
    if (warp == 0) {
      int64_t a = 0;
      for (int64_t e0 = 0; e0 < t; e0 += 32 * 8) {
        uint64_t s[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t j = e0 + q * 32 + lane;
          s[q] = j < t ? ld_poll(&status[j]) : FLAG_A;
        }
        bool miss = false;
#pragma unroll
        for (int q = 0; q < 8; ++q) miss |= (s[q] >> 62) == 0;
        while (__any_sync(~0u, miss)) {
          miss = false;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if ((s[q] >> 62) == 0) s[q] = ld_poll(&status[e0 + q * 32 + lane]);
            miss |= (s[q] >> 62) == 0;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) if (e0 + q * 32 + lane < t) a += int64_t(s[q] & VAL_MASK);
      }
#pragma unroll
      for (int q = 16; q; q >>= 1) a += __shfl_xor_sync(~0u, a, q);
      E = a;
      if (lane == 0) { sE = a; __threadfence_block(); sEready = 1; }
    } else {
      while (!sEready) {}
      E = sE;
    }
    haveE = true;
  };
  const int ngroups = (cnt + 31) / 32;
  while (true) {
    int g = 0;
    if (lane == 0) g = atomicAdd(&snext, 1);
    g = __shfl_sync(~0u, g, 0);
    if (g >= ngroups) break;
    const int e = g * 32 + lane;
    const int64_t B = sLx[g * 32];
    const int T = int(sLx[min(g * 32 + 32, cnt)] - B);
    const int ex = int(sLx[min(e, cnt)] - B);
    const int64_t d = (e < cnt ? sD[e] : 0) + B;
#pragma unroll 1
    for (int m0 = 0; m0 < T; m0 += 32 * K) {
      uint64_t v[K];
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m0 + q * 32 < T) {
          int lo = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const int ee = __shfl_sync(~0u, ex, lo + s);
            if (ee <= m) lo += s;
          }
          const int64_t dd = __shfl_sync(~0u, d, lo);
          if (m < T) v[q] = pool[dd + m];
        }
      }
      if (!haveE) getE();
      uint64_t* ob = out + E + B;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < T) st8<1>(ob + m, v[q], 0);
      }
    }
  }
  if (!haveE) getE();
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int e = tid * RPT + i;
    if (e < cnt) P[rec0 + e] = int(E + sLx[e]);
  }
  if (rec0 + cnt >= n && tid == 0) {
    P[n] = int(E + A);
    *total = E + A;
  }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(s)), "l"(g), "r"(bytes), "r"(su32(bar)) : "memory");
}

// TMA-bulk gather with the prefix given: a warp per group of 32 records, NS groups in flight per warp,
// each record's 16-byte-aligned covering span copied by one bulk op into the warp's stage
template <int NS, int NW, int STAGE>
__global__ void __launch_bounds__(NW * 32, 1) tma_gather(int64_t n, const int* __restrict__ lens,
    const int64_t* __restrict__ off, const int64_t* __restrict__ P, const uint64_t* __restrict__ pool,
    uint64_t* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t dsm_t[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* stage = dsm_t + warp * NS * STAGE;
  __shared__ uint64_t bars[NW][NS];
  __shared__ int sEx[NW][NS][33];
  __shared__ int sBase[NW][NS][32];
  __shared__ int64_t sB[NW][NS];
  if (lane < NS) mb_init(&bars[warp][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t ngroups = (n + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * NW;
  const int64_t g0 = (int64_t)blockIdx.x * NW + warp;
  const int64_t mine = g0 < ngroups ? (ngroups - g0 + nw - 1) / nw : 0;
  auto issue = [&](int64_t i) {  // the warp's i-th group into stage i % NS
    const int st = int(i % NS);
    const int64_t g = g0 + i * nw;
    const int64_t r = g * 32 + lane;
    const int len = r < n ? lens[r] : 0;
    const int64_t o = r < n ? off[r] : 0;
    const int64_t a = (o * 8) & ~int64_t(15), b = ((o + len) * 8 + 15) & ~int64_t(15);
    const int bytes = len ? int(b - a) : 0;
    int x = bytes, e = len;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int y = __shfl_up_sync(~0u, x, s), z = __shfl_up_sync(~0u, e, s);
      if (lane >= s) { x += y; e += z; }
    }
    const int tot = __shfl_sync(~0u, x, 31);
    sEx[warp][st][lane] = e - len;
    if (lane == 31) sEx[warp][st][32] = e;
    sBase[warp][st][lane] = (x - bytes) + int((o * 8) & 15);
    if (lane == 0) { sB[warp][st] = P[g * 32]; mb_expect(&bars[warp][st], uint32_t(tot)); }
    __syncwarp();
    if (bytes) bulk_g2s(stage + st * STAGE + (x - bytes), reinterpret_cast<const uint8_t*>(pool) + a, bytes, &bars[warp][st]);
  };
  for (int64_t i = 0; i < NS - 1 && i < mine; ++i) issue(i);
  for (int64_t i = 0; i < mine; ++i) {
    if (i + NS - 1 < mine) issue(i + NS - 1);
    const int st = int(i % NS);
    mb_wait(&bars[warp][st], uint32_t((i / NS) & 1));
    const int T = sEx[warp][st][32];
    const int ex = sEx[warp][st][lane], base = sBase[warp][st][lane];
    const int64_t B = sB[warp][st];
    const uint8_t* sg = stage + st * STAGE;
    for (int m0 = 0; m0 < T; m0 += 32) {
      const int m = m0 + lane;
      int lo = 0;
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const int ee = __shfl_sync(~0u, ex, lo + s);
        if (ee <= m) lo += s;
      }
      const int bs = __shfl_sync(~0u, base, lo), es = __shfl_sync(~0u, ex, lo);
      if (m < T) __stcs(out + B + m, *reinterpret_cast<const uint64_t*>(sg + bs + (m - es) * 8));
    }
    __syncwarp();
  }
}

int main(int argc, char** argv) {
  const int64_t n = 1000000;
  const int inorder = argc > 1 ? atoi(argv[1]) : 0;
  std::mt19937_64 rng(7);
  std::vector<int> lens(n);
  for (auto& l : lens) l = rng() % 21;
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  if (!inorder) std::shuffle(order.begin(), order.end(), rng);
  std::vector<int64_t> off(n);
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    off[order[i]] = pos;
    pos += lens[order[i]] + rng() % 4;
  }
  const int64_t pool_len = pos;
  std::vector<uint64_t> pool(pool_len);
  for (auto& p : pool) p = rng();
  std::vector<int64_t> P(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) P[i + 1] = P[i] + lens[i];
  const int64_t M = P[n];
  std::vector<uint64_t> want(M);
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < lens[i]; ++j) want[P[i] + j] = pool[off[i] + j];
  printf("records %lld members %lld pool %lld inorder %d\n", (long long)n, (long long)M, (long long)pool_len, inorder);

  int *dl; int64_t *doff, *dP; uint64_t *dpool, *dout; uint4* fl;
  const int64_t FL = 512ll << 20;
  CK(cudaMalloc(&dl, n * 4)); CK(cudaMalloc(&doff, n * 8)); CK(cudaMalloc(&dP, (n + 1) * 8));
  CK(cudaMalloc(&dpool, pool_len * 8)); CK(cudaMalloc(&dout, M * 8 + 4096)); CK(cudaMalloc(&fl, FL));
  CK(cudaMemcpy(dl, lens.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(doff, off.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dP, P.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dpool, pool.data(), pool_len * 8, cudaMemcpyHostToDevice));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const double algo = n * 16.0 + M * 16.0;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto run = [&](const char* name, auto launch, bool check) {
    float best = 1e9, sum = 0; int reps = 10;
    for (int i = 0; i < 3; ++i) launch();
    for (int i = 0; i < reps; ++i) {
      flush_k<<<nsm * 4, 512>>>(fl, FL / 16, i);
      CK(cudaEventRecord(a));
      launch();
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms); sum += ms;
    }
    // back-to-back (no flush)
    CK(cudaEventRecord(a));
    for (int i = 0; i < 20; ++i) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float bb; CK(cudaEventElapsedTime(&bb, a, b)); bb /= 20;
    CK(cudaGetLastError());
    bool ok = true;
    if (check) {
      std::vector<uint64_t> got(M);
      CK(cudaMemcpy(got.data(), dout, M * 8, cudaMemcpyDeviceToHost));
      ok = got == want;
      CK(cudaMemset(dout, 0, M * 8));
    }
    printf("%-34s cold mean %7.2f us best %7.2f us  b2b %7.2f us  frac(b2b) %.3f %s\n", name, sum / reps * 1e3,
           best * 1e3, bb * 1e3, algo / (bb * 1e-3) / 6546.9e9, check ? (ok ? "OK" : "MISMATCH") : "");
  };
  run("copy 16B (members*8 bytes)", [&] { copy_k<<<nsm * 8, 256>>>(M / 2, (const uint4*)dpool, (uint4*)dout); }, false);
#define G(K, POL, SP, GRID)                                                                                      \
  run("gather K" #K " pol" #POL " sp" #SP " grid" #GRID, [&] {                                                    \
    gather_k<K, POL, SP><<<nsm * GRID, 256>>>(n, dl, doff, dP, dpool, dout);                                      \
  }, true);
  G(12, 0, 0, 8)
  G(20, 0, 0, 8)
  G(12, 1, 0, 8)
  G(12, 2, 0, 8)
  G(12, 1, 1, 8)
  G(12, 2, 1, 8)
  G(12, 0, 1, 8)
  G(12, 1, 2, 8)
  G(20, 1, 1, 8)
  G(12, 1, 1, 4)
  G(12, 1, 1, 16)
  G(8, 1, 1, 8)


  {
    cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
    printf("l2 %d persistingMax %d accessPolicyMaxWindow %d\n", prop.l2CacheSize, prop.persistingL2CacheMaxSize, prop.accessPolicyMaxWindowSize);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize));
    G(12, 1, 1, 8)
    G(12, 0, 1, 8)
    cudaStreamAttrValue av = {};
    av.accessPolicyWindow.base_ptr = dpool;
    av.accessPolicyWindow.num_bytes = std::min<size_t>(pool_len * 8, prop.accessPolicyMaxWindowSize);
    av.accessPolicyWindow.hitRatio = 1.0f;
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &av));
    G(12, 0, 1, 8)
    G(12, 0, 0, 8)
    av.accessPolicyWindow.num_bytes = 0;
    CK(cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &av));
    CK(cudaCtxResetPersistingL2Cache());
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
  }
  int* dPo; unsigned* dtk; int64_t* dtot;
  const int64_t maxtiles = (n + 31) / 32, SL = 64 + maxtiles * 8;
  CK(cudaMalloc(&dPo, (n + 1) * 4)); CK(cudaMalloc(&dtk, SL * 8 * 64)); CK(cudaMalloc(&dtot, 16));
  int launch_no = 0;
#define F(K, MB, SP, GPW) FD(K, MB, SP, GPW, 0, 8, 0)
#define FD(K, MB, SP, GPW, DBG, NW, OWN)                                                                          \
  launch_no = 0; CK(cudaMemset(dtk, 0, SL * 8 * 64));                                                \
  run("fused K" #K " minb" #MB " sp" #SP " gpw" #GPW " nw" #NW " own" #OWN, [&] {                                          \
    const int64_t nt = (n + NW * 32 * GPW - 1) / (NW * 32 * GPW);                                            \
    unsigned* tk = (unsigned*)((char*)dtk + (launch_no % 64) * SL * 8);                              \
    if (launch_no % 64 == 63) cudaMemsetAsync(dtk, 0, SL * 8 * 64);                                  \
    ++launch_no;                                                                                     \
    fused_k<K, MB, SP, GPW, DBG, NW, OWN><<<nt, NW * 32>>>(n, dl, doff, dpool, dout, dPo, tk, (uint64_t*)((char*)tk + 64), dtot); \
  }, true);

  {
    // two kernels: cub exclusive scan of the lengths into int64, then the prefix-given gather
    void* tmp = nullptr; size_t tb = 0;
    cub::TransformInputIterator<int64_t, cub::CastOp<int64_t>, const int*> it(dl, cub::CastOp<int64_t>());
    cub::DeviceScan::ExclusiveSum(tmp, tb, it, dP, n + 1);
    CK(cudaMalloc(&tmp, tb));
    run("cub scan only", [&] { cub::DeviceScan::ExclusiveSum(tmp, tb, it, dP, n + 1); }, false);
    run("cub scan + gather K12 grid8", [&] {
      cub::DeviceScan::ExclusiveSum(tmp, tb, it, dP, n + 1);
      gather_k<12, 0, 1><<<nsm * 8, 256>>>(n, dl, doff, dP, dpool, dout);
    }, true);
  }

#define TG(NS, NW, STAGE)                                                                                       \
  {                                                                                                             \
    const size_t smem = (size_t)NS * NW * STAGE;                                                                \
    CK(cudaFuncSetAttribute(tma_gather<NS, NW, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
    run("tma gather ns" #NS " nw" #NW, [&] { tma_gather<NS, NW, STAGE><<<nsm, NW * 32, smem>>>(n, dl, doff, dP, dpool, dout); }, true); \
  }
  TG(4, 8, 6144)
  TG(8, 4, 6144)
  TG(3, 10, 6144)
  TG(2, 16, 6144)
  run("gather K12 pol0 sp1 grid489", [&] { gather_k<12, 0, 1><<<489, 256>>>(n, dl, doff, dP, dpool, dout); }, true);
  F(12, 4, 1, 8)
  FD(12, 4, 1, 8, 4, 8, 0)
  FD(12, 4, 1, 7, 4, 8, 0)
  FD(12, 4, 1, 8, 4, 8, 2)
  run("gather_o K12", [&] { gather_o<12><<<nsm * 8, 256>>>(n, dl, doff, dP, dpool, dout); }, true);
  run("gather_o K16", [&] { gather_o<16><<<nsm * 8, 256>>>(n, dl, doff, dP, dpool, dout); }, true);

#define FC(K, NS, NW, GPW, MINB)                                                                      \
  {                                                                                                  \
    const size_t smem = (size_t)NW * NS * K * 32 * 8 + (size_t)NW * GPW * 32 * 12;                   \
    CK(cudaFuncSetAttribute(fused_cp<K, NS, NW, GPW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fused_cp<K, NS, NW, GPW, MINB>, NW * 32, smem)); \
    printf("occ %d smem %zu\n", occ, smem);                                                         \
    launch_no = 0; CK(cudaMemset(dtk, 0, SL * 8 * 64));                                              \
    run("fcp K" #K " ns" #NS " nw" #NW " gpw" #GPW, [&] {                                            \
      const int64_t nt = (n + NW * 32 * GPW - 1) / (NW * 32 * GPW);                                  \
      unsigned* tk = (unsigned*)((char*)dtk + (launch_no % 64) * SL * 8);                            \
      if (launch_no % 64 == 63) cudaMemsetAsync(dtk, 0, SL * 8 * 64);                                \
      ++launch_no;                                                                                   \
      fused_cp<K, NS, NW, GPW, MINB><<<nt, NW * 32, smem>>>(n, dl, doff, dpool, dout, dPo, tk, (uint64_t*)((char*)tk + 64), dtot); \
    }, true);                                                                                        \
  }

#define FW(K, GPW, MINB, PF, CPS)                                                                     \
  launch_no = 0; CK(cudaMemset(dtk, 0, SL * 8 * 64));                                                \
  run("fw K" #K " gpw" #GPW " minb" #MINB " pf" #PF " cps" #CPS, [&] {                               \
    unsigned* tk = (unsigned*)((char*)dtk + (launch_no % 64) * SL * 8);                              \
    if (launch_no % 64 == 63) cudaMemsetAsync(dtk, 0, SL * 8 * 64);                                  \
    ++launch_no;                                                                                     \
    fused_w<K, GPW, MINB, PF><<<nsm * CPS, 256>>>(n, dl, doff, dpool, dout, dPo, tk, (uint64_t*)((char*)tk + 64), dtot); \
  }, true);

#define FB(K, MINB, RPT, CPS)                                                                         \
  launch_no = 0; CK(cudaMemset(dtk, 0, SL * 8 * 64));                                                \
  run("fb K" #K " minb" #MINB " rpt" #RPT " cps" #CPS, [&] {                                         \
    int64_t br = (n + nsm * CPS - 1) / (nsm * CPS); br = (br + 31) / 32 * 32;                        \
    if (br > 256 * RPT) br = 256 * RPT;                                                              \
    const int64_t nb = (n + br - 1) / br;                                                            \
    unsigned* tk = (unsigned*)((char*)dtk + (launch_no % 64) * SL * 8);                              \
    if (launch_no % 64 == 63) cudaMemsetAsync(dtk, 0, SL * 8 * 64);                                  \
    ++launch_no;                                                                                     \
    fused_b<K, MINB, RPT><<<nb, 256>>>(n, dl, doff, dpool, dout, dPo, tk, (uint64_t*)((char*)tk + 64), dtot, br); \
  }, true);
  {
    std::vector<int> gp(n + 1);
    CK(cudaMemcpy(gp.data(), dPo, (n + 1) * 4, cudaMemcpyDeviceToHost));
    bool ok = true;
    for (int64_t i = 0; i <= n; ++i) ok &= gp[i] == (int)P[i];
    printf("fused prefix %s\n", ok ? "OK" : "MISMATCH");
  }
  return 0;
}
