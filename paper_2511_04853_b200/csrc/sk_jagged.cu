// Jagged-collection packer (K4): single-pass exclusive prefix sum with
// decoupled look-back, then a load-balanced gather of variable-length member
// lists into packed per-field pools.
//
// Reference: Collection.jagged_fill (collection.py:537-556) computes
// pv[1:] = np.cumsum(lengths, int64).astype(index dtype) and
// np.concatenate(segments); import_external (transfer.py:297-320) does the same
// for multi-leaf members. Both walk the segments in a Python loop.
#include <algorithm>

#include "sk_internal.cuh"

namespace sk {
namespace jag {

constexpr int SCAN_NT = 256;
constexpr int SCAN_IT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IT;  // 4096 lengths per CTA

constexpr uint64_t FLAG_A = 1ull << 62;  // tile aggregate published
constexpr uint64_t FLAG_P = 2ull << 62;  // inclusive prefix published
constexpr uint64_t VAL_MASK = (1ull << 62) - 1;

__device__ __forceinline__ int64_t load_int(const void* p, int type, int64_t i) {
  switch (type) {
    case SK_U8: case SK_BOOL: return static_cast<const uint8_t*>(p)[i];
    case SK_U16: return static_cast<const uint16_t*>(p)[i];
    case SK_U32: return static_cast<const uint32_t*>(p)[i];
    case SK_I32: return static_cast<const int32_t*>(p)[i];
    default: return static_cast<const int64_t*>(p)[i];
  }
}

// int64 -> index dtype by truncation, exactly numpy astype on the cumsum
__device__ __forceinline__ void store_int(void* p, int type, int64_t i, int64_t v) {
  switch (type) {
    case SK_U8: case SK_BOOL: static_cast<uint8_t*>(p)[i] = static_cast<uint8_t>(v); break;
    case SK_U16: static_cast<uint16_t*>(p)[i] = static_cast<uint16_t>(v); break;
    case SK_U32: case SK_I32: static_cast<uint32_t*>(p)[i] = static_cast<uint32_t>(v); break;
    default: static_cast<int64_t*>(p)[i] = v; break;
  }
}

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// padded smem index: one int64 of padding per 16 keeps the per-thread
// consecutive reads at a 2-way (64-bit) bank pattern
__device__ __forceinline__ int pad(int e) { return e + (e >> 4); }

__global__ void __launch_bounds__(SCAN_NT) scan_kernel(int64_t n, const void* __restrict__ lens, int lens_type,
                                                       void* __restrict__ out, int out_type, uint64_t* status,
                                                       unsigned int* ticket, int64_t* total_out,
                                                       int64_t* __restrict__ out64) {
  __shared__ int64_t s[SCAN_TILE + SCAN_TILE / 16];
  __shared__ int64_t warp_tot[SCAN_NT / 32];
  __shared__ int64_t s_excl;
  __shared__ unsigned int s_tile;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);  // dynamic tile order: look-back never waits on an unscheduled CTA
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t base = tile * SCAN_TILE;

#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    const int e = i * SCAN_NT + tid;
    const int64_t idx = base + e;
    s[pad(e)] = idx < n ? load_int(lens, lens_type, idx) : 0;
  }
  __syncthreads();
  int64_t loc[SCAN_IT];
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    acc += s[pad(tid * SCAN_IT + i)];
    loc[i] = acc;
  }
  // block-wide exclusive scan of the per-thread totals
  int64_t x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  int64_t warp_off = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < SCAN_NT / 32; ++w) {
    if (w < warp) warp_off += warp_tot[w];
    agg += warp_tot[w];
  }
  const int64_t thread_excl = warp_off + x - acc;

  if (warp == 0) {
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_release(&status[0], FLAG_P | (static_cast<uint64_t>(agg) & VAL_MASK));
    } else {
      if (lane == 0) st_release(&status[tile], FLAG_A | (static_cast<uint64_t>(agg) & VAL_MASK));
      int64_t end = tile - 1;  // look back over [end-31, end]
      while (true) {
        const int64_t idx = end - lane;
        uint64_t st = idx >= 0 ? ld_acquire(&status[idx]) : FLAG_P;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_acquire(&status[idx]);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        int64_t v = static_cast<int64_t>(st & VAL_MASK);
        if (pmask) {
          const int first_p = __ffs(pmask) - 1;  // nearest predecessor with a full prefix
          if (lane > first_p) v = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (pmask) break;
        end -= 32;
      }
      if (lane == 0) st_release(&status[tile], FLAG_P | (static_cast<uint64_t>(excl + agg) & VAL_MASK));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  const int64_t off = s_excl + thread_excl;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) s[pad(tid * SCAN_IT + i)] = off + loc[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    const int e = i * SCAN_NT + tid;
    const int64_t idx = base + e;
    if (idx < n) {
      const int64_t v = s[pad(e)];
      store_int(out, out_type, idx + 1, v);
      if (out64) out64[idx + 1] = v;  // non-wrapped copy for the gather
      if (idx == n - 1 && total_out) *total_out = v;
    }
  }
  if (tile == 0 && tid == 0) {
    store_int(out, out_type, 0, 0);
    if (out64) out64[0] = 0;
  }
}

// ---- scatter ------------------------------------------------------------------------

constexpr int SC_NT = 256;
constexpr int SC_IT = 8;
constexpr int SC_TILE = SC_NT * SC_IT;  // output members per CTA
constexpr int SC_CMAX = 1024;           // records staged in smem per CTA
constexpr int SC_MAXF = 8;

struct ScatterArgs {
  int64_t n;
  const void* prefix;
  int prefix_type;
  const int64_t* src_off;
  const uint8_t* src_pool;
  int64_t member_stride;
  int64_t total;             // members to gather, or the capacity bound when total_dev is set
  const int64_t* total_dev;  // device-resident total (fused pack): gather min(*total_dev, total)
  int nfields;
  int aligned;  // all member fields naturally aligned
  int64_t field_off[SC_MAXF];
  int32_t field_size[SC_MAXF];
  uint8_t* dst[SC_MAXF];
};

// last record c in [lo, hi) with prefix[c] <= j
__device__ __forceinline__ int64_t search_global(const ScatterArgs& A, int64_t lo, int64_t hi, int64_t j) {
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (load_int(A.prefix, A.prefix_type, mid) <= j) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Same answer as search_global, found by a whole warp: each round the 32
// lanes probe 32 evenly spaced records and keep the sub-range after the last
// probe that is <= j, so 1M records need 4 rounds of parallel loads instead
// of 20 dependent ones. All lanes return the result.
__device__ __forceinline__ int64_t search_warp(const ScatterArgs& A, int64_t lo, int64_t hi, int64_t j) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool ok = p < hi && load_int(A.prefix, A.prefix_type, p) <= j;
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    const int last = 31 - __clz(mask);  // lane 0 always qualifies (prefix[lo] <= j)
    const int64_t nlo = lo + last * step;
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  const int64_t p = lo + lane;
  const bool ok = p < hi && load_int(A.prefix, A.prefix_type, p) <= j;
  const unsigned mask = __ballot_sync(0xffffffffu, ok);
  return lo + (31 - __clz(mask));
}

__device__ __forceinline__ uint64_t load_member(const uint8_t* p, int isz, bool aligned) {
  if (aligned) {
    switch (isz) {
      case 1: return *p;
      case 2: return *reinterpret_cast<const uint16_t*>(p);
      case 4: return *reinterpret_cast<const uint32_t*>(p);
      default: return *reinterpret_cast<const uint64_t*>(p);
    }
  }
  uint64_t v = 0;
  for (int i = 0; i < isz; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

__device__ __forceinline__ void store_member(uint8_t* p, uint64_t v, int isz) {
  switch (isz) {
    case 1: *p = static_cast<uint8_t>(v); break;
    case 2: *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>(v); break;
    case 4: *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>(v); break;
    default: *reinterpret_cast<uint64_t*>(p) = v; break;
  }
}

// members to gather. Fused pack: the device total if it fits the capacity
// bound, else nothing -- on overflow the (narrow) prefix may have wrapped and
// the host redoes the pack with grown pools, so no search may run over it.
__device__ __forceinline__ int64_t eff_total(const ScatterArgs& A) {
  if (!A.total_dev) return A.total;
  const int64_t t = *A.total_dev;
  return t <= A.total ? t : 0;
}

// one padding word per 32 keeps both the consecutive-per-thread scan reads and
// the strided member reads at <= 2-way bank conflicts
__device__ __forceinline__ int cpad(int e) { return e + (e >> 5); }

// first record of every member tile: starts[b] = last record c with
// prefix[c] <= b * SC_TILE (one warp per tile, all tiles in parallel), and
// starts[ntiles] = the last record holding a member.
__global__ void __launch_bounds__(256) tile_start_kernel(const __grid_constant__ ScatterArgs A, int64_t* starts,
                                                         int64_t ntiles) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (b > ntiles) return;
  const int64_t T = eff_total(A);
  if (T <= 0) return;
  const int64_t j = b * SC_TILE < T ? b * SC_TILE : T - 1;
  const int64_t c = search_warp(A, 0, A.n, j);
  if ((threadIdx.x & 31) == 0) starts[b] = c;
}

__global__ void __launch_bounds__(SC_NT) scatter_kernel(const __grid_constant__ ScatterArgs A,
                                                        const int64_t* __restrict__ starts) {
  __shared__ int64_t sP[SC_CMAX + 1];
  __shared__ int64_t sOff[SC_CMAX];
  __shared__ int32_t sCl[SC_TILE + SC_TILE / 32];  // member -> record (relative), padded
  __shared__ int32_t sWarpMax[SC_NT / 32];
  const int tid = threadIdx.x;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * SC_TILE;
  const int64_t T = eff_total(A);
  if (j0 >= T) return;
  const int64_t j1 = min(j0 + SC_TILE, T);
  // the records covering [j0, j1) lie in [starts[b], starts[b+1]]
  const int64_t lo = starts[blockIdx.x];
  const int64_t cnt = starts[blockIdx.x + 1] - lo + 1;
  const bool staged = cnt <= SC_CMAX;
  if (staged) {
    for (int k = tid; k <= cnt; k += SC_NT) {
      sP[k] = load_int(A.prefix, A.prefix_type, lo + k);
      if (k < cnt) sOff[k] = A.src_off[lo + k];
    }
  }
  __syncthreads();
  if (staged) {
    // record of every member of the tile: mark where each non-empty record
    // starts, then an inclusive max-scan carries the index forward
    const int m = static_cast<int>(j1 - j0);
    for (int e = tid; e < SC_TILE; e += SC_NT) sCl[cpad(e)] = 0;
    __syncthreads();
    for (int k = tid + 1; k < cnt; k += SC_NT) {
      const int64_t s = sP[k] - j0;
      if (s > 0 && s < m && sP[k + 1] > sP[k]) sCl[cpad(static_cast<int>(s))] = k;
    }
    __syncthreads();
    int vals[SC_IT];
    int run = 0;
#pragma unroll
    for (int i = 0; i < SC_IT; ++i) {
      run = max(run, sCl[cpad(tid * SC_IT + i)]);
      vals[i] = run;
    }
    int x = run;  // warp-inclusive max of the per-thread maxima
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) x = max(x, __shfl_up_sync(0xffffffffu, x, o));
    if ((tid & 31) == 31) sWarpMax[tid >> 5] = x;
    const int excl_lane = __shfl_up_sync(0xffffffffu, x, 1);
    __syncthreads();
    int carry = (tid & 31) ? excl_lane : 0;
    for (int w = 0; w < (tid >> 5); ++w) carry = max(carry, sWarpMax[w]);
#pragma unroll
    for (int i = 0; i < SC_IT; ++i) sCl[cpad(tid * SC_IT + i)] = max(vals[i], carry);
    __syncthreads();
  }
  // resolve the source element of each of this thread's members first, then move
  int64_t src[SC_IT];
#pragma unroll
  for (int i = 0; i < SC_IT; ++i) {
    const int64_t j = j0 + i * SC_NT + tid;
    src[i] = -1;
    if (j < j1) {
      int64_t c, pc, oc;
      if (staged) {
        const int a = sCl[cpad(i * SC_NT + tid)];
        pc = sP[a];
        oc = sOff[a];
      } else {
        c = search_global(A, lo, lo + cnt, j);
        pc = load_int(A.prefix, A.prefix_type, c);
        oc = A.src_off[c];
      }
      src[i] = oc + (j - pc);
    }
  }
  const bool al = A.aligned;
  for (int f = 0; f < A.nfields; ++f) {
    const int isz = A.field_size[f];
    const uint8_t* sp = A.src_pool + A.field_off[f];
    uint8_t* dp = A.dst[f];
    uint64_t v[SC_IT];
#pragma unroll
    for (int i = 0; i < SC_IT; ++i)
      v[i] = src[i] >= 0 ? load_member(sp + src[i] * A.member_stride, isz, al) : 0;
#pragma unroll
    for (int i = 0; i < SC_IT; ++i) {
      const int64_t j = j0 + i * SC_NT + tid;
      if (src[i] >= 0) store_member(dp + j * isz, v[i], isz);
    }
  }
}

}  // namespace jag
}  // namespace sk

using namespace sk;

extern "C" {

int sk_jagged_scratch_bytes(int64_t n, size_t* nbytes) {
  if (!nbytes) return set_error(SK_ERR_INVALID, "null out");
  const int64_t tiles = n > 0 ? (n + jag::SCAN_TILE - 1) / jag::SCAN_TILE : 0;
  *nbytes = static_cast<size_t>(16 + tiles * 8);
  return SK_OK;
}

static bool int_type(int t) {
  return t == SK_U8 || t == SK_U16 || t == SK_U32 || t == SK_U64 || t == SK_I32 || t == SK_I64 || t == SK_BOOL;
}

int sk_jagged_scan(int64_t n, const void* lens, int lens_type, void* prefix, int prefix_type, void* scratch,
                   size_t scratch_bytes, int64_t* total_dev, uintptr_t stream) {
  if (n < 0) return set_error(SK_ERR_INVALID, "negative record count");
  if (!int_type(lens_type) || !int_type(prefix_type) || lens_type == SK_BOOL || prefix_type == SK_BOOL)
    return set_error(SK_ERR_INVALID, "jagged lengths and prefix need integer types");
  size_t need = 0;
  sk_jagged_scratch_bytes(n, &need);
  if (scratch_bytes < need) return set_error(SK_ERR_INVALID, "scratch too small: %zu < %zu", scratch_bytes, need);
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  if (n == 0) {
    // P = [0]
    const int isz = dtype_size(prefix_type);
    SK_TRY(cudaMemsetAsync(prefix, 0, isz, s));
    if (total_dev) SK_TRY(cudaMemsetAsync(total_dev, 0, 8, s));
    return SK_OK;
  }
  SK_TRY(cudaMemsetAsync(scratch, 0, need, s));
  const int64_t tiles = (n + jag::SCAN_TILE - 1) / jag::SCAN_TILE;
  unsigned int* ticket = static_cast<unsigned int*>(scratch);
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(scratch) + 16);
  jag::scan_kernel<<<static_cast<unsigned>(tiles), jag::SCAN_NT, 0, s>>>(n, lens, lens_type, prefix, prefix_type,
                                                                          status, ticket, total_dev, nullptr);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

static int scatter_impl(int64_t n, const void* prefix, int prefix_type, const int64_t* src_off, const void* src_pool,
                        int64_t member_stride, int nfields, const int64_t* field_off, const int32_t* field_size,
                        void* const* dst_pools, int64_t total, const int64_t* total_dev, uintptr_t stream,
                        int64_t* starts_buf = nullptr) {
  if (n < 0 || total < 0) return set_error(SK_ERR_INVALID, "negative sizes");
  if (nfields < 1 || nfields > jag::SC_MAXF) return set_error(SK_ERR_INVALID, "nfields %d outside [1, 8]", nfields);
  if (!int_type(prefix_type)) return set_error(SK_ERR_INVALID, "prefix type must be an integer type");
  jag::ScatterArgs A;
  memset(&A, 0, sizeof(A));
  A.n = n;
  A.prefix = prefix;
  A.prefix_type = prefix_type;
  A.src_off = src_off;
  A.src_pool = static_cast<const uint8_t*>(src_pool);
  A.member_stride = member_stride;
  A.total = total;
  A.total_dev = total_dev;
  A.nfields = nfields;
  bool aligned = true;
  for (int f = 0; f < nfields; ++f) {
    const int isz = field_size[f];
    if (isz != 1 && isz != 2 && isz != 4 && isz != 8) return set_error(SK_ERR_INVALID, "member field size %d", isz);
    if (field_off[f] < 0 || field_off[f] + isz > member_stride)
      return set_error(SK_ERR_RANGE, "member field %d outside the member stride", f);
    A.field_off[f] = field_off[f];
    A.field_size[f] = isz;
    A.dst[f] = static_cast<uint8_t*>(dst_pools[f]);
    aligned = aligned && (field_off[f] % isz == 0) && (member_stride % isz == 0) &&
              (reinterpret_cast<uintptr_t>(src_pool) % isz == 0);
  }
  A.aligned = aligned;
  if (total == 0 || n == 0) return SK_OK;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  const int64_t blocks = (total + jag::SC_TILE - 1) / jag::SC_TILE;
  int64_t* starts = starts_buf;
  if (!starts) SK_TRY(cudaMallocAsync(&starts, static_cast<size_t>(blocks + 1) * sizeof(int64_t), s));
  jag::tile_start_kernel<<<static_cast<unsigned>((blocks + 1 + 7) / 8), 256, 0, s>>>(A, starts, blocks);
  SK_TRY(cudaGetLastError());
  jag::scatter_kernel<<<static_cast<unsigned>(blocks), jag::SC_NT, 0, s>>>(A, starts);
  SK_TRY(cudaGetLastError());
  if (!starts_buf) SK_TRY(cudaFreeAsync(starts, s));
  return SK_OK;
}

int sk_jagged_scatter(int64_t n, const void* prefix, int prefix_type, const int64_t* src_off, const void* src_pool,
                      int64_t member_stride, int nfields, const int64_t* field_off, const int32_t* field_size,
                      void* const* dst_pools, int64_t total, uintptr_t stream) {
  return scatter_impl(n, prefix, prefix_type, src_off, src_pool, member_stride, nfields, field_off, field_size,
                      dst_pools, total, nullptr, stream);
}

int sk_jagged_pack(int64_t n, const void* lens, int lens_type, void* prefix, int prefix_type, const int64_t* src_off,
                   const void* src_pool, int64_t member_stride, int nfields, const int64_t* field_off,
                   const int32_t* field_size, void* const* dst_pools, int64_t capacity, void* scratch,
                   size_t scratch_bytes, int64_t* total_dev, uintptr_t stream) {
  if (n < 0 || capacity < 0) return set_error(SK_ERR_INVALID, "negative sizes");
  if (!total_dev) return set_error(SK_ERR_INVALID, "total_dev is required");
  if (!int_type(lens_type) || !int_type(prefix_type) || lens_type == SK_BOOL || prefix_type == SK_BOOL)
    return set_error(SK_ERR_INVALID, "jagged lengths and prefix need integer types");
  size_t need = 0;
  sk_jagged_scratch_bytes(n, &need);
  if (scratch_bytes < need) return set_error(SK_ERR_INVALID, "scratch too small: %zu < %zu", scratch_bytes, need);
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  if (n == 0) {
    SK_TRY(cudaMemsetAsync(prefix, 0, dtype_size(prefix_type), s));
    SK_TRY(cudaMemsetAsync(total_dev, 0, 8, s));
    return SK_OK;
  }
  // a prefix type that can wrap below the capacity needs an int64 copy for the gather
  const int bits = 8 * dtype_size(prefix_type) - ((prefix_type == SK_I32 || prefix_type == SK_I64) ? 1 : 0);
  const bool may_wrap = bits < 63 && capacity >= (int64_t(1) << bits);
  int64_t* p64 = nullptr;
  if (may_wrap) SK_TRY(cudaMallocAsync(&p64, static_cast<size_t>(n + 1) * sizeof(int64_t), s));
  SK_TRY(cudaMemsetAsync(scratch, 0, need, s));
  const int64_t tiles = (n + jag::SCAN_TILE - 1) / jag::SCAN_TILE;
  unsigned int* ticket = static_cast<unsigned int*>(scratch);
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(scratch) + 16);
  jag::scan_kernel<<<static_cast<unsigned>(tiles), jag::SCAN_NT, 0, s>>>(n, lens, lens_type, prefix, prefix_type,
                                                                          status, ticket, total_dev, p64);
  SK_TRY(cudaGetLastError());
  // gather bounded by the pools' capacity; the kernels read the true total on the device
  // the tile-start array lives in the caller's scratch when it is large enough
  const size_t scan_part = (need + 255) & ~size_t(255);
  const size_t starts_need = static_cast<size_t>((capacity + jag::SC_TILE - 1) / jag::SC_TILE + 1) * sizeof(int64_t);
  int64_t* starts = scratch_bytes >= scan_part + starts_need
                        ? reinterpret_cast<int64_t*>(static_cast<uint8_t*>(scratch) + scan_part)
                        : nullptr;
  int rc = capacity ? scatter_impl(n, p64 ? static_cast<const void*>(p64) : prefix, p64 ? SK_I64 : prefix_type,
                                   src_off, src_pool, member_stride, nfields, field_off, field_size, dst_pools,
                                   capacity, total_dev, stream, starts)
                    : SK_OK;
  if (p64) cudaFreeAsync(p64, s);
  return rc;
}

}  // extern "C"
