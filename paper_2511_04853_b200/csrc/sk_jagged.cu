// Jagged-collection packer (K4): exclusive prefix sum of the lengths, then a
// load-balanced gather of variable-length member lists into packed per-field
// pools.
//
// Reference: Collection.jagged_fill (collection.py:537-556) computes
// pv[1:] = np.cumsum(lengths, int64).astype(index dtype) and
// np.concatenate(segments); import_external (transfer.py:297-320) does the same
// for multi-leaf members. Both walk the segments in a Python loop.
//
// Scan: tiles of 4096 lengths. Up to SCAN_DIRECT_TILES tiles it is
// reduce-then-scan (tile sums, then every tile adds up its predecessors' sums
// in parallel: no inter-CTA waiting at all); beyond that a single-pass
// decoupled look-back. In pack mode the scan also emits the gather's work
// split: starts[w] = the record holding member w*W, and 1 + the last non-empty
// record.
//
// sk_jagged_pack with one aligned 4/8-byte member field runs both in ONE
// kernel (pack_reg_kernel, below): 2048-record tiles with decoupled look-back
// and a register gather. 2-4 such fields of an 8/16-byte member record run in
// pack_fused_kernel: per-CTA record blocks whose prefixes come from the
// predecessor blocks' published totals, then per-sub-tile smem tables feeding
// the window gather. The two-kernel path (scan, then gather) serves
// sk_jagged_scan / sk_jagged_scatter and the other member layouts.
//
// Gather: one warp per W = 256 consecutive output members, no block barriers.
// The warp loads its record window (<= 32 records per batch, one per lane),
// ranks the non-empty ones with ballot/popc and marks where each starts with
// redux.or bitmasks; member j's record is then a popc away and its source is
// j + (src_off[c] - P[c]). The next window's loads are in flight while this
// window's members are.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <random>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "sk_internal.cuh"

namespace sk {
namespace jag {

constexpr int SCAN_NT = 256;
constexpr int SCAN_IT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IT;  // 4096 lengths per CTA
constexpr int64_t SCAN_DIRECT_TILES = 4096;   // reduce-then-scan up to 16.7M records

constexpr int W = 256;          // output members per warp task (= the boundary pitch)
constexpr int W_CH = W / 32;    // 32-member chunks per task
constexpr int G_NT = 256;       // gather threads per CTA
constexpr int G_MAXF = 8;

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

__device__ __forceinline__ int dtype_size_dev(int type) {
  switch (type) {
    case SK_U8: case SK_BOOL: return 1;
    case SK_U16: return 2;
    case SK_U32: case SK_I32: return 4;
    default: return 8;
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

// the look-back status words carry their value: nothing else is published
// with them, so relaxed (L2-coherent, no L1 invalidation) access is enough
__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// polling read that must not be served from a stale L1 line: cache-global (L2) access
__device__ __forceinline__ uint64_t ld_poll(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// padded smem index: one int64 of padding per 16 keeps the per-thread
// consecutive reads at a 2-way (64-bit) bank pattern
__device__ __forceinline__ int pad(int e) { return e + (e >> 4); }

// programmatic dependent launch: the next kernel of the chain may be scheduled
// now (its CTAs park in pdl_wait until this grid has completed and flushed)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

struct ScanOut {
  void* out;                 // prefix, index dtype, n + 1 entries
  int out_type;
  int64_t* total;            // device total (optional)
  int64_t* out64;            // non-wrapped int64 copy of the prefix (optional)
  int64_t* starts;           // pack mode: starts[w] = record holding member w*W
  int64_t nstarts;
  unsigned long long* last;  // pack mode: atomicMax of 1 + non-empty record index
};

struct TileScan {
  int64_t loc[SCAN_IT];  // inclusive scan of this thread's 16 consecutive lengths
  int64_t thread_excl;   // exclusive prefix of this thread within the tile
  int64_t agg;           // tile total
};

// lengths of tile `tile` -> smem, per-thread and block-wide scans
__device__ __forceinline__ void tile_scan(int64_t n, const void* lens, int lens_type, int64_t tile, int64_t* s,
                                          int64_t* warp_tot, TileScan& ts) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = tile * SCAN_TILE;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    const int e = i * SCAN_NT + tid;
    const int64_t idx = base + e;
    s[pad(e)] = idx < n ? load_int(lens, lens_type, idx) : 0;
  }
  __syncthreads();
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    acc += s[pad(tid * SCAN_IT + i)];
    ts.loc[i] = acc;
  }
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
  ts.thread_excl = warp_off + x - acc;
  ts.agg = agg;
}

// tile exclusive prefix known: write P[base+1 .. base+4096], the boundaries and the last non-empty record
__device__ __forceinline__ void tile_write(int64_t n, int64_t tile, int64_t tile_excl, const TileScan& ts, int64_t* s,
                                           const ScanOut& O) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t base = tile * SCAN_TILE;
  const int64_t off = tile_excl + ts.thread_excl;
  __syncthreads();  // everyone has read the lengths out of s
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) s[pad(tid * SCAN_IT + i)] = off + ts.loc[i];
  __syncthreads();
  int64_t last = -1;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    const int e = i * SCAN_NT + tid;
    const int64_t idx = base + e;
    if (idx < n) {
      const int64_t v = s[pad(e)];
      store_int(O.out, O.out_type, idx + 1, v);
      if (O.out64) O.out64[idx + 1] = v;
      if (idx == n - 1 && O.total) *O.total = v;
      if (O.starts) {
        const int64_t pv = e ? s[pad(e - 1)] : tile_excl;
        if (v > pv) {
          last = idx;
          const int64_t w1 = min((v - 1) / W, O.nstarts - 1);
          for (int64_t w = (pv + W - 1) / W; w <= w1; ++w) O.starts[w] = idx;
        }
      }
    }
  }
  if (O.starts) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
    if (lane == 0 && last >= 0) atomicMax(O.last, static_cast<unsigned long long>(last + 1));
  }
  if (tile == 0 && tid == 0) {
    store_int(O.out, O.out_type, 0, 0);
    if (O.out64) O.out64[0] = 0;
  }
}

// reduce-then-scan, pass 1: tile sums
__global__ void __launch_bounds__(SCAN_NT) tile_sum_kernel(int64_t n, const void* __restrict__ lens, int lens_type,
                                                           int64_t* __restrict__ agg, unsigned long long* last) {
  __shared__ int64_t red[SCAN_NT / 32];
  pdl_trigger();
  const int tid = threadIdx.x;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * SCAN_TILE;
  int64_t acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IT; ++i) {
    const int64_t idx = base + i * SCAN_NT + tid;
    if (idx < n) acc += load_int(lens, lens_type, idx);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    int64_t t = 0;
#pragma unroll
    for (int w = 0; w < SCAN_NT / 32; ++w) t += red[w];
    agg[blockIdx.x] = t;
    if (blockIdx.x == 0 && last) *last = 0;
  }
}

// reduce-then-scan, pass 2: each tile sums its predecessors' totals in parallel, then scans itself
__global__ void __launch_bounds__(SCAN_NT) tile_apply_kernel(int64_t n, const void* __restrict__ lens, int lens_type,
                                                             const int64_t* __restrict__ agg, const ScanOut O) {
  __shared__ int64_t s[SCAN_TILE + SCAN_TILE / 16];
  __shared__ int64_t warp_tot[SCAN_NT / 32];
  __shared__ int64_t red[SCAN_NT / 32];
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  int64_t pre = 0;
  for (int64_t k = tid; k < tile; k += SCAN_NT) pre += agg[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if ((tid & 31) == 0) red[tid >> 5] = pre;
  TileScan ts;
  tile_scan(n, lens, lens_type, tile, s, warp_tot, ts);  // its barriers also publish red[]
  int64_t excl = 0;
#pragma unroll
  for (int w = 0; w < SCAN_NT / 32; ++w) excl += red[w];
  tile_write(n, tile, excl, ts, s, O);
}

// single pass with decoupled look-back (large n): tiles in ticket order, warp 0
// looks back over 32 predecessors per round
__global__ void __launch_bounds__(SCAN_NT) scan_lookback_kernel(int64_t n, const void* __restrict__ lens,
                                                                int lens_type, uint64_t* status, unsigned int* ticket,
                                                                const ScanOut O) {
  __shared__ int64_t s[SCAN_TILE + SCAN_TILE / 16];
  __shared__ int64_t warp_tot[SCAN_NT / 32];
  __shared__ int64_t s_excl;
  __shared__ unsigned int s_tile;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);  // dynamic tile order: look-back never waits on an unscheduled CTA
  __syncthreads();
  const int64_t tile = s_tile;
  TileScan ts;
  tile_scan(n, lens, lens_type, tile, s, warp_tot, ts);
  if (tid < 32) {
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed(&status[0], FLAG_P | (static_cast<uint64_t>(ts.agg) & VAL_MASK));
    } else {
      if (lane == 0) st_relaxed(&status[tile], FLAG_A | (static_cast<uint64_t>(ts.agg) & VAL_MASK));
      int64_t end = tile - 1;  // look back over [end-31, end]
      while (true) {
        const int64_t idx = end - lane;
        uint64_t st = idx >= 0 ? ld_relaxed(&status[idx]) : FLAG_P;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          if ((st >> 62) == 0) st = ld_relaxed(&status[idx]);
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
      if (lane == 0) st_relaxed(&status[tile], FLAG_P | (static_cast<uint64_t>(excl + ts.agg) & VAL_MASK));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  tile_write(n, tile, s_excl, ts, s, O);
}

// ---- gather -------------------------------------------------------------------------

struct ScatterArgs {
  int64_t n;
  const void* prefix;
  int prefix_type;
  const int64_t* src_off;
  const uint8_t* src_pool;
  int64_t member_stride;
  int64_t total;             // members to gather, or the capacity bound when total_dev is set
  const int64_t* total_dev;  // device-resident total (fused pack): gather min(*total_dev, total)
  const int64_t* bad_dev;    // device-resident count of invalid segments (pack): gather nothing unless 0
  const int64_t* starts;     // starts[w] = record holding member w*W
  const unsigned long long* last_rec;  // 1 + last non-empty record
  int nfields;
  int64_t field_off[G_MAXF];
  int32_t field_size[G_MAXF];
  int32_t aligned[G_MAXF];   // naturally aligned source field: one load per member
  uint8_t* dst[G_MAXF];
};

// Same answer as a binary search for the last record c in [lo, hi) with
// prefix[c] <= j, found by a whole warp: each round the 32 lanes probe 32
// evenly spaced records and keep the sub-range after the last probe that is
// <= j (4 rounds of parallel loads for 1M records). All lanes return it.
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
  if (A.bad_dev && *A.bad_dev) return 0;
  if (!A.total_dev) return A.total;
  const int64_t t = *A.total_dev;
  return t <= A.total ? t : 0;
}

// work split for a prefix computed elsewhere (sk_jagged_scatter):
// starts[w] = last record c with prefix[c] <= w*W (one warp per task), and
// starts[ntasks] = 1 + the record holding the last member (last_rec form).
__global__ void __launch_bounds__(256) task_start_kernel(const __grid_constant__ ScatterArgs A, int64_t* starts,
                                                         int64_t ntasks) {
  pdl_trigger();
  const int64_t w = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (w > ntasks) return;
  const int64_t T = eff_total(A);
  if (T <= 0) return;
  const int64_t j = w < ntasks ? w * W : T - 1;
  const int64_t c = search_warp(A, 0, A.n, j);
  if ((threadIdx.x & 31) == 0) starts[w] = w < ntasks ? c : c + 1;
}

// one lane per record of a window batch: P[c], P[c+1], src_off[c], loaded
// unconditionally from a clamped (always valid) index and kept in the raw
// prefix type, so nothing consumes them before rank time (a predicated load
// merged with defaults would make the compiler wait for it right away)
template <class PT>
struct RecBatch {
  PT p, pn;
  int64_t off;
  int64_t c;  // unclamped record index: valid when c <= hi
};

template <class PT>
__device__ __forceinline__ RecBatch<PT> load_batch(const ScatterArgs& A, int64_t c, int64_t hi) {
  const PT* P = static_cast<const PT*>(A.prefix);
  const int64_t cc = max(min(c, hi), static_cast<int64_t>(0));
  RecBatch<PT> r;
  r.p = P[cc];
  r.pn = P[cc + 1];
  r.off = A.src_off[cc];
  r.c = c;
  return r;
}

__device__ __forceinline__ void task_window(const ScatterArgs& A, int64_t t, int64_t T, int64_t& lo, int64_t& hi) {
  lo = A.starts[t];
  hi = (t + 1) * W < T ? A.starts[t + 1] : static_cast<int64_t>(*A.last_rec) - 1;
}

// rank the batch's non-empty records (sD[rank] = src_off - P) and mark where each starts
template <class PT>
__device__ __forceinline__ void rank_batch(const RecBatch<PT>& r, int64_t hi, int64_t j0, int64_t j1, int64_t* sD,
                                           int& nr, unsigned (&masks)[W_CH]) {
  const int lane = threadIdx.x & 31;
  const int64_t p = static_cast<int64_t>(r.p), pn = static_cast<int64_t>(r.pn);
  const bool ne = r.c <= hi && pn > p && p < j1;
  const unsigned bal = __ballot_sync(0xffffffffu, ne);
  const int rank = nr + __popc(bal & ((1u << lane) - 1u));
  nr += __popc(bal);
  const int s = ne ? static_cast<int>(max(p - j0, static_cast<int64_t>(0))) : -1;
  if (ne) sD[rank] = r.off - p;
#pragma unroll
  for (int k = 0; k < W_CH; ++k)
    masks[k] |= __reduce_or_sync(0xffffffffu, (s >> 5) == k ? 1u << (s & 31) : 0u);
}

template <int MS>
struct MemberWord;
template <>
struct MemberWord<4> {
  using T = uint32_t;
};
template <>
struct MemberWord<8> {
  using T = uint64_t;
};
template <>
struct MemberWord<16> {  // a staged 16-byte member record (RS kernels)
  using T = uint4;
};

// PT: prefix element type. MS: 4 or 8 = one naturally aligned member field of
// that size (straight-line loads/stores); 0 = the generic field table.
template <class PT, int MS>
__global__ void __launch_bounds__(G_NT) gather_kernel(const __grid_constant__ ScatterArgs A) {
  __shared__ int64_t sD_all[G_NT / 32][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t* sD = sD_all[warp];
  pdl_wait();
  const int64_t T = eff_total(A);
  const int64_t ntasks = (T + W - 1) / W;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * (G_NT / 32);
  int64_t t = static_cast<int64_t>(blockIdx.x) * (G_NT / 32) + warp;
  if (t >= ntasks) return;
  const unsigned le_mask = 0xffffffffu >> (31 - lane);

  int64_t lo, hi;
  task_window(A, t, T, lo, hi);
  RecBatch<PT> cur = load_batch<PT>(A, lo + lane, hi);
  int64_t nlo, nhi;
  task_window(A, min(t + stride, ntasks - 1), T, nlo, nhi);

  while (true) {
    const int64_t j0 = t * W;
    const int64_t j1 = min(j0 + W, T);
    unsigned masks[W_CH];
#pragma unroll
    for (int k = 0; k < W_CH; ++k) masks[k] = 0;
    int nr = 0;
    rank_batch(cur, hi, j0, j1, sD, nr, masks);
    for (int64_t c0 = lo + 32; c0 <= hi; c0 += 32)
      rank_batch(load_batch<PT>(A, c0 + lane, hi), hi, j0, j1, sD, nr, masks);
    __syncwarp();
    // next task's window first: its loads fly together with this task's members
    const int64_t tn = t + stride;
    const bool more = tn < ntasks;
    // unconditional (clamped) prefetches: nothing waits on them before the next task
    const RecBatch<PT> nxt = load_batch<PT>(A, nlo + lane, nhi);
    int64_t nnlo, nnhi;
    task_window(A, min(tn + stride, ntasks - 1), T, nnlo, nnhi);
    // source element of each of this lane's members (chunk k: member j0 + 32k + lane)
    int64_t src[W_CH];
    int cum = 0;
#pragma unroll
    for (int k = 0; k < W_CH; ++k) {
      const int64_t j = j0 + 32 * k + lane;
      const int r = cum + __popc(masks[k] & le_mask) - 1;
      src[k] = j < j1 ? j + sD[r] : -1;
      cum += __popc(masks[k]);
    }
    if constexpr (MS != 0) {
      using V = typename MemberWord<MS>::T;
      const uint8_t* sp = A.src_pool + A.field_off[0];
      V* dp = reinterpret_cast<V*>(A.dst[0]);
      V v[W_CH];
#pragma unroll
      for (int k = 0; k < W_CH; ++k)
        v[k] = src[k] >= 0 ? *reinterpret_cast<const V*>(sp + src[k] * A.member_stride) : V(0);
#pragma unroll
      for (int k = 0; k < W_CH; ++k)
        if (src[k] >= 0) dp[j0 + 32 * k + lane] = v[k];
    } else {
      for (int f = 0; f < A.nfields; ++f) {
        const int isz = A.field_size[f];
        const bool al = A.aligned[f];
        const uint8_t* sp = A.src_pool + A.field_off[f];
        uint8_t* dp = A.dst[f];
        uint64_t v[W_CH];
#pragma unroll
        for (int k = 0; k < W_CH; ++k)
          v[k] = src[k] >= 0 ? load_member(sp + src[k] * A.member_stride, isz, al) : 0;
#pragma unroll
        for (int k = 0; k < W_CH; ++k)
          if (src[k] >= 0) store_member(dp + (j0 + 32 * k + lane) * isz, v[k], isz);
      }
    }
    if (!more) break;
    __syncwarp();  // sD is rewritten for the next task
    t = tn;
    lo = nlo;
    hi = nhi;
    cur = nxt;
    nlo = nnlo;
    nhi = nnhi;
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <int MS>
__device__ __forceinline__ void cp_async_member(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(s)), "l"(g), "n"(MS) : "memory");
}

constexpr int GA_WARPS = 8;  // warps per CTA of the async gather

// Async gather for one naturally aligned 4/8-byte member field with a
// 16-byte aligned destination pool. Members go global -> shared with cp.async
// (no registers held per load in flight) into a per-warp double buffer, and
// each task's 256 contiguous output members leave in ONE bulk (TMA) store, so
// every warp keeps two tasks of loads in flight while the previous task drains.
template <class PT, int MS>
__global__ void __launch_bounds__(GA_WARPS * 32) gather_async_kernel(const __grid_constant__ ScatterArgs A) {
  __shared__ __align__(128) uint8_t stage_all[GA_WARPS][2][W * MS];
  __shared__ int64_t sD_all[GA_WARPS][W];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t* sD = sD_all[warp];
  pdl_wait();
  const int64_t T = eff_total(A);
  const int64_t ntasks = (T + W - 1) / W;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * GA_WARPS;
  int64_t t = static_cast<int64_t>(blockIdx.x) * GA_WARPS + warp;
  if (t >= ntasks) return;
  const unsigned le_mask = 0xffffffffu >> (31 - lane);
  const uint8_t* sp = A.src_pool + A.field_off[0];
  uint8_t* dp = A.dst[0];

  // record windows run two tasks ahead of the member loads: (lo0, hi0, b0) is
  // this task, (lo1, hi1, b1) the next one (batch in flight), (lo2, hi2) the
  // one after (starts only)
  // (prefetches past the last task read clamped, valid entries and are never used)
  int64_t lo0, hi0, lo1, hi1, lo2, hi2;
  task_window(A, t, T, lo0, hi0);
  RecBatch<PT> b0 = load_batch<PT>(A, lo0 + lane, hi0);
  task_window(A, min(t + stride, ntasks - 1), T, lo1, hi1);
  RecBatch<PT> b1 = load_batch<PT>(A, lo1 + lane, hi1);
  task_window(A, min(t + 2 * stride, ntasks - 1), T, lo2, hi2);

  // drains task `pt` from buffer `pb`: bulk store of the 16-byte body, lanes store the tail
  auto drain = [&](int64_t pt, int pb) {
    const int64_t pj0 = pt * W;
    const int m = static_cast<int>(min(static_cast<int64_t>(W), T - pj0));
    const int body = (m * MS) & ~15;
    const uint8_t* buf = stage_all[warp][pb];
    fence_proxy_async();
    __syncwarp();
    if (lane == 0 && body) {
      bulk_s2g_plain(dp + pj0 * MS, buf, body);
      bulk_commit();
    }
    for (int e = body / MS + lane; e < m; e += 32)
      *reinterpret_cast<typename MemberWord<MS>::T*>(dp + (pj0 + e) * MS) =
          *reinterpret_cast<const typename MemberWord<MS>::T*>(buf + e * MS);
  };

  int it = 0;
  int64_t prev_t = -1;
  while (true) {
    const int64_t j0 = t * W;
    const int64_t j1 = min(j0 + W, T);
    unsigned masks[W_CH];
#pragma unroll
    for (int k = 0; k < W_CH; ++k) masks[k] = 0;
    int nr = 0;
    rank_batch(b0, hi0, j0, j1, sD, nr, masks);
    for (int64_t c0 = lo0 + 32; c0 <= hi0; c0 += 32)
      rank_batch(load_batch<PT>(A, c0 + lane, hi0), hi0, j0, j1, sD, nr, masks);
    __syncwarp();
    const int b = it & 1;
    uint8_t* buf = stage_all[warp][b];
    // the most recent bulk store (issued one task ago, draining task t - 2) read this buffer
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    int cum = 0;
#pragma unroll
    for (int k = 0; k < W_CH; ++k) {
      const int64_t j = j0 + 32 * k + lane;
      const int r = cum + __popc(masks[k] & le_mask) - 1;
      if (j < j1) cp_async_member<MS>(buf + (32 * k + lane) * MS, sp + (j + sD[r]) * A.member_stride);
      cum += __popc(masks[k]);
    }
    cp_async_commit();
    // window two tasks ahead
    const RecBatch<PT> b2 = load_batch<PT>(A, lo2 + lane, hi2);
    int64_t lo3, hi3;
    task_window(A, min(t + 3 * stride, ntasks - 1), T, lo3, hi3);
    if (prev_t >= 0) {
      cp_async_wait<1>();  // the previous task's members have landed
      drain(prev_t, b ^ 1);
    }
    prev_t = t;
    ++it;
    if (t + stride >= ntasks) break;
    __syncwarp();  // sD is rewritten for the next task
    t += stride;
    lo0 = lo1; hi0 = hi1; b0 = b1;
    lo1 = lo2; hi1 = hi2; b1 = b2;
    lo2 = lo3; hi2 = hi3;
  }
  cp_async_wait<0>();
  drain(prev_t, (it - 1) & 1);
  if (lane == 0) bulk_wait_read<0>();  // shared memory stays valid until the last bulk store has read it
}

// ---- fused pack: one persistent grid, one block of records per CTA --------------------
//
// The records are cut into one contiguous block per CTA (at most MAX_SUB
// sub-tiles of R = 1024 records; larger inputs hand out several blocks per
// CTA by ticket). Per block:
//   1. all threads sum the block's lengths (coalesced) and publish the block
//      total (status word); warp 0 then adds up every predecessor block's
//      published total for the block's exclusive prefix E. Blocks publish
//      after one pass over their own lengths, so this waits on no gather and
//      on no chain of other blocks' prefixes;
//   2. per sub-tile, all threads scan its lengths (4 consecutive records per
//      thread, prefetched into registers while the previous sub-tile
//      gathered) into smem tables -- local exclusive prefix Lx[r] and
//      D[r] = src_off[r] - Lx[r] -- store P[r] = E_sub + Lx[r] truncated to
//      the index dtype, and the warps claim the sub-tile's 256-member output
//      windows one at a time (an smem counter) and gather them from the tables.
// Output windows use the pool's global 256-member alignment: each window's
// 16-byte-aligned body leaves in one bulk store, and a window shared with a
// neighbour sub-tile is split at its ends, the ragged edges stored by lanes.
// Members go global -> shared with cp.async into a per-warp double buffer;
// each warp's pipeline runs on across sub-tiles, so the sub-tile scans hide
// behind members in flight.
// A sub-tile with more than DEFER_PER_REC members per record on average is
// not gathered by its owner: it is queued, and once every sub-tile is
// accounted for all warps of all CTAs share the queued sub-tiles' windows
// (each CTA rebuilds the tables), so skewed lengths cannot serialise on one CTA.

// experiments only (SK_FUSED_DBG & 8): per-CTA timestamps, read by sk_jagged_trace
__device__ unsigned long long g_fused_trace[1024 * 8];

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int F_NW = 8;             // warps per CTA
constexpr int F_NT = 32 * F_NW;
constexpr int F_RPT = 4;            // records per thread of a sub-tile
constexpr int F_R = F_NT * F_RPT;   // records per sub-tile
constexpr int MAX_SUB = 256;        // sub-tiles per block
constexpr int64_t DEFER_PER_REC = 64;
constexpr int DEFER_CHUNK = 16;     // windows per queued-sub-tile work item

struct FusedHdr {
  unsigned int ticket;
  unsigned int finished;  // sub-tiles gathered or queued
  unsigned int ndef;      // queued sub-tiles
  unsigned int pad;
};

struct DeferEntry {
  int64_t rec0;  // first record of the sub-tile
  int64_t cnt;   // its records
  int64_t E, A;
  unsigned long long next;   // next chunk to hand out
  unsigned long long ready;  // = the launch's generation (release) once the fields above are written
  unsigned long long pad[2];
};

struct FusedArgs {
  int64_t n;
  const void* lens;
  int lens_type;
  void* prefix;
  int prefix_type;
  int64_t* total;
  const int64_t* src_off;
  const uint8_t* src;   // pool + field offset
  int64_t member_stride;
  uint8_t* dst;         // 16-byte aligned
  int64_t capacity;
  int64_t block_recs;   // records per block (multiple of 4)
  int64_t nblocks;
  int64_t tiles;        // sub-tiles over all blocks
  FusedHdr* hdr;
  uint64_t* status;     // per block: its total
  DeferEntry* defer;
  // RS kernels (several member fields): the whole member record (member_stride = 8 or 16 bytes) is staged
  // and field f (fsz[f] = 4 or 8 bytes at foff[f]) is split out into pool fdst[f] when the window drains
  int nf;
  int fsz[4];
  int foff[4];
  uint8_t* fdst[4];
  int pvec;             // 4-byte prefix, 16-byte aligned: vector prefix stores
  int lens16;           // 4/8-byte lengths, 16-byte aligned: vector loads in the block sums
  int dbg;              // experiments only (SK_FUSED_DBG): 1 = no gather, 2 = no look-back
  int64_t src_members;  // member records in the source pool: segments must lie inside it
  int64_t* bad;         // += records whose segment does not (their sub-tiles are not gathered)
  unsigned long long gen;  // this launch's queue generation (queue entries are not zeroed between calls)
};

struct __align__(16) TileBuf {
  int64_t D[F_R];           // src_off - Lx
  int64_t Lx[F_R + 2];      // local exclusive prefix; Lx[F_R] = sub-tile total
  int64_t coarse[32];       // Lx[32 k]: the first probe round of the record search
};

struct FusedSmem {
  TileBuf tb;
  int sRec[F_NW][W];        // per warp: rank -> record of the current window
  int64_t warp_tot[F_NW];
  int warp_bad[F_NW];       // the warp holds a record whose segment lies outside the source pool
  int64_t item, E, A;
  int next;                 // next window of the current sub-tile
};

template <int RPT>
struct FRegs {
  int64_t len[RPT], off[RPT];
};

// this thread's records of the sub-tile [r0, r0 + cnt) (clamped loads; masked in the scan)
__device__ __forceinline__ void sub_load(const FusedArgs& F, int64_t r0, int cnt, FRegs<F_RPT>& g) {
  const int e0 = threadIdx.x * F_RPT;
#pragma unroll
  for (int i = 0; i < F_RPT; ++i) {
    const int64_t idx = r0 + min(e0 + i, max(cnt - 1, 0));
    g.len[i] = e0 + i < cnt ? load_int(F.lens, F.lens_type, idx) : 0;
    g.off[i] = F.src_off[idx];
  }
}

// all threads: the loaded sub-tile -> tables; returns the sub-tile total.
// incl[i] = tile-local inclusive prefix of this thread's records.
// `bad` is set when a record of the sub-tile has a negative length or a segment outside the source pool
// (counted into *F.bad when `count` is set); such a sub-tile is not gathered.
__device__ __forceinline__ int64_t sub_scan(const FusedArgs& F, const FRegs<F_RPT>& g, FusedSmem& S,
                                            int64_t (&ex)[F_RPT], bool& bad, bool count) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t acc = 0;
  unsigned nbad = 0;
#pragma unroll
  for (int i = 0; i < F_RPT; ++i) {
    acc += g.len[i];
    // empty segments are valid whatever their offset (an empty list reads nothing)
    nbad += g.len[i] < 0 || (g.len[i] > 0 && (g.off[i] < 0 || g.off[i] > F.src_members - g.len[i]));
  }
  int64_t x = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const unsigned wbad = __reduce_add_sync(0xffffffffu, nbad);
  if (lane == 31) {
    S.warp_tot[warp] = x;
    S.warp_bad[warp] = wbad != 0;
    if (count && wbad) atomicAdd(reinterpret_cast<unsigned long long*>(F.bad), static_cast<unsigned long long>(wbad));
  }
  __syncthreads();
  int64_t woff = 0, agg = 0;
  int anybad = 0;
#pragma unroll
  for (int w = 0; w < F_NW; ++w) {
    if (w < warp) woff += S.warp_tot[w];
    agg += S.warp_tot[w];
    anybad |= S.warp_bad[w];
  }
  bad = anybad != 0;
  int64_t run = woff + x - acc;
  const int e0 = tid * F_RPT;
#pragma unroll
  for (int i = 0; i < F_RPT; ++i) {
    ex[i] = run;
    S.tb.Lx[e0 + i] = run;
    S.tb.D[e0 + i] = g.off[i] - run;
    run += g.len[i];
  }
  if (tid % (32 / F_RPT) == 0) S.tb.coarse[tid / (32 / F_RPT)] = ex[0];
  if (tid == 0) S.tb.Lx[F_R] = agg;
  return agg;
}

// P[r0 + e] = E + Lx[e] for this thread's records e < cnt, truncated to the index dtype
__device__ __forceinline__ void sub_prefix(const FusedArgs& F, int64_t r0, int cnt, int64_t E,
                                           const int64_t (&ex)[F_RPT]) {
  const int e0 = threadIdx.x * F_RPT;
  if (F.pvec && e0 + F_RPT <= cnt) {
    *reinterpret_cast<uint4*>(static_cast<uint32_t*>(F.prefix) + r0 + e0) =
        make_uint4(static_cast<uint32_t>(E + ex[0]), static_cast<uint32_t>(E + ex[1]),
                   static_cast<uint32_t>(E + ex[2]), static_cast<uint32_t>(E + ex[3]));
    return;
  }
#pragma unroll
  for (int i = 0; i < F_RPT; ++i)
    if (e0 + i < cnt) store_int(F.prefix, F.prefix_type, r0 + e0 + i, E + ex[i]);
}

// last record r in [0, F_R) with Lx[r] <= j (the record holding local member j)
__device__ __forceinline__ int table_search(const TileBuf& B, int64_t j) {
  const int lane = threadIdx.x & 31;
  const unsigned m0 = __ballot_sync(0xffffffffu, B.coarse[lane] <= j);
  const int lo = (31 - __clz(m0)) * 32;
  const unsigned m1 = __ballot_sync(0xffffffffu, B.Lx[lo + lane] <= j);
  return lo + (31 - __clz(m1));
}

// stage buffers per warp: F_NS - 1 windows in flight behind the newest (3 and 4 measured slower: the
// extra shared memory comes out of the L1 the shuffled member reads rely on)
constexpr int F_NS = 2;

// a warp's member pipeline: windows whose loads are in flight, each stored
// once F_NS - 1 newer windows have been issued (possibly in a later sub-tile)
struct PendWin {
  int64_t w0, g0, g1;
};
struct FPipe {
  int it = 0;  // windows issued
  int n = 0;   // of those, pending (oldest first)
  PendWin p[F_NS - 1];
};

// RS: split the staged records of the window into the field pools (lanes, coalesced per pool)
template <int MS>
__device__ __forceinline__ void fdrain_split(const FusedArgs& F, const PendWin& p, const uint8_t* buf) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  for (int f = 0; f < F.nf; ++f) {
    const uint8_t* s = buf + F.foff[f];
    if (F.fsz[f] == 8) {
      uint64_t* d = reinterpret_cast<uint64_t*>(F.fdst[f]);
      for (int64_t g = p.g0 + lane; g < p.g1; g += 32) d[g] = *reinterpret_cast<const uint64_t*>(s + (g - p.w0) * MS);
    } else {
      uint32_t* d = reinterpret_cast<uint32_t*>(F.fdst[f]);
      for (int64_t g = p.g0 + lane; g < p.g1; g += 32) d[g] = *reinterpret_cast<const uint32_t*>(s + (g - p.w0) * MS);
    }
  }
  __syncwarp();
}

template <int MS, bool RS>
__device__ __forceinline__ void fdrain(const FusedArgs& F, const PendWin& p, const uint8_t* buf) {
  if constexpr (RS) {
    fdrain_split<MS>(F, p, buf);
    return;
  }
  using V = typename MemberWord<MS>::T;
  const int lane = threadIdx.x & 31;
  const int64_t a0 = (p.g0 * MS + 15) & ~int64_t(15), a1 = (p.g1 * MS) & ~int64_t(15);
  fence_proxy_async();
  __syncwarp();
  if (lane == 0 && a1 > a0) {
    bulk_s2g_plain(F.dst + a0, buf + (a0 - p.w0 * MS), static_cast<uint32_t>(a1 - a0));
    bulk_commit();
  }
  const int64_t h1 = min(a0 / MS, p.g1), t0 = max(a1 / MS, h1);
  for (int64_t g = p.g0 + lane; g < h1; g += 32)
    *reinterpret_cast<V*>(F.dst + g * MS) = *reinterpret_cast<const V*>(buf + (g - p.w0) * MS);
  for (int64_t g = t0 + lane; g < p.g1; g += 32)
    *reinterpret_cast<V*>(F.dst + g * MS) = *reinterpret_cast<const V*>(buf + (g - p.w0) * MS);
}

template <int MS, bool RS>
__device__ __forceinline__ void fflush(const FusedArgs& F, FPipe& pp, uint8_t (*stage)[W * MS]) {
  if (pp.n) {
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < F_NS - 1; ++i)
      if (i < pp.n) fdrain<MS, RS>(F, pp.p[i], stage[(pp.it - pp.n + i) % F_NS]);
    pp.n = 0;
  }
}

// the warp gathers output window k of the tile whose members are [E, E + A)
template <int MS, bool RS>
__device__ __forceinline__ void gather_window(const FusedArgs& F, const TileBuf& B, int64_t E, int64_t A, int64_t k,
                                              int* sRec, uint8_t (*stage)[W * MS], FPipe& pp) {
  const int lane = threadIdx.x & 31;
  const unsigned le_mask = 0xffffffffu >> (31 - lane);
  const int64_t w0 = k * W;
  const int64_t g0 = max(w0, E), g1 = min(w0 + W, E + A);
  const int64_t j0 = g0 - E, j1 = g1 - E;
  const int sh = static_cast<int>(g0 - w0);
  unsigned masks[W_CH];
#pragma unroll
  for (int q = 0; q < W_CH; ++q) masks[q] = 0;
  int nr = 0;
  for (int c0 = table_search(B, j0);; c0 += 32) {
    const int c = min(c0 + lane, F_R);
    const int64_t p = B.Lx[c], pn = B.Lx[c + 1];  // Lx[F_R + 1] is never used: c < F_R is checked
    const bool ne = c0 + lane < F_R && pn > p && p < j1;
    const unsigned bal = __ballot_sync(0xffffffffu, ne);
    const int rank = nr + __popc(bal & (le_mask >> 1));
    nr += __popc(bal);
    const int s = ne ? static_cast<int>(max(p - j0, int64_t(0))) + sh : -1;
    if (ne) sRec[rank] = c;
#pragma unroll
    for (int q = 0; q < W_CH; ++q) masks[q] |= __reduce_or_sync(0xffffffffu, (s >> 5) == q ? 1u << (s & 31) : 0u);
    if (c0 + 32 >= F_R || B.Lx[c0 + 32] >= j1) break;
  }
  __syncwarp();
  uint8_t* buf = stage[pp.it % F_NS];
  // the latest bulk store (window it - F_NS, drained one window ago) read this buffer
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
  int cum = 0;
#pragma unroll
  for (int q = 0; q < W_CH; ++q) {
    const int pos = 32 * q + lane;
    const int r = cum + __popc(masks[q] & le_mask) - 1;
    if (pos >= sh && w0 + pos < g1)
      cp_async_member<MS>(buf + pos * MS, F.src + (w0 + pos - E + B.D[sRec[r]]) * F.member_stride);
    cum += __popc(masks[q]);
  }
  cp_async_commit();
  if (pp.n == F_NS - 1) {
    cp_async_wait<F_NS - 1>();  // the oldest pending window has landed
    fdrain<MS, RS>(F, pp.p[0], stage[(pp.it - pp.n) % F_NS]);
#pragma unroll
    for (int i = 0; i + 1 < F_NS - 1; ++i) pp.p[i] = pp.p[i + 1];
    --pp.n;
  }
#pragma unroll
  for (int i = 0; i < F_NS - 1; ++i)
    if (i == pp.n) pp.p[i] = PendWin{w0, g0, g1};
  ++pp.n;
  ++pp.it;
  __syncwarp();  // sRec is rewritten by the next window
}

__device__ __forceinline__ int64_t first_window(int64_t E) { return E / W; }
__device__ __forceinline__ int64_t end_window(int64_t E, int64_t A) { return (E + A + W - 1) / W; }


// warp 0: exclusive prefix of block `blk` = the sum of every predecessor
// block's published total (256 status words per round, no chain through
// other blocks' prefixes; polls back off while a predecessor is still summing)
__device__ __forceinline__ int64_t pred_sum(const FusedArgs& F, int64_t blk) {
  const int lane = threadIdx.x & 31;
  int64_t acc = 0;
  int spins = 0;
  for (int64_t e0 = 0; e0 < blk; e0 += 256) {
    uint64_t st[8];
    bool missing = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t idx = e0 + q * 32 + lane;
      st[q] = idx < blk ? ld_poll(&F.status[idx]) : FLAG_A;
      missing |= (st[q] >> 62) == 0;
    }
    if ((F.dbg & 8) && e0 == 0 && lane == 0 && blockIdx.x < 1024) g_fused_trace[blockIdx.x * 8 + 6] = gtimer();
    while (__any_sync(0xffffffffu, missing)) {
      ++spins;
      __nanosleep(200);
      missing = false;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if ((st[q] >> 62) == 0) st[q] = ld_poll(&F.status[e0 + q * 32 + lane]);
        missing |= (st[q] >> 62) == 0;
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t idx = e0 + q * 32 + lane;
      if (idx < blk) acc += static_cast<int64_t>(st[q] & VAL_MASK);
    }
  }
  if ((F.dbg & 8) && lane == 0 && blockIdx.x < 1024) g_fused_trace[blockIdx.x * 8 + 7] = spins;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}


template <int MS, bool RS>
__global__ void __launch_bounds__(F_NT, 3) pack_fused_kernel(const __grid_constant__ FusedArgs F) {
  extern __shared__ __align__(128) uint8_t fsm[];
  auto stage_all = reinterpret_cast<uint8_t(*)[F_NS][W * MS]>(fsm);
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(fsm + F_NW * F_NS * W * MS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto stage = stage_all[warp];
  int* sRec = S.sRec[warp];
  FPipe pp;
  FRegs<F_RPT> g;
  auto stamp = [&](int k) {
    if ((F.dbg & 8) && tid == 0 && blockIdx.x < 1024) g_fused_trace[blockIdx.x * 8 + k] = gtimer();
  };
  stamp(0);


  for (int round = 0;; ++round) {
    // the first block is the CTA's own index (CTAs are dispatched in index order, so a block only ever
    // waits on blocks whose CTAs run -- the assumption CUB's single-pass scan makes); later blocks by
    // ticket, which hands out indices past the grid in the order CTAs come back for more
    if (tid == 0) S.item = round == 0 ? blockIdx.x : gridDim.x + atomicAdd(&F.hdr->ticket, 1u);
    __syncthreads();  // also: every warp is done with the previous block's tables
    const int64_t blk = S.item;
    if (blk >= F.nblocks) break;
    const int64_t rec0 = blk * F.block_recs, rec1 = min(F.n, rec0 + F.block_recs);
    const int nsub = static_cast<int>((rec1 - rec0 + F_R - 1) / F_R);
    // 1. the block total, published; the first sub-tile's records load meanwhile
    int64_t acc = 0;
    int64_t rs = rec0;  // records before rs are summed by the vector loop
    if (F.lens16) {
      // 16-byte loads, 8 in flight per thread: the lengths pass is bandwidth-, not latency-bound
      if (dtype_size_dev(F.lens_type) == 4) {
        const bool sgn = F.lens_type == SK_I32;
        const uint4* L = reinterpret_cast<const uint4*>(static_cast<const uint32_t*>(F.lens) + rec0);
        const int64_t nv = (rec1 - rec0) / 4;
#pragma unroll 8
        for (int64_t i = tid; i < nv; i += F_NT) {
          const uint4 v = L[i];
          acc += sgn ? static_cast<int64_t>(static_cast<int32_t>(v.x)) + static_cast<int32_t>(v.y) +
                           static_cast<int32_t>(v.z) + static_cast<int32_t>(v.w)
                     : static_cast<int64_t>(v.x) + v.y + v.z + static_cast<int64_t>(v.w);
        }
        rs = rec0 + nv * 4;
      } else {
        const longlong2* L = reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(F.lens) + rec0);
        const int64_t nv = (rec1 - rec0) / 2;
#pragma unroll 8
        for (int64_t i = tid; i < nv; i += F_NT) {
          const longlong2 v = L[i];
          acc += v.x + v.y;
        }
        rs = rec0 + nv * 2;
      }
    }
    for (int64_t r = rs + tid; r < rec1; r += F_NT) acc += load_int(F.lens, F.lens_type, r);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) S.warp_tot[warp] = acc;
    // nothing is written and no scratch word read before the scratch-zeroing kernel ahead of this one has
    // completed (its trigger came after ITS predecessor completed, so the lengths read above were final)
    if (round == 0) pdl_wait_prior();
    __syncthreads();
    int64_t Ab = 0;
    if (warp == 0) {
#pragma unroll
      for (int w = 0; w < F_NW; ++w) Ab += S.warp_tot[w];
      if (lane == 0) {
        st_relaxed(&F.status[blk], FLAG_A | (static_cast<uint64_t>(Ab) & VAL_MASK));
        // push the total out now: an unfenced store can sit in the SM for microseconds, and every later
        // block waits on it (this thread has no loads in flight, so the fence is quick)
        __threadfence();
      }
    }
    stamp(4);
    // the first sub-tile's records load while warp 0 sums the predecessors
    sub_load(F, rec0, static_cast<int>(min(static_cast<int64_t>(F_R), rec1 - rec0)), g);
    if (warp == 0) {
      const int64_t E = (F.dbg & 2) ? 0 : pred_sum(F, blk);
      stamp(5);
      if (lane == 0) {
        S.E = E;
        if (rec1 == F.n) {  // the block holding the last record
          store_int(F.prefix, F.prefix_type, F.n, E + Ab);
          *F.total = E + Ab;
        }
      }
    }
    __syncthreads();  // S.E, and warp_tot is free again
    stamp(1);
    int64_t run = S.E;
    // 2. sub-tiles: scan, prefix, gather
    for (int sb = 0; sb < nsub; ++sb) {
      const int64_t r0 = rec0 + static_cast<int64_t>(sb) * F_R;
      const int cnt = static_cast<int>(min(static_cast<int64_t>(F_R), rec1 - r0));
      int64_t ex[F_RPT];
      bool bad;
      const int64_t A = sub_scan(F, g, S, ex, bad, true);
      const int64_t E = run;
      run += A;
      sub_prefix(F, r0, cnt, E, ex);
      if (sb + 1 < nsub) {  // the next sub-tile's records fly while this one gathers
        const int64_t r1 = r0 + F_R;
        sub_load(F, r1, static_cast<int>(min(static_cast<int64_t>(F_R), rec1 - r1)), g);
      }
      // past the capacity: not gathered (the caller sees *total > capacity and redoes the pack)
      const bool gather = A > 0 && E + A <= F.capacity && !bad && !(F.dbg & 1);
      const bool queue = gather && A > DEFER_PER_REC * F_R;
      if (tid == 0) {
        if (queue) {
          const unsigned slot = atomicAdd(&F.hdr->ndef, 1u);
          DeferEntry& d = F.defer[slot];
          d.rec0 = r0;
          d.cnt = cnt;
          d.E = E;
          d.A = A;
          d.next = 0;
          __threadfence();
          st_release(&d.ready, F.gen);
        }
        S.next = 0;
      }
      __syncthreads();  // tables and the window counter are ready
      if (gather && !queue) {
        const int64_t k0 = first_window(E);
        const int nwin = static_cast<int>(end_window(E, A) - k0);
        while (true) {
          int k = 0;
          if (lane == 0) k = atomicAdd(&S.next, 1);
          k = __shfl_sync(0xffffffffu, k, 0);
          if (k >= nwin) break;
          gather_window<MS, RS>(F, S.tb, E, A, k0 + k, sRec, stage, pp);
        }
      }
      __syncthreads();  // the tables are rewritten by the next sub-tile
    }
  }

  stamp(2);
  __syncthreads();  // every thread has read S.item (the loop's last ticket) before it is reused
  // queued sub-tiles: help with the entries queued so far. No CTA waits for another to queue or finish
  // anything (an entry queued later is drained by its owner, which runs this loop after queuing it), so
  // the grid needs no co-residency; an entry whose slot is taken but not yet written is being written
  // by a running CTA.
  if (tid == 0) S.item = *reinterpret_cast<volatile unsigned int*>(&F.hdr->ndef);
  __syncthreads();
  const int64_t ndef = S.item;
  int64_t have = -1;
  for (int64_t d = 0; d < ndef; ++d) {
    if (tid == 0)
      while (ld_acquire(&F.defer[d].ready) != F.gen) __nanosleep(64);
    __syncthreads();
    DeferEntry ent;  // published by another CTA: read through L2 (see load_entry)
    ent.rec0 = __ldcg(&F.defer[d].rec0);
    ent.cnt = __ldcg(&F.defer[d].cnt);
    ent.E = __ldcg(&F.defer[d].E);
    ent.A = __ldcg(&F.defer[d].A);
    const int64_t k0 = first_window(ent.E), nwin = end_window(ent.E, ent.A) - k0;
    const int64_t nchunks = (nwin + DEFER_CHUNK - 1) / DEFER_CHUNK;
    while (true) {
      __syncthreads();  // the previous chunk is done with S.item and the tables
      if (tid == 0) S.item = static_cast<int64_t>(atomicAdd(&F.defer[d].next, 1ull));
      __syncthreads();
      const int64_t c = S.item;
      if (c >= nchunks) break;
      if (have != d) {
        sub_load(F, ent.rec0, static_cast<int>(ent.cnt), g);
        int64_t ex[F_RPT];
        bool bad;
        sub_scan(F, g, S, ex, bad, false);
        __syncthreads();
        have = d;
      }
      const int64_t kb = k0 + c * DEFER_CHUNK, ke = min(kb + DEFER_CHUNK, k0 + nwin);
      for (int64_t k = kb + warp; k < ke; k += F_NW)
        gather_window<MS, RS>(F, S.tb, ent.E, ent.A, k, sRec, stage, pp);
    }
  }
  fflush<MS, RS>(F, pp, stage);
  if (lane == 0) bulk_wait_all();
  stamp(3);
}


// ---- fused pack, register gather (one naturally aligned 4/8-byte member field) ----
//
// The default single-pass pack. Tiles of RG_TR = 2048 records are handed out by
// ticket (a CTA holding tile t only ever waits on tiles < t, whose holders are
// running: no co-residency assumption). Per tile:
//   1. every warp loads the lengths and source offsets of its 8 groups of 32
//      records (coalesced, all 16 loads in flight), scans each group with
//      shuffles, and leaves the group-local exclusive prefix and
//      D = src_off - prefix in shared memory; the CTA publishes the tile total;
//   2. a warp gathers its groups: lane i of round q takes group member
//      m = 32 q + i, finds its record by a 5-step shuffle search over the
//      group's prefixes and loads src[D + m] into a register -- up to RG_K
//      rounds (384 members) are in flight per warp before the first store;
//   3. the first store waits for the tile's exclusive prefix E, which warp 0
//      finds by decoupled look-back (32 predecessors per round, stopping at
//      the nearest inclusive prefix) while its own first loads are in flight;
//   4. prefix elements P[r] = E + local prefix are stored, truncated to the
//      index dtype; the tile holding the last record writes P[n] and the total.
// A group of more than RG_BIG members (skewed lengths) is not gathered by its
// warp: it is queued, and every warp that finishes its tile takes 1536-member
// chunks of the queued groups it sees (an entry queued later is drained by its
// owner's CTA, which looks at the queue after all its warps have queued).
// Measured against the cp.async window design below (pack_fused_kernel, kept
// for multi-field member records): 43 vs 50 us on config 3 -- the member
// loads need registers, not shared-memory staging (tools/jag_micro.cu,
// profiles/r02_jagged_redesign.md).

constexpr int RG_NW = 8;
constexpr int RG_GPW = 8;                      // groups of 32 records per warp and tile
constexpr int RG_TR = RG_NW * RG_GPW * 32;     // records per tile
constexpr int RG_K = 12;                       // 32-member rounds in flight per warp
constexpr int64_t RG_BIG = 32 * RG_K * 8;      // group members above which the group is queued
constexpr int64_t RG_CHUNK = 32 * RG_K * 4;    // members per queued-group work item
constexpr int64_t RG_QMAX = 65536;             // queue entries (a full queue: the owner warp gathers itself)

struct RegHdr {
  unsigned int nq;  // queued groups (zeroed by tile 0 before it publishes)
  unsigned int pad[15];
};

// per-tile look-back word: {value, gen << 2 | 1 (value = the tile's total) or | 2 (its inclusive prefix)},
// written and read as ONE 128-bit access (PTX .b128, single-copy atomic). Nothing in the scratch needs
// zeroing between launches: a word counts only when it carries this launch's generation.
struct __align__(16) RegStatus {
  unsigned long long v;
  unsigned long long tag;
};

__device__ __forceinline__ void st_status(RegStatus* p, int64_t v, unsigned long long tag) {
  asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.release.gpu.global.b128 [%0], t; }" ::"l"(p),
               "l"(static_cast<unsigned long long>(v)), "l"(tag)
               : "memory");
}

__device__ __forceinline__ void ld_status(const RegStatus* p, int64_t& v, unsigned long long& tag) {
  unsigned long long a, b;
  asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
               : "=l"(a), "=l"(b)
               : "l"(p)
               : "memory");
  v = static_cast<int64_t>(a);
  tag = b;
}

struct RegEntry {
  int64_t rec0;              // first record of the group
  int64_t out0;              // output member index of its first member
  int64_t T;                 // its members
  unsigned long long next;   // next chunk to hand out
  unsigned long long ready;  // = the launch's generation (release) once the fields above are written
  int cnt;                   // records in the group
  int pad0;
  int64_t pad[2];
};

// a queue entry published by another CTA (release on `ready`, acquired by this warp's lane 0): its fields are
// read through L2 (ld.global.cg) -- the acquire by one lane does not make the other lanes' plain loads skip a
// stale L1 copy of the entry's line
__device__ __forceinline__ RegEntry load_entry(const RegEntry* e) {
  RegEntry r;
  r.rec0 = __ldcg(&e->rec0);
  r.out0 = __ldcg(&e->out0);
  r.T = __ldcg(&e->T);
  r.cnt = __ldcg(&e->cnt);
  r.next = 0;
  r.ready = 0;
  return r;
}

struct RegArgs {
  int64_t n;
  const void* lens;
  int lens_type;
  void* prefix;
  int prefix_type;
  int64_t* total;
  int64_t* bad;         // += records whose segment lies outside the source pool (their tile is not gathered)
  const int64_t* src_off;
  const uint8_t* src;   // pool + field offset
  int64_t member_stride;
  uint8_t* dst;         // MS-aligned
  int64_t capacity;
  int64_t src_members;
  RegHdr* hdr;
  RegStatus* status;    // per tile
  RegEntry* q;
  int64_t qmax;
  unsigned long long gen;
  int gpw;              // groups of 32 records per warp and tile (1..RG_GPW)
};

template <int MS, bool PACKED>
__device__ __forceinline__ typename MemberWord<MS>::T rg_load(const RegArgs& F, int64_t j) {
  if constexpr (PACKED) return reinterpret_cast<const typename MemberWord<MS>::T*>(F.src)[j];
  return *reinterpret_cast<const typename MemberWord<MS>::T*>(F.src + j * F.member_stride);
}

template <int MS>
__device__ __forceinline__ void rg_store(const RegArgs& F, int64_t j, typename MemberWord<MS>::T v) {
  __stcs(reinterpret_cast<typename MemberWord<MS>::T*>(F.dst) + j, v);
}

// tile 0 has zeroed the queue and invalid-record counters of this launch
__device__ __forceinline__ void rg_wait_tile0(const RegArgs& F, unsigned long long gen2) {
  while ((ld_acquire(&F.status[0].tag) & ~3ull) != gen2) __nanosleep(32);
}

// members [m_begin, m_end) of a group of up to 32 records whose group-local exclusive prefixes are `ex`
// (lane = record) and source bases `d` (= src_off - ex): member m of the group goes to dst[out0 + m].
// 64-bit search: such a group may exceed 2^31 members.
template <int MS, bool PACKED>
__device__ __forceinline__ void span_gather(const uint8_t* src, int64_t stride, uint8_t* dst, int64_t ex, int64_t d,
                                            int64_t out0, int64_t m_begin, int64_t m_end) {
  using V = typename MemberWord<MS>::T;
  const int lane = threadIdx.x & 31;
  for (int64_t m0 = m_begin; m0 < m_end; m0 += 32 * RG_K) {
    V v[RG_K];
#pragma unroll
    for (int q = 0; q < RG_K; ++q) {
      const int64_t m = m0 + q * 32 + lane;
      if (m0 + q * 32 < m_end) {
        int lo = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int64_t e = __shfl_sync(0xffffffffu, ex, lo + s);
          if (e <= m) lo += s;
        }
        const int64_t dd = __shfl_sync(0xffffffffu, d, lo);
        if (m < m_end)
          v[q] = PACKED ? reinterpret_cast<const V*>(src)[dd + m] : *reinterpret_cast<const V*>(src + (dd + m) * stride);
      }
    }
#pragma unroll
    for (int q = 0; q < RG_K; ++q) {
      const int64_t m = m0 + q * 32 + lane;
      if (m < m_end) __stcs(reinterpret_cast<V*>(dst) + out0 + m, v[q]);
    }
  }
}

// a queued group's members [m_begin, m_end): its records' prefixes are rebuilt from the lengths
template <int MS, bool PACKED>
__device__ __forceinline__ void rg_gather_big(const RegArgs& F, const RegEntry& ent, int64_t m_begin, int64_t m_end) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ent.rec0 + lane;
  const int64_t len = lane < ent.cnt ? load_int(F.lens, F.lens_type, r) : 0;
  const int64_t off = lane < ent.cnt ? F.src_off[r] : 0;
  int64_t x = len;
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, s);
    if (lane >= s) x += y;
  }
  span_gather<MS, PACKED>(F.src, F.member_stride, F.dst, x - len, off - (x - len), ent.out0, m_begin, m_end);
}

// WIDE: 64-bit or u32 lengths (held as int64 while the loads fly); otherwise int32
template <int MS, bool WIDE, bool PACKED>
__global__ void __launch_bounds__(RG_NW * 32, 4) pack_reg_kernel(const __grid_constant__ RegArgs F) {
  using LT = typename std::conditional<WIDE, int64_t, int32_t>::type;
  using V = typename MemberWord<MS>::T;
  __shared__ int64_t sD[RG_TR];
  __shared__ int64_t sEx[RG_TR];  // group-local exclusive prefix
  __shared__ int64_t sGb[RG_NW * RG_GPW];
  __shared__ int64_t sWt[RG_NW];
  __shared__ int sBad[RG_NW];
  __shared__ int64_t sLb[2][RG_NW];  // look-back round sums per warp (double-buffered by round)
  __shared__ int sLbP[2][RG_NW];     // ... and whether the warp's 32 held an inclusive prefix
  __shared__ unsigned int sNq;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // tiles in block order: a tile waits only on lower-indexed blocks, which in-order dispatch has started
  // (the look-back assumption of CUB's single-pass scan)
  // F.gpw (<= RG_GPW) groups per warp and tile: fewer for small inputs, so the tiles cover the SMs;
  // group slots past it are empty groups
  const int64_t tile_recs = static_cast<int64_t>(RG_NW * 32) * F.gpw;
  const int64_t t = blockIdx.x, rw = t * tile_recs + warp * (F.gpw * 32);
  const unsigned long long gen2 = F.gen << 2;
  // the previous kernel in the stream has completed (lengths final, scratch no longer in use)
  pdl_wait_prior();
  if (t == 0 && tid == 0) {
    F.hdr->nq = 0;
    *F.bad = 0;
    __threadfence();
  }
  // 1. lengths and offsets of this warp's groups, group scans
  LT len[RG_GPW];
  int64_t off[RG_GPW];
#pragma unroll
  for (int k = 0; k < RG_GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    const bool in = k < F.gpw && r < F.n;
    len[k] = in ? static_cast<LT>(load_int(F.lens, F.lens_type, r)) : 0;
    off[k] = in ? F.src_off[r] : 0;
  }
  int64_t wsum = 0;
  unsigned nbad = 0;
#pragma unroll
  for (int k = 0; k < RG_GPW; ++k) {
    // empty segments are valid whatever their offset (an empty list reads nothing)
    nbad += len[k] < 0 || (len[k] > 0 && (off[k] < 0 || off[k] > F.src_members - len[k]));
    int64_t x = len[k];
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, s);
      if (lane >= s) x += y;
    }
    const int e = warp * (RG_GPW * 32) + k * 32 + lane;
    sEx[e] = x - len[k];
    sD[e] = off[k] - (x - len[k]);
    if (lane == 0) sGb[warp * RG_GPW + k] = wsum;
    wsum += __shfl_sync(0xffffffffu, x, 31);
  }
  const unsigned wbad = __reduce_add_sync(0xffffffffu, nbad);
  if (lane == 0) {
    sWt[warp] = wsum;
    sBad[warp] = wbad != 0;
  }
  __syncthreads();
  if (lane == 0 && wbad) {
    if (t != 0) rg_wait_tile0(F, gen2);  // the counter is zeroed by tile 0 (in this CTA: before the barrier)
    atomicAdd(reinterpret_cast<unsigned long long*>(F.bad), static_cast<unsigned long long>(wbad));
  }
  int64_t A = 0, Wo = 0;
  bool bad = false;
#pragma unroll
  for (int w = 0; w < RG_NW; ++w) {
    Wo += w < warp ? sWt[w] : 0;
    A += sWt[w];
    bad |= sBad[w] != 0;
  }
  if (tid == 0) {
    st_status(&F.status[t], A, gen2 | (t == 0 ? 2 : 1));
    __threadfence();  // push the total out now: every later tile looks back at it
  }
  // 3. the tile's exclusive prefix (warp 0 looks back; every warp calls this exactly once)
  bool haveE = false;
  int64_t E = 0;
  // The look-back is shared by all 8 warps: a round reads the 256 nearest unread predecessors (32 per
  // warp), so the last of ~560 tiles needs at most 3 rounds even when every predecessor has published only
  // its total. Every warp calls this exactly once, from the gather loop or after it (two call sites): the
  // rounds are CTA-uniform (decided from shared memory) and use the non-aligned barrier after the warp
  // has reconverged.
  auto get_E = [&]() {
    __syncwarp();
    int64_t acc = 0;
    if (t > 0) {
      for (int64_t base = t - 1, round = 0;; base -= RG_NW * 32, ++round) {
        const int64_t j = base - (warp * 32 + lane);
        int64_t sv = 0;
        unsigned long long f = gen2 | 2;  // before tile 0: an inclusive prefix of 0
        if (j >= 0) ld_status(&F.status[j], sv, f);
        while (__any_sync(0xffffffffu, (f & ~3ull) != gen2)) {
          if ((f & ~3ull) != gen2) ld_status(&F.status[j], sv, f);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, (f & 3) == 2);
        const int pl = pm ? __ffs(pm) - 1 : 32;
        int64_t v = lane <= pl ? sv : 0;
#pragma unroll
        for (int q = 16; q; q >>= 1) v += __shfl_xor_sync(0xffffffffu, v, q);
        if (lane == 0) {
          sLb[round & 1][warp] = v;
          sLbP[round & 1][warp] = pm != 0;
        }
        asm volatile("barrier.sync 1, %0;" ::"n"(RG_NW * 32) : "memory");
        bool found = false;
#pragma unroll
        for (int w = 0; w < RG_NW; ++w) {
          if (!found) {
            acc += sLb[round & 1][w];
            found = sLbP[round & 1][w] != 0;
          }
        }
        if (found) break;
      }
      if (tid == 0) st_status(&F.status[t], acc + A, gen2 | 2);
    } else {
      asm volatile("barrier.sync 1, %0;" ::"n"(RG_NW * 32) : "memory");  // keeps the barrier counts equal
    }
    E = acc;
    haveE = true;
  };
  // 2. the gather (not for a tile holding an invalid segment; no stores past the capacity); groups over
  // RG_BIG members are set aside for the queue
  unsigned big = 0;
#pragma unroll 1
  for (int k = 0; k < RG_GPW && !bad && F.capacity > 0; ++k) {  // capacity 0: the prefix only
    const int g = warp * RG_GPW + k;
    const int64_t g0 = sGb[g];
    const int64_t T = (k + 1 < RG_GPW ? sGb[g + 1] : sWt[warp]) - g0;
    if (T > RG_BIG) {
      big |= 1u << k;
      continue;
    }
    const int e = g * 32 + lane;
    const int ex = static_cast<int>(sEx[e]);  // T <= RG_BIG
    const int64_t d = sD[e];
    const int Ti = static_cast<int>(T);
#pragma unroll 1
    for (int m0 = 0; m0 < Ti; m0 += 32 * RG_K) {
      V v[RG_K];
#pragma unroll
      for (int q = 0; q < RG_K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m0 + q * 32 < Ti) {
          int lo = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const int ee = __shfl_sync(0xffffffffu, ex, lo + s);
            if (ee <= m) lo += s;
          }
          const int64_t dd = __shfl_sync(0xffffffffu, d, lo);
          if (m < Ti) v[q] = rg_load<MS, PACKED>(F, dd + m);
        }
      }
      if (!haveE) get_E();
      if (E + A > F.capacity) break;
      V* ob = reinterpret_cast<V*>(F.dst) + (E + Wo + g0);
#pragma unroll
      for (int q = 0; q < RG_K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < Ti) __stcs(ob + m, v[q]);
      }
    }
  }
  if (!haveE) get_E();
  // the set-aside groups: queued for every warp to share (a full queue: gathered here)
  if (E + A <= F.capacity) {
#pragma unroll 1
    for (; big; big &= big - 1) {
      const int k = __ffs(big) - 1;
      const int g = warp * RG_GPW + k;
      const int64_t g0 = sGb[g];
      RegEntry ent;
      ent.rec0 = rw + k * 32;
      ent.cnt = static_cast<int>(min(static_cast<int64_t>(32), F.n - ent.rec0));
      ent.out0 = E + Wo + g0;
      ent.T = (k + 1 < RG_GPW ? sGb[g + 1] : sWt[warp]) - g0;
      unsigned slot = 0;
      if (lane == 0) {
        rg_wait_tile0(F, gen2);  // the queue counter is zeroed by tile 0
        slot = atomicAdd(&F.hdr->nq, 1u);
      }
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (slot < F.qmax) {
        if (lane == 0) {
          RegEntry& qe = F.q[slot];
          qe.rec0 = ent.rec0;
          qe.cnt = ent.cnt;
          qe.out0 = ent.out0;
          qe.T = ent.T;
          qe.next = 0;
          __threadfence();
          st_release(&qe.ready, F.gen);
        }
      } else {
        rg_gather_big<MS, PACKED>(F, ent, 0, ent.T);
      }
    }
  }
  // 4. prefix elements, truncated to the index dtype
#pragma unroll
  for (int k = 0; k < RG_GPW; ++k) {
    const int64_t r = rw + k * 32 + lane;
    const int e = warp * (RG_GPW * 32) + k * 32 + lane;
    if (k < F.gpw && r < F.n) store_int(F.prefix, F.prefix_type, r, E + Wo + sGb[warp * RG_GPW + k] + sEx[e]);
  }
  if (tid == 0 && (t + 1) * tile_recs >= F.n) {
    store_int(F.prefix, F.prefix_type, F.n, E + A);
    *F.total = E + A;
  }
  // queued groups: every entry queued so far (this CTA's included: the barrier orders its warps' queueing
  // before the count is read). No warp waits for another to queue anything; an entry whose slot is taken
  // but not yet written is being written by a running warp.
  __syncthreads();
  if (tid == 0) {
    rg_wait_tile0(F, gen2);
    sNq = min(static_cast<unsigned>(F.qmax), *reinterpret_cast<volatile unsigned int*>(&F.hdr->nq));
  }
  __syncthreads();
  const unsigned nq = sNq;
  for (unsigned dq = 0; dq < nq; ++dq) {
    if (lane == 0)
      while (ld_acquire(&F.q[dq].ready) != F.gen) __nanosleep(64);
    __syncwarp();
    const RegEntry ent = load_entry(&F.q[dq]);
    const int64_t nch = (ent.T + RG_CHUNK - 1) / RG_CHUNK;
    while (true) {
      unsigned long long c = 0;
      if (lane == 0) c = atomicAdd(&F.q[dq].next, 1ull);
      c = __shfl_sync(0xffffffffu, c, 0);
      if (static_cast<int64_t>(c) >= nch) break;
      const int64_t mb = static_cast<int64_t>(c) * RG_CHUNK;
      rg_gather_big<MS, PACKED>(F, ent, mb, min(ent.T, mb + RG_CHUNK));
    }
  }
}

// ---- gather over a given prefix, register version (sk_jagged_scatter, one 4/8-byte field) ----
//
// A warp takes groups of 32 records (grid-stride): the group's base and end come from the prefix, each
// lane's record offset inside the group from its prefix element, and the members move as in
// pack_reg_kernel (12 register rounds in flight per warp). A group over RG_BIG members is only listed
// (one tagged atomic append, no zeroing launch); scatter_big_kernel, launched right behind, shares the listed groups' 1536-member
// chunks over its whole grid. Nothing waits on anything inside either kernel. tools/jag_micro.cu measured
// this structure at 37.9 us on config 3 (the window gather: 55 us).
struct ScatRegArgs {
  int64_t n;
  const void* prefix;  // non-wrapped
  const int64_t* src_off;
  const uint8_t* src;  // pool + field offset
  int64_t member_stride;
  uint8_t* dst;
  int64_t total;       // members gathered: positions >= total are skipped
  RegEntry* q;         // the listed groups (rec0, cnt, out0, T)
  unsigned long long* nq;  // list length, tagged: (gen & 2^40 - 1) << 24 | count; a stale tag counts as 0
  int64_t qmax;        // > total / (RG_BIG + 1): the list cannot overflow with a valid prefix
  unsigned long long gen;
};

// next list slot: no zeroing of the counter between launches (the word carries this launch's tag)
__device__ __forceinline__ unsigned scat_list_slot(const ScatRegArgs& A) {
  const unsigned long long tag = (A.gen & ((1ull << 40) - 1)) << 24;
  unsigned long long old = atomicAdd(A.nq, 0ull);
  for (;;) {
    const bool mine = (old & ~((1ull << 24) - 1)) == tag;
    const unsigned slot = mine ? static_cast<unsigned>(old & ((1ull << 24) - 1)) : 0u;
    const unsigned long long seen = atomicCAS(A.nq, old, tag | (slot + 1));
    if (seen == old) return slot;
    old = seen;
  }
}

__device__ __forceinline__ unsigned scat_list_len(const ScatRegArgs& A) {
  const unsigned long long w = *A.nq, tag = (A.gen & ((1ull << 40) - 1)) << 24;
  return (w & ~((1ull << 24) - 1)) == tag ? static_cast<unsigned>(w & ((1ull << 24) - 1)) : 0u;
}

template <class PT, int MS, bool PACKED>
__global__ void __launch_bounds__(256, 4) scatter_reg_kernel(const __grid_constant__ ScatRegArgs A) {
  using V = typename MemberWord<MS>::T;
  const int lane = threadIdx.x & 31;
  const PT* P = static_cast<const PT*>(A.prefix);
  const int64_t ngroups = (A.n + 31) / 32;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  pdl_wait_prior();
#pragma unroll 1
  for (int64_t g = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); g < ngroups; g += nw) {
    const int64_t r0 = g * 32, r = r0 + lane;
    const int cnt = static_cast<int>(min(static_cast<int64_t>(32), A.n - r0));
    const int64_t B = static_cast<int64_t>(P[r0]);
    const int64_t Pe = static_cast<int64_t>(P[r0 + cnt]);
    const int64_t T = min(Pe, A.total) - B;  // past the total: not gathered
    if (T <= 0) continue;
    if (T > RG_BIG) {  // listed for scatter_big_kernel
      if (lane == 0) {
        const unsigned slot = scat_list_slot(A);
        if (slot < A.qmax) {  // (only a non-monotone, invalid prefix could overflow the list)
          RegEntry& qe = A.q[slot];
          qe.rec0 = r0;
          qe.cnt = cnt;
          qe.out0 = B;
          qe.T = T;
        }
      }
      continue;
    }
    const int64_t pr = lane < cnt ? static_cast<int64_t>(P[r]) : Pe;
    const int64_t d64 = (lane < cnt ? A.src_off[r] : 0) - (pr - B);
    const int ex = static_cast<int>(pr - B);
    const int Ti = static_cast<int>(T);
#pragma unroll 1
    for (int m0 = 0; m0 < Ti; m0 += 32 * RG_K) {
      V v[RG_K];
#pragma unroll
      for (int q = 0; q < RG_K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m0 + q * 32 < Ti) {
          int lo = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const int ee = __shfl_sync(0xffffffffu, ex, lo + s);
            if (ee <= m) lo += s;
          }
          const int64_t dd = __shfl_sync(0xffffffffu, d64, lo);
          if (m < Ti)
            v[q] = PACKED ? reinterpret_cast<const V*>(A.src)[dd + m]
                          : *reinterpret_cast<const V*>(A.src + (dd + m) * A.member_stride);
        }
      }
      V* ob = reinterpret_cast<V*>(A.dst) + B;
#pragma unroll
      for (int q = 0; q < RG_K; ++q) {
        const int m = m0 + q * 32 + lane;
        if (m < Ti) __stcs(ob + m, v[q]);
      }
    }
  }
}

// the listed groups: every warp of the grid takes 1536-member chunks of each group in turn
template <class PT, int MS, bool PACKED>
__global__ void __launch_bounds__(256) scatter_big_kernel(const __grid_constant__ ScatRegArgs A) {
  const int lane = threadIdx.x & 31;
  const PT* P = static_cast<const PT*>(A.prefix);
  pdl_wait_prior();
  const unsigned nq = min(static_cast<unsigned>(A.qmax), scat_list_len(A));
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (unsigned dq = 0; dq < nq; ++dq) {
    const RegEntry ent = A.q[dq];
    const int64_t nch = (ent.T + RG_CHUNK - 1) / RG_CHUNK;
    if (gw >= nch) continue;
    const int64_t r = ent.rec0 + lane;
    const int64_t Pe = static_cast<int64_t>(P[ent.rec0 + ent.cnt]);
    const int64_t pr = lane < ent.cnt ? static_cast<int64_t>(P[r]) : Pe;
    const int64_t ex = pr - ent.out0, d = (lane < ent.cnt ? A.src_off[r] : 0) - ex;
    for (int64_t c = gw; c < nch; c += nw) {
      const int64_t mb = c * RG_CHUNK;
      span_gather<MS, PACKED>(A.src, A.member_stride, A.dst, ex, d, ent.out0, mb, min(ent.T, mb + RG_CHUNK));
    }
  }
}

// zeroes the fused pack's scratch header + status words; lets the pack's CTAs
// launch (and sum their lengths) meanwhile, but only once everything before it
// in the stream has completed
__global__ void __launch_bounds__(256) scratch_zero_kernel(uint64_t* p, int64_t words, int64_t* extra) {
  pdl_wait_prior();
  pdl_allow_next();
  if (extra && blockIdx.x == 0 && threadIdx.x == 0) *extra = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = 0;
}

template <int MS>
constexpr size_t fused_smem() {
  return static_cast<size_t>(F_NW) * F_NS * W * MS + sizeof(FusedSmem);
}

// segments that read outside the source pool: negative lengths, or a non-empty
// segment [off, off + len) not inside [0, members) -> *bad counts them
__global__ void __launch_bounds__(256) validate_kernel(int64_t n, const void* __restrict__ lens, int lens_type,
                                                       const int64_t* __restrict__ src_off, int64_t members,
                                                       unsigned long long* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned long long cnt = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t len = load_int(lens, lens_type, i);
    if (len < 0) {
      ++cnt;
    } else if (len > 0) {
      const int64_t off = src_off[i];
      cnt += off < 0 || off > members - len;
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}

// shard rebase: P[i] += offset in the index dtype's modular
// arithmetic -- the truncation of (local cumsum + offset) equals the
// truncation of the global cumsum, so a rebased shard prefix is exactly the
// slice of the unsharded one
template <class PT>
__global__ void __launch_bounds__(256) rebase_kernel(int64_t count, PT* __restrict__ p, uint64_t offset) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    p[i] = static_cast<PT>(static_cast<uint64_t>(p[i]) + offset);
}

}  // namespace jag
}  // namespace sk

using namespace sk;

// launch with programmatic stream serialization (the kernel pdl_wait()s before
// touching its predecessor's output)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                   Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

extern "C" {

// fused pack scratch: header, one look-back status word and one queue entry per
// tile
static size_t fused_scratch_bytes(int64_t n) {
  const int64_t t = (n + jag::F_R - 1) / jag::F_R;  // blocks <= t, sub-tiles <= 2 t
  return static_cast<size_t>(64 + ((t * 8 + 63) & ~int64_t(63)) + 2 * t * sizeof(jag::DeferEntry));
}

// register-gather pack scratch: header, one look-back status word per tile, the queue of skewed groups
static int64_t reg_queue_entries(int64_t n) { return std::min<int64_t>(jag::RG_QMAX, (n + 31) / 32); }
// groups per warp: the full RG_GPW once the 8-warp tiles fill 4 CTAs per SM, fewer below that (small inputs
// still spread over the SMs); tiles <= min(n / 256, n / 2048 + 4 * SMs + 1)
static int reg_gpw(int64_t n, int sm_count) {
  const int64_t groups = (n + 31) / 32, warps = static_cast<int64_t>(sm_count) * 4 * jag::RG_NW;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(jag::RG_GPW, (groups + warps - 1) / warps)));
}
static int64_t reg_tiles_max(int64_t n) {  // any device (up to 1024 SMs)
  return std::min<int64_t>((n + 255) / 256, (n + jag::RG_TR - 1) / jag::RG_TR + 4 * 1024 + 1);
}
static size_t reg_status_bytes(int64_t n) { return static_cast<size_t>(reg_tiles_max(n)) * sizeof(jag::RegStatus); }
static size_t reg_scratch_bytes(int64_t n) {
  return 64 + reg_status_bytes(n) + static_cast<size_t>(reg_queue_entries(n)) * sizeof(jag::RegEntry);
}

int sk_jagged_scratch_bytes(int64_t n, size_t* nbytes) {
  if (!nbytes) return set_error(SK_ERR_INVALID, "null out");
  const int64_t tiles = n > 0 ? (n + jag::SCAN_TILE - 1) / jag::SCAN_TILE : 0;
  *nbytes = std::max({static_cast<size_t>(16 + tiles * 8), n > 0 ? fused_scratch_bytes(n) : size_t(0),
                      n > 0 ? reg_scratch_bytes(n) : size_t(0)});
  return SK_OK;
}

static bool int_type(int t) {
  return t == SK_U8 || t == SK_U16 || t == SK_U32 || t == SK_U64 || t == SK_I32 || t == SK_I64 || t == SK_BOOL;
}

// scratch layout: [0] look-back ticket (u32), [8] 1 + last non-empty record, [16..] per-tile status / sums
static int launch_scan(int64_t n, const void* lens, int lens_type, void* scratch, size_t need, const jag::ScanOut& O,
                       cudaStream_t s) {
  const int64_t tiles = (n + jag::SCAN_TILE - 1) / jag::SCAN_TILE;
  uint8_t* sc = static_cast<uint8_t*>(scratch);
  static const int64_t direct_max = [] {
    const char* e = getenv("SK_SCAN_DIRECT_TILES");
    return e ? static_cast<int64_t>(atoll(e)) : jag::SCAN_DIRECT_TILES;
  }();
  if (tiles <= direct_max) {
    int64_t* agg = reinterpret_cast<int64_t*>(sc + 16);
    jag::tile_sum_kernel<<<static_cast<unsigned>(tiles), jag::SCAN_NT, 0, s>>>(
        n, lens, lens_type, agg, O.starts ? O.last : nullptr);
    SK_TRY(cudaGetLastError());
    SK_TRY(launch_pdl(jag::tile_apply_kernel, dim3(static_cast<unsigned>(tiles)), dim3(jag::SCAN_NT), s, n, lens,
                      lens_type, static_cast<const int64_t*>(agg), O));
  } else {
    SK_TRY(cudaMemsetAsync(scratch, 0, need, s));
    jag::scan_lookback_kernel<<<static_cast<unsigned>(tiles), jag::SCAN_NT, 0, s>>>(
        n, lens, lens_type, reinterpret_cast<uint64_t*>(sc + 16), reinterpret_cast<unsigned int*>(sc), O);
  }
  SK_TRY(cudaGetLastError());
  return SK_OK;
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
  jag::ScanOut O{prefix, prefix_type, total_dev, nullptr, nullptr, 0, nullptr};
  return launch_scan(n, lens, lens_type, scratch, need, O, s);
}

// member-field table of the gather
static int gather_args(jag::ScatterArgs* A, int64_t n, const void* prefix, int prefix_type, const int64_t* src_off,
                       const void* src_pool, int64_t member_stride, int nfields, const int64_t* field_off,
                       const int32_t* field_size, void* const* dst_pools, int64_t total, const int64_t* total_dev) {
  if (n < 0 || total < 0) return set_error(SK_ERR_INVALID, "negative sizes");
  if (nfields < 1 || nfields > jag::G_MAXF) return set_error(SK_ERR_INVALID, "nfields %d outside [1, 8]", nfields);
  if (!int_type(prefix_type)) return set_error(SK_ERR_INVALID, "prefix type must be an integer type");
  memset(A, 0, sizeof(*A));
  A->n = n;
  A->prefix = prefix;
  A->prefix_type = prefix_type;
  A->src_off = src_off;
  A->src_pool = static_cast<const uint8_t*>(src_pool);
  A->member_stride = member_stride;
  A->total = total;
  A->total_dev = total_dev;
  A->nfields = nfields;
  for (int f = 0; f < nfields; ++f) {
    const int isz = field_size[f];
    if (isz != 1 && isz != 2 && isz != 4 && isz != 8) return set_error(SK_ERR_INVALID, "member field size %d", isz);
    if (field_off[f] < 0 || field_off[f] + isz > member_stride)
      return set_error(SK_ERR_RANGE, "member field %d outside the member stride", f);
    A->field_off[f] = field_off[f];
    A->field_size[f] = isz;
    A->dst[f] = static_cast<uint8_t*>(dst_pools[f]);
    A->aligned[f] = (field_off[f] % isz == 0) && (member_stride % isz == 0) &&
                    (reinterpret_cast<uintptr_t>(src_pool) % isz == 0);
  }
  return SK_OK;
}


}  // extern "C"

template <class PT, int MS>
static int launch_gather_t(const jag::ScatterArgs& A, int64_t ntasks, cudaStream_t s, const DeviceState* ds) {
  static int occ = 0;
  if (!occ) {
    SK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jag::gather_kernel<PT, MS>, jag::G_NT, 0));
    occ = std::max(occ, 1);
  }
  const int64_t wpb = jag::G_NT / 32;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((ntasks + wpb - 1) / wpb,
                                                              static_cast<int64_t>(ds->sm_count) * occ));
  SK_TRY(launch_pdl(jag::gather_kernel<PT, MS>, dim3(static_cast<unsigned>(grid)), dim3(jag::G_NT), s, A));
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

template <class PT, int MS>
static int launch_gather_async(const jag::ScatterArgs& A, int64_t ntasks, cudaStream_t s, const DeviceState* ds) {
  static int occ = 0;
  if (!occ) {
    SK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jag::gather_async_kernel<PT, MS>,
                                                         jag::GA_WARPS * 32, 0));
    occ = std::max(occ, 1);
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((ntasks + jag::GA_WARPS - 1) / jag::GA_WARPS,
                                                              static_cast<int64_t>(ds->sm_count) * occ));
  SK_TRY(launch_pdl(jag::gather_async_kernel<PT, MS>, dim3(static_cast<unsigned>(grid)), dim3(jag::GA_WARPS * 32), s,
                    A));
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

template <int MS, bool RS>
static int launch_fused_ms(jag::FusedArgs F, uint8_t* scratch, cudaStream_t s, int dev, const DeviceState* ds) {

  constexpr size_t smem = jag::fused_smem<MS>();
  static int occ[64] = {0};
  int& o = occ[dev & 63];
  if (!o) {
    SK_TRY(cudaFuncSetAttribute(jag::pack_fused_kernel<MS, RS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
    SK_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, jag::pack_fused_kernel<MS, RS>, jag::F_NT, smem));
    o = std::max(o, 1);
  }
  // one block of records per CTA (a multiple of 4 records, at least one sub-tile, at most MAX_SUB)
  const int64_t ctas = static_cast<int64_t>(ds->sm_count) * o;
  static const int64_t bpc = [] {  // record blocks per CTA (later ones handed out by ticket)
    const char* e = getenv("SK_FUSED_BPC");
    return e ? std::max<int64_t>(1, atoll(e)) : int64_t(1);
  }();
  int64_t br = (F.n + ctas * bpc - 1) / (ctas * bpc);
  br = std::max<int64_t>(jag::F_R, std::min<int64_t>((br + 3) & ~int64_t(3), int64_t(jag::MAX_SUB) * jag::F_R));
  F.block_recs = br;
  F.nblocks = (F.n + br - 1) / br;
  const int64_t last = F.n - (F.nblocks - 1) * br;
  F.tiles = (F.nblocks - 1) * ((br + jag::F_R - 1) / jag::F_R) + (last + jag::F_R - 1) / jag::F_R;
  F.hdr = reinterpret_cast<jag::FusedHdr*>(scratch);
  F.status = reinterpret_cast<uint64_t*>(scratch + 64);
  const size_t status_bytes = (static_cast<size_t>(F.nblocks) * 8 + 63) & ~size_t(63);
  F.defer = reinterpret_cast<jag::DeferEntry*>(scratch + 64 + status_bytes);
  const int64_t zwords = static_cast<int64_t>((64 + status_bytes) / 8);
  SK_TRY(launch_pdl(jag::scratch_zero_kernel, dim3(static_cast<unsigned>(std::min<int64_t>((zwords + 255) / 256, 64))),
                    dim3(256), s, reinterpret_cast<uint64_t*>(scratch), zwords, F.bad));
  const int64_t grid = std::min<int64_t>(F.nblocks, ctas);
  SK_TRY(launch_pdl_smem(jag::pack_fused_kernel<MS, RS>, dim3(static_cast<unsigned>(grid)), dim3(jag::F_NT), smem, s, F));
  return SK_OK;
}

template <int MS>
static int launch_reg_ms(jag::RegArgs R, uint8_t* scratch, cudaStream_t s, int sm_count) {
  // no scratch zeroing: the kernel's flags carry the launch generation, tile 0 resets the counters
  R.gpw = reg_gpw(R.n, sm_count);
  const int64_t tile_recs = static_cast<int64_t>(jag::RG_NW * 32) * R.gpw;
  const int64_t ntiles = (R.n + tile_recs - 1) / tile_recs;
  if (ntiles > reg_tiles_max(R.n)) return set_error(SK_ERR_INVALID, "jagged pack: %lld tiles exceed the scratch layout", (long long)ntiles);
  R.hdr = reinterpret_cast<jag::RegHdr*>(scratch);
  R.status = reinterpret_cast<jag::RegStatus*>(scratch + 64);
  R.q = reinterpret_cast<jag::RegEntry*>(scratch + 64 + reg_status_bytes(R.n));
  R.qmax = reg_queue_entries(R.n);
  const bool wide = dtype_size(R.lens_type) == 8 || R.lens_type == SK_U32, packed = R.member_stride == MS;
  auto k = wide ? (packed ? jag::pack_reg_kernel<MS, true, true> : jag::pack_reg_kernel<MS, true, false>)
                : (packed ? jag::pack_reg_kernel<MS, false, true> : jag::pack_reg_kernel<MS, false, false>);
  SK_TRY(launch_pdl(k, dim3(static_cast<unsigned>(ntiles)), dim3(jag::RG_NW * 32), s, R));
  return SK_OK;
}

// launch generations for the scratch words that are not zeroed between calls (queue entries, look-back
// words). The scratch may hold words a previous process wrote with its own generations, so the sequence
// starts at a random 61-bit point: a stale word matches a live generation with probability ~2^-61.
static unsigned long long next_generation() {
  static std::atomic<unsigned long long> g{[] {
    std::random_device rd;
    const unsigned long long r = (static_cast<unsigned long long>(rd()) << 32) ^ rd() ^
                                 static_cast<unsigned long long>(
                                     std::chrono::steady_clock::now().time_since_epoch().count());
    return (r & ((1ull << 61) - 1)) | 1;
  }()};
  return (++g) & ((1ull << 62) - 1);  // gen << 2 must not lose bits that matter
}

static bool reg_pack_ok() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SK_JAGGED_REG");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static bool fused_pack_ok() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SK_JAGGED_FUSED");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

static bool async_gather_ok() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SK_JAGGED_ASYNC");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

template <class PT>
static int launch_gather_p(const jag::ScatterArgs& A, int64_t ntasks, cudaStream_t s, const DeviceState* ds) {
  const bool dst16 = reinterpret_cast<uintptr_t>(A.dst[0]) % 16 == 0;
  if (async_gather_ok() && A.nfields == 1 && A.aligned[0] && dst16) {
    if (A.field_size[0] == 8) return launch_gather_async<PT, 8>(A, ntasks, s, ds);
    if (A.field_size[0] == 4) return launch_gather_async<PT, 4>(A, ntasks, s, ds);
  }
  if (A.nfields == 1 && A.aligned[0] && A.field_size[0] == 8) return launch_gather_t<PT, 8>(A, ntasks, s, ds);
  if (A.nfields == 1 && A.aligned[0] && A.field_size[0] == 4) return launch_gather_t<PT, 4>(A, ntasks, s, ds);
  return launch_gather_t<PT, 0>(A, ntasks, s, ds);
}

static int launch_gather(const jag::ScatterArgs& A, int64_t ntasks, cudaStream_t s, int dev) {
  DeviceState* ds = nullptr;
  if (int rc = device_state(dev, &ds)) return rc;
  switch (A.prefix_type) {
    case SK_U8: case SK_BOOL: return launch_gather_p<uint8_t>(A, ntasks, s, ds);
    case SK_U16: return launch_gather_p<uint16_t>(A, ntasks, s, ds);
    case SK_U32: return launch_gather_p<uint32_t>(A, ntasks, s, ds);
    case SK_I32: return launch_gather_p<int32_t>(A, ntasks, s, ds);
    default: return launch_gather_p<int64_t>(A, ntasks, s, ds);
  }
}

template <class PT, int MS, bool PACKED>
static int launch_scatter_reg_t(const jag::ScatRegArgs& R, cudaStream_t s, const DeviceState* ds) {
  const int64_t groups = (R.n + 31) / 32;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((groups + 7) / 8, static_cast<int64_t>(ds->sm_count) * 8));
  SK_TRY(launch_pdl(jag::scatter_reg_kernel<PT, MS, PACKED>, dim3(static_cast<unsigned>(grid)), dim3(256), s, R));
  // the listed groups (usually none: the kernel returns at once); chunks of the largest possible group
  // spread over up to 4 CTAs per SM
  const int64_t chunks = (R.total + jag::RG_CHUNK - 1) / jag::RG_CHUNK;
  const int64_t bgrid = std::max<int64_t>(1, std::min<int64_t>((chunks + 7) / 8, static_cast<int64_t>(ds->sm_count) * 4));
  SK_TRY(launch_pdl(jag::scatter_big_kernel<PT, MS, PACKED>, dim3(static_cast<unsigned>(bgrid)), dim3(256), s, R));
  return SK_OK;
}

template <class PT>
static int launch_scatter_reg_p(const jag::ScatRegArgs& R, int ms, cudaStream_t s, const DeviceState* ds) {
  const bool packed = R.member_stride == ms;
  if (ms == 8)
    return packed ? launch_scatter_reg_t<PT, 8, true>(R, s, ds) : launch_scatter_reg_t<PT, 8, false>(R, s, ds);
  return packed ? launch_scatter_reg_t<PT, 4, true>(R, s, ds) : launch_scatter_reg_t<PT, 4, false>(R, s, ds);
}

// sk_jagged_scatter with one naturally aligned 4/8-byte field: the register gather over the given prefix
static int launch_scatter_reg(const jag::ScatterArgs& A, cudaStream_t s, int dev) {
  DeviceState* ds = nullptr;
  if (int rc = device_state(dev, &ds)) return rc;
  jag::ScatRegArgs R{};
  R.n = A.n;
  R.prefix = A.prefix;
  R.src_off = A.src_off;
  R.src = A.src_pool + A.field_off[0];
  R.member_stride = A.member_stride;
  R.dst = A.dst[0];
  R.total = A.total;
  // every listed group holds more than RG_BIG of the `total` members: the list cannot overflow
  R.qmax = std::min<int64_t>((A.n + 31) / 32, A.total / (jag::RG_BIG + 1) + 1);
  uint8_t* qbuf = nullptr;
  const size_t qbytes = 64 + static_cast<size_t>(R.qmax) * sizeof(jag::RegEntry);
  SK_TRY(cudaMallocAsync(reinterpret_cast<void**>(&qbuf), qbytes, s));
  R.gen = next_generation();  // tags the list counter: nothing is zeroed
  R.nq = reinterpret_cast<unsigned long long*>(qbuf);
  R.q = reinterpret_cast<jag::RegEntry*>(qbuf + 64);
  int rc;
  switch (A.prefix_type) {
    case SK_U8: case SK_BOOL: rc = launch_scatter_reg_p<uint8_t>(R, A.field_size[0], s, ds); break;
    case SK_U16: rc = launch_scatter_reg_p<uint16_t>(R, A.field_size[0], s, ds); break;
    case SK_U32: rc = launch_scatter_reg_p<uint32_t>(R, A.field_size[0], s, ds); break;
    case SK_I32: rc = launch_scatter_reg_p<int32_t>(R, A.field_size[0], s, ds); break;
    case SK_U64: rc = launch_scatter_reg_p<uint64_t>(R, A.field_size[0], s, ds); break;
    default: rc = launch_scatter_reg_p<int64_t>(R, A.field_size[0], s, ds); break;
  }
  SK_TRY(cudaFreeAsync(qbuf, s));
  return rc;
}

extern "C" {

int sk_jagged_scatter(int64_t n, const void* prefix, int prefix_type, const int64_t* src_off, const void* src_pool,
                      int64_t member_stride, int nfields, const int64_t* field_off, const int32_t* field_size,
                      void* const* dst_pools, int64_t total, uintptr_t stream) {
  jag::ScatterArgs A;
  if (int rc = gather_args(&A, n, prefix, prefix_type, src_off, src_pool, member_stride, nfields, field_off,
                           field_size, dst_pools, total, nullptr))
    return rc;
  if (total == 0 || n == 0) return SK_OK;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  if (reg_pack_ok() && nfields == 1 && A.aligned[0] && (A.field_size[0] == 4 || A.field_size[0] == 8) &&
      reinterpret_cast<uintptr_t>(A.dst[0]) % A.field_size[0] == 0)
    return launch_scatter_reg(A, s, dev);
  const int64_t ntasks = (total + jag::W - 1) / jag::W;
  // starts[0..ntasks) from a search over the given prefix, starts[ntasks] = 1 + last non-empty record
  int64_t* starts = nullptr;
  SK_TRY(cudaMallocAsync(&starts, static_cast<size_t>(ntasks + 1) * sizeof(int64_t), s));
  jag::task_start_kernel<<<static_cast<unsigned>((ntasks + 1 + 7) / 8), 256, 0, s>>>(A, starts, ntasks);
  SK_TRY(cudaGetLastError());
  A.starts = starts;
  A.last_rec = reinterpret_cast<const unsigned long long*>(starts + ntasks);
  const int rc = launch_gather(A, ntasks, s, dev);
  SK_TRY(cudaFreeAsync(starts, s));
  return rc;
}

int sk_jagged_validate(int64_t n, const void* lens, int lens_type, const int64_t* src_off, int64_t src_members,
                       int64_t* bad_dev, uintptr_t stream) {
  if (n < 0 || src_members < 0) return set_error(SK_ERR_INVALID, "negative sizes");
  if (!bad_dev) return set_error(SK_ERR_INVALID, "bad_dev is required");
  if (!int_type(lens_type) || lens_type == SK_BOOL) return set_error(SK_ERR_INVALID, "lengths need an integer type");
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  SK_TRY(cudaMemsetAsync(bad_dev, 0, 8, s));
  if (n == 0) return SK_OK;
  DeviceState* ds = nullptr;
  if (int rc = device_state(dev, &ds)) return rc;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, ds->sm_count * 8ll));
  jag::validate_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(n, lens, lens_type, src_off, src_members,
                                                                     reinterpret_cast<unsigned long long*>(bad_dev));
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

int sk_jagged_pack(int64_t n, const void* lens, int lens_type, void* prefix, int prefix_type, const int64_t* src_off,
                   const void* src_pool, int64_t src_members, int64_t member_stride, int nfields,
                   const int64_t* field_off, const int32_t* field_size, void* const* dst_pools, int64_t capacity,
                   void* scratch, size_t scratch_bytes, int64_t* total_dev, uintptr_t stream) {
  if (n < 0 || capacity < 0 || src_members < 0) return set_error(SK_ERR_INVALID, "negative sizes");
  if (!total_dev) return set_error(SK_ERR_INVALID, "total_dev is required");
  if (!int_type(lens_type) || !int_type(prefix_type) || lens_type == SK_BOOL || prefix_type == SK_BOOL)
    return set_error(SK_ERR_INVALID, "jagged lengths and prefix need integer types");
  size_t need = 0;
  sk_jagged_scratch_bytes(n, &need);
  if (scratch_bytes < need) return set_error(SK_ERR_INVALID, "scratch too small: %zu < %zu", scratch_bytes, need);
  jag::ScatterArgs A;
  if (int rc = gather_args(&A, n, nullptr, prefix_type, src_off, src_pool, member_stride, nfields, field_off,
                           field_size, dst_pools, capacity, total_dev))
    return rc;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  cudaStream_t s = resolve_stream(dev, stream);
  if (n == 0) {
    SK_TRY(cudaMemsetAsync(prefix, 0, dtype_size(prefix_type), s));
    SK_TRY(cudaMemsetAsync(total_dev, 0, 16, s));
    return SK_OK;
  }
  // single pass: one aligned 4/8-byte member field into a 16-byte-aligned pool, or (RS) 2-4 naturally
  // aligned 4/8-byte fields of an 8- or 16-byte member record in a record-aligned source pool
  const bool single = nfields == 1 && A.aligned[0] && (A.field_size[0] == 4 || A.field_size[0] == 8) &&
                      reinterpret_cast<uintptr_t>(A.dst[0]) % 16 == 0;
  bool split = nfields >= 2 && nfields <= 4 && (member_stride == 8 || member_stride == 16) &&
               reinterpret_cast<uintptr_t>(src_pool) % member_stride == 0;
  for (int f = 0; f < nfields && split; ++f)
    split = A.aligned[f] && (A.field_size[f] == 4 || A.field_size[f] == 8) &&
            reinterpret_cast<uintptr_t>(A.dst[f]) % A.field_size[f] == 0;
  // single field, MS-aligned destination: the register-gather pack
  if (fused_pack_ok() && reg_pack_ok() && nfields == 1 && A.aligned[0] &&
      (A.field_size[0] == 4 || A.field_size[0] == 8) &&
      reinterpret_cast<uintptr_t>(A.dst[0]) % A.field_size[0] == 0 && reinterpret_cast<uintptr_t>(scratch) % 16 == 0) {
    jag::RegArgs R{};
    R.n = n;
    R.lens = lens;
    R.lens_type = lens_type;
    R.prefix = prefix;
    R.prefix_type = prefix_type;
    R.total = total_dev;
    R.bad = total_dev + 1;
    R.src_off = src_off;
    R.src = A.src_pool + A.field_off[0];
    R.member_stride = member_stride;
    R.dst = A.dst[0];
    R.capacity = capacity;
    R.src_members = src_members;
    R.gen = next_generation();
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    DeviceState* ds = nullptr;
    if (int rc = device_state(dev, &ds)) return rc;
    return A.field_size[0] == 8 ? launch_reg_ms<8>(R, sc, s, ds->sm_count) : launch_reg_ms<4>(R, sc, s, ds->sm_count);
  }
  if (fused_pack_ok() && (single || split)) {
    DeviceState* ds = nullptr;
    if (int rc = device_state(dev, &ds)) return rc;
    jag::FusedArgs F{};
    F.n = n;
    F.lens = lens;
    F.lens_type = lens_type;
    F.prefix = prefix;
    F.prefix_type = prefix_type;
    F.total = total_dev;
    F.src_off = src_off;
    F.src = single ? A.src_pool + A.field_off[0] : A.src_pool;
    F.nf = nfields;
    for (int f = 0; f < nfields && f < 4; ++f) {
      F.fsz[f] = A.field_size[f];
      F.foff[f] = static_cast<int>(A.field_off[f]);
      F.fdst[f] = A.dst[f];
    }
    F.member_stride = member_stride;
    F.dst = A.dst[0];
    F.capacity = capacity;
    F.pvec = dtype_size(prefix_type) == 4 && reinterpret_cast<uintptr_t>(prefix) % 16 == 0;
    F.lens16 = (dtype_size(lens_type) == 4 || dtype_size(lens_type) == 8) && reinterpret_cast<uintptr_t>(lens) % 16 == 0;
    static const int dbg = [] {
      const char* e = getenv("SK_FUSED_DBG");
      return e ? atoi(e) : 0;
    }();
    F.dbg = dbg;
    F.src_members = src_members;
    F.bad = total_dev + 1;
    F.gen = next_generation();
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    if (split)
      return member_stride == 16 ? launch_fused_ms<16, true>(F, sc, s, dev, ds)
                                 : launch_fused_ms<8, true>(F, sc, s, dev, ds);
    return A.field_size[0] == 8 ? launch_fused_ms<8, false>(F, sc, s, dev, ds)
                                : launch_fused_ms<4, false>(F, sc, s, dev, ds);
  }
  // a prefix type that can wrap below the capacity needs an int64 copy for the gather
  const int bits = 8 * dtype_size(prefix_type) - ((prefix_type == SK_I32 || prefix_type == SK_I64) ? 1 : 0);
  const bool may_wrap = bits < 63 && capacity >= (int64_t(1) << bits);
  int64_t* p64 = nullptr;
  if (may_wrap) SK_TRY(cudaMallocAsync(&p64, static_cast<size_t>(n + 1) * sizeof(int64_t), s));
  // the gather's work split: in the caller's scratch when it is large enough
  const int64_t ntasks = capacity ? (capacity + jag::W - 1) / jag::W : 0;
  const size_t scan_part = (need + 255) & ~size_t(255);
  const size_t starts_need = static_cast<size_t>(ntasks + 1) * sizeof(int64_t);
  int64_t* starts = scratch_bytes >= scan_part + starts_need
                        ? reinterpret_cast<int64_t*>(static_cast<uint8_t*>(scratch) + scan_part)
                        : nullptr;
  const bool own_starts = ntasks && !starts;
  if (own_starts) SK_TRY(cudaMallocAsync(&starts, starts_need, s));
  unsigned long long* last_rec = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(scratch) + 8);
  jag::ScanOut O{prefix, prefix_type, total_dev, p64, ntasks ? starts : nullptr, ntasks, last_rec};
  int rc = sk_jagged_validate(n, lens, lens_type, src_off, src_members, total_dev + 1, stream);
  if (rc == SK_OK) rc = launch_scan(n, lens, lens_type, scratch, need, O, s);
  // gather bounded by the pools' capacity; the kernel reads the true total on the device
  if (rc == SK_OK && ntasks) {
    A.prefix = p64 ? static_cast<const void*>(p64) : prefix;
    A.prefix_type = p64 ? SK_I64 : prefix_type;
    A.starts = starts;
    A.last_rec = last_rec;
    A.bad_dev = total_dev + 1;
    rc = launch_gather(A, ntasks, s, dev);
  }
  if (own_starts) cudaFreeAsync(starts, s);
  if (p64) cudaFreeAsync(p64, s);
  return rc;
}

}  // extern "C"

template <class PT>
static int launch_rebase(int64_t count, void* p, int64_t offset, cudaStream_t s, const DeviceState* ds) {
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, ds->sm_count * 8ll));
  jag::rebase_kernel<PT><<<static_cast<unsigned>(blocks), 256, 0, s>>>(count, static_cast<PT*>(p),
                                                                        static_cast<uint64_t>(offset));
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

// experiments only: the fused pack's per-CTA timestamps (SK_FUSED_DBG & 8)
extern "C" int sk_jagged_trace(void* host, size_t bytes) {
  SK_TRY(cudaDeviceSynchronize());
  SK_TRY(cudaMemcpyFromSymbol(host, jag::g_fused_trace, std::min(bytes, sizeof(jag::g_fused_trace))));
  return SK_OK;
}

extern "C" int sk_jagged_rebase(int64_t count, void* prefix, int prefix_type, int64_t offset, uintptr_t stream) {
  if (count < 0) return set_error(SK_ERR_INVALID, "negative count");
  if (!int_type(prefix_type) || prefix_type == SK_BOOL) return set_error(SK_ERR_INVALID, "prefix needs an integer type");
  if (count == 0 || offset == 0) return SK_OK;
  if (!prefix) return set_error(SK_ERR_INVALID, "null prefix");
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  DeviceState* ds = nullptr;
  if (int rc = device_state(dev, &ds)) return rc;
  cudaStream_t s = resolve_stream(dev, stream);
  switch (prefix_type) {
    case SK_U8: return launch_rebase<uint8_t>(count, prefix, offset, s, ds);
    case SK_U16: return launch_rebase<uint16_t>(count, prefix, offset, s, ds);
    case SK_U32: case SK_I32: return launch_rebase<uint32_t>(count, prefix, offset, s, ds);
    default: return launch_rebase<uint64_t>(count, prefix, offset, s, ds);
  }
}
