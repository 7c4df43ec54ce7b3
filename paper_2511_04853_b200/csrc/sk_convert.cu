// Layout-conversion engine (K1 aos->planes, K2 planes->aos, K3 ->aosoa with
// subset/reorder/cast) and the host<->device transfer pipeline.
//
// Reference behaviour being replaced: transfer.py:171-236 (_per_leaf_execute)
// streams the packed AoS struct once per leaf with numpy strided gathers and
// stages every plane through host buffers. Here one persistent kernel moves
// each record exactly once through shared memory:
//
//   TMA bulk load (cp.async.bulk g2s, mbarrier ring of `stages` tiles)
//     -> in-smem transposition (word moves for 4-byte-aligned fields,
//        funnel-shift element moves + numpy-exact casts for the rest)
//     -> TMA bulk store (cp.async.bulk s2g, double-buffered output tile)
//
// A tile holds R records in the source representation: a packed AoS run, or
// one R-element segment per field (planes), or R/T AoSoA tiles. Global traffic
// is exactly the algorithmic bytes: every source byte is read once, every
// destination byte written once, all through 16-byte-aligned bulk transfers.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "sk_internal.cuh"

namespace sk {
namespace conv {

constexpr int NT = 256;
constexpr int MAX_WORDS = 256;     // word table -> AoS strides up to 1 KiB use word moves
constexpr int TILE_TARGET = 49152; // in+out bytes per tile (sweep: profiles/r01_sweep.md)
constexpr int MAX_STAGES = 4;

enum { MODE_ELEM = 0, MODE_WORD_A2P = 1, MODE_WORD_P2A = 2 };
enum { EPI_NONE = 0, EPI_SENSOR = 1 };

struct FieldPlan {
  uint8_t st, dt, sisz, disz;
  uint8_t wordable;
  uint8_t op;        // element-path specialisation (ELEM_*), chosen on the host
  uint8_t sal, dal;  // source / destination element always naturally aligned in smem
  int32_t sloc;  // AOS: offset in record; PLANES: smem segment offset; AOSOA: block offset in tile
  int32_t dloc;
  const uint8_t* splane;
  uint8_t* dplane;
};

struct Plan {
  int64_t n;
  int64_t ntiles;
  int32_t R;
  int32_t src_kind, dst_kind;
  int32_t src_stride, dst_stride;  // AOS record bytes / AOSOA tile bytes
  int32_t src_lshift, dst_lshift;  // log2(lanes) for AOSOA
  // smem element address of record r of a field, branch-free for every kind:
  //   ((r >> lshift) * A) + ((r & msk) * itemsize) + loc
  //   AOS: A = stride, msk = 0;  PLANES: A = 0, msk = ~0;  AOSOA: A = tile, msk = T-1
  int32_t src_A, dst_A, src_msk, dst_msk;
  int32_t in_tile_bytes, out_tile_bytes;
  int32_t in_stage_stride, out_stage_stride;
  int32_t stages;
  int32_t nfields;
  int32_t mode;
  int32_t words_per_rec;
  int32_t bulk_in, bulk_out;
  int32_t zero_out;
  int32_t epi;
  int32_t epi_seg[7];       // sensor: counts, energy, noisy, A, B, nA, nB (out-tile segment offsets)
  int32_t extra_loc;        // epilogue output segment (sensor noise)
  uint8_t* extra_plane;
  const uint8_t* src;
  uint8_t* dst;
  int32_t smem_bar_off, smem_tab_off, smem_in_off, smem_out_off, smem_total;
  int32_t n_elem;           // fields moved by the element path, their indices, records split
  int32_t elem_chunks;
  uint8_t elem_idx[SK_MAX_FIELDS];
  int32_t cache_hint;       // 0 none, 1 evict_first on loads and stores, 2 loads only
  FieldPlan f[SK_MAX_FIELDS];
  int32_t wtab[MAX_WORDS];  // (segment byte base << 4) | element size ; -1 = not a word-moved word
};

static_assert(sizeof(Plan) < 4000, "kernel parameter block must stay under 4 KB");

// ---------------------------------------------------------------------------------
// element access in shared memory (any alignment) and numpy-exact casts

__device__ __forceinline__ uint64_t lds_any(const uint8_t* p, int isz) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
  const uint32_t sh = static_cast<uint32_t>(a & 3) * 8u;
  const uint32_t w0 = w[0];
  const uint32_t w1 = w[1];
  const uint32_t lo = __funnelshift_r(w0, w1, sh);
  if (isz == 8) {
    const uint32_t hi = __funnelshift_r(w1, w[2], sh);
    return (static_cast<uint64_t>(hi) << 32) | lo;
  }
  if (isz == 4) return lo;
  if (isz == 2) return lo & 0xffffu;
  return lo & 0xffu;
}

__device__ __forceinline__ void sts_any(uint8_t* p, uint64_t v, int isz) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if ((a & (isz - 1)) == 0) {
    switch (isz) {
      case 1: *p = static_cast<uint8_t>(v); return;
      case 2: *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>(v); return;
      case 4: *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>(v); return;
      default: *reinterpret_cast<uint64_t*>(p) = v; return;
    }
  }
  if ((a & 1) == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (2 * i < isz) reinterpret_cast<uint16_t*>(p)[i] = static_cast<uint16_t>(v >> (16 * i));
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if (i < isz) p[i] = static_cast<uint8_t>(v >> (8 * i));
}

__device__ __forceinline__ bool is_signed_int(int t) { return t == SK_I32 || t == SK_I64; }
__device__ __forceinline__ bool is_float(int t) { return t == SK_F32 || t == SK_F64; }

// raw bits of the source element -> raw bits of the destination element,
// following numpy astype (IEEE RNE, integer wrap, x86 NaN payload rules).
__device__ __forceinline__ uint64_t cast_bits(uint64_t v, int st, int dt) {
  if (st == dt) return v;
  if (st == SK_F64 && dt == SK_F32) {
    const uint64_t exp = (v >> 52) & 0x7ff;
    const uint64_t man = v & 0xfffffffffffffull;
    if (exp == 0x7ff && man != 0) {  // NaN: cvtsd2ss keeps the top payload bits, sets quiet bit
      const uint32_t sign = static_cast<uint32_t>(v >> 63) << 31;
      return sign | 0x7fc00000u | static_cast<uint32_t>(man >> 29);
    }
    return __float_as_uint(__double2float_rn(__longlong_as_double(static_cast<long long>(v))));
  }
  if (st == SK_F32 && dt == SK_F64) {
    const uint32_t u = static_cast<uint32_t>(v);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) {  // NaN: cvtss2sd quiets, keeps payload
      const uint64_t sign = static_cast<uint64_t>(u >> 31) << 63;
      return sign | 0x7ff8000000000000ull | (static_cast<uint64_t>(u & 0x7fffffu) << 29);
    }
    return static_cast<uint64_t>(__double_as_longlong(static_cast<double>(__uint_as_float(u))));
  }
  if (st == SK_BOOL) v = (v & 0xff) ? 1 : 0;
  if (dt == SK_BOOL) {
    if (is_float(st)) {
      const double x = st == SK_F32 ? static_cast<double>(__uint_as_float(static_cast<uint32_t>(v)))
                                    : __longlong_as_double(static_cast<long long>(v));
      return x != 0.0 ? 1 : 0;  // NaN != 0 -> True, as numpy
    }
    return v ? 1 : 0;
  }
  // integer source: widen to a 64-bit value
  int64_t iv;
  if (st == SK_I32) iv = static_cast<int32_t>(static_cast<uint32_t>(v));
  else iv = static_cast<int64_t>(v);  // unsigned widths arrive zero-extended; I64/U64 raw
  if (dt == SK_F32) {
    float f = st == SK_U64 ? __ull2float_rn(v) : __ll2float_rn(iv);
    return __float_as_uint(f);
  }
  if (dt == SK_F64) {
    double x = st == SK_U64 ? __ull2double_rn(v) : __ll2double_rn(iv);
    return static_cast<uint64_t>(__double_as_longlong(x));
  }
  // integer destination: two's-complement wrap to the destination width
  const uint64_t u = static_cast<uint64_t>(iv);
  switch (dt) {
    case SK_U8: return u & 0xff;
    case SK_U16: return u & 0xffff;
    case SK_U32: case SK_I32: return u & 0xffffffffull;
    default: return u;
  }
}

__device__ __forceinline__ uint32_t rec_addr(int kind, int32_t loc, int isz, int32_t stride, int lshift, int r) {
  if (kind == SK_KIND_AOS) return static_cast<uint32_t>(r * stride + loc);
  if (kind == SK_KIND_PLANES) return static_cast<uint32_t>(loc + r * isz);
  return static_cast<uint32_t>((r >> lshift) * stride + loc + (r & ((1 << lshift) - 1)) * isz);
}

// ---------------------------------------------------------------------------------
// tile regions: global address + byte count for tile t with `rows` records

__device__ __forceinline__ int64_t tile_bytes_kind(int kind, int rows, int isz, int stride, int lshift) {
  if (kind == SK_KIND_AOS) return static_cast<int64_t>(rows) * stride;
  if (kind == SK_KIND_PLANES) return static_cast<int64_t>(rows) * isz;
  return static_cast<int64_t>((rows + (1 << lshift) - 1) >> lshift) * stride;
}

// cooperative copy between global and shared memory (tail tiles, peer pointers,
// misaligned planes). 16-byte moves when both sides allow it, 4 loads in flight.
__device__ __forceinline__ void coop_copy(uint8_t* dst, const uint8_t* src, int64_t bytes) {
  const int tid = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 15) == 0) {
    const int64_t nv = bytes >> 4;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    int64_t i = tid;
    for (; i + 3 * NT < nv; i += 4 * NT) {
      uint4 a = s[i], b = s[i + NT], c = s[i + 2 * NT], e = s[i + 3 * NT];
      d[i] = a; d[i + NT] = b; d[i + 2 * NT] = c; d[i + 3 * NT] = e;
    }
    for (; i < nv; i += NT) d[i] = s[i];
  } else if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 3) == 0) {
    const int64_t nw = bytes >> 2;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int64_t i = tid; i < nw; i += NT) d[i] = s[i];
  } else {
    for (int64_t i = tid; i < bytes; i += NT) dst[i] = src[i];
  }
}

__device__ __forceinline__ void g2s(const Plan& P, void* s, const void* g, uint32_t bytes, uint64_t* bar,
                                    uint64_t pol) {
  if (P.cache_hint) bulk_g2s(s, g, bytes, bar, pol);
  else bulk_g2s_plain(s, g, bytes, bar);
}

__device__ __forceinline__ void s2g(const Plan& P, void* g, const void* s, uint32_t bytes, uint64_t pol) {
  if (P.cache_hint == 1) bulk_s2g(g, s, bytes, pol);
  else bulk_s2g_plain(g, s, bytes);
}

__device__ void issue_bulk_load(const Plan& P, int64_t t, uint8_t* in, uint64_t* bar, uint64_t pol) {
  const int64_t r0 = t * P.R;
  mbar_expect_tx(bar, static_cast<uint32_t>(P.in_tile_bytes));
  if (P.src_kind == SK_KIND_PLANES) {
    for (int i = 0; i < P.nfields; ++i) {
      const FieldPlan& F = P.f[i];
      g2s(P, in + F.sloc, F.splane + r0 * F.sisz, static_cast<uint32_t>(P.R * F.sisz), bar, pol);
    }
  } else {
    const int64_t off = P.src_kind == SK_KIND_AOS ? r0 * P.src_stride : (r0 >> P.src_lshift) * P.src_stride;
    g2s(P, in, P.src + off, static_cast<uint32_t>(P.in_tile_bytes), bar, pol);
  }
}

__device__ void coop_load(const Plan& P, int64_t t, int rows, uint8_t* in) {
  const int64_t r0 = t * P.R;
  if (P.src_kind == SK_KIND_PLANES) {
    for (int i = 0; i < P.nfields; ++i) {
      const FieldPlan& F = P.f[i];
      coop_copy(in + F.sloc, F.splane + r0 * F.sisz, static_cast<int64_t>(rows) * F.sisz);
    }
  } else {
    const int64_t off = P.src_kind == SK_KIND_AOS ? r0 * P.src_stride : (r0 >> P.src_lshift) * P.src_stride;
    coop_copy(in, P.src + off, tile_bytes_kind(P.src_kind, rows, 0, P.src_stride, P.src_lshift));
  }
}

__device__ void issue_bulk_store(const Plan& P, int64_t t, const uint8_t* out, uint64_t pol) {
  const int64_t r0 = t * P.R;
  if (P.dst_kind == SK_KIND_PLANES) {
    for (int i = 0; i < P.nfields; ++i) {
      const FieldPlan& F = P.f[i];
      s2g(P, F.dplane + r0 * F.disz, out + F.dloc, static_cast<uint32_t>(P.R * F.disz), pol);
    }
  } else {
    const int64_t off = P.dst_kind == SK_KIND_AOS ? r0 * P.dst_stride : (r0 >> P.dst_lshift) * P.dst_stride;
    s2g(P, P.dst + off, out, static_cast<uint32_t>(P.out_tile_bytes), pol);
  }
  if (P.extra_plane) s2g(P, P.extra_plane + r0 * 4, out + P.extra_loc, static_cast<uint32_t>(P.R * 4), pol);
}

__device__ void coop_store(const Plan& P, int64_t t, int rows, const uint8_t* out) {
  const int64_t r0 = t * P.R;
  if (P.dst_kind == SK_KIND_PLANES) {
    for (int i = 0; i < P.nfields; ++i) {
      const FieldPlan& F = P.f[i];
      coop_copy(F.dplane + r0 * F.disz, out + F.dloc, static_cast<int64_t>(rows) * F.disz);
    }
  } else {
    const int64_t off = P.dst_kind == SK_KIND_AOS ? r0 * P.dst_stride : (r0 >> P.dst_lshift) * P.dst_stride;
    coop_copy(P.dst + off, out, tile_bytes_kind(P.dst_kind, rows, 0, P.dst_stride, P.dst_lshift));
  }
  if (P.extra_plane) coop_copy(P.extra_plane + r0 * 4, out + P.extra_loc, static_cast<int64_t>(rows) * 4);
}

// ---------------------------------------------------------------------------------
// element path: one specialised loop per (size, alignment, cast) class; the
// class is chosen on the host (FieldPlan::op/sal/dal) and dispatched once per
// field, so the per-element body is a handful of instructions.

enum { ELEM_GENERIC = 0, ELEM_MOVE = 1, ELEM_F64_F32 = 2, ELEM_F32_F64 = 3 };

template <int SZ>
__device__ __forceinline__ uint64_t lds_al(const uint8_t* p) {
  if (SZ == 1) return *p;
  if (SZ == 2) return *reinterpret_cast<const uint16_t*>(p);
  if (SZ == 4) return *reinterpret_cast<const uint32_t*>(p);
  return *reinterpret_cast<const uint64_t*>(p);
}

template <int SZ>
__device__ __forceinline__ void sts_al(uint8_t* p, uint64_t v) {
  if (SZ == 1) *p = static_cast<uint8_t>(v);
  else if (SZ == 2) *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>(v);
  else if (SZ == 4) *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>(v);
  else *reinterpret_cast<uint64_t*>(p) = v;
}

template <int CV>
__device__ __forceinline__ uint64_t convert_op(uint64_t v) {
  if (CV == ELEM_F64_F32) return cast_bits(v, SK_F64, SK_F32);
  if (CV == ELEM_F32_F64) return cast_bits(v, SK_F32, SK_F64);
  return v;
}

// One warp moves records [r0, r1) of one field: lane l takes r0 + l, r0 + l + 32, ...
template <int SI, int DI, int CV, bool SAL, bool DAL>
__device__ __forceinline__ void elem_loop(const Plan& P, const FieldPlan& F, const uint8_t* __restrict__ in,
                                          uint8_t* __restrict__ out, int r0, int r1) {
  const int sl = P.src_lshift, dl = P.dst_lshift, sA = P.src_A, dA = P.dst_A, sm = P.src_msk, dm = P.dst_msk;
  const int sloc = F.sloc, dloc = F.dloc;
#pragma unroll 8
  for (int r = r0 + static_cast<int>(threadIdx.x & 31); r < r1; r += 32) {
    const uint32_t sa = static_cast<uint32_t>((r >> sl) * sA + (r & sm) * SI + sloc);
    const uint32_t da = static_cast<uint32_t>((r >> dl) * dA + (r & dm) * DI + dloc);
    const uint64_t v = convert_op<CV>(SAL ? lds_al<SI>(in + sa) : lds_any(in + sa, SI));
    if (DAL) sts_al<DI>(out + da, v);
    else sts_any(out + da, v, DI);
  }
}

template <int SI, int DI, int CV>
__device__ __forceinline__ void elem_aligned(const Plan& P, const FieldPlan& F, const uint8_t* in, uint8_t* out,
                                             int r0, int r1) {
  if (F.sal) {
    if (F.dal) elem_loop<SI, DI, CV, true, true>(P, F, in, out, r0, r1);
    else elem_loop<SI, DI, CV, true, false>(P, F, in, out, r0, r1);
  } else {
    if (F.dal) elem_loop<SI, DI, CV, false, true>(P, F, in, out, r0, r1);
    else elem_loop<SI, DI, CV, false, false>(P, F, in, out, r0, r1);
  }
}

__device__ __noinline__ void elem_generic(const Plan& P, const FieldPlan& F, const uint8_t* in, uint8_t* out,
                                          int r0, int r1) {
  const int st = F.st, dt = F.dt, sisz = F.sisz, disz = F.disz;
  for (int r = r0 + static_cast<int>(threadIdx.x & 31); r < r1; r += 32) {
    const uint32_t sa = static_cast<uint32_t>((r >> P.src_lshift) * P.src_A + (r & P.src_msk) * sisz + F.sloc);
    const uint32_t da = static_cast<uint32_t>((r >> P.dst_lshift) * P.dst_A + (r & P.dst_msk) * disz + F.dloc);
    sts_any(out + da, cast_bits(lds_any(in + sa, sisz), st, dt), disz);
  }
}

__device__ __forceinline__ void elem_field(const Plan& P, const FieldPlan& F, const uint8_t* in, uint8_t* out,
                                           int r0, int r1) {
  switch (F.op) {
    case ELEM_MOVE:
      switch (F.sisz) {
        case 1: elem_aligned<1, 1, ELEM_MOVE>(P, F, in, out, r0, r1); break;
        case 2: elem_aligned<2, 2, ELEM_MOVE>(P, F, in, out, r0, r1); break;
        case 4: elem_aligned<4, 4, ELEM_MOVE>(P, F, in, out, r0, r1); break;
        default: elem_aligned<8, 8, ELEM_MOVE>(P, F, in, out, r0, r1); break;
      }
      break;
    case ELEM_F64_F32: elem_aligned<8, 4, ELEM_F64_F32>(P, F, in, out, r0, r1); break;
    case ELEM_F32_F64: elem_aligned<4, 8, ELEM_F32_F64>(P, F, in, out, r0, r1); break;
    default: elem_generic(P, F, in, out, r0, r1); break;
  }
}

// ---------------------------------------------------------------------------------
// in-smem transposition

__device__ __forceinline__ void transform(const Plan& P, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                          int rows, const int32_t* __restrict__ wtab) {
  const int tid = threadIdx.x;
  if (P.mode != MODE_ELEM) {
    // word moves: iterate over the words of the AoS side (conflict-free there);
    // the planes side is staggered 16 B per segment so 8 lanes x 4 records hit
    // distinct banks.
    const int wpr = P.words_per_rec;
    const int total = rows * wpr;
    int r = tid / wpr;
    int q = tid - r * wpr;
    const int dr = NT / wpr;
    const int dq = NT - dr * wpr;
    if (dq == 0) {
      // NT is a multiple of the record's word count: every word this thread
      // touches sits at the same record slot q, so the table entry is loop
      // invariant and the loop is a pure, unrolled LDS->STS stream (4 loads in
      // flight per thread).
      const int e = wtab[q];
      if (e >= 0) {
        const int base = e >> 4, isz = e & 15;
        if (P.mode == MODE_WORD_A2P) {
          const uint32_t* in32 = reinterpret_cast<const uint32_t*>(in);
          int w = tid;
          for (; w + 3 * NT < total; w += 4 * NT, r += 4 * dr) {
            const uint32_t v0 = in32[w], v1 = in32[w + NT], v2 = in32[w + 2 * NT], v3 = in32[w + 3 * NT];
            *reinterpret_cast<uint32_t*>(out + base + r * isz) = v0;
            *reinterpret_cast<uint32_t*>(out + base + (r + dr) * isz) = v1;
            *reinterpret_cast<uint32_t*>(out + base + (r + 2 * dr) * isz) = v2;
            *reinterpret_cast<uint32_t*>(out + base + (r + 3 * dr) * isz) = v3;
          }
          for (; w < total; w += NT, r += dr) *reinterpret_cast<uint32_t*>(out + base + r * isz) = in32[w];
        } else {
          uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
          int w = tid;
          for (; w + 3 * NT < total; w += 4 * NT, r += 4 * dr) {
            const uint32_t v0 = *reinterpret_cast<const uint32_t*>(in + base + r * isz);
            const uint32_t v1 = *reinterpret_cast<const uint32_t*>(in + base + (r + dr) * isz);
            const uint32_t v2 = *reinterpret_cast<const uint32_t*>(in + base + (r + 2 * dr) * isz);
            const uint32_t v3 = *reinterpret_cast<const uint32_t*>(in + base + (r + 3 * dr) * isz);
            out32[w] = v0;
            out32[w + NT] = v1;
            out32[w + 2 * NT] = v2;
            out32[w + 3 * NT] = v3;
          }
          for (; w < total; w += NT, r += dr) out32[w] = *reinterpret_cast<const uint32_t*>(in + base + r * isz);
        }
      }
    } else if (P.mode == MODE_WORD_A2P) {
      const uint32_t* in32 = reinterpret_cast<const uint32_t*>(in);
      for (int w = tid; w < total; w += NT) {
        const int e = wtab[q];
        if (e >= 0) *reinterpret_cast<uint32_t*>(out + (e >> 4) + r * (e & 15)) = in32[w];
        q += dq;
        r += dr;
        if (q >= wpr) { q -= wpr; ++r; }
      }
    } else {
      uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
      for (int w = tid; w < total; w += NT) {
        const int e = wtab[q];
        if (e >= 0) out32[w] = *reinterpret_cast<const uint32_t*>(in + (e >> 4) + r * (e & 15));
        q += dq;
        r += dr;
        if (q >= wpr) { q -= wpr; ++r; }
      }
    }
  }
  if (!P.n_elem) return;
  // element moves: work items (field, record chunk) spread over the warps, so
  // each warp dispatches once per item and walks a long, unrolled record loop
  const int warp = tid >> 5;
  const int chunks = P.elem_chunks;
  const int items = P.n_elem * chunks;
  for (int it = warp; it < items; it += NT / 32) {
    const int fi = P.elem_idx[it / chunks];
    const int c = it - (it / chunks) * chunks;
    const int r0 = (rows * c) / chunks, r1 = (rows * (c + 1)) / chunks;
    elem_field(P, P.f[fi], in, out, r0, r1);
  }
}

// case-study kernel applied to the converted planes tile (detector/schemas.py:29-41)
__device__ __forceinline__ void sensor_epilogue(const Plan& P, uint8_t* out, int rows) {
  for (int r = threadIdx.x; r < rows; r += NT) {
    const uint64_t c = *reinterpret_cast<const uint64_t*>(out + P.epi_seg[0] + r * 8);
    const float a = *reinterpret_cast<const float*>(out + P.epi_seg[3] + r * 4);
    const float b = *reinterpret_cast<const float*>(out + P.epi_seg[4] + r * 4);
    const float na = *reinterpret_cast<const float*>(out + P.epi_seg[5] + r * 4);
    const float nb = *reinterpret_cast<const float*>(out + P.epi_seg[6] + r * 4);
    const uint8_t noisy = out[P.epi_seg[2] + r];
    const float e = sensor_energy(c, a, b);
    *reinterpret_cast<float*>(out + P.epi_seg[1] + r * 4) = e;
    *reinterpret_cast<float*>(out + P.extra_loc + r * 4) = sensor_noise(e, na, nb, noisy != 0);
  }
}

// ---------------------------------------------------------------------------------
// the persistent pipelined kernel

__global__ void __launch_bounds__(NT) convert_kernel(const __grid_constant__ Plan P) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.smem_bar_off);
  int32_t* wtab = reinterpret_cast<int32_t*>(smem + P.smem_tab_off);
  uint8_t* in0 = smem + P.smem_in_off;
  uint8_t* out0 = smem + P.smem_out_off;
  const int tid = threadIdx.x;
  const int S = P.stages;

  if (tid < S) mbar_init(&bars[tid], 1);
  if (P.mode != MODE_ELEM)
    for (int i = tid; i < P.words_per_rec; i += NT) wtab[i] = P.wtab[i];
  if (tid == 0) fence_mbar_init();
  __syncthreads();

  const int64_t first = blockIdx.x;
  const int64_t step = gridDim.x;
  if (first >= P.ntiles) return;
  const int64_t my_tiles = (P.ntiles - first + step - 1) / step;
  const uint64_t pol_in = policy_evict_first();
  const uint64_t pol_out = policy_evict_first();
  const int64_t last_tile = P.ntiles - 1;
  const int last_rows = static_cast<int>(P.n - last_tile * P.R);

  auto tile_bulk_in = [&](int64_t t) { return P.bulk_in && (t != last_tile || last_rows == P.R); };

  if (tid == 0) {
    for (int s = 0; s < S && s < my_tiles; ++s) {
      const int64_t t = first + s * step;
      if (tile_bulk_in(t)) issue_bulk_load(P, t, in0 + s * P.in_stage_stride, &bars[s], pol_in);
    }
  }

  uint32_t phase_bits = 0;
  int slot = 0;
  for (int64_t it = 0; it < my_tiles; ++it) {
    const int64_t t = first + it * step;
    const int rows = t == last_tile ? last_rows : P.R;
    uint8_t* in = in0 + slot * P.in_stage_stride;
    uint8_t* out = out0 + static_cast<int>(it & 1) * P.out_stage_stride;
    const bool bin = tile_bulk_in(t);
    if (bin) {
      mbar_wait(&bars[slot], (phase_bits >> slot) & 1u);
      phase_bits ^= 1u << slot;
    } else {
      coop_load(P, t, rows, in);
    }
    if (tid == 0) bulk_wait_read<1>();  // out[it&1] no longer read by the store of tile it-2
    __syncthreads();
    if (P.zero_out || (rows < P.R && P.dst_kind == SK_KIND_AOSOA)) {
      uint32_t* o32 = reinterpret_cast<uint32_t*>(out);
      for (int i = tid; i < (P.out_tile_bytes >> 2); i += NT) o32[i] = 0;
      __syncthreads();
    }
    transform(P, in, out, rows, wtab);
    if (P.epi == EPI_SENSOR) {
      __syncthreads();
      sensor_epilogue(P, out, rows);
    }
    const bool bout = P.bulk_out && rows == P.R;
    if (bout) fence_proxy_async();
    __syncthreads();
    if (bout) {
      if (tid == 0) {
        issue_bulk_store(P, t, out, pol_out);
        bulk_commit();
      }
    } else {
      coop_store(P, t, rows, out);
    }
    if (tid == 0 && it + S < my_tiles) {
      const int64_t tn = first + (it + S) * step;
      if (tile_bulk_in(tn)) issue_bulk_load(P, tn, in, &bars[slot], pol_in);
    }
    if (++slot == S) slot = 0;
  }
  if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------------
// host-side planning

static bool cast_supported(int st, int dt) {
  if (st == dt) return true;
  const bool sf = st == SK_F32 || st == SK_F64;
  const bool df = dt == SK_F32 || dt == SK_F64;
  if (sf && !df) return dt == SK_BOOL;  // float->int is undefined in numpy for out-of-range; refuse
  return true;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}

static int64_t lcm64(int64_t a, int64_t b) { return a / gcd64(a, b) * b; }

static int log2_exact(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return (1 << l) == v ? l : -1;
}

static inline int32_t align_up(int32_t v, int32_t a) { return (v + a - 1) / a * a; }

// Validate a descriptor; fills per-kind geometry used by both the planner and
// the transfer pipeline.
int validate(const sk_conv_desc& d, int64_t* granule, int64_t* in_rec_x1000, int64_t* out_rec_x1000) {
  if (d.n < 0) return set_error(SK_ERR_INVALID, "negative record count %lld", (long long)d.n);
  if (d.nfields < 1 || d.nfields > SK_MAX_FIELDS)
    return set_error(SK_ERR_INVALID, "nfields %d outside [1, %d]", d.nfields, SK_MAX_FIELDS);
  if (d.flags != 0) return set_error(SK_ERR_INVALID, "flags must be 0");
  int64_t g = 16;
  for (int side = 0; side < 2; ++side) {
    const int kind = side ? d.dst_kind : d.src_kind;
    const int64_t stride = side ? d.dst_stride : d.src_stride;
    const int lanes = side ? d.dst_lanes : d.src_lanes;
    const void* base = side ? static_cast<const void*>(d.dst) : d.src;
    if (kind < SK_KIND_AOS || kind > SK_KIND_AOSOA) return set_error(SK_ERR_INVALID, "bad endpoint kind %d", kind);
    if (kind != SK_KIND_PLANES && !base && d.n) return set_error(SK_ERR_INVALID, "null %s base pointer", side ? "dst" : "src");
    if (kind == SK_KIND_AOS && (stride < 1 || stride > (1 << 20)))
      return set_error(SK_ERR_INVALID, "AoS record stride %lld outside [1, 1 MiB]", (long long)stride);
    if (kind == SK_KIND_AOSOA) {
      if (lanes < 1 || lanes > 1024 || log2_exact(lanes) < 0)
        return set_error(SK_ERR_INVALID, "AoSoA lanes %d must be a power of two in [1, 1024]", lanes);
      if (stride < 1 || stride > (1 << 22)) return set_error(SK_ERR_INVALID, "AoSoA tile stride %lld invalid", (long long)stride);
      g = lcm64(g, lanes);
    }
  }
  int64_t in_rec = 0, out_rec = 0;  // x1000 to keep AoSoA fractions
  if (d.src_kind == SK_KIND_AOS) in_rec = d.src_stride * 1000;
  if (d.src_kind == SK_KIND_AOSOA) in_rec = d.src_stride * 1000 / d.src_lanes;
  if (d.dst_kind == SK_KIND_AOS) out_rec = d.dst_stride * 1000;
  if (d.dst_kind == SK_KIND_AOSOA) out_rec = d.dst_stride * 1000 / d.dst_lanes;
  std::vector<uint8_t> cover;
  if (d.dst_kind != SK_KIND_PLANES) cover.assign(static_cast<size_t>(d.dst_stride), 0);
  for (int i = 0; i < d.nfields; ++i) {
    const sk_field& f = d.fields[i];
    const int sisz = dtype_size(f.src_type), disz = dtype_size(f.dst_type);
    if (!sisz || !disz) return set_error(SK_ERR_INVALID, "field %d: bad type codes %d -> %d", i, f.src_type, f.dst_type);
    if (!cast_supported(f.src_type, f.dst_type))
      return set_error(SK_ERR_UNSUPPORTED, "field %d: cast %d -> %d is not supported (float->int)", i, f.src_type,
                       f.dst_type);
    // source geometry
    if (d.src_kind == SK_KIND_PLANES) {
      if (!f.src_plane && d.n) return set_error(SK_ERR_INVALID, "field %d: null src plane", i);
      in_rec += sisz * 1000;
    } else {
      const int64_t span = d.src_kind == SK_KIND_AOS ? sisz : static_cast<int64_t>(sisz) * d.src_lanes;
      if (f.src_off < 0 || f.src_off + span > d.src_stride)
        return set_error(SK_ERR_RANGE, "field %d: source bytes [%lld, %lld) outside stride %lld", i,
                         (long long)f.src_off, (long long)(f.src_off + span), (long long)d.src_stride);
    }
    if (d.dst_kind == SK_KIND_PLANES) {
      if (!f.dst_plane && d.n) return set_error(SK_ERR_INVALID, "field %d: null dst plane", i);
      out_rec += disz * 1000;
    } else {
      const int64_t span = d.dst_kind == SK_KIND_AOS ? disz : static_cast<int64_t>(disz) * d.dst_lanes;
      if (f.dst_off < 0 || f.dst_off + span > d.dst_stride)
        return set_error(SK_ERR_RANGE, "field %d: destination bytes [%lld, %lld) outside stride %lld", i,
                         (long long)f.dst_off, (long long)(f.dst_off + span), (long long)d.dst_stride);
      for (int64_t b = f.dst_off; b < f.dst_off + span; ++b) {
        if (cover[b]) return set_error(SK_ERR_INVALID, "field %d overlaps another destination field", i);
        cover[b] = 1;
      }
    }
  }
  *granule = g;
  *in_rec_x1000 = in_rec;
  *out_rec_x1000 = out_rec;
  return SK_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Opt-in shared memory and resident CTAs per SM for a dynamic smem size,
// cached per device (these runtime queries cost microseconds per call, which
// matters for small conversions).
static int occupancy_for(int smem) {
  static std::mutex mu;
  static int max_set[64] = {0};
  static std::vector<std::pair<int, int>> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& e : cache[dev])
    if (e.first == smem) return e.second;
  if (smem > max_set[dev]) {
    cudaFuncSetAttribute(convert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    max_set[dev] = smem;
  }
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, convert_kernel, NT, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  cudaGetLastError();
  if (cache[dev].size() < 256) cache[dev].push_back({smem, per_sm});
  return per_sm;
}

// Tiling knobs; defaults are the measured best on B200 (profiles/), the
// environment overrides exist for sweeps (SK_TILE_BYTES, SK_STAGES, SK_CTAS,
// SK_CACHE_HINT).
struct Tunables {
  int tile_bytes = TILE_TARGET;
  int max_stages = MAX_STAGES;
  int ctas_per_sm = 4;
  int cache_hint = 1;
};

static int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  const int x = atoi(v);
  return x < lo ? lo : (x > hi ? hi : x);
}

static Tunables tunables() {
  Tunables t;
  t.tile_bytes = env_int("SK_TILE_BYTES", t.tile_bytes, 1024, 65536);
  t.max_stages = env_int("SK_STAGES", t.max_stages, 1, 8);
  t.ctas_per_sm = env_int("SK_CTAS", t.ctas_per_sm, 1, 8);
  t.cache_hint = env_int("SK_CACHE_HINT", t.cache_hint, 0, 2);
  return t;
}

// Build the kernel plan. `in_bulk_ok`/`out_bulk_ok` veto bulk copies (peer or
// host pointers); alignment is checked here.
int make_plan(const sk_conv_desc& d, const DeviceState& ds, bool in_bulk_ok, bool out_bulk_ok, int epi, Plan* out,
              int* grid) {
  int64_t g, in_rec, out_rec;
  int rc = validate(d, &g, &in_rec, &out_rec);
  if (rc) return rc;
  Plan& P = *out;
  memset(&P, 0, sizeof(P));
  P.n = d.n;
  P.src_kind = d.src_kind;
  P.dst_kind = d.dst_kind;
  P.src_stride = static_cast<int32_t>(d.src_stride);
  P.dst_stride = static_cast<int32_t>(d.dst_stride);
  P.src_lshift = d.src_kind == SK_KIND_AOSOA ? log2_exact(d.src_lanes) : 0;
  P.dst_lshift = d.dst_kind == SK_KIND_AOSOA ? log2_exact(d.dst_lanes) : 0;
  P.nfields = d.nfields;
  P.src = static_cast<const uint8_t*>(d.src);
  P.dst = static_cast<uint8_t*>(d.dst);
  P.epi = epi;
  if (epi == EPI_SENSOR) out_rec += 4000;

  // records per tile: multiple of the granule, in + out bytes of a tile ~tile_bytes
  // (the sweeps in profiles/ put the optimum at a fixed smem footprint per tile,
  // whatever the in/out split: 24+24 KB for Obj8, ~40+10 KB for a 60->16 B AoSoA)
  const Tunables tun = tunables();
  P.cache_hint = tun.cache_hint;
  const int64_t rec = std::max<int64_t>(std::max(in_rec, out_rec), 1000);
  const int64_t rec_sum = std::max<int64_t>(in_rec + out_rec, 1000);
  int64_t R = (static_cast<int64_t>(tun.tile_bytes) * 1000 / rec_sum) / g * g;
  R = std::max<int64_t>(R, g);
  R = std::min<int64_t>(R, std::max<int64_t>(g, 4096));
  P.R = static_cast<int32_t>(R);
  P.ntiles = d.n ? (d.n + R - 1) / R : 0;

  // in tile layout
  int32_t cur = 0;
  for (int i = 0; i < d.nfields; ++i) {
    const sk_field& f = d.fields[i];
    FieldPlan& F = P.f[i];
    F.st = static_cast<uint8_t>(f.src_type);
    F.dt = static_cast<uint8_t>(f.dst_type);
    F.sisz = static_cast<uint8_t>(dtype_size(f.src_type));
    F.disz = static_cast<uint8_t>(dtype_size(f.dst_type));
    F.splane = static_cast<const uint8_t*>(f.src_plane);
    F.dplane = static_cast<uint8_t*>(f.dst_plane);
    if (d.src_kind == SK_KIND_PLANES) {
      F.sloc = cur;
      cur = align_up(cur + static_cast<int32_t>(R) * F.sisz, 16) + 16;  // 16 B stagger between segments
    } else {
      F.sloc = static_cast<int32_t>(f.src_off);
    }
  }
  if (d.src_kind == SK_KIND_AOS) P.in_tile_bytes = static_cast<int32_t>(R * d.src_stride);
  else if (d.src_kind == SK_KIND_AOSOA) P.in_tile_bytes = static_cast<int32_t>((R >> P.src_lshift) * d.src_stride);
  else P.in_tile_bytes = cur;  // includes stagger; bulk expect_tx uses the exact sum below
  int32_t in_exact = P.in_tile_bytes;
  if (d.src_kind == SK_KIND_PLANES) {
    in_exact = 0;
    for (int i = 0; i < d.nfields; ++i) in_exact += static_cast<int32_t>(R) * P.f[i].sisz;
  }
  // out tile layout
  cur = 0;
  for (int i = 0; i < d.nfields; ++i) {
    FieldPlan& F = P.f[i];
    if (d.dst_kind == SK_KIND_PLANES) {
      F.dloc = cur;
      cur = align_up(cur + static_cast<int32_t>(R) * F.disz, 16) + 16;
    } else {
      F.dloc = static_cast<int32_t>(d.fields[i].dst_off);
    }
  }
  int32_t out_bytes;
  if (d.dst_kind == SK_KIND_AOS) out_bytes = static_cast<int32_t>(R * d.dst_stride);
  else if (d.dst_kind == SK_KIND_AOSOA) out_bytes = static_cast<int32_t>((R >> P.dst_lshift) * d.dst_stride);
  else out_bytes = cur;
  if (epi == EPI_SENSOR) {
    P.extra_loc = align_up(out_bytes, 16);
    out_bytes = P.extra_loc + static_cast<int32_t>(R) * 4;
  }
  P.out_tile_bytes = align_up(out_bytes, 16);

  // branch-free element addressing + per-field element-path class
  auto side_geo = [](int kind, int64_t stride, int32_t* A, int32_t* msk, int lanes) {
    if (kind == SK_KIND_AOS) { *A = static_cast<int32_t>(stride); *msk = 0; }
    else if (kind == SK_KIND_PLANES) { *A = 0; *msk = -1; }
    else { *A = static_cast<int32_t>(stride); *msk = lanes - 1; }
  };
  side_geo(d.src_kind, d.src_stride, &P.src_A, &P.src_msk, d.src_lanes);
  side_geo(d.dst_kind, d.dst_stride, &P.dst_A, &P.dst_msk, d.dst_lanes);
  auto always_aligned = [](int kind, int64_t stride, int32_t loc, int isz) {
    if (kind == SK_KIND_PLANES) return true;  // segments are 16-byte aligned
    return stride % isz == 0 && loc % isz == 0;
  };
  for (int i = 0; i < d.nfields; ++i) {
    FieldPlan& F = P.f[i];
    F.sal = always_aligned(d.src_kind, d.src_stride, F.sloc, F.sisz);
    F.dal = always_aligned(d.dst_kind, d.dst_stride, F.dloc, F.disz);
    F.op = F.st == F.dt ? ELEM_MOVE
                        : (F.st == SK_F64 && F.dt == SK_F32) ? ELEM_F64_F32
                        : (F.st == SK_F32 && F.dt == SK_F64) ? ELEM_F32_F64 : ELEM_GENERIC;
  }

  // word moves
  P.mode = MODE_ELEM;
  if (d.src_kind == SK_KIND_AOS && d.dst_kind == SK_KIND_PLANES && d.src_stride % 4 == 0 &&
      d.src_stride <= 4 * MAX_WORDS) {
    P.mode = MODE_WORD_A2P;
    P.words_per_rec = static_cast<int32_t>(d.src_stride / 4);
  } else if (d.src_kind == SK_KIND_PLANES && d.dst_kind == SK_KIND_AOS && d.dst_stride % 4 == 0 &&
             d.dst_stride <= 4 * MAX_WORDS) {
    P.mode = MODE_WORD_P2A;
    P.words_per_rec = static_cast<int32_t>(d.dst_stride / 4);
  }
  if (P.mode != MODE_ELEM) {
    for (int q = 0; q < MAX_WORDS; ++q) P.wtab[q] = -1;
    int nword = 0;
    for (int i = 0; i < d.nfields; ++i) {
      FieldPlan& F = P.f[i];
      const int64_t aos_off = P.mode == MODE_WORD_A2P ? d.fields[i].src_off : d.fields[i].dst_off;
      const int isz = F.sisz;
      if (F.st != F.dt || (isz != 4 && isz != 8) || (aos_off & 3)) continue;
      // a word of the AoS record read by two fields cannot be a single move
      bool clash = false;
      for (int m = 0; m < isz / 4; ++m)
        if (P.wtab[aos_off / 4 + m] != -1) clash = true;
      if (clash) continue;
      const int32_t seg = P.mode == MODE_WORD_A2P ? F.dloc : F.sloc;
      for (int m = 0; m < isz / 4; ++m) P.wtab[aos_off / 4 + m] = ((seg + 4 * m) << 4) | isz;
      F.wordable = 1;
      ++nword;
    }
    if (!nword) P.mode = MODE_ELEM;
  }
  P.n_elem = 0;
  for (int i = 0; i < d.nfields; ++i)
    if (!P.f[i].wordable) P.elem_idx[P.n_elem++] = static_cast<uint8_t>(i);
  // at least two work items per warp so a slow field does not idle the others
  P.elem_chunks = P.n_elem ? std::max(1, (2 * (NT / 32) + P.n_elem - 1) / P.n_elem) : 1;

  // destination bytes covered by no field are written as zero
  if (d.dst_kind != SK_KIND_PLANES) {
    int64_t covered = 0;
    for (int i = 0; i < d.nfields; ++i)
      covered += d.dst_kind == SK_KIND_AOS ? P.f[i].disz : static_cast<int64_t>(P.f[i].disz) * d.dst_lanes;
    P.zero_out = covered != d.dst_stride;
  }

  // bulk eligibility: 16-byte aligned bases, strides and sizes
  bool bin = in_bulk_ok;
  if (d.src_kind == SK_KIND_PLANES) {
    for (int i = 0; i < d.nfields; ++i) bin = bin && aligned16(P.f[i].splane);
  } else {
    bin = bin && aligned16(d.src) && (d.src_kind == SK_KIND_AOS || d.src_stride % 16 == 0);
  }
  bool bout = out_bulk_ok;
  if (d.dst_kind == SK_KIND_PLANES) {
    for (int i = 0; i < d.nfields; ++i) bout = bout && aligned16(P.f[i].dplane);
  } else {
    bout = bout && aligned16(d.dst) && (d.dst_kind == SK_KIND_AOS || d.dst_stride % 16 == 0);
  }
  P.bulk_in = bin;
  P.bulk_out = bout;
  P.in_tile_bytes = in_exact;  // bytes a full tile brings in (tx count)
  // in-tile allocation span (segments incl. stagger)
  int32_t in_span = in_exact;
  if (d.src_kind == SK_KIND_PLANES) {
    in_span = 0;
    for (int i = 0; i < d.nfields; ++i)
      in_span = std::max(in_span, P.f[i].sloc + static_cast<int32_t>(R) * P.f[i].sisz);
  }
  P.in_stage_stride = align_up(in_span + 16, 128);
  P.out_stage_stride = align_up(P.out_tile_bytes + 16, 128);

  // shared memory budget: `ctas` CTAs per SM (228 KB per SM, 1 KB reserved per CTA)
  const int32_t fixed = 128 /*barriers*/ + (P.mode != MODE_ELEM ? 4 * MAX_WORDS : 0);
  const int32_t optin = ds.max_smem_optin > 0 ? ds.max_smem_optin : 232448;
  int ctas = tun.ctas_per_sm;
  int stages = 0;
  for (; ctas >= 1; --ctas) {
    const int32_t budget = std::min(optin, 233472 / ctas - 1024);
    stages = (budget - fixed - 2 * P.out_stage_stride) / std::max(P.in_stage_stride, 1);
    if (stages >= 2 || ctas == 1) break;
  }
  if (stages < 1)
    return set_error(SK_ERR_UNSUPPORTED, "records too large for the shared-memory tile (%lld B)",
                     (long long)rec / 1000);
  P.stages = std::min(stages, tun.max_stages);
  P.smem_bar_off = 0;
  P.smem_tab_off = 128;
  P.smem_in_off = align_up(fixed, 128);
  P.smem_out_off = P.smem_in_off + P.stages * P.in_stage_stride;
  P.smem_total = P.smem_out_off + 2 * P.out_stage_stride;

  const int per_sm = occupancy_for(P.smem_total);
  const int64_t want = static_cast<int64_t>(ds.sm_count) * std::min(per_sm, std::max(ctas, 1));
  *grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, P.ntiles)));
  return SK_OK;
}

int launch(const Plan& P, int grid, cudaStream_t s) {
  if (P.ntiles == 0) return SK_OK;
  convert_kernel<<<grid, NT, P.smem_total, s>>>(P);
  SK_TRY(cudaGetLastError());
  return SK_OK;
}

// ---------------------------------------------------------------------------------
// placement discovery + the host<->device pipeline

enum Loc { LOC_DEVICE = 0, LOC_PEER = 1, LOC_HOST = 2 };

static int classify(const void* p, int device, int* loc, int* owner) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes");
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    *owner = a.device;
    *loc = a.device == device ? LOC_DEVICE : LOC_PEER;
  } else {
    *owner = -1;
    *loc = LOC_HOST;
  }
  return SK_OK;
}

static int side_location(const sk_conv_desc& d, bool dst, int device, int* loc) {
  const int kind = dst ? d.dst_kind : d.src_kind;
  int l0 = -1, owner = -1;
  auto visit = [&](const void* p) -> int {
    if (!p) return SK_OK;
    int l, o;
    int rc = classify(p, device, &l, &o);
    if (rc) return rc;
    if (l0 == -1) { l0 = l; owner = o; return SK_OK; }
    if (l != l0 || o != owner)
      return set_error(SK_ERR_INVALID, "%s fields live in different memory placements", dst ? "destination" : "source");
    return SK_OK;
  };
  if (kind == SK_KIND_PLANES) {
    for (int i = 0; i < d.nfields; ++i) {
      int rc = visit(dst ? d.fields[i].dst_plane : d.fields[i].src_plane);
      if (rc) return rc;
    }
  } else {
    int rc = visit(dst ? d.dst : d.src);
    if (rc) return rc;
  }
  if (l0 == LOC_PEER) {
    int rc = sk_peer_enable(device, owner);
    if (rc) return rc;
  }
  *loc = l0 < 0 ? LOC_DEVICE : l0;
  return SK_OK;
}

// bytes of `rows` records of one side, and per-field chunk offsets in staging
static int64_t side_bytes(const sk_conv_desc& d, bool dst, int64_t rows, std::vector<int64_t>* field_off) {
  const int kind = dst ? d.dst_kind : d.src_kind;
  const int64_t stride = dst ? d.dst_stride : d.src_stride;
  const int lanes = dst ? d.dst_lanes : d.src_lanes;
  if (kind == SK_KIND_AOS) return rows * stride;
  if (kind == SK_KIND_AOSOA) return (rows + lanes - 1) / lanes * stride;
  int64_t cur = 0;
  if (field_off) field_off->assign(d.nfields, 0);
  for (int i = 0; i < d.nfields; ++i) {
    if (field_off) (*field_off)[i] = cur;
    const int isz = dtype_size(dst ? d.fields[i].dst_type : d.fields[i].src_type);
    cur = (cur + rows * isz + 255) / 256 * 256;
  }
  return cur;
}

// shift a side of the descriptor to start at record r0 (r0 is a granule multiple)
static void offset_side(sk_conv_desc* d, bool dst, int64_t r0) {
  const int kind = dst ? d->dst_kind : d->src_kind;
  if (kind == SK_KIND_PLANES) {
    for (int i = 0; i < d->nfields; ++i) {
      sk_field& f = d->fields[i];
      if (dst) f.dst_plane = static_cast<uint8_t*>(f.dst_plane) + r0 * dtype_size(f.dst_type);
      else f.src_plane = static_cast<const uint8_t*>(f.src_plane) + r0 * dtype_size(f.src_type);
    }
    return;
  }
  const int64_t stride = dst ? d->dst_stride : d->src_stride;
  const int lanes = dst ? d->dst_lanes : d->src_lanes;
  const int64_t off = kind == SK_KIND_AOS ? r0 * stride : r0 / lanes * stride;
  if (dst) d->dst = static_cast<uint8_t*>(d->dst) + off;
  else d->src = static_cast<const uint8_t*>(d->src) + off;
}

// point a side of the descriptor at a staging chunk
static void stage_side(sk_conv_desc* d, bool dst, uint8_t* base, const std::vector<int64_t>& foff) {
  const int kind = dst ? d->dst_kind : d->src_kind;
  if (kind == SK_KIND_PLANES) {
    for (int i = 0; i < d->nfields; ++i) {
      if (dst) d->fields[i].dst_plane = base + foff[i];
      else d->fields[i].src_plane = base + foff[i];
    }
  } else if (dst) {
    d->dst = base;
  } else {
    d->src = base;
  }
}

// copy `rows` records of one side between host memory (at record r0 of the
// original descriptor) and a staging chunk
static int copy_side(const sk_conv_desc& orig, bool dst, int64_t r0, int64_t rows, uint8_t* stage,
                     const std::vector<int64_t>& foff, bool to_device, cudaStream_t s) {
  const int kind = dst ? orig.dst_kind : orig.src_kind;
  if (kind == SK_KIND_PLANES) {
    for (int i = 0; i < orig.nfields; ++i) {
      const sk_field& f = orig.fields[i];
      const int isz = dtype_size(dst ? f.dst_type : f.src_type);
      uint8_t* host = static_cast<uint8_t*>(const_cast<void*>(dst ? f.dst_plane : f.src_plane)) + r0 * isz;
      if (to_device) SK_TRY(cudaMemcpyAsync(stage + foff[i], host, rows * isz, cudaMemcpyHostToDevice, s));
      else SK_TRY(cudaMemcpyAsync(host, stage + foff[i], rows * isz, cudaMemcpyDeviceToHost, s));
    }
    return SK_OK;
  }
  const int64_t stride = dst ? orig.dst_stride : orig.src_stride;
  const int lanes = dst ? orig.dst_lanes : orig.src_lanes;
  const int64_t off = kind == SK_KIND_AOS ? r0 * stride : r0 / lanes * stride;
  const int64_t bytes = side_bytes(orig, dst, rows, nullptr);
  uint8_t* host = static_cast<uint8_t*>(const_cast<void*>(dst ? orig.dst : orig.src)) + off;
  if (to_device) SK_TRY(cudaMemcpyAsync(stage, host, bytes, cudaMemcpyHostToDevice, s));
  else SK_TRY(cudaMemcpyAsync(host, stage, bytes, cudaMemcpyDeviceToHost, s));
  return SK_OK;
}

constexpr int64_t CHUNK_TARGET = 32ll << 20;  // bytes of the larger side per pipeline chunk
constexpr int NSLOT = 2;

int run(const sk_conv_desc& d, int device, cudaStream_t s, int epi, float* extra, const int* epi_fields) {
  DeviceState* ds = nullptr;
  int rc = device_state(device, &ds);
  if (rc) return rc;
  int64_t g, in_rec, out_rec;
  rc = validate(d, &g, &in_rec, &out_rec);
  if (rc) return rc;
  if (d.n == 0) return SK_OK;
  int src_loc, dst_loc;
  rc = side_location(d, false, device, &src_loc);
  if (rc) return rc;
  rc = side_location(d, true, device, &dst_loc);
  if (rc) return rc;

  auto plan_and_launch = [&](const sk_conv_desc& dk, float* extra_k, cudaStream_t st) -> int {
    Plan P;
    int grid = 1;
    int r = make_plan(dk, *ds, src_loc != LOC_PEER, dst_loc != LOC_PEER, epi, &P, &grid);
    if (r) return r;
    if (epi == EPI_SENSOR) {
      for (int k = 0; k < 7; ++k) P.epi_seg[k] = P.f[epi_fields[k]].dloc;
      P.extra_plane = reinterpret_cast<uint8_t*>(extra_k);
    }
    return launch(P, grid, st);
  };

  if (src_loc != LOC_HOST && dst_loc != LOC_HOST) return plan_and_launch(d, extra, s);

  // staged pipeline: chunk k: [H2D src chunk] -> convert -> [D2H dst chunk]
  const bool sh = src_loc == LOC_HOST, dh = dst_loc == LOC_HOST;
  const int64_t per = std::max<int64_t>(std::max(sh ? in_rec : 0, dh ? out_rec : 0), 1000);
  int64_t C = (CHUNK_TARGET * 1000 / per) / g * g;
  C = std::max<int64_t>(C, g);
  C = std::min<int64_t>(C, (d.n + g - 1) / g * g);
  std::vector<int64_t> in_foff, out_foff;
  const int64_t in_slot = sh ? (side_bytes(d, false, C, &in_foff) + 255) / 256 * 256 : 0;
  const int64_t out_slot = dh ? (side_bytes(d, true, C, &out_foff) + 255) / 256 * 256 : 0;
  const int64_t extra_slot = (dh && epi == EPI_SENSOR) ? (C * 4 + 255) / 256 * 256 : 0;
  const size_t need = static_cast<size_t>(NSLOT * (in_slot + out_slot + extra_slot));
  if (ds->staging_bytes < need) {
    SK_TRY(cudaStreamSynchronize(ds->stream));
    SK_TRY(cudaStreamSynchronize(ds->copy_in));
    SK_TRY(cudaStreamSynchronize(ds->copy_out));
    if (ds->staging) SK_TRY(cudaFree(ds->staging));
    ds->staging = nullptr;
    ds->staging_bytes = 0;
    SK_TRY(cudaMalloc(&ds->staging, need));
    ds->staging_bytes = need;
  }
  uint8_t* base = static_cast<uint8_t*>(ds->staging);
  cudaEvent_t start, in_ready[NSLOT], in_free[NSLOT], out_ready[NSLOT], out_free[NSLOT];
  SK_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  for (int k = 0; k < NSLOT; ++k) {
    SK_TRY(cudaEventCreateWithFlags(&in_ready[k], cudaEventDisableTiming));
    SK_TRY(cudaEventCreateWithFlags(&in_free[k], cudaEventDisableTiming));
    SK_TRY(cudaEventCreateWithFlags(&out_ready[k], cudaEventDisableTiming));
    SK_TRY(cudaEventCreateWithFlags(&out_free[k], cudaEventDisableTiming));
  }
  // the helper streams start after everything already queued on s
  SK_TRY(cudaEventRecord(start, s));
  SK_TRY(cudaStreamWaitEvent(ds->copy_in, start, 0));
  SK_TRY(cudaStreamWaitEvent(ds->copy_out, start, 0));
  const int64_t nchunks = (d.n + C - 1) / C;
  for (int64_t k = 0; k < nchunks; ++k) {
    const int slot = static_cast<int>(k % NSLOT);
    const int64_t r0 = k * C;
    const int64_t rows = std::min(C, d.n - r0);
    uint8_t* sin = base + slot * (in_slot + out_slot + extra_slot);
    uint8_t* sout = sin + in_slot;
    float* sextra = reinterpret_cast<float*>(sout + out_slot);
    sk_conv_desc dk = d;
    dk.n = rows;
    if (sh) {
      if (k >= NSLOT) SK_TRY(cudaStreamWaitEvent(ds->copy_in, in_free[slot], 0));
      rc = copy_side(d, false, r0, rows, sin, in_foff, true, ds->copy_in);
      if (rc) return rc;
      SK_TRY(cudaEventRecord(in_ready[slot], ds->copy_in));
      SK_TRY(cudaStreamWaitEvent(s, in_ready[slot], 0));
      stage_side(&dk, false, sin, in_foff);
    } else {
      offset_side(&dk, false, r0);
    }
    float* ek = extra ? extra + r0 : nullptr;
    if (dh) {
      if (k >= NSLOT) SK_TRY(cudaStreamWaitEvent(s, out_free[slot], 0));
      stage_side(&dk, true, sout, out_foff);
      if (epi == EPI_SENSOR) ek = sextra;
    } else {
      offset_side(&dk, true, r0);
    }
    rc = plan_and_launch(dk, ek, s);
    if (rc) return rc;
    if (sh) SK_TRY(cudaEventRecord(in_free[slot], s));
    if (dh) {
      SK_TRY(cudaEventRecord(out_ready[slot], s));
      SK_TRY(cudaStreamWaitEvent(ds->copy_out, out_ready[slot], 0));
      rc = copy_side(d, true, r0, rows, sout, out_foff, false, ds->copy_out);
      if (rc) return rc;
      if (epi == EPI_SENSOR && extra)
        SK_TRY(cudaMemcpyAsync(extra + r0, sextra, rows * 4, cudaMemcpyDefault, ds->copy_out));
      SK_TRY(cudaEventRecord(out_free[slot], ds->copy_out));
    }
  }
  if (dh) SK_TRY(cudaStreamWaitEvent(s, out_free[(nchunks - 1) % NSLOT], 0));
  cudaEventDestroy(start);
  for (int k = 0; k < NSLOT; ++k) {
    cudaEventDestroy(in_ready[k]);
    cudaEventDestroy(in_free[k]);
    cudaEventDestroy(out_ready[k]);
    cudaEventDestroy(out_free[k]);
  }
  return SK_OK;
}

}  // namespace conv
}  // namespace sk

using namespace sk;

extern "C" {

int sk_convert(const sk_conv_desc* desc, int device, uintptr_t stream) {
  if (!desc) return set_error(SK_ERR_INVALID, "null descriptor");
  DeviceState* ds = nullptr;
  int rc = device_state(device, &ds);
  if (rc) return rc;
  return conv::run(*desc, device, resolve_stream(device, stream), conv::EPI_NONE, nullptr, nullptr);
}

int sk_convert_plan(const sk_conv_desc* desc, int device, int* records_per_tile, int* stages, int* mode,
                    size_t* smem_bytes, int* grid) {
  if (!desc) return set_error(SK_ERR_INVALID, "null descriptor");
  DeviceState* ds = nullptr;
  int rc = device_state(device, &ds);
  if (rc) return rc;
  conv::Plan P;
  int g = 0;
  rc = conv::make_plan(*desc, *ds, true, true, conv::EPI_NONE, &P, &g);
  if (rc) return rc;
  if (records_per_tile) *records_per_tile = P.R;
  if (stages) *stages = P.stages;
  if (mode) *mode = P.mode | (P.bulk_in ? 4 : 0) | (P.bulk_out ? 8 : 0);
  if (smem_bytes) *smem_bytes = static_cast<size_t>(P.smem_total);
  if (grid) *grid = g;
  return SK_OK;
}

int sk_sensor_convert_calibrate(const sk_conv_desc* desc, int f_counts, int f_energy, int f_noisy, int f_a, int f_b,
                                int f_na, int f_nb, float* noise, int device, uintptr_t stream) {
  if (!desc) return set_error(SK_ERR_INVALID, "null descriptor");
  if (desc->dst_kind != SK_KIND_PLANES)
    return set_error(SK_ERR_UNSUPPORTED, "fused sensor kernel writes per_field planes only");
  const int fi[7] = {f_counts, f_energy, f_noisy, f_a, f_b, f_na, f_nb};
  const int want[7] = {SK_U64, SK_F32, SK_BOOL, SK_F32, SK_F32, SK_F32, SK_F32};
  for (int k = 0; k < 7; ++k) {
    if (fi[k] < 0 || fi[k] >= desc->nfields) return set_error(SK_ERR_INVALID, "sensor field index %d out of range", fi[k]);
    if (desc->fields[fi[k]].dst_type != want[k] || desc->fields[fi[k]].src_type != want[k])
      return set_error(SK_ERR_INVALID, "sensor field %d has type %d, expected %d", fi[k], desc->fields[fi[k]].dst_type,
                       want[k]);
  }
  if (!noise && desc->n) return set_error(SK_ERR_INVALID, "null noise plane");
  DeviceState* ds = nullptr;
  int rc = device_state(device, &ds);
  if (rc) return rc;
  return conv::run(*desc, device, resolve_stream(device, stream), conv::EPI_SENSOR, noise, fi);
}

}  // extern "C"
