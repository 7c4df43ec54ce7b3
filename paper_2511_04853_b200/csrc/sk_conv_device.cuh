// The conversion kernel framework (persistent CTA, TMA bulk ring, in-smem
// transposition, bulk stores). Compiled ahead of time by sk_convert.cu and,
// as source text, by NVRTC for record-signature-specialised transforms
// (sk_rtc.cu) -- keep it free of host-only headers.
#pragma once

#include "sk_device.cuh"

namespace sk {
namespace conv {

constexpr int NT = 256;
constexpr int MAX_WORDS = 256;     // word table -> AoS strides up to 1 KiB use word moves
constexpr int TILE_TARGET = 49152; // in+out bytes per tile (sweep: profiles/r01_sweep.md)
constexpr int MAX_STAGES = 4;
constexpr int MAX_SUBWORD = 16;    // AoS words made of 1-/2-byte fields the word path splits / assembles

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
  int32_t wtab[MAX_WORDS];  // (segment byte base << 4) | element size ; -1 = not a word-moved word;
                            // -2 - k = sub-word slot k of btab
  // sub-word slots: a word of the AoS record holding 1-/2-byte fields, moved as
  // one word and split (A2P) / assembled (P2A); parts (base << 4) | (size << 2) | byte, -1 unused
  int32_t btab[MAX_SUBWORD][4];
  int32_t issue_lanes;           // 32: warp 0 issues the bulk segment copies in parallel; 1: thread 0 alone
  int32_t nsub;                  // sub-word slots in use and the record word each one is
  int32_t bword[MAX_SUBWORD];
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

// issued by P.issue_lanes threads (thread 0 alone, or the 32 lanes of warp 0):
// lane 0 arms the barrier, then every lane sends its share of the segments
template <int NL>
static __device__ __forceinline__ void issue_bulk_load(const Plan& P, int64_t t, uint8_t* in, uint64_t* bar,
                                                       uint64_t pol) {
  const int lane = NL > 1 ? (threadIdx.x & 31) : 0;
  constexpr int nl = NL;
  const int64_t r0 = t * P.R;
  if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(P.in_tile_bytes));
  if (nl > 1) __syncwarp();
  if (P.src_kind == SK_KIND_PLANES) {
    for (int i = lane; i < P.nfields; i += nl) {
      const FieldPlan& F = P.f[i];
      g2s(P, in + F.sloc, F.splane + r0 * F.sisz, static_cast<uint32_t>(P.R * F.sisz), bar, pol);
    }
  } else if (lane == 0) {
    const int64_t off = P.src_kind == SK_KIND_AOS ? r0 * P.src_stride : (r0 >> P.src_lshift) * P.src_stride;
    g2s(P, in, P.src + off, static_cast<uint32_t>(P.in_tile_bytes), bar, pol);
  }
}

static __device__ void coop_load(const Plan& P, int64_t t, int rows, uint8_t* in) {
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

// same issuing threads; each commits its own bulk group
template <int NL>
static __device__ __forceinline__ void issue_bulk_store(const Plan& P, int64_t t, const uint8_t* out, uint64_t pol) {
  const int lane = NL > 1 ? (threadIdx.x & 31) : 0;
  constexpr int nl = NL;
  const int64_t r0 = t * P.R;
  if (P.dst_kind == SK_KIND_PLANES) {
    for (int i = lane; i < P.nfields; i += nl) {
      const FieldPlan& F = P.f[i];
      s2g(P, F.dplane + r0 * F.disz, out + F.dloc, static_cast<uint32_t>(P.R * F.disz), pol);
    }
  } else if (lane == 0) {
    const int64_t off = P.dst_kind == SK_KIND_AOS ? r0 * P.dst_stride : (r0 >> P.dst_lshift) * P.dst_stride;
    s2g(P, P.dst + off, out, static_cast<uint32_t>(P.out_tile_bytes), pol);
  }
  if (P.extra_plane && lane == nl - 1)
    s2g(P, P.extra_plane + r0 * 4, out + P.extra_loc, static_cast<uint32_t>(P.R * 4), pol);
  bulk_commit();
}

static __device__ void coop_store(const Plan& P, int64_t t, int rows, const uint8_t* out) {
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

static __device__ __noinline__ void elem_generic(const Plan& P, const FieldPlan& F, const uint8_t* in, uint8_t* out,
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
// sub-word slots of the word path

// plane-side byte address of element r of a field at `base`: a planes segment
// (GEO false) or an AoSoA tile block (GEO true)
template <bool GEO>
__device__ __forceinline__ int paddr(int base, int r, int isz, int lsh, int A, int msk) {
  if (GEO) return base + ((r >> lsh) * A) + ((r & msk) * isz);
  return base + r * isz;
}

template <bool GEO>
__device__ __forceinline__ void subword_put(uint32_t v, uint8_t* out, int r, int32_t p, int lsh, int A, int msk) {
  if (p < 0) return;
  const int base = p >> 4, sz = (p >> 2) & 3, sh = (p & 3) * 8;
  if (sz == 1) out[paddr<GEO>(base, r, 1, lsh, A, msk)] = static_cast<uint8_t>(v >> sh);
  else *reinterpret_cast<uint16_t*>(out + paddr<GEO>(base, r, 2, lsh, A, msk)) = static_cast<uint16_t>(v >> sh);
}

template <bool GEO>
__device__ __forceinline__ uint32_t subword_get(const uint8_t* in, int r, int32_t p, int lsh, int A, int msk) {
  if (p < 0) return 0u;
  const int base = p >> 4, sz = (p >> 2) & 3, sh = (p & 3) * 8;
  const uint32_t x =
      sz == 1 ? static_cast<uint32_t>(in[paddr<GEO>(base, r, 1, lsh, A, msk)])
              : static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(in + paddr<GEO>(base, r, 2, lsh, A, msk)));
  return x << sh;
}

// A2P: AoS words -> planes / AoSoA; P2A: planes / AoSoA -> AoS words.
template <bool A2P, bool GEO>
__device__ __forceinline__ void word_moves(const Plan& P, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                           int rows, const int32_t* __restrict__ wtab) {
  const int tid = threadIdx.x;
  const int lsh = A2P ? P.dst_lshift : P.src_lshift;
  const int A = A2P ? P.dst_A : P.src_A;
  const int msk = A2P ? P.dst_msk : P.src_msk;
  const int wpr = P.words_per_rec;
  const int total = rows * wpr;
  const int per = NT / wpr;   // records per pass when every active thread owns one word slot
  const int nta = per * wpr;  // active threads in that mode
  if (per >= 1 && 4 * nta >= 3 * NT) {
    // fixed word slot per thread (all NT threads when NT is a multiple of the
    // record's word count, else the largest multiple): every word this thread
    // touches sits at the same record slot q, so the table entry is loop
    // invariant and the loop is a pure, unrolled LDS->STS stream (4 loads in
    // flight per thread). Sub-word slots are left to their own pass.
    if (tid >= nta) return;
    int r = tid / wpr;
    const int q = tid - r * wpr;
    const int e = wtab[q];
    if (e < 0) return;
    const int base = e >> 4, isz = e & 15;
    int w = tid;
    if (A2P) {
      const uint32_t* in32 = reinterpret_cast<const uint32_t*>(in);
      for (; w + 3 * nta < total; w += 4 * nta, r += 4 * per) {
        const uint32_t v0 = in32[w], v1 = in32[w + nta], v2 = in32[w + 2 * nta], v3 = in32[w + 3 * nta];
        *reinterpret_cast<uint32_t*>(out + paddr<GEO>(base, r, isz, lsh, A, msk)) = v0;
        *reinterpret_cast<uint32_t*>(out + paddr<GEO>(base, r + per, isz, lsh, A, msk)) = v1;
        *reinterpret_cast<uint32_t*>(out + paddr<GEO>(base, r + 2 * per, isz, lsh, A, msk)) = v2;
        *reinterpret_cast<uint32_t*>(out + paddr<GEO>(base, r + 3 * per, isz, lsh, A, msk)) = v3;
      }
      for (; w < total; w += nta, r += per)
        *reinterpret_cast<uint32_t*>(out + paddr<GEO>(base, r, isz, lsh, A, msk)) = in32[w];
    } else {
      uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
      for (; w + 3 * nta < total; w += 4 * nta, r += 4 * per) {
        const uint32_t v0 = *reinterpret_cast<const uint32_t*>(in + paddr<GEO>(base, r, isz, lsh, A, msk));
        const uint32_t v1 = *reinterpret_cast<const uint32_t*>(in + paddr<GEO>(base, r + per, isz, lsh, A, msk));
        const uint32_t v2 = *reinterpret_cast<const uint32_t*>(in + paddr<GEO>(base, r + 2 * per, isz, lsh, A, msk));
        const uint32_t v3 = *reinterpret_cast<const uint32_t*>(in + paddr<GEO>(base, r + 3 * per, isz, lsh, A, msk));
        out32[w] = v0;
        out32[w + nta] = v1;
        out32[w + 2 * nta] = v2;
        out32[w + 3 * nta] = v3;
      }
      for (; w < total; w += nta, r += per)
        out32[w] = *reinterpret_cast<const uint32_t*>(in + paddr<GEO>(base, r, isz, lsh, A, msk));
    }
    return;
  }
  int r = tid / wpr;
  int q = tid - r * wpr;
  const int dr = NT / wpr;
  const int dq = NT - dr * wpr;
  for (int w = tid; w < total; w += NT) {
    const int e = wtab[q];
    if (e >= 0) {
      const int a = paddr<GEO>(e >> 4, r, e & 15, lsh, A, msk);
      if (A2P) *reinterpret_cast<uint32_t*>(out + a) = reinterpret_cast<const uint32_t*>(in)[w];
      else reinterpret_cast<uint32_t*>(out)[w] = *reinterpret_cast<const uint32_t*>(in + a);
    }
    q += dq;
    r += dr;
    if (q >= wpr) { q -= wpr; ++r; }
  }
}

// sub-word slots as their own pass over (record, slot) pairs on all threads
// (inside the fixed-slot loop only a few lanes per warp would own such a slot
// and every warp would run both loops back to back); uncovered bytes of an
// assembled word come out zero (the zero_out contract)
template <bool A2P, bool GEO>
__device__ __forceinline__ void subword_moves(const Plan& P, const uint8_t* __restrict__ in,
                                              uint8_t* __restrict__ out, int rows) {
  const int lsh = A2P ? P.dst_lshift : P.src_lshift;
  const int A = A2P ? P.dst_A : P.src_A;
  const int msk = A2P ? P.dst_msk : P.src_msk;
  const int wpr = P.words_per_rec, ns = P.nsub;
  const int pairs = rows * ns;
  for (int i = threadIdx.x; i < pairs; i += NT) {
    const int r = i / ns, k = i - r * ns;
    const int32_t* pt = P.btab[k];
    if (A2P) {
      const uint32_t v = reinterpret_cast<const uint32_t*>(in)[r * wpr + P.bword[k]];
#pragma unroll
      for (int j = 0; j < 4; ++j) subword_put<GEO>(v, out, r, pt[j], lsh, A, msk);
    } else {
      uint32_t v = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) v |= subword_get<GEO>(in, r, pt[j], lsh, A, msk);
      reinterpret_cast<uint32_t*>(out)[r * wpr + P.bword[k]] = v;
    }
  }
}

// ---------------------------------------------------------------------------------
// in-smem transposition

__device__ __forceinline__ void transform(const Plan& P, const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                          int rows, const int32_t* __restrict__ wtab) {
  const int tid = threadIdx.x;
  if (P.mode != MODE_ELEM) {
    // word moves; the non-AoS side is planes (segment + r * size) or AoSoA
    // tiles ((r >> lshift) * tile + (r & lanes-1) * size + block)
    const bool a2p = P.mode == MODE_WORD_A2P;
    const bool geo = a2p ? P.dst_kind == SK_KIND_AOSOA : P.src_kind == SK_KIND_AOSOA;
    if (a2p) {
      if (geo) word_moves<true, true>(P, in, out, rows, wtab);
      else word_moves<true, false>(P, in, out, rows, wtab);
    } else {
      if (geo) word_moves<false, true>(P, in, out, rows, wtab);
      else word_moves<false, false>(P, in, out, rows, wtab);
    }
  }
  if (P.nsub) {
    const bool a2p = P.mode == MODE_WORD_A2P;
    const bool geo = a2p ? P.dst_kind == SK_KIND_AOSOA : P.src_kind == SK_KIND_AOSOA;
    if (a2p) {
      if (geo) subword_moves<true, true>(P, in, out, rows);
      else subword_moves<true, false>(P, in, out, rows);
    } else {
      if (geo) subword_moves<false, true>(P, in, out, rows);
      else subword_moves<false, false>(P, in, out, rows);
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

// The transposition is a policy: GenericTransform (word + element paths driven
// by the Plan at run time) is compiled ahead of time; sk_rtc.cu generates
// record-signature-specialised transforms and compiles them with NVRTC.
struct GenericTransform {
  static constexpr bool kFusedEpilogue = false;
  __device__ __forceinline__ static void run(const Plan& P, const uint8_t* in, uint8_t* out, int rows,
                                             const int32_t* wtab) {
    transform(P, in, out, rows, wtab);
  }
};

// NL: threads that issue the bulk segment copies (1: thread 0; 32: warp 0), a
// compile-time choice so the single-issuer loop stays exactly a plain loop
template <class T, int NL>
__device__ __forceinline__ void convert_body(const Plan& P) {
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
  // back-to-back conversions: the next one's CTAs may start their prologue as ours retire; nothing global
  // (plan tables come from the kernel parameter) is touched before the previous kernel has completed
  pdl_allow_next();
  pdl_wait_prior();

  const int64_t first = blockIdx.x;
  const int64_t step = gridDim.x;
  if (first >= P.ntiles) return;
  const int64_t my_tiles = (P.ntiles - first + step - 1) / step;
  const uint64_t pol_in = policy_evict_first();
  const uint64_t pol_out = policy_evict_first();
  const int64_t last_tile = P.ntiles - 1;
  const int last_rows = static_cast<int>(P.n - last_tile * P.R);

  auto tile_bulk_in = [&](int64_t t) { return P.bulk_in && (t != last_tile || last_rows == P.R); };

  const bool issuer = tid < NL;
  if (issuer) {
    for (int s = 0; s < S && s < my_tiles; ++s) {
      const int64_t t = first + s * step;
      if (tile_bulk_in(t)) issue_bulk_load<NL>(P, t, in0 + s * P.in_stage_stride, &bars[s], pol_in);
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
    if (issuer) bulk_wait_read<1>();  // out[it&1] no longer read by the store of tile it-2 (every issuer)
    __syncthreads();
    if (P.zero_out || (rows < P.R && P.dst_kind == SK_KIND_AOSOA)) {
      uint32_t* o32 = reinterpret_cast<uint32_t*>(out);
      for (int i = tid; i < (P.out_tile_bytes >> 2); i += NT) o32[i] = 0;
      __syncthreads();
    }
    T::run(P, in, out, rows, wtab);
    if (P.epi == EPI_SENSOR && !T::kFusedEpilogue) {
      __syncthreads();
      sensor_epilogue(P, out, rows);
    }
    const bool bout = P.bulk_out && rows == P.R;
    if (bout) fence_proxy_async();
    __syncthreads();
    if (bout) {
      if (issuer) issue_bulk_store<NL>(P, t, out, pol_out);
    } else {
      coop_store(P, t, rows, out);
    }
    if (issuer && it + S < my_tiles) {
      const int64_t tn = first + (it + S) * step;
      if (tile_bulk_in(tn)) issue_bulk_load<NL>(P, tn, in, &bars[slot], pol_in);
    }
    if (++slot == S) slot = 0;
  }
  if (issuer) bulk_wait_all();
}

template <class T>
__global__ void __launch_bounds__(NT) convert_kernel_t(const __grid_constant__ Plan P) {
  if (P.issue_lanes == 32) convert_body<T, 32>(P);
  else convert_body<T, 1>(P);
}

}  // namespace conv
}  // namespace sk
