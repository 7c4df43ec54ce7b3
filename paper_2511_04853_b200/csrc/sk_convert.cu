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
#include "sk_conv_device.cuh"

namespace sk {
namespace conv {

#define convert_kernel convert_kernel_t<GenericTransform>

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
  int cache_hint = 0;  // evict_first hints: neutral at 1e9 records, costly when the data could stay in L2
  bool tile_set = false;  // SK_TILE_BYTES given: no per-signature tile choice
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
  t.tile_set = getenv("SK_TILE_BYTES") && *getenv("SK_TILE_BYTES");
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
  // many fields -> many small segment transfers per tile: smaller tiles, more CTAs per SM
  // (Particle, 18 fields: 0.68 -> 0.71 of the copy peak; <= 12 fields keep the larger tile)
  // the fused case study (30 B Sensor records -> planes + energy + noise) measured best at 40 KB tiles on real
  // events (tools/time_sensor.py: 123 us vs 128.5 us at 48 KB; 36 and 44 KB are worse -- the record-group
  // rounding of R matters more than the size)
  // odd-stride packed records into planes (Sensor, 30 B: record groups of 2) measured best with 64 KB tiles,
  // which the smem budget turns into one CTA per SM with 4 stages: 0.85 -> 0.93 of the copy peak
  // (tools/time_paths.py, tools/time_sensor.py); the reverse direction and even strides lose with them
  const bool odd_a2p = d.src_kind == SK_KIND_AOS && d.dst_kind == SK_KIND_PLANES && d.src_stride % 4 != 0;
  const int tile_bytes = tun.tile_set           ? tun.tile_bytes
                         : d.nfields > 12       ? 32768
                         : epi == EPI_SENSOR    ? 40960
                         : odd_a2p              ? 65536
                                                : tun.tile_bytes;
  int64_t R = (static_cast<int64_t>(tile_bytes) * 1000 / rec_sum) / g * g;
  R = std::max<int64_t>(R, g);
  R = std::min<int64_t>(R, std::max<int64_t>(g, 4096));
  // small problems: shrink the tile so the tiles fill whole rounds of the
  // persistent grid (1M Obj8 records = 2.25 target tiles per CTA would
  // otherwise run 3 rounds with the last one a quarter full)
  if (d.n > 0) {
    const int64_t est_grid = static_cast<int64_t>(ds.sm_count) * std::max(tun.ctas_per_sm, 1);
    const int64_t tiles0 = (d.n + R - 1) / R;
    const int64_t rounds = (tiles0 + est_grid - 1) / est_grid;
    if (rounds <= 16 && tiles0 > est_grid) {
      int64_t Rb = (d.n + est_grid * rounds - 1) / (est_grid * rounds);
      Rb = (Rb + g - 1) / g * g;
      if (Rb >= std::min<int64_t>(R, 256)) R = std::min(R, Rb);
    }
  }
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
  // The non-AoS side is planes, or (AoSoA -> AoS only) AoSoA tiles whose
  // stride keeps words aligned. AoS -> AoSoA stays on the element /
  // specialised path: AoSoA field blocks sit at multiples of the lane count x
  // size, so a record's word slots would all hit one smem bank (planes get a
  // 16-byte stagger per segment instead); measured 0.82 vs 0.96 specialised.
  P.mode = MODE_ELEM;
  const bool src_colw = d.src_kind == SK_KIND_PLANES || (d.src_kind == SK_KIND_AOSOA && d.src_stride % 4 == 0);
  const bool dst_colw = d.dst_kind == SK_KIND_PLANES;
  if (d.src_kind == SK_KIND_AOS && dst_colw && d.src_stride % 4 == 0 && d.src_stride <= 4 * MAX_WORDS) {
    P.mode = MODE_WORD_A2P;
    P.words_per_rec = static_cast<int32_t>(d.src_stride / 4);
  } else if (src_colw && d.dst_kind == SK_KIND_AOS && d.dst_stride % 4 == 0 && d.dst_stride <= 4 * MAX_WORDS) {
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
      const int32_t cloc = P.mode == MODE_WORD_A2P ? F.dloc : F.sloc;  // planes segment / AoSoA block
      if (F.st != F.dt || (isz != 4 && isz != 8) || (aos_off & 3) || (cloc & 3)) continue;
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
    // 1-/2-byte fields inside one AoS word: the word is moved once and split /
    // assembled in registers (Particle's noisy_count[4] u8 slots share a word)
    for (int q = 0; q < MAX_SUBWORD; ++q)
      for (int k = 0; k < 4; ++k) P.btab[q][k] = -1;
    int nsub = 0;
    for (int i = 0; i < d.nfields; ++i) {
      FieldPlan& F = P.f[i];
      const int64_t aos_off = P.mode == MODE_WORD_A2P ? d.fields[i].src_off : d.fields[i].dst_off;
      const int isz = F.sisz;
      const int32_t cloc = P.mode == MODE_WORD_A2P ? F.dloc : F.sloc;
      if (F.st != F.dt || (isz != 1 && isz != 2) || (aos_off & 3) + isz > 4 || (aos_off & (isz - 1)) ||
          (cloc & (isz - 1)))
        continue;
      int32_t& slot = P.wtab[aos_off / 4];
      if (slot >= 0) continue;
      if (slot == -1) {
        if (nsub == MAX_SUBWORD) continue;
        P.bword[nsub] = static_cast<int32_t>(aos_off / 4);
        slot = -2 - nsub++;
      }
      int32_t* parts = P.btab[-2 - slot];
      int k = 0;
      while (k < 4 && parts[k] != -1) ++k;
      if (k == 4) continue;
      const int32_t seg = P.mode == MODE_WORD_A2P ? F.dloc : F.sloc;
      parts[k] = (seg << 4) | (isz << 2) | static_cast<int32_t>(aos_off & 3);
      F.wordable = 1;
      ++nword;
    }
    P.nsub = nsub;
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
  // who issues the per-segment bulk copies, measured per path on B200
  // (profiles/r01_path_survey.md): the 32 lanes of warp 0 in parallel for
  // word-mode AoS <-> planes (Obj8 0.97 -> 0.99, Track/Particle planes->AoS
  // +3-5%); thread 0 alone for element-mode and AoSoA-side plans (Sensor
  // planes->AoS 0.94 -> 1.00, AoSoA->AoS 0.78 -> 0.84)
  {
    const bool word_planes = (P.mode == MODE_WORD_A2P && d.dst_kind == SK_KIND_PLANES) ||
                             (P.mode == MODE_WORD_P2A && d.src_kind == SK_KIND_PLANES);
    P.issue_lanes = word_planes ? 32 : 1;
    if (const char* e = getenv("SK_ISSUE_LANES")) P.issue_lanes = atoi(e) == 32 ? 32 : 1;
  }
  P.in_tile_bytes = in_exact;  // bytes a full tile brings in (tx count)
  // in-tile allocation span (segments incl. stagger)
  int32_t in_span = in_exact;
  if (d.src_kind == SK_KIND_PLANES) {
    in_span = 0;
    for (int i = 0; i < d.nfields; ++i)
      in_span = std::max(in_span, P.f[i].sloc + static_cast<int32_t>(R) * P.f[i].sisz);
  }
  // +128: a specialised transform may read/write one 4-byte-aligned record
  // group (<= 128 B) past the last record of a tail tile
  P.in_stage_stride = align_up(in_span + 128, 128);
  P.out_stage_stride = align_up(P.out_tile_bytes + 128, 128);

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

int launch_specialized(const sk_conv_desc& d, const Plan& P, const DeviceState& ds, const int* epi_fields,
                       cudaStream_t s, bool* launched);  // sk_rtc.cu

// programmatic stream serialization (PDL): a conversion queued right behind
// another kernel overlaps its launch and prologue with that kernel's tail
// (SK_PDL=0 turns it off)
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SK_PDL");
    return !(e && *e == '0');
  }();
  return on;
}

int launch(const Plan& P, int grid, cudaStream_t s) {
  if (P.ntiles == 0) return SK_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = P.smem_total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  SK_TRY(cudaLaunchKernelEx(&cfg, convert_kernel, P));
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

// Peer-device sides (NVLink through peer access or a CUDA IPC mapping) use the same TMA bulk copies as
// local HBM: cp.async.bulk takes any global address, and the copy engine of the SM pulls the remote
// lines over NVLink. SK_PEER_BULK=0 falls back to cooperative 16-byte loads/stores for peer sides.
static bool peer_bulk() {
  static const bool on = [] {
    const char* e = getenv("SK_PEER_BULK");
    return !(e && e[0] == '0');
  }();
  return on;
}

constexpr int64_t CHUNK_TARGET = 32ll << 20;  // bytes of the larger side per pipeline chunk
// (splitting one 5.7 MB event into 4 chunks measured slower: 0.151 -> 0.163 ms per event)
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
    int r = make_plan(dk, *ds, src_loc != LOC_PEER || peer_bulk(), dst_loc != LOC_PEER || peer_bulk(), epi, &P,
                      &grid);
    if (r) return r;
    if (epi == EPI_SENSOR) {
      for (int k = 0; k < 7; ++k) P.epi_seg[k] = P.f[epi_fields[k]].dloc;
      P.extra_plane = reinterpret_cast<uint8_t*>(extra_k);
    }
    bool spec = false;
    r = launch_specialized(dk, P, *ds, epi_fields, st, &spec);
    if (r || spec) return r;
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
    if (ds->staging) retire_or_free_staging(device, ds->staging);
    ds->staging = nullptr;
    ds->staging_bytes = 0;
    SK_TRY(cudaMalloc(&ds->staging, need));
    ds->staging_bytes = need;
  }
  uint8_t* base = static_cast<uint8_t*>(ds->staging);
  // the pipeline's events live with the device state (created once; every use is stream-ordered on the
  // device's own helper streams, like the staging buffer)
  static_assert(1 + 4 * NSLOT <= 9, "pipe_events");
  if (!ds->pipe_events[0])
    for (cudaEvent_t& e : ds->pipe_events) SK_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t start = ds->pipe_events[0];
  cudaEvent_t* in_ready = ds->pipe_events + 1;
  cudaEvent_t* in_free = in_ready + NSLOT;
  cudaEvent_t* out_ready = in_free + NSLOT;
  cudaEvent_t* out_free = out_ready + NSLOT;
  // the helper streams start after everything already queued on s
  SK_TRY(cudaEventRecord(start, s));
  // fork only the helper streams that get work (an idle fork would be an
  // unjoined stream inside a CUDA-graph capture)
  if (sh) SK_TRY(cudaStreamWaitEvent(ds->copy_in, start, 0));
  if (dh) SK_TRY(cudaStreamWaitEvent(ds->copy_out, start, 0));
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
