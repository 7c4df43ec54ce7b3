// Particle reconstruction on the B200.
//
// Reference: reconstruct_arrays (detector/reconstruct.py:53-136) walks seeds
// (ratio > 5) in descending energy / ascending index; an unconsumed seed takes
// the unconsumed ratio > 2 cells of its grid-clipped 5x5 window. The walk is
// sequential, but two seeds interact only when their windows overlap
// (Chebyshev distance <= 4). So the walk is a dependency graph: a seed's
// BLOCKERS are the candidates of higher priority within distance 4, and a
// seed may be processed as soon as every blocker is decided (processed, or
// consumed by another particle) -- with exactly the sequential walk's outcome,
// because every seed that could touch its window is then final and no seed of
// lower priority can touch it first (it would have this seed as a blocker).
//
//  1. tile_kernel: one CTA per 32x32 cell tile of an event stages energy and
//     noise of the tile plus a 4-cell halo in shared memory, marks the
//     candidates and writes each one's blocker list (offsets inside its 9x9
//     neighbourhood) -- the only 81-cell scan of the whole run.
//  2. pass_kernel, repeated: over the candidates still pending, one thread per
//     candidate walks its blocker list from where the last pass stopped; a
//     candidate whose blockers are all decided is processed by its warp right
//     away (window, contributors, sums), one that still waits goes to the next
//     pass's list. Processing publishes its cell flags with release ordering
//     and readers check them with acquire ordering, so a pass also resolves
//     chains whose blockers finish earlier in the same launch.
//
// Per-particle sums run in one thread in the reference's order (f64, no FMA,
// row-major contributors), so the attributes are bit-identical; particles are
// finally ordered by priority per event. The one approximation: the reference
// squares deviations with Python's `x ** 2` (glibc pow) and this kernel with
// x * x; profiles/r02_pow_check.md shows no f32 variance of the benchmark
// events differs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "sk_internal.cuh"


namespace sk {
namespace reco {

constexpr int NT = 256;
constexpr int MAXC = 25;  // contributors per particle (5x5 window)

// Programmatic dependent launch: every kernel of a run is launched with programmatic stream
// serialisation, waits for its predecessor's results (griddepcontrol.wait) before it reads anything and
// lets its successor be scheduled right away, so the launch gap between the many short kernels of a
// reconstruction overlaps the previous kernel's tail.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
static cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// per-cell flags
constexpr uint8_t PENDING = 1;   // a candidate not decided yet
constexpr uint8_t CONSUMED = 2;  // taken by a particle (a consumed candidate is decided)

struct Slot {  // one reconstructed particle, before ordering
  float energy, x, y, xvar, yvar;
  float sig[4], ec[4];
  uint8_t nc[4];
  int32_t nsens;
  int32_t event;   // -1: a seed found consumed at its turn (a hole)
  int64_t origin;  // seed flat index inside its event
  float key_e;     // priority: energy desc, then origin asc
};

// [1] ready seeds of this round [2] next round's list size [3] this round's list size
// [4] slots taken [5] CTAs finished in the current kernel [6] rounds that saw work [7] contributors
// [8] the tile pass's list sizes: candidates without blockers (low 32 bits), the others (high 32 bits)
constexpr int C_READY = 1, C_NEXT = 2, C_CUR = 3, C_SLOTS = 4, C_DONE = 5, C_PASSES = 6, C_CONTRIB = 7,
              C_TILE = 8, NCOUNTERS = 16;

struct Args {
  int64_t w, h, n;  // n = cells per event
  int nevents;
  const float* energy;
  const float* noise;
  const uint8_t* type;
  const uint8_t* noisy;
  uint8_t* flags;
  int64_t cand_cap;  // capacity of the lists
  int64_t* list[2];  // candidates (cells) still pending
  int64_t* ready;    // this round's ready seeds (cells)
  Slot* slots;
  uint64_t* contrib;  // MAXC per slot
  int64_t slot_cap;
  unsigned long long* counters;
  unsigned long long* event_count;
};

// ---- 1. tiles: flags, candidates and their blockers ------------------------------------

constexpr int TX = 56, TY = 40, HALO = 4, HX = TX + 2 * HALO, HY = TY + 2 * HALO;  // a halo tile of 64 x 48

// One CTA per tile. Each candidate's 81-cell neighbourhood is scanned by one
// warp (lane l looks at cells l, l + 32, l + 64 of the 9x9 square, row-major),
// the blockers collected with three ballots. Candidates without blockers are
// ready for the first round, the others start the first pending list. Index
// math inside an event is 32-bit (events hold fewer than 2^31 cells).
// the 80 cells of a 9x9 square around its centre, nearest ring first, as offsets in the HX = 64 wide halo
// tile (dy * 64 + dx; negative = a smaller cell index in the same event)
__constant__ int16_t kRing[80] = {
    -65, -64, -63, -1, 1, 63, 64, 65,
    -130, -129, -128, -127, -126, -66, -62, -2, 2, 62, 66, 126, 127, 128, 129, 130,
    -195, -194, -193, -192, -191, -190, -189, -131, -125, -67, -61, -3, 3, 61, 67, 125, 131, 189, 190, 191, 192,
    193, 194, 195,
    -260, -259, -258, -257, -256, -255, -254, -253, -252, -196, -188, -132, -124, -68, -60, -4, 4, 60, 68, 124,
    132, 188, 196, 252, 253, 254, 255, 256, 257, 258, 259, 260};

// numpy's f32 `e / z > 5` (SEED_THRESHOLD, reconstruct.py:62-66) without the division: the rounded
// quotient exceeds 5 iff the exact one exceeds the midpoint 5 + 2^-22 between 5 and the next float (a tie
// rounds to 5, whose significand is even). z * (5 + 2^-22) is exact in f64 (24 x 25 significant bits), so
// for z != 0 the test is one f64 product and compare, with the inequality flipped for z < 0. z = +-0: e / z
// is an infinity of the sign of e XOR z (> 5 iff that is +inf), or NaN for e = 0; NaN anywhere: false.
__device__ __forceinline__ bool seed_ratio(float e, float z) {
  const double t = static_cast<double>(z) * (5.0 + 0x1p-22);
  if (z > 0.0f) return static_cast<double>(e) > t;
  if (z < 0.0f) return static_cast<double>(e) < t;
  if (z == 0.0f) return e != 0.0f && e == e && ((e > 0.0f) != static_cast<bool>(signbit(z)));
  return false;  // z is NaN
}

template <bool VEC>
__global__ void __launch_bounds__(NT, 5) tile_kernel(Args A, int tiles_x, int tiles_per_event) {
  pdl_enter();
  __shared__ __align__(16) float se[HY * HX];
  __shared__ __align__(16) uint8_t sc[HY * HX];
  __shared__ uint16_t cl[TX * TY];   // the tile's candidates (halo index)
  __shared__ uint16_t cls[TX * TY];  // their list (bit 15) and position in it
  __shared__ int s_cnt[NT / 32];
  __shared__ int s_nl[2];
  __shared__ int s_total;
  __shared__ unsigned long long s_lb;
  const int ev = blockIdx.x / tiles_per_event;
  const int tile = blockIdx.x - ev * tiles_per_event;
  const int ty0 = (tile / tiles_x) * TY, tx0 = (tile % tiles_x) * TX;
  const int w = static_cast<int>(A.w), h = static_cast<int>(A.h);
  const int64_t base = static_cast<int64_t>(ev) * A.n;
  const float* E = A.energy + base;
  const float* NZ = A.noise + base;
  uint8_t* F = A.flags + base;
  if (threadIdx.x < 2) s_nl[threadIdx.x] = 0;
  if constexpr (VEC) {
    // w % 4 == 0 and 16-byte aligned planes: a thread loads 4 cells at once (a group of 4 is wholly
    // inside or outside the grid, wholly interior or halo), all of its rows in flight together
    constexpr int G4 = HX / 4, RG = NT / G4, RPT = HY / RG;
    static_assert(NT % G4 == 0 && HY % RG == 0, "tile shape");
    const int c4 = threadIdx.x % G4, rg = threadIdx.x / G4;
    const int hx = c4 * 4, x = tx0 - HALO + hx;
    const bool xin = x >= 0 && x < w, xint = hx >= HALO && hx < HALO + TX;
    float4 e[RPT], z[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int y = ty0 - HALO + rg + r * RG;
      const bool in = xin && y >= 0 && y < h;
      e[r] = in ? *reinterpret_cast<const float4*>(E + static_cast<int64_t>(y) * w + x) : make_float4(0, 0, 0, 0);
      z[r] = in ? *reinterpret_cast<const float4*>(NZ + static_cast<int64_t>(y) * w + x) : make_float4(1, 1, 1, 1);
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int hy = rg + r * RG, y = ty0 - HALO + hy;
      const bool in = xin && y >= 0 && y < h;
      // numpy f32 division (IEEE); NaN is no candidate
      const uint32_t cand = in ? (static_cast<uint32_t>(seed_ratio(e[r].x, z[r].x)) |
                                  static_cast<uint32_t>(seed_ratio(e[r].y, z[r].y)) << 8 |
                                  static_cast<uint32_t>(seed_ratio(e[r].z, z[r].z)) << 16 |
                                  static_cast<uint32_t>(seed_ratio(e[r].w, z[r].w)) << 24)
                               : 0u;
      if (in && xint && hy >= HALO && hy < HALO + TY)  // PENDING == 1: the candidate bytes are the flags
        *reinterpret_cast<uint32_t*>(F + static_cast<int64_t>(y) * w + x) = cand;
      *reinterpret_cast<float4*>(&se[hy * HX + hx]) = e[r];
      *reinterpret_cast<uint32_t*>(&sc[hy * HX + hx]) = cand;
    }
  } else {
    // a warp loads whole halo rows (HX = 2 x 32 lanes), all of its rows in flight at once
    constexpr int RPW = HY / (NT / 32);  // rows per warp
    static_assert(HY % (NT / 32) == 0 && HX == 64, "tile shape");
    const int lane0 = threadIdx.x & 31, wid0 = threadIdx.x >> 5;
    float e[RPW][2], nz[RPW][2];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int y = ty0 - HALO + wid0 + r * (NT / 32);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const int x = tx0 - HALO + ch * 32 + lane0;
        const bool in = y >= 0 && y < h && x >= 0 && x < w;
        e[r][ch] = in ? E[static_cast<int64_t>(y) * w + x] : 0.0f;
        nz[r][ch] = in ? NZ[static_cast<int64_t>(y) * w + x] : 1.0f;
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int hy = wid0 + r * (NT / 32), y = ty0 - HALO + hy;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const int hx = ch * 32 + lane0, x = tx0 - HALO + hx;
        const bool in = y >= 0 && y < h && x >= 0 && x < w;
        const bool cand = in && seed_ratio(e[r][ch], nz[r][ch]);  // numpy f32 e / z > 5; NaN: no candidate
        if (in && hy >= HALO && hy < HALO + TY && hx >= HALO && hx < HALO + TX)
          F[static_cast<int64_t>(y) * w + x] = cand ? PENDING : 0;  // read by the rounds (later launches)
        se[hy * HX + hx] = e[r][ch];
        sc[hy * HX + hx] = cand;
      }
    }
  }
  __syncthreads();
  // compact the tile's candidates (row-major order) into cl
  constexpr int PER = (TX * TY + NT - 1) / NT;  // a contiguous run of interior cells per thread
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int mine = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int j = threadIdx.x * PER + k, iy = j / TX, ix = j - iy * TX;
    if (j < TX * TY) mine += sc[(iy + HALO) * HX + ix + HALO];
  }
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_cnt[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < NT / 32; ++k) {
      const int v = s_cnt[k];
      s_cnt[k] = t;
      t += v;
    }
    s_total = t;
  }
  __syncthreads();
  const int total = s_total;
  if (!total) return;
  {
    int pos = s_cnt[wid] + incl - mine;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = threadIdx.x * PER + k, iy = j / TX, ix = j - iy * TX;
      const int hc = (iy + HALO) * HX + ix + HALO;
      if (j < TX * TY && sc[hc]) cl[pos++] = static_cast<uint16_t>(hc);
    }
  }
  __syncthreads();
  // is each candidate the top priority among the candidates of its 9x9 neighbourhood? Eight lanes per
  // candidate walk the neighbourhood nearest ring first, 8 cells a step, and stop at the first candidate of
  // higher priority (usually in the first ring): four candidates per warp, every warp busy
  static_assert(HX == 64, "kRing assumes a 64-wide halo tile");
  const int sub = lane & 7, grp = lane >> 3;
  int ring[10];
#pragma unroll
  for (int it = 0; it < 10; ++it) ring[it] = kRing[it * 8 + sub];
  for (int q0 = wid * 4; q0 < total; q0 += NT / 8) {
    const int q = q0 + grp;
    const bool have = q < total;
    const int hc = have ? cl[q] : HALO * HX + HALO;
    const float ec = se[hc];
    bool top = have;
#pragma unroll
    for (int it = 0; it < 10; ++it) {
      const int d = ring[it];
      const float eq = se[hc + d];
      const bool blk = top && sc[hc + d] && (eq > ec || (d < 0 && eq == ec));
      const unsigned b = __ballot_sync(0xffffffffu, blk);
      if ((b >> (grp * 8)) & 0xffu) top = false;
      if (!__any_sync(0xffffffffu, top)) break;
    }
    if (have && sub == 0) {
      const int which = top ? 0 : 1;  // 0: no blockers, ready for the first round
      cls[q] = static_cast<uint16_t>(atomicAdd(&s_nl[which], 1) | (which << 15));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0)  // both lists' places with one atomic
    s_lb = atomicAdd(&A.counters[C_TILE],
                     static_cast<unsigned long long>(s_nl[1]) << 32 | static_cast<unsigned long long>(s_nl[0]));
  __syncthreads();
  const int64_t cap = A.cand_cap;
  for (int q = threadIdx.x; q < total; q += NT) {  // no blockers: ready for the first round; the others: the
    const int which = cls[q] >> 15, li = cls[q] & 0x7fff;  // first pending list (cells, both)
    const int64_t at = static_cast<int64_t>(which ? s_lb >> 32 : s_lb & 0xffffffffull) + li;
    if (at >= cap) continue;  // over capacity: counted, the host grows the lists and runs again
    const int hc = cl[q], iy = hc / HX - HALO, ix = hc % HX - HALO;
    (which ? A.list[0] : A.ready)[at] = base + (ty0 + iy) * w + tx0 + ix;
  }
}

// ---- 2. rounds: check, then process ---------------------------------------------------------
//
// check_kernel: one thread per candidate of the pending list walks its blocker
// list from where the last round stopped (8 blocker flags in flight); a
// candidate consumed meanwhile drops out, one with a pending blocker goes to
// the next list, the rest are ready. process_kernel then processes the ready
// seeds, whose windows are pairwise disjoint, spread over every warp of the
// grid. Kernel boundaries order the two, so plain loads and stores suffice.
// The last CTA out of each kernel does the round's bookkeeping, so the host
// queues rounds without looking in between (an empty round returns at once).
constexpr int PNT = 128;
constexpr int PW = PNT / 32;

struct WinSmem {  // window values of 32 seeds of one warp
  float e[32][25], r[32][25];
  uint8_t t[32][25], nz[32][25];
  unsigned mask[32];
  int64_t seed[32];
  int64_t slot[32];
  int ev[32], sy[32], sx[32];  // the seed's event and position in it
};

// seed j's particle from its window values, into its slot: f64 sums in the reference's row-major
// contributor order, no FMA, rounded once to f32 (reconstruct.py:84-117)
__device__ void particle_sums(const Args& A, const WinSmem& S, int j) {
  const int64_t s = S.seed[j];
  const int ev = S.ev[j], sy = S.sy[j], sx = S.sx[j];
  const int64_t loc = static_cast<int64_t>(sy) * A.w + sx;
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
  Slot& P = A.slots[S.slot[j]];
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
}

__device__ __forceinline__ bool higher(const Args& A, int64_t q, int64_t c) {
  const float eq = A.energy[q], ec = A.energy[c];
  return eq > ec || (eq == ec && q < c);
}

// bit 0 of each byte of v, in byte order
__device__ __forceinline__ uint32_t low_bits8(uint64_t v) {
  return static_cast<uint32_t>(((v & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56);
}

// Is pending candidate c blocked, i.e. is a pending candidate of higher priority within distance 4?
// The 81 flags come in with two aligned 8-byte loads per row (all in flight together) and are reduced to
// an 81-bit mask of pending neighbours (bit = row * 9 + column of the 9x9 square); their energies are
// then fetched 8 at a time, stopping at the first one of higher priority.
__device__ bool blocked(const Args& A, int64_t c) {
  const int w = static_cast<int>(A.w), h = static_cast<int>(A.h);
  const int64_t ev = c / A.n, base = ev * A.n;
  const int loc = static_cast<int>(c - base), cy = loc / w, cx = loc - cy * w;
  const int x0 = max(0, cx - 4), len = min(w - 1, cx + 4) - x0 + 1, shift = x0 - (cx - 4);
  uint64_t lo[9], hi[9];
  int off[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    const int y = cy - 4 + r;
    lo[r] = hi[r] = 0;
    off[r] = 0;
    if (y >= 0 && y < h) {
      const uintptr_t start = reinterpret_cast<uintptr_t>(A.flags + base + static_cast<int64_t>(y) * w + x0);
      const uint64_t* al = reinterpret_cast<const uint64_t*>(start & ~uintptr_t(7));
      off[r] = static_cast<int>(start & 7);
      lo[r] = al[0];
      hi[r] = al[1];  // the flags allocation is padded: this may read up to 15 bytes past the last cell
    }
  }
  uint32_t m[3] = {0, 0, 0};
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    uint32_t row = ((low_bits8(lo[r]) | (low_bits8(hi[r]) << 8)) >> off[r]) & ((1u << len) - 1u);
    row <<= shift;  // into the 9-wide frame
    if (r == 4) row &= ~(1u << 4);  // the candidate itself
    const int b = r * 9;  // bits b .. b + 8 of the 81-bit mask
    if (b < 32) {
      m[0] |= row << b;
      if (b + 9 > 32) m[1] |= row >> (32 - b);
    } else if (b < 64) {
      m[1] |= row << (b - 32);
      if (b + 9 > 64) m[2] |= row >> (64 - b);
    } else {
      m[2] |= row << (b - 64);
    }
  }
  const float ec = A.energy[c];
  while (m[0] | m[1] | m[2]) {
    int js[8];
    float eq[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int j = -1;
      if (m[0]) {
        j = __ffs(m[0]) - 1;
        m[0] &= m[0] - 1;
      } else if (m[1]) {
        j = 31 + __ffs(m[1]);
        m[1] &= m[1] - 1;
      } else if (m[2]) {
        j = 63 + __ffs(m[2]);
        m[2] &= m[2] - 1;
      }
      js[u] = j;
      eq[u] = j >= 0 ? A.energy[base + static_cast<int64_t>(cy - 4 + j / 9) * w + (cx - 4 + j % 9)] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (js[u] >= 0 && (eq[u] > ec || (js[u] < 40 && eq[u] == ec))) return true;  // j < 40: smaller cell index
  }
  return false;
}

// true in the one CTA that finishes last (every other CTA of the grid is done)
__device__ __forceinline__ bool last_cta(unsigned long long* done) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  return s_last;
}

__global__ void __launch_bounds__(NT) check_kernel(Args A, int parity) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(A.counters[C_CUR]);
  if (m == 0) return;  // converged: nothing to check, nothing to book
  const int64_t* cur = A.list[parity];
  int64_t* nxt = A.list[parity ^ 1];
  const int64_t stride = static_cast<int64_t>(gridDim.x) * NT;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * NT + (threadIdx.x & ~31); i0 < m; i0 += stride) {
    const int64_t i = i0 + lane;
    const bool have = i < m;
    const int64_t c = have ? cur[i] : 0;
    const bool pend = have && (A.flags[c] & PENDING);  // most were consumed by the previous round
    const bool ok = pend && !blocked(A, c);
    const bool wait = pend && !ok;
    const unsigned wm = __ballot_sync(0xffffffffu, wait), rm = __ballot_sync(0xffffffffu, ok);
    const unsigned below = (1u << lane) - 1u;
    unsigned long long wb = 0, rb = 0;
    if (lane == 0) {
      if (wm) wb = atomicAdd(&A.counters[C_NEXT], static_cast<unsigned long long>(__popc(wm)));
      if (rm) rb = atomicAdd(&A.counters[C_READY], static_cast<unsigned long long>(__popc(rm)));
    }
    wb = __shfl_sync(0xffffffffu, wb, 0);
    rb = __shfl_sync(0xffffffffu, rb, 0);
    if (wait) nxt[wb + __popc(wm & below)] = c;
    if (ok) A.ready[rb + __popc(rm & below)] = c;
  }
  if (last_cta(&A.counters[C_DONE]) && threadIdx.x == 0) {
    A.counters[C_PASSES] += m != 0;
    // C_NEXT was built by every CTA's atomics in this kernel: read and reset it atomically (a plain load
    // may be served a stale L1 line)
    A.counters[C_CUR] = atomicExch(&A.counters[C_NEXT], 0ull);
    A.counters[C_DONE] = 0;
  }
}

// A warp takes up to 32 ready seeds at a time: for each in turn, lane l < 25
// examines window cell (l / 5 - 2, l % 5 - 2) -- every load in one round trip,
// the taken cells marked consumed, the contributor list written, the values
// kept in shared memory -- then lane j adds up seed j's contributors.
__global__ void __launch_bounds__(PNT) process_kernel(Args A, int first) {
  pdl_enter();
  __shared__ WinSmem W[PW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WinSmem& S = W[wid];
  // the first round's ready seeds come from the tile pass
  const int64_t nready = first ? min(static_cast<int64_t>(A.counters[C_TILE] & 0xffffffffull), A.cand_cap)
                               : static_cast<int64_t>(A.counters[C_READY]);
  if (nready == 0 && !first) return;  // an empty round
  const int64_t slot0 = static_cast<int64_t>(A.counters[C_SLOTS]);
  const int w = static_cast<int>(A.w), h = static_cast<int>(A.h);
  // seeds per warp batch: spread over every warp of the grid (the window step is serial per warp)
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * PW;
  const int64_t per = max(static_cast<int64_t>(1), min(static_cast<int64_t>(32), (nready + nwarps - 1) / nwarps));
  const int64_t stride = nwarps * per;
  for (int64_t k0 = (static_cast<int64_t>(blockIdx.x) * PW + wid) * per; k0 < nready; k0 += stride) {
    const int nb = static_cast<int>(min(per, nready - k0));
    // lane j owns seed j of the batch: one load and one 64-bit division each, shared by shuffles
    const int64_t my_s = lane < nb ? A.ready[k0 + lane] : 0;
    const int64_t my_ev = my_s / A.n;
    const int my_loc = static_cast<int>(my_s - my_ev * A.n);
    const int my_sy = my_loc / w;
    const int my_sx = my_loc - my_sy * w;
    const int dy = lane / 5 - 2, dx = lane % 5 - 2;
    constexpr int G = 4;  // windows whose loads are in flight together (the windows are disjoint)
    for (int j0 = 0; j0 < nb; j0 += G) {
      float e[G], z[G];
      uint8_t fl[G], ty[G], nzv[G];
      int64_t fc[G];
      bool inw[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g;
        const int sy = __shfl_sync(0xffffffffu, my_sy, j & 31), sx = __shfl_sync(0xffffffffu, my_sx, j & 31);
        const int64_t ev = __shfl_sync(0xffffffffu, my_ev, j & 31);
        const int y = sy + dy, x = sx + dx;
        inw[g] = j < nb && lane < 25 && y >= 0 && y < h && x >= 0 && x < w;
        fc[g] = ev * A.n + (inw[g] ? y * w + x : sy * w + sx);
        fl[g] = j < nb ? A.flags[fc[g]] : 0;
        e[g] = j < nb ? A.energy[fc[g]] : 0.0f;
        z[g] = j < nb ? A.noise[fc[g]] : 1.0f;
        ty[g] = j < nb ? A.type[fc[g]] & 3 : 0;
        nzv[g] = j < nb ? A.noisy[fc[g]] != 0 : 0;
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int j = j0 + g;
        if (j >= nb) break;
        const int64_t p = slot0 + k0 + j;
        const float r32 = __fdiv_rn(e[g], z[g]);
        const bool take = inw[g] && !(fl[g] & CONSUMED) && r32 > 2.0f;
        if (take) A.flags[fc[g]] = CONSUMED;  // clears PENDING: a consumed candidate is decided, so is the seed
        const unsigned mask = __ballot_sync(0xffffffffu, take);
        const int64_t ev = __shfl_sync(0xffffffffu, my_ev, j & 31);
        if (take && p < A.slot_cap)  // contributor list, row-major: rank of this lane among the taken ones
          A.contrib[p * MAXC + __popc(mask & ((1u << lane) - 1u))] = static_cast<uint64_t>(fc[g] - ev * A.n);
        if (lane < 25) {
          S.e[j][lane] = e[g];
          S.r[j][lane] = r32;
          S.t[j][lane] = ty[g];
          S.nz[j][lane] = nzv[g];
        }
        if (lane == 0) {
          S.mask[j] = mask;
          S.slot[j] = p;
        }
      }
    }
    if (lane < nb) {
      S.seed[lane] = my_s;
      S.ev[lane] = static_cast<int>(my_ev);
      S.sy[lane] = my_sy;
      S.sx[lane] = my_sx;
    }
    __syncwarp();
    const bool mine = lane < nb && S.slot[lane] < A.slot_cap;
    if (mine) {
      particle_sums(A, S, lane);
      atomicAdd(&A.event_count[S.ev[lane]], 1ull);
    }
    const unsigned nc = __reduce_add_sync(0xffffffffu, mine ? static_cast<unsigned>(__popc(S.mask[lane])) : 0u);
    if (lane == 0 && nc) atomicAdd(&A.counters[C_CONTRIB], static_cast<unsigned long long>(nc));
    __syncwarp();  // the window buffers are reused by the next batch
  }
  if (last_cta(&A.counters[C_DONE]) && threadIdx.x == 0) {
    A.counters[C_SLOTS] += nready;
    A.counters[C_READY] = 0;
    if (first) A.counters[C_CUR] = min(static_cast<int64_t>(A.counters[C_TILE] >> 32), A.cand_cap);
    A.counters[C_DONE] = 0;
  }
}

// ---- 3. ordering -------------------------------------------------------------------------

// event offsets: exclusive prefix of the per-event particle counts (one CTA, a thread per event run)
__global__ void __launch_bounds__(NT) event_offsets_kernel(const unsigned long long* counts, int nevents,
                                                            int64_t* off, int64_t* cnt, unsigned long long* cursor) {
  pdl_enter();
  __shared__ int64_t s_part[NT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int per = (nevents + NT - 1) / NT, lo = min(nevents, static_cast<int>(threadIdx.x) * per),
            hi = min(nevents, lo + per);
  int64_t t = 0;
  for (int e = lo; e < hi; ++e) t += static_cast<int64_t>(counts[e]);
  int64_t incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_part[wid] = incl;
  __syncthreads();
  int64_t before = 0;
  for (int k = 0; k < wid; ++k) before += s_part[k];
  int64_t run = before + incl - t;
  for (int e = lo; e < hi; ++e) {
    off[e] = run;
    cnt[e] = static_cast<int64_t>(counts[e]);
    cursor[e] = 0;
    run += static_cast<int64_t>(counts[e]);
  }
}

// bucket particles by event, then rank by priority inside the event
__global__ void bucket_kernel(const Slot* slots, const unsigned long long* nslots, int64_t cap,
                              const int64_t* event_off, unsigned long long* cursor, int64_t* order, int32_t* lens,
                              int64_t nlens) {
  pdl_enter();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * NT + threadIdx.x; i < nlens;
       i += static_cast<int64_t>(gridDim.x) * NT)
    lens[i] = 0;  // the write sets the particles' contributor counts; the rest of the capacity packs nothing
  const int64_t np = min(static_cast<int64_t>(*nslots), cap);
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
                                                   const int64_t* event_cnt, const int64_t* order, OutArgs O,
                                                   int64_t cap) {
  pdl_enter();
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
    const int64_t o = b + rank;
    if (!have || q || o >= cap) continue;  // (past the output's capacity: the caller grows it, writes again)
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

// ---- host side ---------------------------------------------------------------------------

// Device workspace of one run. Kept per device between runs (grow-only) so a
// steady stream of calls allocates nothing; a run that finds the cache taken
// (another handle alive) allocates its own.
struct Workspace {
  int device = -1;
  void* mem = nullptr;
  cudaEvent_t released = nullptr;  // recorded on the releasing stream: the next user waits for it
  size_t bytes = 0;
  int64_t cells = 0, cand_cap = 0, slot_cap = 0;
  int nevents = 0;
  void* aux = nullptr;  // the write's temporaries: contributor counts / offsets, the packer's scratch
  size_t aux_bytes = 0;
};

static std::mutex g_ws_mu;
static Workspace g_ws[64];
static bool g_ws_busy[64];

struct Handle {
  int device = 0;
  int64_t w = 0, h = 0, n = 0;
  int nevents = 0;
  int64_t np = 0;      // particles
  int64_t nslots = 0;  // particle slots written, holes (skipped seeds) included
  Workspace ws;
  bool cached = false;  // ws belongs to the per-device cache
  Args A;
  int64_t ncontrib = 0;
  int64_t* order = nullptr;  // particle slots bucketed by event
  int64_t* ev_off = nullptr;
  int64_t* ev_cnt = nullptr;
  unsigned long long* cursor = nullptr;
  std::vector<int64_t> counts;
};

static size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

static size_t ws_bytes(int64_t cells, int64_t cand_cap, int64_t slot_cap, int nevents) {
  return al256(static_cast<size_t>(cells) + 16) +
         3 * al256(static_cast<size_t>(cand_cap) * 8) + al256(static_cast<size_t>(slot_cap) * sizeof(Slot)) +
         al256(static_cast<size_t>(slot_cap) * MAXC * 8) + al256(NCOUNTERS * 8) + al256(static_cast<size_t>(nevents + 1) * 8) +
         al256(static_cast<size_t>(slot_cap) * 8) + 3 * al256(static_cast<size_t>(nevents + 1) * 8);
}

static void carve(Handle* H) {
  uint8_t* p = static_cast<uint8_t*>(H->ws.mem);
  Args& A = H->A;
  A.flags = p; p += al256(static_cast<size_t>(H->ws.cells) + 16);  // + 16: blocked() reads whole words
  A.list[0] = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.cand_cap) * 8);
  A.list[1] = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.cand_cap) * 8);
  A.ready = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.cand_cap) * 8);
  A.slots = reinterpret_cast<Slot*>(p); p += al256(static_cast<size_t>(H->ws.slot_cap) * sizeof(Slot));
  A.contrib = reinterpret_cast<uint64_t*>(p); p += al256(static_cast<size_t>(H->ws.slot_cap) * MAXC * 8);
  A.counters = reinterpret_cast<unsigned long long*>(p); p += al256(NCOUNTERS * 8);
  A.event_count = reinterpret_cast<unsigned long long*>(p); p += al256(static_cast<size_t>(H->ws.nevents + 1) * 8);
  H->order = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.slot_cap) * 8);
  H->ev_off = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.nevents + 1) * 8);
  H->ev_cnt = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(H->ws.nevents + 1) * 8);
  H->cursor = reinterpret_cast<unsigned long long*>(p);
  A.cand_cap = H->ws.cand_cap;
  A.slot_cap = H->ws.slot_cap;
}

// a workspace for `cells` cells, at least the given capacities
static int acquire_ws(Handle* H, int64_t cand_cap, int64_t slot_cap, cudaStream_t s) {
  const int dev = H->device;
  if (!H->ws.mem && dev >= 0 && dev < 64) {
    std::lock_guard<std::mutex> g(g_ws_mu);
    if (!g_ws_busy[dev]) {
      g_ws_busy[dev] = true;
      H->cached = true;
      H->ws = g_ws[dev];
      g_ws[dev] = Workspace();
    }
  }
  Workspace& W = H->ws;
  if (W.released) {  // work queued by the previous user (e.g. the pack of its contributor pool) comes first
    SK_TRY(cudaStreamWaitEvent(s, W.released, 0));
  }
  cand_cap = std::max(cand_cap, W.cand_cap);
  slot_cap = std::max(slot_cap, W.slot_cap);
  const int64_t cells = std::max(H->n * H->nevents, W.cells);
  const int nev = std::max(H->nevents, W.nevents);
  if (W.mem && cells == W.cells && cand_cap == W.cand_cap && slot_cap == W.slot_cap && nev == W.nevents) {
    carve(H);
    return SK_OK;
  }
  if (W.mem) cudaFreeAsync(W.mem, s);
  cudaEvent_t ev = W.released;
  void* aux = W.aux;
  const size_t aux_bytes = W.aux_bytes;
  W = Workspace();
  W.released = ev;
  W.aux = aux;
  W.aux_bytes = aux_bytes;
  const size_t bytes = ws_bytes(cells, cand_cap, slot_cap, nev);
  cudaError_t e = cudaMallocAsync(&W.mem, bytes, s);
  if (e != cudaSuccess) {
    W.mem = nullptr;
    return cuda_fail(e, "cudaMallocAsync(reconstruction workspace)");
  }
  W.device = dev;
  W.bytes = bytes;
  W.cells = cells;
  W.cand_cap = cand_cap;
  W.slot_cap = slot_cap;
  W.nevents = nev;
  carve(H);
  return SK_OK;
}

static void release_ws(Handle* H, cudaStream_t s) {
  if (!H->ws.mem) return;
  if (H->cached) {
    if (!H->ws.released) cudaEventCreateWithFlags(&H->ws.released, cudaEventDisableTiming);
    if (H->ws.released) cudaEventRecord(H->ws.released, s);
    std::lock_guard<std::mutex> g(g_ws_mu);
    g_ws[H->device] = H->ws;
    g_ws_busy[H->device] = false;
  } else {
    cudaFreeAsync(H->ws.mem, s);
    if (H->ws.aux) cudaFreeAsync(H->ws.aux, s);
    if (H->ws.released) cudaEventDestroy(H->ws.released);
  }
  H->ws = Workspace();
}

static int process_grid(const DeviceState* ds, int device) {
  static int per_sm[64] = {0};
  int& occ = per_sm[device & 63];
  if (!occ && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, process_kernel, PNT, 0) != cudaSuccess || occ < 1))
    occ = 1;
  return ds->sm_count * occ;
}

// Queue the write of the particles (reference order) and of their contributor lists into `out`: event
// offsets, bucketing and ranking on the device, then the jagged packer over `out`'s whole particle capacity
// (contributor counts past the particles are zero). Sizes are read on the device, so this can be queued
// before the host knows them; whatever does not fit the capacities is dropped and reported by the caller.
static int queue_write(Handle* H, const sk_reco_out* out, cudaStream_t s, const DeviceState* ds, unsigned chunks) {
  const int64_t pcap = std::max<int64_t>(out->particle_capacity, 0);
  size_t scan = 0;
  sk_jagged_scratch_bytes(pcap, &scan);
  const size_t scratch = al256(scan) + static_cast<size_t>((std::max<int64_t>(out->pool_capacity, 0) + 255) / 256 + 1) * 8;
  const size_t need = al256(static_cast<size_t>(pcap) * 4) + al256(static_cast<size_t>(pcap) * 8) + al256(16) + scratch;
  Workspace& W = H->ws;
  if (W.aux_bytes < need) {
    if (W.aux) cudaFreeAsync(W.aux, s);
    W.aux = nullptr;
    W.aux_bytes = 0;
    cudaError_t e = cudaMallocAsync(&W.aux, need, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(reconstruction write scratch)");
    W.aux_bytes = need;
  }
  uint8_t* p = static_cast<uint8_t*>(W.aux);
  int32_t* lens = reinterpret_cast<int32_t*>(p); p += al256(static_cast<size_t>(pcap) * 4);
  int64_t* offs = reinterpret_cast<int64_t*>(p); p += al256(static_cast<size_t>(pcap) * 8);
  int64_t* total = reinterpret_cast<int64_t*>(p); p += al256(16);
  void* pack_scratch = p;
  SK_TRY(launch(event_offsets_kernel, dim3(1), dim3(NT), s, H->A.event_count, H->nevents, H->ev_off, H->ev_cnt,
                H->cursor));
  SK_TRY(launch(bucket_kernel, dim3(ds->sm_count * 4), dim3(NT), s, H->A.slots, &H->A.counters[C_SLOTS],
                H->A.slot_cap, H->ev_off, H->cursor, H->order, lens, pcap));
  OutArgs O;
  O.energy = out->energy; O.x = out->x; O.y = out->y; O.xvar = out->x_variance; O.yvar = out->y_variance;
  O.origin = out->origin;
  for (int t = 0; t < 4; ++t) {
    O.sig[t] = out->significance[t];
    O.ec[t] = out->e_contribution[t];
    O.nc[t] = out->noisy_count[t];
  }
  O.lens = lens;
  O.offsets = offs;
  if (H->nevents && chunks)
    SK_TRY(launch(write_kernel, dim3(H->nevents, chunks), dim3(NT), s, H->A.slots, H->ev_off, H->ev_cnt, H->order, O,
                  pcap));
  const int64_t field_off = 0;
  const int32_t field_size = 8;
  void* dst = out->sensor_pool;
  return sk_jagged_pack(pcap, lens, SK_I32, out->sensor_prefix, out->sensor_prefix_type, offs, H->A.contrib,
                        H->A.slot_cap * MAXC, 8, 1, &field_off, &field_size, &dst, out->pool_capacity, pack_scratch,
                        scratch, total, reinterpret_cast<uintptr_t>(s));
}

}  // namespace reco
}  // namespace sk

using namespace sk;

extern "C" {

int sk_reco_run(int64_t w, int64_t h, int nevents, const float* energy, const float* noise, const uint8_t* type,
                const uint8_t* noisy, const sk_reco_out* out, int device, uintptr_t stream, void** handle,
                int64_t* nparticles, int64_t* ncontributors, int* rounds, int* written) {
  if (!handle || w < 1 || h < 1 || nevents < 0) return set_error(SK_ERR_INVALID, "bad reconstruction arguments");
  if (w * h >= (int64_t(1) << 31) || w * h * nevents >= (int64_t(1) << 32))
    return set_error(SK_ERR_INVALID, "%d events of %lld cells: too many cells for one run", nevents,
                     static_cast<long long>(w * h));
  if (written) *written = 0;
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
  reco::Args& A = H->A;
  memset(&A, 0, sizeof(A));
  A.w = w; A.h = h; A.n = H->n; A.nevents = nevents;
  A.energy = energy; A.noise = noise; A.type = type; A.noisy = noisy;
  // first guess at the capacities (the benchmark events hold ~4% candidates, ~7% of them particles);
  // the run counts what it needed and is repeated once with that if it did not fit
  int64_t cand_cap = std::max<int64_t>(4096, total / 16), slot_cap = std::max<int64_t>(1024, total / 64);
  const int tiles_x = static_cast<int>((w + reco::TX - 1) / reco::TX);
  const int tiles_per_event = tiles_x * static_cast<int>((h + reco::TY - 1) / reco::TY);
  const int cgrid = ds->sm_count * 8;
  const bool vec = w % 4 == 0 && ((reinterpret_cast<uintptr_t>(energy) | reinterpret_cast<uintptr_t>(noise)) & 15) == 0;
  const int pgrid = reco::process_grid(ds, device);
  unsigned long long cnt[reco::NCOUNTERS] = {0};
  std::vector<unsigned long long> ec(nevents > 0 ? nevents : 1);
  auto fail = [&](int code) {
    reco::release_ws(H, s);
    delete H;
    return code;
  };
  for (int attempt = 0;; ++attempt) {
    rc = reco::acquire_ws(H, cand_cap, slot_cap, s);
    if (rc) {
      delete H;
      return rc;
    }
    SK_TRY(cudaMemsetAsync(A.counters, 0, reco::NCOUNTERS * 8, s));
    SK_TRY(cudaMemsetAsync(A.event_count, 0, static_cast<size_t>(nevents + 1) * 8, s));
    const dim3 tgrid(static_cast<unsigned>(nevents) * tiles_per_event);
    if (total) SK_TRY(reco::launch(vec ? reco::tile_kernel<true> : reco::tile_kernel<false>, tgrid, dim3(reco::NT), s, A,
                                   tiles_x, tiles_per_event));
    SK_TRY(reco::launch(reco::process_kernel, dim3(pgrid), dim3(reco::PNT), s, A, 1));  // candidates without blockers
    // rounds are queued without a host check in between (a round with nothing pending returns at once):
    // 6 (full events converge in 4-5), then 4 more at a time until nothing is pending. The write into `out`
    // is queued behind them, so one host synchronisation covers the whole reconstruction.
    int launched = 0;
    for (;;) {
      const int batch = launched ? 4 : 6;
      for (int k = 0; k < batch; ++k, ++launched) {
        SK_TRY(reco::launch(reco::check_kernel, dim3(cgrid), dim3(reco::NT), s, A, launched & 1));
        SK_TRY(reco::launch(reco::process_kernel, dim3(pgrid), dim3(reco::PNT), s, A, 0));
      }
      SK_TRY(cudaGetLastError());
      if (out && (rc = reco::queue_write(H, out, s, ds, 8))) return fail(rc);
      SK_TRY(cudaMemcpyAsync(cnt, A.counters, sizeof(cnt), cudaMemcpyDeviceToHost, s));
      if (nevents) SK_TRY(cudaMemcpyAsync(ec.data(), A.event_count, nevents * 8, cudaMemcpyDeviceToHost, s));
      SK_TRY(cudaStreamSynchronize(s));
      const int64_t n_top = static_cast<int64_t>(cnt[reco::C_TILE] & 0xffffffffull);
      const int64_t n_rest = static_cast<int64_t>(cnt[reco::C_TILE] >> 32);
      const bool over = n_top > A.cand_cap || n_rest > A.cand_cap || static_cast<int64_t>(cnt[reco::C_SLOTS]) > A.slot_cap;
      if (over || cnt[reco::C_CUR] == 0) break;
      if (launched > static_cast<int>(std::min<int64_t>(n_top + n_rest, 1 << 30)) + 16)
        return fail(set_error(SK_ERR_CUDA, "reconstruction made no progress"));  // a round decides >= 1 seed
    }
    const int64_t n_top = static_cast<int64_t>(cnt[reco::C_TILE] & 0xffffffffull);
    const int64_t n_rest = static_cast<int64_t>(cnt[reco::C_TILE] >> 32);
    if (n_top <= A.cand_cap && n_rest <= A.cand_cap && static_cast<int64_t>(cnt[reco::C_SLOTS]) <= A.slot_cap) break;
    if (attempt) return fail(set_error(SK_ERR_CUDA, "reconstruction workspace overflow"));  // cannot happen
    cand_cap = std::max({cand_cap, n_top, n_rest});
    slot_cap = std::max<int64_t>(slot_cap, n_top + n_rest);  // at most one slot per candidate
  }
  H->counts.assign(nevents, 0);
  int64_t np = 0;
  for (int i = 0; i < nevents; ++i) {
    H->counts[i] = static_cast<int64_t>(ec[i]);
    np += H->counts[i];
  }
  H->np = np;
  H->nslots = static_cast<int64_t>(cnt[reco::C_SLOTS]);
  H->ncontrib = static_cast<int64_t>(cnt[reco::C_CONTRIB]);
  if (H->nslots != np)  // a slot without a particle: the contributor pool would not match the counts
    return fail(set_error(SK_ERR_CUDA, "reconstruction left particle slots empty"));
  if (nparticles) *nparticles = H->np;
  if (ncontributors) *ncontributors = H->ncontrib;
  if (rounds) *rounds = static_cast<int>(cnt[reco::C_PASSES]);
  if (written) *written = out && H->np <= out->particle_capacity && H->ncontrib <= out->pool_capacity;
  *handle = H;
  return SK_OK;
}

int sk_reco_event_counts(void* handle, int64_t* counts) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H) return set_error(SK_ERR_INVALID, "null handle");
  for (int i = 0; i < H->nevents; ++i) counts[i] = H->counts[i];
  return SK_OK;
}

int sk_reco_write(void* handle, const sk_reco_out* out, uintptr_t stream) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H || !out) return set_error(SK_ERR_INVALID, "null handle or output");
  if (out->particle_capacity < H->np || out->pool_capacity < H->ncontrib)
    return set_error(SK_ERR_RANGE, "output holds %lld particles / %lld contributors, the run has %lld / %lld",
                     static_cast<long long>(out->particle_capacity), static_cast<long long>(out->pool_capacity),
                     static_cast<long long>(H->np), static_cast<long long>(H->ncontrib));
  DeviceState* ds = nullptr;
  int rc = device_state(H->device, &ds);
  if (rc) return rc;
  cudaStream_t s = resolve_stream(H->device, stream);
  int64_t mmax = 0;
  for (int i = 0; i < H->nevents; ++i) mmax = std::max(mmax, H->counts[i]);
  const unsigned chunks =
      static_cast<unsigned>(std::min<int64_t>((mmax + reco::RANK_PER_CTA - 1) / reco::RANK_PER_CTA, 65535));
  return reco::queue_write(H, out, s, ds, std::max(chunks, 1u));
}

int sk_reco_free(void* handle, uintptr_t stream) {
  auto* H = static_cast<reco::Handle*>(handle);
  if (!H) return SK_OK;
  cudaStream_t s = resolve_stream(H->device, stream);
  reco::release_ws(H, s);
  delete H;
  return SK_OK;
}

}  // extern "C"
