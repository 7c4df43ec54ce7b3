// Record-signature specialisation of the conversion engine (NVRTC).
//
// The ahead-of-time kernel reads field offsets and types from the Plan at run
// time, so records whose fields are not 4-byte aligned (Sensor, 30 B) or need a
// cast go through per-element funnel-shift reads in shared memory. For such a
// signature this file generates a transform in which one thread owns a group
// of G records that is 4-byte aligned in the AoS tile (G = 4 / gcd(stride, 4)):
// it loads the group's words once (conflict-free, the group stride is odd in
// words or vector-aligned), extracts every field with compile-time shifts /
// funnel shifts, applies compile-time casts, and writes the G values of each
// field with one vector store. The reverse direction assembles the group's
// words from vector loads of the planes. The case-study epilogue is fused into
// the same pass (values never leave registers). The kernel framework (TMA ring,
// bulk stores) is the same source as the ahead-of-time build; NVRTC compiles
// it for sm_100a once per signature and the cubin is cached in-process.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "sk_internal.cuh"
#include "sk_conv_device.cuh"
#include "sk_rtc_sources.inc"

namespace sk {
namespace conv {

// ---- NVRTC, loaded on demand ---------------------------------------------------------

typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;

struct Nvrtc {
  bool ok = false;
  std::string why;
  nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*log)(nvrtcProgram_t, char*);
  nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*cubin)(nvrtcProgram_t, char*);
  nvrtcResult_t (*add_name)(nvrtcProgram_t, const char*);
  nvrtcResult_t (*lowered)(nvrtcProgram_t, const char*, const char**);
  nvrtcResult_t (*destroy)(nvrtcProgram_t*);
};

static Nvrtc& nvrtc() {
  static Nvrtc n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
  void* h = nullptr;
  for (const char* nm : names)
    if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) {
    n.why = "libnvrtc not found";
    return n;
  }
  bool all = true;
  auto sym = [&](const char* s) {
    void* p = dlsym(h, s);
    all = all && p;
    return p;
  };
  n.create = reinterpret_cast<decltype(n.create)>(sym("nvrtcCreateProgram"));
  n.compile = reinterpret_cast<decltype(n.compile)>(sym("nvrtcCompileProgram"));
  n.log_size = reinterpret_cast<decltype(n.log_size)>(sym("nvrtcGetProgramLogSize"));
  n.log = reinterpret_cast<decltype(n.log)>(sym("nvrtcGetProgramLog"));
  n.cubin_size = reinterpret_cast<decltype(n.cubin_size)>(sym("nvrtcGetCUBINSize"));
  n.cubin = reinterpret_cast<decltype(n.cubin)>(sym("nvrtcGetCUBIN"));
  n.add_name = reinterpret_cast<decltype(n.add_name)>(sym("nvrtcAddNameExpression"));
  n.lowered = reinterpret_cast<decltype(n.lowered)>(sym("nvrtcGetLoweredName"));
  n.destroy = reinterpret_cast<decltype(n.destroy)>(sym("nvrtcDestroyProgram"));
  n.ok = all;
  if (!all) n.why = "libnvrtc lacks required symbols";
  return n;
}

// ---- code generation -------------------------------------------------------------------

static const char* ctype(int t) {
  switch (t) {
    case SK_BOOL: case SK_U8: return "uint8_t";
    case SK_U16: return "uint16_t";
    case SK_U32: case SK_I32: case SK_F32: return "uint32_t";
    default: return "uint64_t";
  }
}

static int gcd_int(int a, int b) {
  while (b) { int t = a % b; a = b; b = t; }
  return a;
}

// value bits (as uint64_t expression) of `isz` bytes at group byte offset b
static std::string extract(int b, int isz) {
  std::ostringstream o;
  const int k = b / 4, sh = b % 4;
  auto word4 = [&](int bb) {
    const int kk = bb / 4, s = bb % 4;
    std::ostringstream w;
    if (s == 0) w << "W" << kk;
    else w << "__funnelshift_r(W" << kk << ", W" << kk + 1 << ", " << 8 * s << ")";
    return w.str();
  };
  if (isz == 8) {
    o << "((static_cast<uint64_t>(" << word4(b + 4) << ") << 32) | static_cast<uint64_t>(" << word4(b) << "))";
  } else if (isz == 4) {
    o << "static_cast<uint64_t>(" << word4(b) << ")";
  } else {
    const unsigned mask = isz == 2 ? 0xffffu : 0xffu;
    if (sh + isz <= 4)
      o << "static_cast<uint64_t>((W" << k << " >> " << 8 * sh << ") & 0x" << std::hex << mask << std::dec << "u)";
    else
      o << "static_cast<uint64_t>(" << word4(b) << " & 0x" << std::hex << mask << std::dec << "u)";
  }
  return o.str();
}

// a vector store of G consecutive values of `dsz` bytes (value names v_<f>_<i>)
static void emit_group_store(std::ostringstream& o, const std::string& addr, int f, int G, int dsz,
                             const std::string& val_prefix) {
  const int bytes = G * dsz;
  auto val = [&](int i) { return val_prefix + std::to_string(f) + "_" + std::to_string(i); };
  o << "        if (full) {\n";
  if (G == 1) {
    o << "          *reinterpret_cast<" << (dsz == 1 ? "uint8_t" : dsz == 2 ? "uint16_t" : dsz == 4 ? "uint32_t"
                                                                                     : "uint64_t")
      << "*>(" << addr << ") = static_cast<" << (dsz == 8 ? "uint64_t" : dsz == 4 ? "uint32_t" : dsz == 2 ? "uint16_t"
                                                                                                    : "uint8_t")
      << ">(" << val(0) << ");\n";
  } else if (bytes <= 8) {
    const char* wt = bytes == 2 ? "uint16_t" : bytes == 4 ? "uint32_t" : "uint64_t";
    o << "          *reinterpret_cast<" << wt << "*>(" << addr << ") = static_cast<" << wt << ">(";
    for (int i = 0; i < G; ++i) o << (i ? " | " : "") << "(" << val(i) << " << " << 8 * dsz * i << ")";
    o << ");\n";
  } else {
    // 16 or 32 bytes: uint4 stores built from 32-bit lanes
    const int nq = bytes / 16;
    for (int q = 0; q < nq; ++q) {
      o << "          { uint4 q; ";
      for (int l = 0; l < 4; ++l) {
        const int byte0 = q * 16 + l * 4;  // 4-byte lane: part of one value (dsz >= 4 here)
        const int i = byte0 / dsz, within = byte0 % dsz;
        o << "q." << "xyzw"[l] << " = static_cast<uint32_t>(" << val(i) << " >> " << 8 * within << "); ";
      }
      o << "*reinterpret_cast<uint4*>(" << addr << " + " << q * 16 << ") = q; }\n";
    }
  }
  o << "        } else {\n";
  for (int i = 0; i < G; ++i) {
    const char* st = dsz == 1 ? "uint8_t" : dsz == 2 ? "uint16_t" : dsz == 4 ? "uint32_t" : "uint64_t";
    o << "          if (r0 + " << i << " < rows) *reinterpret_cast<" << st << "*>(" << addr << " + " << i * dsz
      << ") = static_cast<" << st << ">(" << val(i) << ");\n";
  }
  o << "        }\n";
}

struct Spec {
  std::string source;
  std::string key;
};

// AoS source (any destination kind whose G consecutive records are contiguous
// per field: PLANES, or AOSOA with lanes % G == 0) or PLANES source -> AoS.
// Neither side AoS (PLANES <-> AOSOA, AOSOA <-> AOSOA): one thread moves 4
// consecutive records of every field -- 4 typed shared-memory loads, a
// compile-time cast, one vector store of the 4 values (both layouts keep 4
// consecutive records of a field contiguous when the AoSoA width is a
// multiple of 4).
static bool generate_blocks(const sk_conv_desc& d, const Plan& P, Spec* out) {
  constexpr int G = 4;
  auto kind_ok = [&](int kind, int64_t lanes, int64_t stride, bool dst) {
    if (kind == SK_KIND_PLANES) return true;
    if (kind != SK_KIND_AOSOA || lanes % G || stride % 16) return false;
    for (int f = 0; f < d.nfields; ++f)
      if ((dst ? d.fields[f].dst_off : d.fields[f].src_off) % 16) return false;
    return true;
  };
  if (P.epi || !kind_ok(d.src_kind, d.src_lanes, d.src_stride, false) ||
      !kind_ok(d.dst_kind, d.dst_lanes, d.dst_stride, true) ||
      (d.src_kind == SK_KIND_PLANES && d.dst_kind == SK_KIND_PLANES))
    return false;
  std::ostringstream k;
  k << "b1|" << d.src_kind << "," << d.dst_kind << "," << d.src_lanes << "," << d.dst_lanes << ","
    << (d.src_kind == SK_KIND_AOSOA ? d.src_stride : 0) << "," << (d.dst_kind == SK_KIND_AOSOA ? d.dst_stride : 0);
  for (int i = 0; i < d.nfields; ++i) k << "|" << d.fields[i].src_type << "," << d.fields[i].dst_type;
  std::ostringstream o;
  o << "#include \"sk_conv_device.cuh\"\nnamespace sk {\nnamespace conv {\n";
  o << "struct SpecTransform {\n  static constexpr bool kFusedEpilogue = false;\n";
  o << "  __device__ __forceinline__ static void run(const Plan& P, const uint8_t* __restrict__ in, "
       "uint8_t* __restrict__ out, int rows, const int32_t*) {\n";
  o << "    const int ngroups = (rows + " << G - 1 << ") / " << G << ";\n";
  o << "#pragma unroll 1\n    for (int g = threadIdx.x; g < ngroups; g += NT) {\n";
  o << "      const int r0 = g * " << G << ";\n      const bool full = r0 + " << G << " <= rows;\n";
  for (int f = 0; f < d.nfields; ++f) {
    const sk_field& F = d.fields[f];
    const int ssz = dtype_size(F.src_type);
    const char* st = ctype(F.src_type);
    o << "      {\n        const uint8_t* s = in + P.f[" << f << "].sloc + ";
    if (d.src_kind == SK_KIND_PLANES)
      o << "r0 * " << ssz << ";\n";
    else
      o << "(r0 >> " << P.src_lshift << ") * " << d.src_stride << " + (r0 & " << d.src_lanes - 1 << ") * " << ssz
        << ";\n";
    for (int i = 0; i < G; ++i)
      o << "        const uint64_t v" << f << "_" << i << " = cast_bits((full || r0 + " << i << " < rows) ? "
        << "static_cast<uint64_t>(*reinterpret_cast<const " << st << "*>(s + " << i * ssz << ")) : 0ull, "
        << F.src_type << ", " << F.dst_type << ");\n";
    const int dsz = dtype_size(F.dst_type);
    std::ostringstream addr;
    if (d.dst_kind == SK_KIND_PLANES)
      addr << "(out + P.f[" << f << "].dloc + r0 * " << dsz << ")";
    else
      addr << "(out + P.f[" << f << "].dloc + (r0 >> " << P.dst_lshift << ") * " << d.dst_stride << " + (r0 & "
           << d.dst_lanes - 1 << ") * " << dsz << ")";
    emit_group_store(o, addr.str(), f, G, dsz, "v");
    o << "      }\n";
  }
  o << "    }\n  }\n};\n}  // namespace conv\n}  // namespace sk\n";
  out->source = o.str();
  out->key = k.str();
  return true;
}

static bool generate(const sk_conv_desc& d, const Plan& P, const int* epi_fields, Spec* out) {
  const bool a2x = d.src_kind == SK_KIND_AOS && (d.dst_kind == SK_KIND_PLANES || d.dst_kind == SK_KIND_AOSOA);
  const bool p2a = (d.src_kind == SK_KIND_PLANES || d.src_kind == SK_KIND_AOSOA) && d.dst_kind == SK_KIND_AOS;
  if (d.src_kind != SK_KIND_AOS && d.dst_kind != SK_KIND_AOS) return generate_blocks(d, P, out);
  if (!a2x && !p2a) return false;
  const int S = static_cast<int>(a2x ? d.src_stride : d.dst_stride);
  const int G = 4 / gcd_int(S, 4);
  const int GB = G * S, GW = GB / 4;
  if (GB > 128) return false;
  if (a2x && d.dst_kind == SK_KIND_AOSOA) {  // G lanes of a tile must be one aligned vector per field
    if ((d.dst_lanes % G) != 0 || d.dst_stride % 16) return false;
    for (int f = 0; f < d.nfields; ++f)
      if (d.fields[f].dst_off % 16) return false;
  }
  if (P.epi && !a2x) return false;

  std::ostringstream k;  // the signature: everything the generated code bakes in
  k << "v1|" << d.src_kind << "," << d.dst_kind << "," << S << "," << G << "," << P.epi << "," << d.src_lanes << ","
    << (d.src_kind == SK_KIND_AOSOA ? d.src_stride : 0);
  for (int i = 0; i < d.nfields; ++i)
    k << "|" << d.fields[i].src_type << "," << d.fields[i].dst_type << "," << d.fields[i].src_off << ","
      << d.fields[i].dst_off;
  if (P.epi)
    for (int i = 0; i < 7; ++i) k << "|e" << epi_fields[i];

  std::ostringstream o;
  o << "#include \"sk_conv_device.cuh\"\nnamespace sk {\nnamespace conv {\n";
  o << "struct SpecTransform {\n  static constexpr bool kFusedEpilogue = " << (P.epi ? "true" : "false") << ";\n";
  o << "  __device__ __forceinline__ static void run(const Plan& P, const uint8_t* __restrict__ in, "
       "uint8_t* __restrict__ out, int rows, const int32_t*) {\n";
  o << "    const int ngroups = (rows + " << G - 1 << ") / " << G << ";\n";
  o << "#pragma unroll 1\n    for (int g = threadIdx.x; g < ngroups; g += NT) {\n";
  o << "      const int r0 = g * " << G << ";\n      const bool full = r0 + " << G << " <= rows;\n";
  if (a2x) {
    o << "      const uint32_t* w = reinterpret_cast<const uint32_t*>(in) + g * " << GW << ";\n";
    if (GW % 4 == 0) {
      // an even group stride in words puts many lanes on one bank: 16-byte loads cut the conflicts 4x
      for (int q = 0; q < GW / 4; ++q) {
        o << "      const uint4 Q" << q << " = reinterpret_cast<const uint4*>(w)[" << q << "];\n";
        for (int l = 0; l < 4; ++l) o << "      const uint32_t W" << 4 * q + l << " = Q" << q << "." << "xyzw"[l] << ";\n";
      }
    } else {
      for (int q = 0; q < GW; ++q) o << "      const uint32_t W" << q << " = w[" << q << "];\n";
    }
    // extract + cast every field of every record
    for (int f = 0; f < d.nfields; ++f) {
      const sk_field& F = d.fields[f];
      const int ssz = dtype_size(F.src_type);
      for (int i = 0; i < G; ++i)
        o << "      const uint64_t v" << f << "_" << i << " = cast_bits(" << extract(i * S + static_cast<int>(F.src_off), ssz)
          << ", " << F.src_type << ", " << F.dst_type << ");\n";
    }
    int e_energy = -1;
    if (P.epi) {
      const int* fi = epi_fields;  // counts, energy, noisy, A, B, nA, nB
      e_energy = fi[1];
      for (int i = 0; i < G; ++i) {
        auto v = [&](int idx) { return "v" + std::to_string(fi[idx]) + "_" + std::to_string(i); };
        o << "      const float e_" << i << " = sensor_energy(" << v(0) << ", __uint_as_float(static_cast<uint32_t>("
          << v(3) << ")), __uint_as_float(static_cast<uint32_t>(" << v(4) << ")));\n";
        o << "      const uint64_t ve" << e_energy << "_" << i << " = __float_as_uint(e_" << i << ");\n";
        o << "      const uint64_t vn0_" << i << " = __float_as_uint(sensor_noise(e_" << i
          << ", __uint_as_float(static_cast<uint32_t>(" << v(5) << ")), __uint_as_float(static_cast<uint32_t>("
          << v(6) << ")), (" << v(2) << " & 0xffu) != 0));\n";
      }
    }
    for (int f = 0; f < d.nfields; ++f) {
      const int dsz = dtype_size(d.fields[f].dst_type);
      std::ostringstream addr;
      if (d.dst_kind == SK_KIND_PLANES)
        addr << "(out + P.f[" << f << "].dloc + r0 * " << dsz << ")";
      else
        addr << "(out + (r0 >> P.dst_lshift) * P.dst_A + (r0 & P.dst_msk) * " << dsz << " + P.f[" << f << "].dloc)";
      o << "      {\n";
      emit_group_store(o, addr.str(), f, G, dsz, f == e_energy ? "ve" : "v");
      o << "      }\n";
    }
    if (P.epi) {
      o << "      {\n";
      emit_group_store(o, "(out + P.extra_loc + r0 * 4)", 0, G, 4, "vn");
      o << "      }\n";
    }
  } else {
    // planes -> AoS: vector-load the G values of each field, assemble words
    for (int f = 0; f < d.nfields; ++f) {
      const sk_field& F = d.fields[f];
      const int ssz = dtype_size(F.src_type);
      const char* st = ctype(F.src_type);
      for (int i = 0; i < G; ++i) {
        // planes: loc + r * size; AoSoA blocks (lanes, tile baked in): (r >> log2 lanes) * tile + (r & lanes-1) * size + loc
        std::ostringstream a;
        if (d.src_kind == SK_KIND_PLANES)
          a << "(r0 + " << i << ") * " << ssz;
        else
          a << "((r0 + " << i << ") >> " << P.src_lshift << ") * " << d.src_stride << " + ((r0 + " << i
            << ") & " << d.src_lanes - 1 << ") * " << ssz;
        o << "      const uint64_t r" << f << "_" << i << " = (full || r0 + " << i << " < rows) ? static_cast<uint64_t>("
          << "*reinterpret_cast<const " << st << "*>(in + P.f[" << f << "].sloc + " << a.str() << ")) : 0ull;\n";
      }
      for (int i = 0; i < G; ++i)
        o << "      const uint64_t v" << f << "_" << i << " = cast_bits(r" << f << "_" << i << ", " << F.src_type << ", "
          << F.dst_type << ");\n";
    }
    o << "      uint32_t* w = reinterpret_cast<uint32_t*>(out) + g * " << GW << ";\n";
    const bool vec = GW % 4 == 0;  // an even group stride in words: 16-byte stores (4x fewer bank conflicts)
    for (int q = 0; q < GW; ++q) {
      std::ostringstream expr;
      bool any = false;
      for (int f = 0; f < d.nfields; ++f) {
        const int dsz = dtype_size(d.fields[f].dst_type);
        for (int i = 0; i < G; ++i) {
          const int start = i * S + static_cast<int>(d.fields[f].dst_off), end = start + dsz;
          const int lo = std::max(start, 4 * q), hi = std::min(end, 4 * q + 4);
          if (lo >= hi) continue;
          const int len = hi - lo;
          const unsigned long long mask = len == 4 ? 0xffffffffull : ((1ull << (8 * len)) - 1);
          expr << (any ? " | " : "") << "(static_cast<uint32_t>((v" << f << "_" << i << " >> " << 8 * (lo - start)
               << ") & 0x" << std::hex << mask << std::dec << "ull) << " << 8 * (lo - 4 * q) << ")";
          any = true;
        }
      }
      if (vec)
        o << "      const uint32_t O" << q << " = " << (any ? expr.str() : std::string("0u")) << ";\n";
      else
        o << "      w[" << q << "] = " << (any ? expr.str() : std::string("0u")) << ";\n";
      if (vec && q % 4 == 3)
        o << "      reinterpret_cast<uint4*>(w)[" << q / 4 << "] = make_uint4(O" << q - 3 << ", O" << q - 2 << ", O" << q - 1
          << ", O" << q << ");\n";
    }
  }
  o << "    }\n  }\n};\n}  // namespace conv\n}  // namespace sk\n";
  out->source = o.str();
  out->key = k.str();
  return true;
}

// ---- compile + cache -------------------------------------------------------------------

struct Compiled {
  bool ok = false;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  // kernel attributes and occupancy are per device: a signature first launched on cuda:1 must set its
  // dynamic shared memory limit there too
  int max_smem_set[64] = {};
  std::vector<std::pair<int64_t, int>> occ;  // (device << 32 | smem) -> CTAs per SM
};

static std::mutex g_mu;
static std::map<std::string, Compiled>* g_cache = new std::map<std::string, Compiled>();

static bool compile(const Spec& spec, Compiled* c) {
  Nvrtc& nv = nvrtc();
  if (!nv.ok) return false;
  const char* hdrs[] = {kSrc_sk_device_cuh, kSrc_sk_conv_device_cuh, kSrc_soakit_b200_h};
  const char* hnames[] = {kSrc_sk_device_cuh_name, kSrc_sk_conv_device_cuh_name, kSrc_soakit_b200_h_name};
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, spec.source.c_str(), "sk_spec.cu", 3, hdrs, hnames) != 0) return false;
  const char* name_expr = "sk::conv::convert_kernel_t<sk::conv::SpecTransform>";
  nv.add_name(prog, name_expr);
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo"};
  const int rc = nv.compile(prog, 4, opts);
  if (rc != 0) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    nv.log(prog, &log[0]);
    fprintf(stderr, "[soakit_b200] NVRTC specialisation failed (falling back to the generic kernel):\n%s\n",
            log.c_str());
    nv.destroy(&prog);
    return false;
  }
  const char* lowered = nullptr;
  nv.lowered(prog, name_expr, &lowered);
  std::string lname = lowered ? lowered : "";
  size_t nbin = 0;
  nv.cubin_size(prog, &nbin);
  std::vector<char> bin(nbin);
  nv.cubin(prog, bin.data());
  nv.destroy(&prog);
  if (cudaLibraryLoadData(&c->lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (cudaLibraryGetKernel(&c->kernel, c->lib, lname.c_str()) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  c->ok = true;
  return true;
}

static bool specialise_enabled() {
  const char* v = getenv("SK_SPECIALIZE");
  return !(v && v[0] == '0');
}

// Launch the signature-specialised kernel for this plan when it applies.
// *launched = false means: not eligible / unavailable, use the generic kernel.
bool pdl_enabled();  // sk_convert.cu

int launch_specialized(const sk_conv_desc& d, const Plan& P, const DeviceState& ds, const int* epi_fields,
                       cudaStream_t s, bool* launched) {
  *launched = false;
  if (!specialise_enabled() || P.ntiles == 0) return SK_OK;
  // pure word mode is already at the copy roofline -- except out of AoSoA tiles (0.83 vs 0.93+ specialised)
  static const bool force = [] {
    const char* v = getenv("SK_SPECIALIZE");
    return v && v[0] == '2';
  }();
  // word mode with sub-word slots (1-/2-byte fields) in a 16-byte-multiple record (Particle's 64 B with
  // noisy_count[4]) loses to the record-group transform: 0.70 -> 0.88 / 0.92 for Particle AoS <-> planes; in
  // odd-stride records (Sensor, 30 B) word mode stays ahead (planes -> AoS 1.00 vs 0.76)
  const int64_t aos_stride = d.src_kind == SK_KIND_AOS ? d.src_stride : d.dst_kind == SK_KIND_AOS ? d.dst_stride : 0;
  const bool subword_even = P.nsub > 0 && aos_stride % 16 == 0;
  if (P.n_elem == 0 && !P.epi && d.src_kind != SK_KIND_AOSOA && !subword_even && !force) return SK_OK;
  Spec spec;
  if (!generate(d, P, epi_fields, &spec)) return SK_OK;
  Compiled* c = nullptr;
  int dev = 0;
  SK_TRY(cudaGetDevice(&dev));
  dev &= 63;
  const int64_t occ_key = (static_cast<int64_t>(dev) << 32) | static_cast<int64_t>(P.smem_total);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache->find(spec.key);
    if (it == g_cache->end()) {
      Compiled fresh;
      compile(spec, &fresh);  // failures are cached too: one attempt per signature
      it = g_cache->emplace(spec.key, fresh).first;
    }
    c = &it->second;
    if (!c->ok) return SK_OK;
    if (P.smem_total > c->max_smem_set[dev]) {
      if (cudaKernelSetAttributeForDevice(c->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P.smem_total,
                                          dev) != cudaSuccess) {
        cudaGetLastError();
        return SK_OK;
      }
      c->max_smem_set[dev] = P.smem_total;
    }
  }
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const auto& e : c->occ)
      if (e.first == occ_key) per_sm = e.second;
  }
  if (!per_sm) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(c->kernel), NT,
                                                      P.smem_total) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(g_mu);
    c->occ.push_back({occ_key, per_sm});
  }
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(ds.sm_count) * per_sm, P.ntiles));
  void* args[] = {const_cast<Plan*>(&P)};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = P.smem_total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  SK_TRY(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(c->kernel), args));
  *launched = true;
  return SK_OK;
}

}  // namespace conv
}  // namespace sk

// ---- diagnostic entry point: generate + compile without a GPU ---------------------------

namespace sk {
namespace conv {
int make_plan(const sk_conv_desc& d, const DeviceState& ds, bool in_bulk_ok, bool out_bulk_ok, int epi, Plan* out,
              int* grid);  // sk_convert.cu
}  // namespace conv
}  // namespace sk

extern "C" int sk_convert_specialize_check(const sk_conv_desc* desc, const int* epi_fields, char* source_out,
                                           size_t capacity, size_t* source_len) {
  using namespace sk;
  using namespace sk::conv;
  if (!desc) return set_error(SK_ERR_INVALID, "null descriptor");
  DeviceState ds;  // a B200's geometry; nothing is launched
  ds.sm_count = 148;
  ds.max_smem_optin = 232448;
  Plan P;
  int grid = 0;
  const int epi = epi_fields ? EPI_SENSOR : EPI_NONE;
  int rc = make_plan(*desc, ds, true, true, epi, &P, &grid);
  cudaGetLastError();
  if (rc) return rc;
  Spec spec;
  if (!generate(*desc, P, epi_fields, &spec))
    return set_error(SK_ERR_UNSUPPORTED, "descriptor is not eligible for signature specialisation");
  if (source_len) *source_len = spec.source.size();
  if (source_out && capacity) {
    const size_t n = std::min(capacity - 1, spec.source.size());
    memcpy(source_out, spec.source.data(), n);
    source_out[n] = '\0';
  }
  Nvrtc& nv = nvrtc();
  if (!nv.ok) return set_error(SK_ERR_UNSUPPORTED, "NVRTC unavailable: %s", nv.why.c_str());
  const char* hdrs[] = {kSrc_sk_device_cuh, kSrc_sk_conv_device_cuh, kSrc_soakit_b200_h};
  const char* hnames[] = {kSrc_sk_device_cuh_name, kSrc_sk_conv_device_cuh_name, kSrc_soakit_b200_h_name};
  nvrtcProgram_t prog = nullptr;
  if (nv.create(&prog, spec.source.c_str(), "sk_spec.cu", 3, hdrs, hnames) != 0)
    return set_error(SK_ERR_CUDA, "nvrtcCreateProgram failed");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false"};
  const int crc = nv.compile(prog, 3, opts);
  if (crc != 0) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string log(n, '\0');
    nv.log(prog, &log[0]);
    nv.destroy(&prog);
    return set_error(SK_ERR_CUDA, "NVRTC compile failed: %s", log.c_str());
  }
  nv.destroy(&prog);
  return SK_OK;
}
