/*
 * soakit_b200.h -- C-ABI boundary of the B200-native layout-conversion and
 * transfer engine (libsoakit_b200.so).
 *
 * The reference (soakit 0.1.0, pure Python + numpy) has no native boundary;
 * its hot path is reached through three Python registries. Every entry point
 * below replaces one reference function on that path; the citation after each
 * declaration names it. The Python host package (paper_2511_04853_b200) binds
 * these with ctypes; INTEGRATION.md shows the binding a soakit maintainer would
 * add.
 *
 * Conventions
 *   - every entry point returns an int status, SK_OK == 0;
 *     sk_last_error() returns a thread-local message for the last failure;
 *   - the caller owns every pointer; nothing is retained after return except
 *     in-flight asynchronous work on the given stream;
 *   - streams are cudaStream_t values passed as uintptr_t (0 = the library's
 *     per-device stream, see sk_stream_default);
 *   - sizes are bytes unless the name says records/elements.
 */
#ifndef SOAKIT_B200_H
#define SOAKIT_B200_H

#ifndef __CUDACC_RTC__ /* the library also compiles its kernels at run time (NVRTC) */
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to soakit exceptions in one place, _native.py) -- */
enum {
  SK_OK = 0,
  SK_ERR_ALLOC = 1,       /* -> AllocationError          (memctx.py:115-123, 188-193) */
  SK_ERR_RANGE = 2,       /* -> CopyError                (memctx.py:259-264)          */
  SK_ERR_UNSUPPORTED = 3, /* -> UnsupportedTransferError (transfer.py:113-116)        */
  SK_ERR_INVALID = 4,     /* -> SoakitError (bad descriptor / argument)               */
  SK_ERR_CUDA = 5,        /* -> MemoryContextError (any other CUDA runtime failure)   */
  SK_ERR_NO_DEVICE = 6    /* -> MemoryContextError (no usable B200 / driver)          */
};

/* ---- scalar type codes; order follows schema.py:37 _SCALAR_CODES -------- */
enum {
  SK_BOOL = 0, SK_U8 = 1, SK_U16 = 2, SK_U32 = 3, SK_U64 = 4,
  SK_I32 = 5, SK_I64 = 6, SK_F32 = 7, SK_F64 = 8
};

/* ---- endpoint kinds of a conversion ------------------------------------- */
enum {
  SK_KIND_AOS = 0,    /* packed records, stride = record bytes (layouts.py:573-598)     */
  SK_KIND_PLANES = 1, /* one contiguous plane per field (layouts.py:459-460, 545-546)   */
  SK_KIND_AOSOA = 2   /* tiles of T lanes; per tile one T-element block per field       */
};

#define SK_MAX_FIELDS 64

/* One field (one slot of one leaf) of a conversion. */
typedef struct sk_field {
  int32_t src_type;      /* SK_BOOL..SK_F64 */
  int32_t dst_type;      /* == src_type for raw moves; else a numpy-astype cast */
  int64_t src_off;       /* AOS: byte offset in the record; AOSOA: byte offset of the
                            field's block inside a tile; PLANES: unused */
  int64_t dst_off;
  const void* src_plane; /* PLANES: address of element 0 of this field's plane */
  void* dst_plane;
} sk_field;

/* A whole-collection conversion: records [0, n) of src -> records [0, n) of dst. */
typedef struct sk_conv_desc {
  int64_t n;             /* records */
  int32_t src_kind;      /* SK_KIND_* */
  int32_t dst_kind;
  const void* src;       /* AOS/AOSOA base (record/tile 0); NULL for PLANES */
  void* dst;
  int64_t src_stride;    /* AOS: record stride; AOSOA: tile stride (bytes) */
  int64_t dst_stride;
  int32_t src_lanes;     /* AOSOA lanes per tile (power of two, 1..1024) */
  int32_t dst_lanes;
  int32_t nfields;       /* 1..SK_MAX_FIELDS */
  int32_t flags;         /* reserved, 0 */
  sk_field fields[SK_MAX_FIELDS];
} sk_conv_desc;

#ifndef __CUDACC_RTC__
/* ---- diagnostics ---------------------------------------------------------- */
const char* sk_last_error(void);
int sk_version(void);                     /* 0x00MMmmpp */
int sk_device_count(int* count);
int sk_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                   size_t* total_mem);

/* ---- memory context plugin (memctx.py:91-156, 288-298) -------------------- */
/* Device allocation, stream-ordered on the device's library stream.
   Replaces MemoryContext.allocate/deallocate (memctx.py:115-133). */
int sk_malloc(int device, size_t nbytes, void** out);
int sk_free(int device, void* ptr);
/* Page-locked host allocation for the "pinned" context (no reference analog:
   the reference only has pageable numpy buffers, memctx.py:120). */
int sk_host_alloc_pinned(size_t nbytes, void** out);
int sk_host_free_pinned(void* ptr);
int sk_host_register(void* ptr, size_t nbytes);   /* pin existing host memory */
int sk_host_unregister(void* ptr);

/* Streams and events (plumbing; the reference is synchronous, memctx.py:316). */
int sk_stream_default(int device, uintptr_t* stream);
int sk_stream_sync(uintptr_t stream);
int sk_device_sync(int device);
int sk_event_create(uintptr_t* event);
int sk_event_destroy(uintptr_t event);
int sk_event_record(uintptr_t event, uintptr_t stream);
int sk_event_elapsed_ms(uintptr_t start, uintptr_t stop, float* ms);

/* memset (MemoryContext.memset, memctx.py:135-143). */
int sk_memset_async(void* dst, int byte, size_t nbytes, uintptr_t stream);
/* Byte copy between any two placements (host, pinned, device, peer device);
   replaces _default_copier (memctx.py:350-360) for every context pair that
   touches a device. Ranges must not overlap (use sk_memmove_async). */
int sk_memcpy_async(void* dst, const void* src, size_t nbytes, uintptr_t stream);
/* Overlap-safe copy inside one allocation: the memmove contract of
   memcopy_with_context (memctx.py:314-316, 356-357; test_acceptance.py:558-583). */
int sk_memmove_async(void* dst, const void* src, size_t nbytes, uintptr_t stream);
/* Batched row moves of one layout splice (LayoutInstance insert / erase /
   resize, layouts.py:298-367): every stream of a size tag shifts its tail and
   zero-fills new rows in two launches, instead of one copy per plane. Each
   op moves `bytes` from src to dst (memmove semantics: an op may overlap
   itself); src == NULL zero-fills dst. Zero fills apply after every move has
   read its source; distinct ops' destinations must not overlap. Device
   memory only (host buffers are spliced on the host). */
typedef struct sk_move {
  void* dst;
  const void* src;
  uint64_t bytes;
} sk_move;
int sk_move_batch_async(const sk_move* ops, int count, uintptr_t stream);
/* Enable NVLink peer access from `device` to `peer` (idempotent). */
int sk_peer_enable(int device, int peer);

/* ---- transfer-spec plugin: the conversion engine (transfer.py:171-236) ----- */
/* K1 aos->planes, K2 planes->aos, K3 ->aosoa with subset/reorder/cast, and
   any other kind pair. Placement of the src/dst pointers is discovered from the
   pointers: all on `device` -> one kernel launch; src and/or dst in host memory
   -> chunked pipeline (H2D copy | convert | D2H copy on separate streams, the
   conversion never runs on the CPU); src on a peer device -> the kernel on
   `device` pulls the bytes over NVLink. Replaces _per_leaf_execute's
   per-leaf gather + staging (transfer.py:182-233). */
int sk_convert(const sk_conv_desc* desc, int device, uintptr_t stream);
/* CUDA-graph capture of the device's library stream: everything enqueued on
   it (and on the pipeline's helper streams) between begin and end -- e.g. a
   whole transfer with its chunked copies and conversion launches -- becomes
   one executable graph replayed with a single launch. Operations that cannot
   be captured (pageable-host copies, synchronisation) make end fail. */
int sk_capture_begin(int device);
int sk_capture_end(int device, void** graph_exec);
int sk_graph_launch(void* graph_exec, int device);
int sk_graph_destroy(void* graph_exec);
/* Diagnostic: generate the record-signature-specialised transform the engine
   would JIT (NVRTC) for `desc` (epi_fields: the 7 sensor field indices of the
   fused case-study path, or NULL), copy its source to source_out, and compile
   it for sm_100a without launching. SK_ERR_UNSUPPORTED: not eligible. */
int sk_convert_specialize_check(const sk_conv_desc* desc, const int* epi_fields,
                                char* source_out, size_t capacity, size_t* source_len);
/* Dry run: validates `desc` and reports the tiling the engine would use. */
int sk_convert_plan(const sk_conv_desc* desc, int device, int* records_per_tile,
                    int* stages, int* mode, size_t* smem_bytes, int* grid);

/* ---- jagged packer (collection.py:537-556, transfer.py:297-320) ------------ */
/* Scratch needed by sk_jagged_scan for n records. */
int sk_jagged_scratch_bytes(int64_t n, size_t* nbytes);
/* Exclusive prefix sum of n segment lengths into prefix[0..n] (prefix[0] = 0),
   computed in int64 and stored truncated to prefix_type exactly like
   np.cumsum(int64).astype(index dtype) (collection.py:554). Single pass,
   decoupled look-back. *total_dev receives the int64 grand total (device ptr). */
int sk_jagged_scan(int64_t n, const void* lens, int lens_type, void* prefix,
                   int prefix_type, void* scratch, size_t scratch_bytes,
                   int64_t* total_dev, uintptr_t stream);
/* Gather every record's members from a source pool into packed per-field pools:
   member j of record i (j < len_i) is read from
   src_pool + (src_off[i] + j) * member_stride + field_off[f] and written to
   dst_pools[f][prefix[i] + j]. prefix must be the non-wrapped prefix (pass an
   SK_I64 prefix when the index type wrapped). Replaces np.concatenate over the
   segments (collection.py:546-556) and the multi-leaf split (transfer.py:301-320). */
int sk_jagged_scatter(int64_t n, const void* prefix, int prefix_type,
                      const int64_t* src_off, const void* src_pool,
                      int64_t member_stride, int nfields, const int64_t* field_off,
                      const int32_t* field_size, void* const* dst_pools,
                      int64_t total, uintptr_t stream);

/* Validation of a pack's inputs: *bad_dev (device int64, zeroed first) counts
   the records with a negative length or a non-empty segment
   [src_off, src_off + len) outside [0, src_members) of the source pool. The
   reference raises before it mutates anything (np.asarray of each segment,
   collection.py:546); callers with device-resident inputs run this first. */
int sk_jagged_validate(int64_t n, const void* lens, int lens_type, const int64_t* src_off,
                       int64_t src_members, int64_t* bad_dev, uintptr_t stream);
/* scan + gather in one call with no host round trip: the gather is
   sized by the pools' `capacity` (members) and reads the true total on the
   device, so it is complete iff total <= capacity. total_dev points at TWO
   device int64: [0] the total, [1] the count of invalid records (as
   sk_jagged_validate; src_pool holds src_members member records). The caller
   reads both afterwards: invalid records -> nothing was gathered for their
   sub-tiles (the prefix is written regardless), raise; total > capacity ->
   grow the pools and gather again with sk_jagged_scatter. One naturally
   aligned 4/8-byte member field (a 16-byte-aligned scratch) runs as ONE
   launch: 2048-record tiles, register gather, 128-bit look-back words tagged
   with the launch generation (nothing in the scratch is zeroed between
   calls). 2-4 such fields of an 8/16-byte member record (16-byte-aligned
   pool) run as one kernel behind a scratch-zeroing launch. Either kernel
   needs no co-residency of its CTAs beyond in-order dispatch (a CTA only
   waits on lower-indexed blocks' published totals). Other member layouts run
   validate, scan and gather back to
   back. Scratch: at least sk_jagged_scratch_bytes; with
   (ceil(capacity / 256) + 1) * 8 more bytes after it (256-aligned) the
   two-kernel path allocates nothing (the scan writes the gather's work split
   there). The scratch is not retained after the call's work completes. */
int sk_jagged_pack(int64_t n, const void* lens, int lens_type, void* prefix,
                   int prefix_type, const int64_t* src_off, const void* src_pool,
                   int64_t src_members, int64_t member_stride, int nfields,
                   const int64_t* field_off, const int32_t* field_size,
                   void* const* dst_pools, int64_t capacity, void* scratch,
                   size_t scratch_bytes, int64_t* total_dev, uintptr_t stream);
/* Sharded jagged collections (no reference counterpart -- the
   reference has no sharding): after each shard packed locally and the shard
   totals were exclusive-scanned across ranks, prefix[0..count) += offset in
   the index dtype's modular arithmetic, which makes the shard's prefix the
   exact slice of the unsharded np.cumsum(...).astype(idx)
   (collection.py:553-554). */
int sk_jagged_rebase(int64_t count, void* prefix, int prefix_type, int64_t offset,
                     uintptr_t stream);

/* Diagnostics only: the fused pack's per-CTA timestamps (globaltimer ns:
   start, block prefix known, blocks done, exit), recorded when the
   environment variable SK_FUSED_DBG has bit 8 set. */
int sk_jagged_trace(void* host, size_t bytes);

/* ---- behavior plugin: the case-study per-object kernel (detector/schemas.py) */
/* energy = A * f32(counts) + B, two f32 roundings, no FMA
   (calibrate_collection, detector/schemas.py:29-33). */
int sk_sensor_calibrate(int64_t n, const uint64_t* counts, const float* a,
                        const float* b, float* energy, uintptr_t stream);
/* noise = nA * sqrt(max(E, 0)) + nB, doubled where noisy
   (noise_for_collection, detector/schemas.py:36-41). */
int sk_sensor_noise(int64_t n, const float* energy, const float* na,
                    const float* nb, const uint8_t* noisy, float* noise,
                    uintptr_t stream);
/* Fused transfer + case study: AoS sensor records (30 B, SENSOR_AOS_DTYPE,
   detector/baselines.py:19-35) -> per_field planes with energy computed and the
   noise column written, one pass over HBM. `desc` is an AOS->PLANES conversion
   of the Sensor plan; field indices name the leaves inside desc->fields. */
int sk_sensor_convert_calibrate(const sk_conv_desc* desc, int f_counts,
                                int f_energy, int f_noisy, int f_a, int f_b,
                                int f_na, int f_nb, float* noise, int device,
                                uintptr_t stream);

/* Deterministic sensor events on the device (detector/events.py:85-133):
   nevents events of w*h cells, event e drawn from the splitmix64 stream of
   seeds[e] (host array). Per cell: type = draw0 & 3, counts = draw1 & 15,
   noisy = draw2 % 50 == 0, calibration parameters by type from draws 0..15;
   then n_dep deposits per event add int(amp * footprint[dy][dx]) to a 5x5
   window (footprint25 = the reference's exp(-(dx^2+dy^2)/2.88) table, row
   major, passed from the host so every bit matches the reference's libm).
   Writes per_field planes of nevents*w*h records; energy is zeroed. */
int sk_sensor_generate(int64_t w, int64_t h, const uint64_t* seeds, int nevents,
                       int64_t n_dep, const double* footprint25, uint8_t* type,
                       uint64_t* counts, uint8_t* noisy, float* a, float* b, float* na,
                       float* nb, float* energy, uintptr_t stream);

/* Particle reconstruction (reconstruct_arrays, detector/reconstruct.py:53-136)
   over nevents calibrated events of w x h cells (energy/noise/type/noisy
   planes, event-major). Round-synchronous parallel greedy over the seeds'
   blockers: same particles in the same order as the reference's sequential
   seed walk. The output is per_field planes of a Particle collection
   (reconstruct.py:172-194): the attribute planes (the 4-wide arrays as 4 slot
   planes each), the sensor lists' prefix plane (particle_capacity + 1 entries
   of sensor_prefix_type) and pool (u64 cell indices inside the event). */
typedef struct sk_reco_out {
  float* energy;
  float* x;
  float* y;
  uint64_t* origin;
  float* x_variance;
  float* y_variance;
  float* significance[4];
  float* e_contribution[4];
  uint8_t* noisy_count[4];
  void* sensor_prefix;
  int sensor_prefix_type;
  uint64_t* sensor_pool;
  int64_t particle_capacity; /* rows of each particle plane */
  int64_t pool_capacity;     /* cells of sensor_pool */
} sk_reco_out;
/* Runs the reconstruction; with `out`, the write into it is queued behind the
   rounds, and one host synchronisation covers both. *written = 1 when the
   particles and their sensor lists fit out's capacities; otherwise grow the
   output to *nparticles / *ncontributors and call sk_reco_write. The handle
   keeps the particles and per-event counts until sk_reco_free. */
int sk_reco_run(int64_t w, int64_t h, int nevents, const float* energy,
                const float* noise, const uint8_t* type, const uint8_t* noisy,
                const sk_reco_out* out, int device, uintptr_t stream, void** handle,
                int64_t* nparticles, int64_t* ncontributors, int* rounds,
                int* written);
int sk_reco_event_counts(void* handle, int64_t* counts);
/* Queue the write into an output large enough for the run (SK_ERR_RANGE otherwise). */
int sk_reco_write(void* handle, const sk_reco_out* out, uintptr_t stream);
int sk_reco_free(void* handle, uintptr_t stream);

/* ---- synthetic inputs ------------------------------------------------------- */
/* Fill nbytes of device memory with splitmix64(seed, first_word + word index)
   bits (counter-based, so a shard starting at 8-byte word `first_word` of the
   global image regenerates exactly its slice): the seeded synthetic record
   images the benches convert. */
int sk_fill_random(void* dst, size_t nbytes, uint64_t seed, uint64_t first_word,
                   uintptr_t stream);
/* Count the bytes where a[i] != b[i] into *mismatches (device memory; zeroed
   first, on the stream): full-size identity checks of round trips (AoS ->
   planes -> AoS) without copying the collections to the host. A verification
   utility, not a reference interface. */
int sk_compare_bytes(const void* a, const void* b, size_t nbytes, unsigned long long* mismatches,
                     uintptr_t stream);

/* ---- multi-GPU shards: CUDA IPC for cross-process peer pulls --- */
/* cudaMalloc'd (IPC-exportable) device memory; pool allocations from sk_malloc
   cannot be exported through cudaIpcGetMemHandle. */
int sk_malloc_shareable(int device, size_t nbytes, void** out);
int sk_free_shareable(int device, void* ptr);
int sk_ipc_handle_size(size_t* nbytes);
int sk_ipc_get_handle(void* dev_ptr, void* handle_out);
int sk_ipc_open_handle(int device, const void* handle, void** dev_ptr);
int sk_ipc_close_handle(int device, void* dev_ptr);
#endif /* !__CUDACC_RTC__ */

#ifdef __cplusplus
}
#endif

#endif /* SOAKIT_B200_H */
