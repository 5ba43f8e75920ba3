/* lopc.h — C-ABI of liblopc.so, the B200 (sm_100a) LOPC hot path.
 *
 * LOPC (arxiv 2603.26968, PAPER.md): error-bounded quantization (§IV.A,
 * P:109-116), local-order repair of subbins to a fixpoint (§IV.B, Alg. 1
 * P:127-154, Alg. 2), chunked lossless coding (§IV.C)
 * and the matching decoder.  Readings of silent passages and
 * the stream format are in DESIGN.md §3-§4.
 *
 * Conventions for every entry point:
 *  - Grid: dims[0..ndims-1] slowest -> fastest, ndims in {2,3}; values are
 *    row-major with the last dim contiguous (G3).  Each dim and the product
 *    N must be <= 2^40.  N = 0 is allowed (header-only stream).
 *  - dtype: LOPC_F32 or LOPC_F64.
 *  - Buffers are owned by the caller.  The library never frees or retains a
 *    caller pointer after return.  `in`/`out` may be device pointers or host
 *    pointers (pinned or pageable); host buffers are staged through the
 *    workspace with cudaMemcpyAsync inside the call.  All other pointers
 *    (workspace) are device pointers.
 *  - The *_ex calls take an explicit workspace (device memory, >= the size the
 *    matching *_workspace_bytes function returns, 256-byte aligned) and a
 *    cudaStream_t (passed as void*; NULL = legacy default stream).  The plain
 *    calls use a grow-only internal workspace on the current device and the
 *    legacy default stream.  No allocation happens inside *_ex.
 *  - Every call blocks until its result code is known (one device->host read
 *    of the status block at the end, into a pinned slot owned by the calling
 *    host thread).
 *  - Concurrency: calls on different streams with different
 *    workspaces are independent and may run at the same time from different
 *    host threads.  Everything a call writes on the host side is per thread
 *    (status slot, lopc_last_stats, lopc_last_error_string, the side streams
 *    and events of the host-I/O decompress pipeline, the plain calls'
 *    workspace pool), keyed by device.  lopc_set_timing and
 *    lopc_set_repair_engine are process-wide settings.
 *  - Return value: LOPC_OK (0) or a negative LOPC_E_* code.  On LOPC_E_NOSPACE
 *    from a compress call, *out_bytes holds the size required.  Output buffer
 *    contents are unspecified on error.
 *  - Determinism: the same (x, dims, dtype, eps) gives the same bytes for any
 *    launch configuration, stream or GPU (the repair result is the unique least
 *    fixpoint; chunk payloads are placed by a prefix sum).
 *  - NaN, +-Inf and values whose bin exceeds BINMAX (2^31-2 for f32, 2^50 for
 *    f64) are not errors: they are stored losslessly (escapes, G8-G11).
 */
#ifndef LOPC_H
#define LOPC_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define LOPC_ABI_VERSION 1

typedef enum { LOPC_F32 = 0, LOPC_F64 = 1 } lopc_dtype;

enum {
  LOPC_OK = 0,
  LOPC_E_ARG = -1,      /* null pointer, bad dtype, eps not finite / not in [2^-900, 2^1000] */
  LOPC_E_SHAPE = -2,    /* ndims not 2/3, a dim or N > 2^40 */
  LOPC_E_NOSPACE = -3,  /* output or workspace too small */
  LOPC_E_CORRUPT = -4,  /* malformed stream (header, size table or payload) */
  LOPC_E_VERSION = -5,  /* stream version != 1 */
  LOPC_E_CUDA = -6,     /* CUDA runtime error (message: lopc_last_error_string) */
  LOPC_E_NCCL = -7,     /* NCCL failure in the multi-GPU slab mode */
  LOPC_E_INTERNAL = -8  /* a self-check failed (bound re-check a4, subbin overflow, pass cap) */
};

/* Worst-case stream size: 64 + 8C + 2 * 16384 * C bytes, C = ceil(N / (16384/k))
 * (16 kB chunks; raw fallback per payload, reading G23). */
size_t lopc_compress_bound(int ndims, const uint64_t* dims, int dtype);

/* Workspace bytes for lopc_compress_ex.  host_io != 0 adds room to stage a
 * host input (N*k) and a host output (lopc_compress_bound). */
size_t lopc_compress_workspace_bytes(int ndims, const uint64_t* dims, int dtype, int host_io);

/* Workspace bytes for lopc_decompress_ex of a stream of in_bytes bytes that
 * decodes to out_bytes bytes; host_io != 0 adds staging for both. */
size_t lopc_decompress_workspace_bytes(size_t in_bytes, size_t out_bytes, int host_io);

/* Compress x (N values of dtype) with absolute error bound eps (ABS; for NOA
 * the caller passes eps = rel * (max - min)): quantization to bins
 * b = floor(x/eps + 1/2) with the exact double-check (§IV.A, G6-G9),
 * flags and the repair of the subbins to the least fixpoint (§IV.B, Alg. 1
 * P:127-154, Alg. 2; "as low as possible"), the bound
 * self-check a4, and the chunk pipelines DIFF-NB-BIT-RZE (bins,
 * P:90-91) and BIT-RZE_k-RZE_1 (subbins) placed by one
 * prefix sum.  Stream format: DESIGN.md §4.  *out_bytes: in = the
 * capacity of out, out = bytes written (or required, on LOPC_E_NOSPACE).
 * Errors: E_ARG (null in/out/out_bytes, eps outside [2^-900, 2^1000]),
 * E_SHAPE, E_NOSPACE (out or workspace too small), E_CUDA, E_INTERNAL. */
int lopc_compress(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                  size_t* out_bytes);
int lopc_compress_ex(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                     size_t* out_bytes, void* workspace, size_t workspace_bytes, void* stream);

/* Decompress a stream of in_bytes bytes into out (capacity out_capacity
 * bytes, must hold N*k): the inverse chunk pipelines, then per point the
 * value whose key is key(lo(b)) + s ("subbin 0 decodes to the lowest
 * representable value within the bin"; escapes bit-exact, G10); the
 * decoder is "embarrassingly parallel".  The header and size table
 * are validated before any payload is read; corrupt streams return
 * LOPC_E_CORRUPT (LOPC_E_VERSION for a version != 1) without
 * partial-output guarantees; E_NOSPACE if out_capacity < N*k. */
int lopc_decompress(const void* in, size_t in_bytes, void* out, size_t out_capacity);
int lopc_decompress_ex(const void* in, size_t in_bytes, void* out, size_t out_capacity, void* workspace,
                       size_t workspace_bytes, void* stream);

/* Host-side parse of a stream header (host pointer, >= 64
 * bytes).  dims3 gets (d0, d1, d2) with d0 = 1 for 2D.  Any output pointer
 * may be NULL.  E_CORRUPT for a short or malformed header, E_VERSION. */
int lopc_stream_info(const void* host_hdr, size_t n, int* ndims, uint64_t* dims3, int* dtype, double* eps,
                     uint64_t* n_elems, uint32_t* n_chunks);

/* Parity/diagnostic hook: run steps a1-a3 only (Alg. 1 P:137-146,
 * Alg. 2) and copy the flags (as u16, Alg. 1 loop 2, slot order
 * G2) and the final subbins (u32) into the given device buffers (N entries
 * each; either may be NULL).  Device input only (E_ARG otherwise).  Uses the
 * lopc_compress_ex workspace. */
int lopc_repair_ex(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, uint16_t* flags_out,
                   uint32_t* subbins_out, void* workspace, size_t workspace_bytes, void* stream);

/* Statistics of the calling host thread's last compress/decompress call. */
typedef struct {
  uint64_t n_elems;
  uint64_t n_chunks;
  uint64_t n_tiles;
  uint64_t sweep_passes;      /* repair passes (engine 0: tile passes of k_tiles; 1/2: k_sweep passes) */
  uint64_t worklist_points;   /* engine 0: tiles processed over all passes; 1/2: worklist points */
  uint64_t inner_iters;       /* sum of tile-local relaxation rounds in the dense pass */
  uint64_t escapes;
  uint64_t bin_bytes;
  uint64_t sub_bytes;
  uint64_t total_bytes;
  uint32_t max_subbin;
  uint32_t timing_valid;      /* 1 if the ms_* fields were measured (lopc_set_timing) */
  float ms_h2d;               /* host->device staging */
  float ms_quant_repair;      /* k_quant_flags (a1 + a2) */
  float ms_sweep;             /* k_sweep */
  float ms_encode;            /* k_encode */
  float ms_decode;            /* k_decode */
  float ms_d2h;               /* device->host staging */
  float ms_total;             /* whole call on the stream */
  uint64_t raised;            /* engine 0: subbins changed, summed over passes; 1/2: raises */
  uint32_t pass_items[16];    /* engine 0: tiles of pass q at [q]; 1/2: [1] dense tiles, [q>1] worklist points */
  uint64_t phase_cycles[16];  /* diagnostic (lopc_set_timing(2)): SM cycles per codec phase, summed over chunks */
  float ms_place;             /* compress: k_chunk_scan + k_place; decompress: k_chunk_scan */
  uint32_t launches;          /* kernels this library launched in the call */
  float pass_us[16];          /* diagnostic (lopc_set_timing(2)): k_sweep pass q ended pass_us[q] us after its start */
  uint32_t tma;               /* 1 if k_quant_flags loaded its halo boxes with TMA (LOPC_NO_TMA=1 disables) */
} lopc_stats;

int lopc_last_stats(lopc_stats* out);

/* Enable (1) / disable (0) per-kernel CUDA-event timing in lopc_stats; 2 also
 * records per-phase clocks of the codec kernels (diagnostic, slower). */
void lopc_set_timing(int enable);

/* Repair schedule (process-wide; NEXT f2 ablation).  0 (default): exact
 * tile fixpoints over alternating half-shifted tilings with subbin bit planes
 * (lopc_tiles.cuh), falling back to 2 when a subbin exceeds 254; 1: the
 * paper's point worklist from the first pass (Alg. 2 over every point, then
 * the points whose inputs rose); 2: round 1's dense tile pass
 * then point-worklist passes (u32 subbins).  All reach the same unique least
 * fixpoint (reading G14), hence the same bytes.  Slab mode repairs with
 * the tile engine for engine 0 (re-running every rank on engine 2 when a
 * subbin exceeds 8 planes anywhere) and with engine 2 otherwise.
 * E_ARG for another value. */
int lopc_set_repair_engine(int engine);

/* Test switch (process-wide): force != 0 makes k_quant_flags and k_sweep
 * use their int64 index builds on every grid (they are otherwise used only
 * from N >= 2^31 - 2^24, e.g. the cfg5 slabs at N > 1), so the parity suite
 * covers them on small grids.  Results are identical by construction. */
int lopc_set_index64(int force);

/* Decoder (process-wide): 1 (default) = one CTA per chunk decodes both
 * streams and reconstructs from its own shared memory (k_decode1); 2 = the
 * two streams of a chunk in a 2-CTA cluster, reconstructing through
 * distributed shared memory (k_decode).  Same output.  E_ARG otherwise. */
int lopc_set_decoder(int decoder);

/* Message for a return code; lopc_last_error_string() adds CUDA / NCCL
 * detail of the calling thread's last failure. */
const char* lopc_strerror(int code);
const char* lopc_last_error_string(void);

int lopc_abi_version(void);

/* ---- Checker (SURVEY §8(d.1) k_check; NEXT f3 error statistics) ------------
 * x, y: device arrays of the same grid.  order_violations: star edges
 * {p, p+e} (each once) with non-NaN x at both ends whose SoS order (ord, then
 * index) differs in y (or y is NaN there).  bound_violations: escaped points
 * not bit-identical, or regular points without 0 <= x - y <= eps exactly.
 * max_abs_err / sum_sq_err over the regular points (PSNR = 20 log10(range) -
 * 10 log10(sum_sq_err / n_regular)).  Uses the first 256 bytes of workspace. */
typedef struct {
  uint64_t order_violations;
  uint64_t bound_violations;
  uint64_t n_regular;
  double max_abs_err;
  double sum_sq_err;
} lopc_check_result;
int lopc_check(const void* x, const void* y, int ndims, const uint64_t* dims, int dtype, double eps,
               lopc_check_result* res, void* workspace, size_t workspace_bytes, void* stream);

/* Critical-point preservation (NEXT f3; Table III semantics): PL
 * critical points of x and y under SoS on the Freudenthal triangulation
 * (lower link empty = minimum, upper empty = maximum, one component each =
 * regular, else saddle; G5, G27).  false_positives: regular in x, critical in
 * y; false_negatives: the reverse; false_types: critical in both with
 * different types; pair_mismatches: (#lower, #upper) link components differ.
 * Vertices where x is NaN are skipped and NaN neighbours leave the link.
 * Device arrays; first 256 bytes of workspace. */
typedef struct {
  uint64_t false_positives;
  uint64_t false_negatives;
  uint64_t false_types;
  uint64_t pair_mismatches;
  uint64_t critical_x;
  uint64_t critical_y;
} lopc_critical_result;
int lopc_critical_points(const void* x, const void* y, int ndims, const uint64_t* dims, int dtype,
                         lopc_critical_result* res, void* workspace, size_t workspace_bytes, void* stream);

/* ---- NOA error bound on the device (row a0) ---------------
 * lopc_value_range: min and max over the finite values of x (device pointer,
 * one read pass; NaN and +-Inf skipped), returned as doubles, and their count.
 * Uses the first 256 bytes of `workspace`.  Blocks (one 24-byte D2H read).
 * lopc_noa_eps: eps = rel * (max - min) in double, or rel if there is no
 * finite value or max == min (P:112 NOA).  lopc_compress_noa = both, then
 * lopc_compress_ex with that eps (reported in *eps_used); workspace as for
 * lopc_compress_ex. */
int lopc_value_range(const void* in, int ndims, const uint64_t* dims, int dtype, double* vmin, double* vmax,
                     uint64_t* n_finite, void* workspace, size_t workspace_bytes, void* stream);
double lopc_noa_eps(double vmin, double vmax, uint64_t n_finite, double rel);
int lopc_compress_noa(const void* in, int ndims, const uint64_t* dims, int dtype, double rel, void* out,
                      size_t* out_bytes, double* eps_used, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Multi-GPU slab mode -----------------------------------
 * The grid is split into R contiguous element ranges [b_r, b_{r+1}) of the
 * linear order, rank r owning range r (one rank per GPU, one process each).
 * Every inner boundary b_r must be a multiple of W = 16384/k (each chunk has
 * one owner) and every range except the first and last must hold at least
 * H = d1*d2 + d2 + 1 (3D) / d2 + 1 (2D) elements (halos come from adjacent
 * ranks only); lopc_slab_partition gives a valid chunk-balanced split.
 * lopc_compress_slab runs the repair on the rank's range plus its halo, then
 * exchanges the halo subbins with rank r-1 / r+1 after every round until no
 * subbin changes on any rank (one NCCL send/recv pair per neighbour and one
 * u64 allreduce per round; the least fixpoint is unique, so the result is
 * the single-GPU one), then encodes the rank's chunks.  Output per rank
 * (out_local): its size-table slice (8 bytes per owned chunk) followed by its
 * payload slice.  The single-GPU stream is
 *   header(total) ‖ table slices in rank order ‖ payload slices in rank order,
 * and *payload_offset is where this rank's payload slice starts in it.
 * Device pointers only (in_slab, out_local, workspace).  Errors are agreed
 * across ranks (every rank returns the worst code): at entry (an allgather of
 * the ranges and local checks), after every repair round (the round's
 * allreduce carries a failure count, so a rank that fails locally keeps
 * taking part in the collectives and all ranks stop together) and at exit
 * (an allgather of sizes and codes).  A subbin above 8 planes on any rank
 * (tile engine) is agreed the same way and every rank re-runs the call on
 * the u32 engine internally (same bytes).  A failing NCCL call itself returns
 * LOPC_E_NCCL at once; the communicator is then unusable.  A NULL comm means
 * world = 1.  SURVEY §8(e); the exchange is the one of Alg. 2's sweeps
 * across slab boundaries.
 */
typedef struct lopc_comm lopc_comm;

/* NCCL unique id (128 bytes) for lopc_comm_create; make it on one rank and
 * broadcast it (e.g. torch.distributed.broadcast_object_list). */
int lopc_comm_unique_id(void* id128);
/* NCCL communicator on the current CUDA device (libnccl.so.2 via dlopen: the
 * copy the process already loaded, e.g. torch's).  Collective over ranks. */
int lopc_comm_create(lopc_comm** comm, int world, int rank, const void* id128);
int lopc_comm_destroy(lopc_comm* comm);

/* Default partition: world+1 chunk-aligned bounds, chunk-balanced.  Host only. */
int lopc_slab_partition(int ndims, const uint64_t* dims, int dtype, int world, uint64_t* bounds);
/* Host-side geometry of one range (for tests/bindings): info8 = {box start
 * B0, box points, H, ghosts below, ghosts above, points sent down, points
 * sent up, owned chunks}.  has_lo / has_hi: a neighbour exists below/above. */
int lopc_slab_info(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end, int has_lo,
                   int has_hi, uint64_t* info8);
size_t lopc_slab_workspace_bytes(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end);
/* Worst-case out_local bytes of a range. */
size_t lopc_slab_bound(int ndims, const uint64_t* dims, int dtype, uint64_t e_begin, uint64_t e_end);
/* The 64-byte stream header for a stream of total_bytes (host buffer). */
int lopc_write_header(void* hdr64, int ndims, const uint64_t* dims, int dtype, double eps, uint64_t total_bytes);

int lopc_compress_slab(lopc_comm* comm, const void* in_slab, int ndims, const uint64_t* dims, int dtype, double eps,
                       uint64_t e_begin, uint64_t e_end, void* out_local, size_t* out_local_bytes,
                       uint64_t* payload_offset, uint64_t* total_bytes, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Decode the chunks of [e_begin, e_end) from a rank's out_local (table slice
 * ‖ payload slice, local_bytes long), given the stream header (host).  No
 * communication.  out_slab receives e_end - e_begin values. */
size_t lopc_decompress_slab_workspace_bytes(uint64_t n_chunks_local);
int lopc_decompress_slab(const void* hdr64_host, const void* local, size_t local_bytes, uint64_t e_begin,
                         uint64_t e_end, void* out_slab, size_t out_capacity, void* workspace, size_t workspace_bytes,
                         void* stream);

/* Test hook (single device): the slab algorithm for nslabs ranges (bounds:
 * nslabs+1 entries) in one call, halos exchanged by device copies, writing
 * the whole stream to out (device).  Allocates its own scratch. */
int lopc_compress_slabs_local(const void* in, int ndims, const uint64_t* dims, int dtype, double eps, int nslabs,
                              const uint64_t* bounds, void* out, size_t* out_bytes);

#ifdef __cplusplus
}
#endif
#endif
