/* lopc_ref.h — CPU ORACLE for the LOPC hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liblopc_ref.so.  The product library
 * (include/lopc.h, paper_2603_26968_b200/csrc) shares no code, header,
 * table or constant with this file.
 *
 * Every function is a plain, single-threaded implementation of what
 * PAPER.md (arxiv 2603.26968) defines; readings of silent/ambiguous
 * passages are the G-items of DESIGN.md §3.
 * All pointers are HOST pointers owned by the caller.
 *
 * Error codes (int return): 0 ok, -1 bad argument, -2 bad shape,
 * -3 output too small, -4 corrupt stream, -5 version, -8 internal
 * (self-check failed).  Codes equal LOPC_* in include/lopc.h by
 * specification, not by sharing a header.
 */
#ifndef LOPC_REF_H
#define LOPC_REF_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* dtype: 0 = float32, 1 = float64.  dims[0..ndims-1] slowest -> fastest,
 * ndims in {2,3}, row-major with the last dim contiguous (G3). */

/* --- O5 / O6: scalar quantizer primitives ------------- */
/* bin of x (x given as its double value; for f32 data pass (double)xf).
 * returns 1 and *b if regular (finite, |b| <= BINMAX), 0 if escaped.   */
int lopc_ref_bin(double x, double eps, int dtype, int64_t* b);
/* lo(b): smallest dtype value >= (b - 1/2) * eps, exactly (as a double). */
double lopc_ref_lo(int64_t b, double eps, int dtype);
/* ord(): monotone map of a value's bits to an integer (O3). */
int64_t lopc_ref_ord(uint64_t bits, int dtype);

/* --- Whole-field steps (Alg. 1, Alg. 2, O5-O10) ------------------------ */
/* bins[i] = b or INT64_MIN for escaped points. */
int lopc_ref_quantize(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                      int64_t* bins);
/* flags[i]: bit j set iff star slot j of i is a lower same-bin neighbour
 * (Alg. 1 loop 2).  Slot order O2/G2.  */
int lopc_ref_flags(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                   uint16_t* flags);
/* least fixpoint by SoS-sorted DP (O9).  s[i] for escaped points = 0.  */
int lopc_ref_subbins(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                     uint32_t* s);
/* the paper's Alg. 1 + Alg. 2 with dual worklists and stamps, serial.
 * stats[0] = iterations, stats[1] = raises (points whose subbin rose). */
int lopc_ref_subbins_alg12(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                           uint32_t* s, uint64_t* stats);
/* synchronous Jacobi sweeps.  stats[0] = sweeps including the final
 * no-change sweep, stats[1] = point updates, stats[2] = sum of increments. */
int lopc_ref_subbins_jacobi(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                            uint32_t* s, uint64_t* stats);
/* O10 reconstruction from (x, s): xhat. */
int lopc_ref_reconstruct(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                         const uint32_t* s, void* xhat);

/* --- Stream (format v1) ---------------------------------- */
size_t lopc_ref_compress_bound(int ndims, const uint64_t* dims, int dtype);
int lopc_ref_compress(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                      void* out, size_t* out_bytes /* in: capacity, out: written/required */);
int lopc_ref_decompress(const void* in, size_t in_bytes, void* out, size_t out_capacity);
/* header parse: returns 0 and fills fields, or an error code. */
int lopc_ref_stream_info(const void* in, size_t n, int* ndims, uint64_t* dims3, int* dtype,
                         double* eps, uint64_t* n_elems, uint32_t* n_chunks);
/* per-chunk sizes (u32 pairs) of a stream: copies 2*C u32 into sizes. */
int lopc_ref_chunk_sizes(const void* in, size_t n, uint32_t* sizes, uint32_t cap_pairs);

/* one chunk (elements [c*W, min((c+1)W, n))) from x and a given subbin
 * field s: out (>= 32768 B) gets bin payload then subbin payload. */
int lopc_ref_encode_chunk(const void* x, uint64_t n, int dtype, double eps, const uint32_t* s, uint64_t c,
                          void* out, uint32_t* sizes2);

/* O12 for one chunk c: payloads = its bin payload (bin_size bytes) then its
 * subbin payload (sub_size bytes); writes elements [cW, min((c+1)W, n)) of
 * out (the whole field's buffer).  0 or E_CORRUPT / E_INTERNAL. */
int lopc_ref_decode_chunk(const void* payloads, uint32_t bin_size, uint32_t sub_size, uint32_t c, uint64_t n,
                          int dtype, double eps, void* out);

/* --- Lossless stages (G17-G21) ---------------------- */
void lopc_ref_diffnb(const void* words, size_t W, int k, void* out);
void lopc_ref_undiffnb(const void* in, size_t W, int k, void* words);
void lopc_ref_bitshuffle(const void* words, size_t W, int k, void* out);
void lopc_ref_unbitshuffle(const void* in, size_t W, int k, void* words);
/* RZE_g over L bytes; returns output length. out must hold L + L/g bytes. */
size_t lopc_ref_rze(const void* in, size_t L, int g, void* out);
/* inverse: reads at most in_len bytes; returns bytes consumed or -1. */
long lopc_ref_unrze(const void* in, size_t in_len, size_t L, int g, void* out);

/* --- Checkers (O13) ----------------------------------------------------- */
/* number of star edges whose SoS order differs between x and y (edges
 * touching NaN in x are skipped). */
uint64_t lopc_ref_order_violations(const void* x, const void* y, int ndims, const uint64_t* dims,
                                   int dtype);
/* number of points violating: escaped -> bit-identical; regular ->
 * 0 <= x - y <= eps in exact arithmetic. */
uint64_t lopc_ref_bound_violations(const void* x, const void* y, uint64_t n, int dtype, double eps);
/* Row a0 (NOA): min and max over the finite values (as doubles) and
 * their count; eps = rel * (max - min) computed in double, or rel when there
 * is no finite value or max == min (the caller's convention). */
uint64_t lopc_ref_value_range(const void* x, uint64_t n, int dtype, double* vmin, double* vmax);
double lopc_ref_noa_eps(const void* x, uint64_t n, int dtype, double rel);
/* Bellman certificate: number of points where s != max(0, max_arcs s(n)+w). */
uint64_t lopc_ref_certify(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                          const uint32_t* s);

#ifdef __cplusplus
}
#endif
#endif
