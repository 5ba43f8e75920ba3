/* lopc_omp.c — NEXT f4: the multi-core CPU baseline (OpenMP, blocked), test
 * and bench infrastructure beside the single-thread oracle.  NOT the product
 * path.  Same definitions as lopc_ref.c (whose scalar primitives and chunk
 * encoder it calls): bins by lopc_ref_bin (O5), the least fixpoint by
 * parallel in-place relaxation sweeps over z-plane / row blocks (the paper's
 * "OMP" schedule: every point re-evaluated each sweep until no change;
 * monotone, so any order reaches the unique fixpoint O9), chunks encoded in
 * parallel by lopc_ref_encode_chunk, payloads placed by one serial scan.
 * Parity: tests/test_oracle_omp.py requires the oracle's exact bytes. */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "lopc_ref.h"

static uint64_t bits_of(const void* x, uint64_t i, int dtype) {
  if (dtype == 0) {
    uint32_t u;
    memcpy(&u, (const uint8_t*)x + 4 * i, 4);
    return u;
  }
  uint64_t u;
  memcpy(&u, (const uint8_t*)x + 8 * i, 8);
  return u;
}

static double val_of(const void* x, uint64_t i, int dtype) {
  if (dtype == 0) {
    float f;
    memcpy(&f, (const uint8_t*)x + 4 * i, 4);
    return (double)f;
  }
  double d;
  memcpy(&d, (const uint8_t*)x + 8 * i, 8);
  return d;
}

int lopc_omp_compress(const void* x, int ndims, const uint64_t* dims, int dtype, double eps, void* out,
                      size_t* out_bytes, int threads, uint64_t* sweeps_out) {
  if (ndims != 2 && ndims != 3) return -2;
  if (threads > 0) omp_set_num_threads(threads);
  const int64_t d0 = ndims == 3 ? (int64_t)dims[0] : 1, d1 = (int64_t)dims[ndims - 2], d2 = (int64_t)dims[ndims - 1];
  const int64_t n = d0 * d1 * d2, plane = d1 * d2;
  const int k = dtype ? 8 : 4;
  const uint64_t W = 16384 / k, C = ((uint64_t)n + W - 1) / W;
  const size_t cap = *out_bytes;
  int64_t* bin = malloc(sizeof(int64_t) * (n ? n : 1));
  int64_t* ord = malloc(sizeof(int64_t) * (n ? n : 1));
  uint32_t* s = calloc(n ? n : 1, 4);
  uint8_t* chunks = malloc(32768 * (C ? C : 1));
  uint32_t* sz = malloc(8 * (C ? C : 1));
  if (!bin || !ord || !s || !chunks || !sz) return -8;
  /* a1: exact bins (INT64_MIN = escaped) and ord keys */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    int64_t b;
    bin[i] = lopc_ref_bin(val_of(x, i, dtype), eps, dtype, &b) ? b : INT64_MIN;
    ord[i] = lopc_ref_ord(bits_of(x, i, dtype), dtype);
  }
  /* star offsets (Kuhn/Freudenthal, G1): e in {0,1}^r \ 0 and -e */
  int ez[14], ey[14], ex[14], D = ndims == 3 ? 7 : 3;
  for (int j = 0; j < D; j++) {
    int e = j + 1;
    ez[j] = ndims == 3 ? (e >> 2) & 1 : 0;
    ey[j] = (e >> 1) & 1;
    ex[j] = e & 1;
    ez[j + D] = -ez[j];
    ey[j + D] = -ey[j];
    ex[j + D] = -ex[j];
  }
  /* a2 + a3: in-place relaxation sweeps over blocks of planes (rows in 2D) */
  uint64_t sweeps = 0;
  int changed = 1;
  while (changed) {
    changed = 0;
    sweeps++;
#pragma omp parallel for schedule(static) reduction(| : changed)
    for (int64_t p = 0; p < n; p++) {
      if (bin[p] == INT64_MIN) continue;
      const int64_t z = p / plane, r = p - z * plane, y = r / d2, xx = r - y * d2;
      uint32_t best = 0;
      for (int j = 0; j < 2 * D; j++) {
        const int64_t qz = z + ez[j], qy = y + ey[j], qx = xx + ex[j];
        if (qz < 0 || qz >= d0 || qy < 0 || qy >= d1 || qx < 0 || qx >= d2) continue;
        const int64_t q = (qz * d1 + qy) * d2 + qx;
        if (bin[q] != bin[p]) continue;  /* escaped q: INT64_MIN != regular bin */
        if (!(ord[q] < ord[p] || (ord[q] == ord[p] && q < p))) continue;
        const uint32_t v = __atomic_load_n(&s[q], __ATOMIC_RELAXED) + (q > p ? 1u : 0u);
        best = v > best ? v : best;
      }
      if (best > __atomic_load_n(&s[p], __ATOMIC_RELAXED)) {
        __atomic_store_n(&s[p], best, __ATOMIC_RELAXED);
        changed = 1;
      }
    }
  }
  /* a5/a6: chunks in parallel */
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (int64_t c = 0; c < (int64_t)C; c++)
    if (lopc_ref_encode_chunk(x, (uint64_t)n, dtype, eps, s, (uint64_t)c, chunks + 32768 * c, sz + 2 * c)) bad = 1;
  /* a7: header, table, payloads */
  uint64_t total = 64 + 8 * C;
  for (uint64_t c = 0; c < C; c++) total += (uint64_t)sz[2 * c] + sz[2 * c + 1];
  int rc = 0;
  if (bad) {
    rc = -8;
  } else if (total > cap) {
    rc = -3;
  } else {
    uint8_t* o = out;
    memset(o, 0, 64);
    memcpy(o, "LOPC", 4);
    const uint16_t ver = 1;
    memcpy(o + 4, &ver, 2);
    o[6] = (uint8_t)dtype;
    o[7] = (uint8_t)ndims;
    const uint64_t d3[3] = {(uint64_t)d0, (uint64_t)d1, (uint64_t)d2};
    memcpy(o + 8, d3, 24);
    memcpy(o + 32, &eps, 8);
    const uint64_t nn = (uint64_t)n;
    memcpy(o + 40, &nn, 8);
    const uint32_t cb = 16384, c32 = (uint32_t)C;
    memcpy(o + 48, &cb, 4);
    memcpy(o + 52, &c32, 4);
    memcpy(o + 56, &total, 8);
    memcpy(o + 64, sz, 8 * C);
    uint64_t off = 64 + 8 * C;
    for (uint64_t c = 0; c < C; c++) {
      const uint64_t len = (uint64_t)sz[2 * c] + sz[2 * c + 1];
      memcpy(o + off, chunks + 32768 * c, len);
      off += len;
    }
  }
  *out_bytes = total;
  if (sweeps_out) *sweeps_out = sweeps;
  free(bin);
  free(ord);
  free(s);
  free(chunks);
  free(sz);
  return rc;
}

/* Whole-stream chunk check for fields too large for the single-thread oracle
 * (cfg5 rank slab, 1 G points): every chunk c is encoded by the oracle's own
 * chunk encoder (lopc_ref_encode_chunk, a5/a6) from (x, eps, s) and compared
 * byte for byte with the stream under test: its size-table entry and its
 * payloads at the offsets the table's exclusive scan gives (a7), plus the
 * header fields and the total length.  s must already be certified as the
 * least fixpoint by lopc_ref_certify (O9: the Bellman certificate proves it
 * IS the oracle's subbins), which makes this the oracle's stream.  Returns the
 * number of mismatching chunks (+1 for a header / length mismatch), or
 * (uint64_t)-1 on allocation failure; the first bad chunk index goes to
 * *first_bad (or UINT64_MAX). */
uint64_t lopc_omp_check_chunks(const void* x, uint64_t n, int dtype, double eps, const uint32_t* s,
                               const void* stream, uint64_t stream_bytes, uint64_t* first_bad) {
  const int k = dtype ? 8 : 4;
  const uint64_t W = 16384 / k, C = (n + W - 1) / W;
  const uint8_t* st = (const uint8_t*)stream;
  *first_bad = UINT64_MAX;
  uint64_t bad = 0;
  if (stream_bytes < 64 + 8 * C) return 1 + C;
  uint64_t hn, htotal;
  uint32_t hc;
  double heps;
  memcpy(&hn, st + 40, 8);
  memcpy(&hc, st + 52, 4);
  memcpy(&htotal, st + 56, 8);
  memcpy(&heps, st + 32, 8);
  if (memcmp(st, "LOPC", 4) || hn != n || hc != C || htotal != stream_bytes || heps != eps || st[6] != dtype) bad++;
  uint64_t* off = malloc(8 * (C ? C : 1));
  if (!off) return (uint64_t)-1;
  uint64_t o = 64 + 8 * C;
  for (uint64_t c = 0; c < C; c++) {
    uint32_t bs, ss;
    memcpy(&bs, st + 64 + 8 * c, 4);
    memcpy(&ss, st + 64 + 8 * c + 4, 4);
    off[c] = o;
    o += (uint64_t)bs + ss;
  }
  if (o != stream_bytes) bad++;
  uint64_t first = UINT64_MAX;
#pragma omp parallel
  {
    uint8_t* buf = malloc(32768);
    uint64_t my_first = UINT64_MAX, my_bad = 0;
#pragma omp for schedule(dynamic, 64)
    for (int64_t ci = 0; ci < (int64_t)C; ci++) {
      const uint64_t c = (uint64_t)ci;
      uint32_t sz[2];
      int ok = buf && lopc_ref_encode_chunk(x, n, dtype, eps, s, c, buf, sz) == 0;
      if (ok) {
        uint32_t bs, ss;
        memcpy(&bs, st + 64 + 8 * c, 4);
        memcpy(&ss, st + 64 + 8 * c + 4, 4);
        ok = bs == sz[0] && ss == sz[1] && off[c] + bs + ss <= stream_bytes &&
             memcmp(st + off[c], buf, (size_t)bs + ss) == 0;
      }
      if (!ok) {
        my_bad++;
        if (c < my_first) my_first = c;
      }
    }
#pragma omp critical
    {
      bad += my_bad;
      if (my_first < first) first = my_first;
    }
    free(buf);
  }
  *first_bad = first;
  free(off);
  return bad;
}

/* Multi-core decompress (f4 baseline, paired with lopc_omp_compress so the
 * two CPU baselines time the same round trip): header parse and the size
 * table's exclusive scan serially, then every chunk by lopc_ref_decode_chunk
 * in parallel.  Same return codes as lopc_ref_decompress. */
int lopc_omp_decompress(const void* in, size_t in_bytes, void* out, size_t out_capacity, int threads) {
  if (threads > 0) omp_set_num_threads(threads);
  int nd, dt;
  uint64_t d3[3], n;
  uint32_t C;
  double eps;
  int rc = lopc_ref_stream_info(in, in_bytes, &nd, d3, &dt, &eps, &n, &C);
  if (rc) return rc;
  const int k = dt ? 8 : 4;
  if (out_capacity < n * (uint64_t)k) return -3;
  const uint8_t* st = (const uint8_t*)in;
  uint64_t* off = malloc(8 * (C ? C : 1));
  uint32_t* sz = malloc(8 * (C ? C : 1));
  if (!off || !sz) return -8;
  uint64_t o = 64 + 8ull * C;
  for (uint32_t c = 0; c < C; c++) {
    memcpy(sz + 2 * c, st + 64 + 8ull * c, 8);
    if (sz[2 * c] < 4 || sz[2 * c] > 16384 || (sz[2 * c] & 3) || sz[2 * c + 1] < 4 || sz[2 * c + 1] > 16384 ||
        (sz[2 * c + 1] & 3))
      rc = -4;
    off[c] = o;
    o += (uint64_t)sz[2 * c] + sz[2 * c + 1];
  }
  if (!rc && o != in_bytes) rc = -4;
  if (!rc) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
    for (int64_t c = 0; c < (int64_t)C; c++)
      if (lopc_ref_decode_chunk(st + off[c], sz[2 * c], sz[2 * c + 1], (uint32_t)c, n, dt, eps, out)) bad = 1;
    if (bad) rc = -4;
  }
  free(off);
  free(sz);
  return rc;
}
