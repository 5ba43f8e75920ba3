/* lopc_ref.c — CPU ORACLE for the LOPC hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded C implementation of what PAPER.md
 * (arxiv 2603.26968, "LOPC") defines.  Each function cites the passage
 * it follows as P:<line> and the DESIGN.md reading (G-items,
 * restated from SURVEY §8(c.3)) where the paper is silent.
 *
 * Shares no code with the product (include/lopc.h, csrc/).  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
 * may load it.  Compile with -O2 -ffp-contract=off (no FMA contraction,
 * no fast-math): fma() is called explicitly only for the TwoProduct error
 * term of lo().
 *
 * Pins (tests/test_oracle_*.py): exact rationals for bin/lo, the paper's
 * worked example, the golden 3x4 grid (tests/golden), the chain
 * closed forms, DP == Alg.2 == Jacobi, the Bellman
 * certificate, brute-force critical points (Table III), SPEC stage
 * examples.  The stream bytes themselves are our format:
 * parity of the exact bytes is unpinned w.r.t. the paper; each stage is
 * pinned by worked examples and inverse round trips.
 */
#include "lopc_ref.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define E_ARG (-1)
#define E_SHAPE (-2)
#define E_NOSPACE (-3)
#define E_CORRUPT (-4)
#define E_VERSION (-5)
#define E_INTERNAL (-8)

#define CHUNK_BYTES 16384u /* "16kB chunks" P:90, G22 */
#define HDR_BYTES 64u

/* ------------------------------------------------------------------ */
/* O3: ord() — the SoS value key ("Simulation of Simplicity";     */
/* P:164 tie breaker on the index, G4).                                */
/* ------------------------------------------------------------------ */
int64_t lopc_ref_ord(uint64_t bits, int dtype) {
  if (dtype == 0) {
    uint32_t u = (uint32_t)bits;
    if ((u & 0x80000000u) == 0) return (int64_t)u;
    return -(int64_t)(u & 0x7fffffffu);
  }
  if ((bits & 0x8000000000000000ull) == 0) return (int64_t)bits;
  return -(int64_t)(bits & 0x7fffffffffffffffull);
}

static uint64_t unord(int64_t o, int dtype) {
  if (dtype == 0) {
    if (o >= 0) return (uint64_t)(uint32_t)o;
    return (uint64_t)(0x80000000u | (uint32_t)(-o));
  }
  if (o >= 0) return (uint64_t)o;
  return 0x8000000000000000ull | (uint64_t)(-o);
}

static uint64_t bits_at(const void* x, uint64_t i, int dtype) {
  if (dtype == 0) {
    uint32_t u;
    memcpy(&u, (const uint8_t*)x + 4 * i, 4);
    return u;
  }
  uint64_t u;
  memcpy(&u, (const uint8_t*)x + 8 * i, 8);
  return u;
}

static double value_at(const void* x, uint64_t i, int dtype) {
  if (dtype == 0) {
    float f;
    memcpy(&f, (const uint8_t*)x + 4 * i, 4);
    return (double)f;
  }
  double d;
  memcpy(&d, (const uint8_t*)x + 8 * i, 8);
  return d;
}

/* ------------------------------------------------------------------ */
/* O6: lo(b) = the smallest dtype value >= (b - 1/2) eps, exactly.     */
/* "subbin 0 decodes to the lowest representable value within   */
/* the bin".  a = b - 1/2 is exact (|b| <= 2^51); a*eps = p + e        */
/* exactly (TwoProduct, e = fma(a, eps, -p)); no underflow because     */
/* eps >= 2^-900 (argument check).                                     */
/* ------------------------------------------------------------------ */
double lopc_ref_lo(int64_t b, double eps, int dtype) {
  double a = (double)b - 0.5;
  double p = a * eps;
  double e = fma(a, eps, -p);
  if (dtype == 1) {
    /* smallest double >= p + e */
    if (e > 0) return nextafter(p, INFINITY);
    return p;
  }
  /* smallest float >= p + e (G7: eps is never rounded to f32) */
  float f = (float)p;
  if ((double)f < p) {
    f = nextafterf(f, INFINITY);
  } else if ((double)f == p && e > 0) {
    f = nextafterf(f, INFINITY);
  }
  return (double)f;
}

/* ------------------------------------------------------------------ */
/* O5: b = floor(x/eps + 1/2) in exact arithmetic ("multiplying  */
/* the value by 1/eps and rounding the result to the nearest integer"; */
/* G6: half-up, bins [(b-1/2)eps, (b+1/2)eps)).  Written as: estimate, */
/* then step until lo(b) <= x < lo(b+1), which for a dtype value x is  */
/* the same condition.  Regular iff finite and |b| <= BINMAX (G8/G9).  */
/* ------------------------------------------------------------------ */
static double binmax_of(int dtype) { return dtype == 0 ? 2147483646.0 : 1125899906842624.0; }

int lopc_ref_bin(double x, double eps, int dtype, int64_t* bout) {
  if (!isfinite(x)) return 0;
  double binmax = binmax_of(dtype);
  double t = x / eps;
  if (!(fabs(t) <= 2.0 * binmax)) return 0; /* certainly |b| > BINMAX */
  int64_t b = (int64_t)floor(t + 0.5);
  while (x < lopc_ref_lo(b, eps, dtype)) b--;
  while (x >= lopc_ref_lo(b + 1, eps, dtype)) b++;
  if ((double)b > binmax || (double)b < -binmax) return 0;
  *bout = b;
  return 1;
}

/* ------------------------------------------------------------------ */
/* O1/O2: grid and Kuhn/Freudenthal star (G1, G2, G25).          */
/* ------------------------------------------------------------------ */
typedef struct {
  int r;       /* 2 or 3 */
  int D;       /* number of +e offsets: 3 (2D) or 7 (3D) */
  int64_t d[3]; /* z, y, x extents (2D: d[0] = 1) */
  uint64_t n;
  int off[7][3]; /* (dz, dy, dx) */
} grid_t;

static int make_grid(int ndims, const uint64_t* dims, grid_t* g) {
  if (ndims != 2 && ndims != 3) return E_SHAPE;
  g->r = ndims;
  if (ndims == 2) {
    g->d[0] = 1;
    g->d[1] = (int64_t)dims[0];
    g->d[2] = (int64_t)dims[1];
    static const int o2[3][3] = {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}};
    g->D = 3;
    memcpy(g->off, o2, sizeof(o2));
  } else {
    g->d[0] = (int64_t)dims[0];
    g->d[1] = (int64_t)dims[1];
    g->d[2] = (int64_t)dims[2];
    static const int o3[7][3] = {{0, 0, 1}, {0, 1, 0}, {0, 1, 1}, {1, 0, 0},
                                 {1, 0, 1}, {1, 1, 0}, {1, 1, 1}};
    g->D = 7;
    memcpy(g->off, o3, sizeof(o3));
  }
  for (int a = 0; a < 3; a++)
    if (g->d[a] < 0 || (uint64_t)g->d[a] > (1ull << 40)) return E_SHAPE;
  g->n = (uint64_t)g->d[0] * (uint64_t)g->d[1] * (uint64_t)g->d[2];
  if (g->n > (1ull << 40)) return E_SHAPE;
  return 0;
}

/* neighbour of p through star slot j (j < D: +offset j; else -offset j-D).
 * returns 1 and *q if in bounds. */
static int neighbour(const grid_t* g, uint64_t p, int j, uint64_t* q) {
  int64_t x = (int64_t)(p % (uint64_t)g->d[2]);
  int64_t y = (int64_t)((p / (uint64_t)g->d[2]) % (uint64_t)g->d[1]);
  int64_t z = (int64_t)(p / ((uint64_t)g->d[2] * (uint64_t)g->d[1]));
  int sgn = j < g->D ? 1 : -1;
  int jj = j < g->D ? j : j - g->D;
  z += sgn * g->off[jj][0];
  y += sgn * g->off[jj][1];
  x += sgn * g->off[jj][2];
  if (z < 0 || y < 0 || x < 0 || z >= g->d[0] || y >= g->d[1] || x >= g->d[2]) return 0;
  *q = ((uint64_t)z * (uint64_t)g->d[1] + (uint64_t)y) * (uint64_t)g->d[2] + (uint64_t)x;
  return 1;
}

static int check_eps(double eps) {
  if (!(eps > 0) || !isfinite(eps)) return E_ARG;
  if (eps < ldexp(1.0, -900) || eps > ldexp(1.0, 1000)) return E_ARG;
  return 0;
}

/* Per-point state of Alg. 1 loop 1: bin (INT64_MIN if escaped), ord. */
typedef struct {
  grid_t g;
  int dtype;
  int64_t* bin;
  int64_t* ord;
} field_t;

static void field_free(field_t* f) {
  free(f->bin);
  free(f->ord);
  f->bin = f->ord = NULL;
}

static int field_init(field_t* f, const void* x, int ndims, const uint64_t* dims, int dtype,
                      double eps) {
  memset(f, 0, sizeof(*f));
  if (dtype != 0 && dtype != 1) return E_ARG;
  int rc = check_eps(eps);
  if (rc) return rc;
  rc = make_grid(ndims, dims, &f->g);
  if (rc) return rc;
  f->dtype = dtype;
  uint64_t n = f->g.n;
  f->bin = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  f->ord = (int64_t*)malloc((n ? n : 1) * sizeof(int64_t));
  if (!f->bin || !f->ord) {
    field_free(f);
    return E_INTERNAL;
  }
  /* Alg. 1 line 2: p_bin <- quantized input */
  for (uint64_t i = 0; i < n; i++) {
    int64_t b;
    if (lopc_ref_bin(value_at(x, i, dtype), eps, dtype, &b))
      f->bin[i] = b;
    else
      f->bin[i] = INT64_MIN;
    f->ord[i] = lopc_ref_ord(bits_at(x, i, dtype), dtype);
  }
  return 0;
}

/* n precedes p in the SoS total order (G4: ties go to the
 * lower index). */
static int sos_less(const field_t* f, uint64_t n, uint64_t p) {
  if (f->ord[n] != f->ord[p]) return f->ord[n] < f->ord[p];
  return n < p;
}

/* O8: arc n -> p iff both regular, same bin, n precedes p (Alg. 1 lines
 * 9-10, "same bin" and "n < p with tie breaker"). */
static int is_arc(const field_t* f, uint64_t n, uint64_t p) {
  if (f->bin[n] == INT64_MIN || f->bin[p] == INT64_MIN) return 0;
  if (f->bin[n] != f->bin[p]) return 0;
  return sos_less(f, n, p);
}

static uint16_t flags_of(const field_t* f, uint64_t p) {
  uint16_t m = 0;
  for (int j = 0; j < 2 * f->g.D; j++) {
    uint64_t q;
    if (neighbour(&f->g, p, j, &q) && is_arc(f, q, p)) m |= (uint16_t)(1u << j);
  }
  return m;
}

int lopc_ref_quantize(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                      int64_t* bins) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  memcpy(bins, f.bin, f.g.n * sizeof(int64_t));
  field_free(&f);
  return 0;
}

int lopc_ref_flags(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                   uint16_t* flags) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  for (uint64_t p = 0; p < f.g.n; p++) flags[p] = flags_of(&f, p);
  field_free(&f);
  return 0;
}

/* ------------------------------------------------------------------ */
/* O9: the least fixpoint of s(p) = max(0, max_{n->p} s(n) + w),       */
/* w = [idx n > idx p] (Alg. 2 "tie"; rules (1)/(2)).    */
/* The arcs follow the SoS order, so processing points in ascending    */
/* SoS order is a topological order of the DAG ("acyclic"); one  */
/* pass gives the least solution ("as low as possible").        */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t ord;
  uint64_t idx;
} key_t;

static int key_cmp(const void* a, const void* b) {
  const key_t* ka = (const key_t*)a;
  const key_t* kb = (const key_t*)b;
  if (ka->ord != kb->ord) return ka->ord < kb->ord ? -1 : 1;
  if (ka->idx != kb->idx) return ka->idx < kb->idx ? -1 : 1;
  return 0;
}

static int dp_fixpoint(const field_t* f, uint32_t* s) {
  uint64_t n = f->g.n, m = 0;
  key_t* keys = (key_t*)malloc((n ? n : 1) * sizeof(key_t));
  if (!keys) return E_INTERNAL;
  for (uint64_t i = 0; i < n; i++) {
    s[i] = 0;
    if (f->bin[i] != INT64_MIN) {
      keys[m].ord = f->ord[i];
      keys[m].idx = i;
      m++;
    }
  }
  qsort(keys, m, sizeof(key_t), key_cmp);
  int rc = 0;
  for (uint64_t t = 0; t < m; t++) {
    uint64_t p = keys[t].idx;
    uint64_t best = 0;
    for (int j = 0; j < 2 * f->g.D; j++) {
      uint64_t q;
      if (neighbour(&f->g, p, j, &q) && is_arc(f, q, p)) {
        uint64_t v = (uint64_t)s[q] + (q > p ? 1u : 0u);
        if (v > best) best = v;
      }
    }
    if (best >= 0xffffffffull) {
      rc = E_INTERNAL; /* G28 overflow guard */
      break;
    }
    s[p] = (uint32_t)best;
  }
  free(keys);
  return rc;
}

int lopc_ref_subbins(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                     uint32_t* s) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  rc = dp_fixpoint(&f, s);
  field_free(&f);
  return rc;
}

/* ------------------------------------------------------------------ */
/* The paper's own schedule, serial: Alg. 1 + Alg. 2       */
/* with dual worklists and iteration stamps.       */
/* ------------------------------------------------------------------ */
int lopc_ref_subbins_alg12(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                           uint32_t* s, uint64_t* stats) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  uint64_t n = f.g.n;
  uint16_t* flags = (uint16_t*)malloc((n ? n : 1) * sizeof(uint16_t));
  uint64_t* wl1 = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* wl2 = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* stamp = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
  if (!flags || !wl1 || !wl2 || !stamp) {
    rc = E_INTERNAL;
    goto out;
  }
  /* Alg. 1 lines 1-12: subbin <- 0, flags */
  for (uint64_t p = 0; p < n; p++) {
    s[p] = 0;
    flags[p] = flags_of(&f, p);
  }
  /* line 13: worklist1 <- all input points */
  uint64_t n1 = n, n2, iter = 0, raises = 0;
  for (uint64_t p = 0; p < n; p++) wl1[p] = p;
  while (n1 > 0) { /* line 14 */
    iter++;
    n2 = 0; /* line 15: worklist2 <- empty */
    for (uint64_t t = 0; t < n1; t++) { /* Alg. 2 line 1 */
      uint64_t p = wl1[t];
      uint64_t n_max = 0;
      for (int j = 0; j < 2 * f.g.D; j++) { /* lines 3-4, using p_flags */
        uint64_t q;
        if (!(flags[p] & (1u << j))) continue;
        neighbour(&f.g, p, j, &q);
        uint64_t tie = q > p ? 1u : 0u; /* line 5 */
        uint64_t val = s[q];            /* line 6 */
        if (val + tie > n_max) n_max = val + tie;
      }
      if (n_max >= 0xffffffffull) {
        rc = E_INTERNAL;
        goto out;
      }
      if (s[p] < n_max) { /* line 10: atomicMax(p_subbin, n_max) < n_max */
        s[p] = (uint32_t)n_max;
        raises++;
        /* line 11: enqueue p's greater same-bin neighbours, once per
         * iteration (stamps) */
        for (int j = 0; j < 2 * f.g.D; j++) {
          uint64_t q;
          if (neighbour(&f.g, p, j, &q) && is_arc(&f, p, q) && stamp[q] != iter) {
            stamp[q] = iter;
            wl2[n2++] = q;
          }
        }
      }
    }
    uint64_t* tmp = wl1; /* line 17: swap */
    wl1 = wl2;
    wl2 = tmp;
    n1 = n2;
  }
  if (stats) {
    stats[0] = iter;
    stats[1] = raises;
  }
out:
  free(flags);
  free(wl1);
  free(wl2);
  free(stamp);
  field_free(&f);
  return rc;
}

/* Synchronous (Jacobi) sweeps of the same relaxation: the workload
 * characterisation of SURVEY §8(d.5). */
int lopc_ref_subbins_jacobi(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                            uint32_t* s, uint64_t* stats) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  uint64_t n = f.g.n;
  uint32_t* nxt = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!nxt) {
    field_free(&f);
    return E_INTERNAL;
  }
  for (uint64_t p = 0; p < n; p++) s[p] = 0;
  uint64_t sweeps = 0, updates = 0, incr = 0;
  for (;;) {
    sweeps++;
    uint64_t changed = 0;
    for (uint64_t p = 0; p < n; p++) {
      uint64_t best = s[p];
      for (int j = 0; j < 2 * f.g.D; j++) {
        uint64_t q;
        if (neighbour(&f.g, p, j, &q) && is_arc(&f, q, p)) {
          uint64_t v = (uint64_t)s[q] + (q > p ? 1u : 0u);
          if (v > best) best = v;
        }
      }
      if (best >= 0xffffffffull) {
        rc = E_INTERNAL;
        goto out;
      }
      nxt[p] = (uint32_t)best;
      if (best != s[p]) {
        changed++;
        incr += best - s[p];
      }
    }
    memcpy(s, nxt, n * sizeof(uint32_t));
    updates += changed;
    if (changed == 0) break;
  }
  if (stats) {
    stats[0] = sweeps;
    stats[1] = updates;
    stats[2] = incr;
  }
out:
  free(nxt);
  field_free(&f);
  return rc;
}

/* O10: regular -> the value whose ord is ord(lo(b)) + s; escaped ->
 * x bit-for-bit (G10/G11). */
static uint64_t decode_point(int64_t b, uint64_t s, double eps, int dtype) {
  double lo = lopc_ref_lo(b, eps, dtype);
  uint64_t lobits;
  if (dtype == 0) {
    float lf = (float)lo;
    uint32_t u;
    memcpy(&u, &lf, 4);
    lobits = u;
  } else {
    memcpy(&lobits, &lo, 8);
  }
  int64_t o = lopc_ref_ord(lobits, dtype) + (int64_t)s;
  return unord(o, dtype);
}

int lopc_ref_reconstruct(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                         const uint32_t* s, void* xhat) {
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  int k = dtype == 0 ? 4 : 8;
  for (uint64_t i = 0; i < f.g.n; i++) {
    uint64_t v =
        f.bin[i] == INT64_MIN ? bits_at(x, i, dtype) : decode_point(f.bin[i], s[i], eps, dtype);
    memcpy((uint8_t*)xhat + (size_t)k * i, &v, (size_t)k); /* little-endian host */
  }
  field_free(&f);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Lossless stages.  Words are k-byte little-endian integers.           */
/* ------------------------------------------------------------------ */
static uint64_t word_get(const uint8_t* p, int k) {
  uint64_t v = 0;
  for (int b = 0; b < k; b++) v |= (uint64_t)p[b] << (8 * b);
  return v;
}
static void word_put(uint8_t* p, int k, uint64_t v) {
  for (int b = 0; b < k; b++) p[b] = (uint8_t)(v >> (8 * b));
}
static uint64_t mask_k(int k) { return k == 8 ? ~0ull : ((1ull << (8 * k)) - 1); }

/* DIFFNB_k: "delta encoded ... converted to negabinary" (G18,
 * G19): d[i] = w[i] - w[i-1] mod 2^(8k), w[-1] = 0; u = (d + M) xor M,
 * M = 0xAA..A. */
void lopc_ref_diffnb(const void* words, size_t W, int k, void* out) {
  const uint8_t* in = (const uint8_t*)words;
  uint8_t* o = (uint8_t*)out;
  uint64_t msk = mask_k(k), M = 0xAAAAAAAAAAAAAAAAull & msk, prev = 0;
  for (size_t i = 0; i < W; i++) {
    uint64_t w = word_get(in + i * k, k);
    uint64_t d = (w - prev) & msk;
    prev = w;
    word_put(o + i * k, k, ((d + M) & msk) ^ M);
  }
}

void lopc_ref_undiffnb(const void* in, size_t W, int k, void* words) {
  const uint8_t* p = (const uint8_t*)in;
  uint8_t* o = (uint8_t*)words;
  uint64_t msk = mask_k(k), M = 0xAAAAAAAAAAAAAAAAull & msk, prev = 0;
  for (size_t i = 0; i < W; i++) {
    uint64_t u = word_get(p + i * k, k);
    uint64_t d = ((u ^ M) - M) & msk;
    prev = (prev + d) & msk;
    word_put(o + i * k, k, prev);
  }
}

/* BIT_k: "group the first bit of every value together, then all the
 * second bits, and so on" (Fig. 1; G20): plane j (j = 0 LSB)
 * holds bit j of words 0..W-1, packed LSB-first; W % 8 == 0. */
void lopc_ref_bitshuffle(const void* words, size_t W, int k, void* out) {
  const uint8_t* in = (const uint8_t*)words;
  uint8_t* o = (uint8_t*)out;
  size_t plane = W / 8;
  memset(o, 0, W * (size_t)k);
  for (size_t i = 0; i < W; i++) {
    uint64_t w = word_get(in + i * k, k);
    for (int j = 0; j < 8 * k; j++)
      if ((w >> j) & 1u) o[(size_t)j * plane + i / 8] |= (uint8_t)(1u << (i % 8));
  }
}

void lopc_ref_unbitshuffle(const void* in, size_t W, int k, void* words) {
  const uint8_t* p = (const uint8_t*)in;
  uint8_t* o = (uint8_t*)words;
  size_t plane = W / 8;
  for (size_t i = 0; i < W; i++) {
    uint64_t w = 0;
    for (int j = 0; j < 8 * k; j++)
      if ((p[(size_t)j * plane + i / 8] >> (i % 8)) & 1u) w |= 1ull << j;
    word_put(o + i * k, k, w);
  }
}

/* RZE_g: "a bitmap in which each bit corresponds to a word in the input
 * and indicates whether the word is zero.  All zero words are then
 * removed ... the bitmap, which itself is repeatedly compressed with a
 * similar algorithm that identifies repeating words" (Fig. 2;
 * G21).  Level sizes are static functions of L. */
static int rze_levels(size_t nwords, size_t* sz) {
  int top = 0;
  sz[0] = (nwords + 7) / 8;
  while (sz[top] > 8) {
    sz[top + 1] = (sz[top] + 7) / 8;
    top++;
  }
  return top;
}

size_t lopc_ref_rze(const void* in, size_t L, int g, void* out) {
  const uint8_t* p = (const uint8_t*)in;
  uint8_t* o = (uint8_t*)out;
  size_t n = L / (size_t)g;
  size_t sz[16];
  int top = rze_levels(n, sz);
  uint8_t* B[16];
  for (int i = 0; i <= top; i++) B[i] = (uint8_t*)calloc(sz[i] ? sz[i] : 1, 1);
  /* B0: bit i = word i is non-zero */
  for (size_t i = 0; i < n; i++) {
    int nz = 0;
    for (int b = 0; b < g; b++) nz |= p[i * g + b] != 0;
    if (nz) B[0][i / 8] |= (uint8_t)(1u << (i % 8));
  }
  /* B_{i+1}: bit t = B_i[t] differs from B_i[t-1] (B_i[-1] = 0) */
  for (int i = 0; i < top; i++)
    for (size_t t = 0; t < sz[i]; t++) {
      uint8_t prev = t ? B[i][t - 1] : 0;
      if (B[i][t] != prev) B[i + 1][t / 8] |= (uint8_t)(1u << (t % 8));
    }
  size_t w = 0;
  memcpy(o, B[top], sz[top]);
  w += sz[top];
  for (int i = top - 1; i >= 0; i--) /* K_i: bytes of B_i marked in B_{i+1} */
    for (size_t t = 0; t < sz[i]; t++)
      if ((B[i + 1][t / 8] >> (t % 8)) & 1u) o[w++] = B[i][t];
  for (size_t i = 0; i < n; i++) /* the non-zero words, in order */
    if ((B[0][i / 8] >> (i % 8)) & 1u) {
      memcpy(o + w, p + i * g, (size_t)g);
      w += (size_t)g;
    }
  for (int i = 0; i <= top; i++) free(B[i]);
  return w;
}

long lopc_ref_unrze(const void* in, size_t in_len, size_t L, int g, void* out) {
  const uint8_t* p = (const uint8_t*)in;
  uint8_t* o = (uint8_t*)out;
  size_t n = L / (size_t)g;
  size_t sz[16];
  int top = rze_levels(n, sz);
  uint8_t* B[16];
  for (int i = 0; i <= top; i++) B[i] = (uint8_t*)calloc(sz[i] ? sz[i] : 1, 1);
  long rc = -1;
  size_t r = 0;
  if (sz[top] > in_len) goto done;
  memcpy(B[top], p, sz[top]);
  r = sz[top];
  for (int i = top - 1; i >= 0; i--)
    for (size_t t = 0; t < sz[i]; t++) {
      if ((B[i + 1][t / 8] >> (t % 8)) & 1u) {
        if (r >= in_len) goto done;
        B[i][t] = p[r++];
      } else {
        B[i][t] = t ? B[i][t - 1] : 0;
      }
    }
  for (size_t i = 0; i < n; i++) {
    if ((B[0][i / 8] >> (i % 8)) & 1u) {
      if (r + (size_t)g > in_len) goto done;
      memcpy(o + i * g, p + r, (size_t)g);
      r += (size_t)g;
    } else {
      memset(o + i * g, 0, (size_t)g);
    }
  }
  rc = (long)r;
done:
  for (int i = 0; i <= top; i++) free(B[i]);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Chunk pipelines (P:192 bins: lossless PFPL portion; P:209-210       */
/* subbins: BIT_k RZE_k RZE_1) and container v1.        */
/* ------------------------------------------------------------------ */
static size_t pad4(size_t v) { return (v + 3) & ~(size_t)3; }

/* bin payload of one chunk: RZE_1(BIT_k(DIFFNB_k(words))) or raw. */
static size_t encode_bin_chunk(const uint8_t* words, int k, uint8_t* dst, uint8_t* t1,
                               uint8_t* t2, uint8_t* t3) {
  size_t W = CHUNK_BYTES / (size_t)k;
  lopc_ref_diffnb(words, W, k, t1);
  lopc_ref_bitshuffle(t1, W, k, t2);
  size_t len = lopc_ref_rze(t2, CHUNK_BYTES, 1, t3);
  if (pad4(len) >= CHUNK_BYTES) { /* raw fallback (G23) */
    memcpy(dst, words, CHUNK_BYTES);
    return CHUNK_BYTES;
  }
  memcpy(dst, t3, len);
  memset(dst + len, 0, pad4(len) - len);
  return pad4(len);
}

/* subbin payload: u16 L' | RZE_1(RZE_k(BIT_k(words))) or raw. */
static size_t encode_sub_chunk(const uint8_t* words, int k, uint8_t* dst, uint8_t* t1,
                               uint8_t* t2, uint8_t* t3) {
  size_t W = CHUNK_BYTES / (size_t)k;
  lopc_ref_bitshuffle(words, W, k, t1);
  size_t l1 = lopc_ref_rze(t1, CHUNK_BYTES, k, t2);
  size_t l2 = lopc_ref_rze(t2, l1, 1, t3);
  if (pad4(2 + l2) >= CHUNK_BYTES) {
    memcpy(dst, words, CHUNK_BYTES);
    return CHUNK_BYTES;
  }
  dst[0] = (uint8_t)(l1 & 0xff);
  dst[1] = (uint8_t)(l1 >> 8);
  memcpy(dst + 2, t3, l2);
  memset(dst + 2 + l2, 0, pad4(2 + l2) - (2 + l2));
  return pad4(2 + l2);
}

static void put_u16(uint8_t* p, uint16_t v) {
  p[0] = (uint8_t)v;
  p[1] = (uint8_t)(v >> 8);
}
static void put_u32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static void put_u64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; i++) p[i] = (uint8_t)(v >> (8 * i));
}
static uint16_t get_u16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get_u32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; i++) v |= (uint32_t)p[i] << (8 * i);
  return v;
}
static uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; i++) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

static uint64_t n_chunks(uint64_t n, int k) {
  uint64_t W = CHUNK_BYTES / (uint64_t)k;
  return (n + W - 1) / W;
}

size_t lopc_ref_compress_bound(int ndims, const uint64_t* dims, int dtype) {
  grid_t g;
  if (make_grid(ndims, dims, &g) || (dtype != 0 && dtype != 1)) return 0;
  uint64_t C = n_chunks(g.n, dtype == 0 ? 4 : 8);
  return HDR_BYTES + 8 * C + 2 * CHUNK_BYTES * C;
}

int lopc_ref_compress(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                      void* out, size_t* out_bytes) {
  if (!out_bytes) return E_ARG;
  field_t f;
  int rc = field_init(&f, x, ndims, dims, dtype, eps);
  if (rc) return rc;
  uint64_t n = f.g.n;
  int k = dtype == 0 ? 4 : 8;
  uint64_t W = CHUNK_BYTES / (uint64_t)k, C = n_chunks(n, k);
  uint32_t* s = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  uint8_t* buf = (uint8_t*)malloc(HDR_BYTES + 8 * C + 2 * CHUNK_BYTES * C);
  uint8_t *bw = (uint8_t*)malloc(CHUNK_BYTES), *sw = (uint8_t*)malloc(CHUNK_BYTES);
  uint8_t *t1 = (uint8_t*)malloc(CHUNK_BYTES), *t2 = (uint8_t*)malloc(2 * CHUNK_BYTES),
          *t3 = (uint8_t*)malloc(2 * CHUNK_BYTES);
  if (!s || !buf || !bw || !sw || !t1 || !t2 || !t3) {
    rc = E_INTERNAL;
    goto out;
  }
  rc = dp_fixpoint(&f, s);
  if (rc) goto out;
  /* a4: bound self-check (SPEC verify_encode): the
   * decoded value must satisfy lo(b) <= xhat <= x for regular points. */
  for (uint64_t i = 0; i < n; i++) {
    if (f.bin[i] == INT64_MIN) continue;
    uint64_t xh = decode_point(f.bin[i], s[i], eps, dtype);
    int64_t oh = lopc_ref_ord(xh, dtype);
    if (oh > f.ord[i]) {
      rc = E_INTERNAL;
      goto out;
    }
  }
  uint8_t* tab = buf + HDR_BYTES;
  size_t w = HDR_BYTES + 8 * C;
  for (uint64_t c = 0; c < C; c++) {
    memset(bw, 0, CHUNK_BYTES); /* words past N are 0 (G23) */
    memset(sw, 0, CHUNK_BYTES);
    for (uint64_t i = c * W; i < n && i < (c + 1) * W; i++) {
      uint64_t bwv, swv;
      if (f.bin[i] == INT64_MIN) { /* O7/G10: sentinel + raw bits */
        bwv = dtype == 0 ? 0x80000000ull : 0x8000000000000000ull;
        swv = bits_at(x, i, dtype);
      } else {
        bwv = (uint64_t)f.bin[i] & mask_k(k);
        swv = s[i];
      }
      word_put(bw + (i - c * W) * k, k, bwv);
      word_put(sw + (i - c * W) * k, k, swv);
    }
    size_t bs = encode_bin_chunk(bw, k, buf + w, t1, t2, t3);
    w += bs;
    size_t ss = encode_sub_chunk(sw, k, buf + w, t1, t2, t3);
    w += ss;
    put_u32(tab + 8 * c, (uint32_t)bs);
    put_u32(tab + 8 * c + 4, (uint32_t)ss);
  }
  /* header */
  memset(buf, 0, HDR_BYTES);
  memcpy(buf, "LOPC", 4);
  put_u16(buf + 4, 1);
  buf[6] = (uint8_t)dtype;
  buf[7] = (uint8_t)ndims;
  put_u64(buf + 8, (uint64_t)f.g.d[0]);
  put_u64(buf + 16, (uint64_t)f.g.d[1]);
  put_u64(buf + 24, (uint64_t)f.g.d[2]);
  uint64_t eb;
  memcpy(&eb, &eps, 8);
  put_u64(buf + 32, eb);
  put_u64(buf + 40, n);
  put_u32(buf + 48, CHUNK_BYTES);
  put_u32(buf + 52, (uint32_t)C);
  put_u64(buf + 56, (uint64_t)w);
  if (*out_bytes < w) {
    *out_bytes = w;
    rc = E_NOSPACE;
    goto out;
  }
  memcpy(out, buf, w);
  *out_bytes = w;
out:
  free(s);
  free(buf);
  free(bw);
  free(sw);
  free(t1);
  free(t2);
  free(t3);
  field_free(&f);
  return rc;
}

/* One chunk's two payloads from x and a subbin field s (used to check a GPU
 * stream chunk by chunk after the Bellman certificate has shown that s is
 * the fixpoint).  out receives bin payload then subbin
 * payload; sizes2 = {bin_size, sub_size}. */
int lopc_ref_encode_chunk(const void* x, uint64_t n, int dtype, double eps, const uint32_t* s, uint64_t c,
                          void* out, uint32_t* sizes2) {
  if ((dtype != 0 && dtype != 1) || check_eps(eps)) return E_ARG;
  int k = dtype == 0 ? 4 : 8;
  uint64_t W = CHUNK_BYTES / (uint64_t)k;
  if (c * W >= n) return E_ARG;
  uint8_t *bw = (uint8_t*)calloc(CHUNK_BYTES, 1), *sw = (uint8_t*)calloc(CHUNK_BYTES, 1);
  uint8_t *t1 = (uint8_t*)malloc(CHUNK_BYTES), *t2 = (uint8_t*)malloc(2 * CHUNK_BYTES),
          *t3 = (uint8_t*)malloc(2 * CHUNK_BYTES);
  int rc = 0;
  if (!bw || !sw || !t1 || !t2 || !t3) {
    rc = E_INTERNAL;
    goto out;
  }
  for (uint64_t i = c * W; i < n && i < (c + 1) * W; i++) {
    int64_t b;
    uint64_t bwv, swv;
    if (lopc_ref_bin(value_at(x, i, dtype), eps, dtype, &b)) {
      bwv = (uint64_t)b & mask_k(k);
      swv = s[i];
    } else {
      bwv = dtype == 0 ? 0x80000000ull : 0x8000000000000000ull;
      swv = bits_at(x, i, dtype);
    }
    word_put(bw + (i - c * W) * k, k, bwv);
    word_put(sw + (i - c * W) * k, k, swv);
  }
  sizes2[0] = (uint32_t)encode_bin_chunk(bw, k, (uint8_t*)out, t1, t2, t3);
  sizes2[1] = (uint32_t)encode_sub_chunk(sw, k, (uint8_t*)out + sizes2[0], t1, t2, t3);
out:
  free(bw);
  free(sw);
  free(t1);
  free(t2);
  free(t3);
  return rc;
}

int lopc_ref_stream_info(const void* in, size_t nbytes, int* ndims, uint64_t* dims3, int* dtype,
                         double* eps, uint64_t* n_elems, uint32_t* n_chunks_out) {
  const uint8_t* p = (const uint8_t*)in;
  if (nbytes < HDR_BYTES) return E_CORRUPT;
  if (memcmp(p, "LOPC", 4) != 0) return E_CORRUPT;
  if (get_u16(p + 4) != 1) return E_VERSION;
  int dt = p[6], nd = p[7];
  if ((dt != 0 && dt != 1) || (nd != 2 && nd != 3)) return E_CORRUPT;
  uint64_t d[3] = {get_u64(p + 8), get_u64(p + 16), get_u64(p + 24)};
  if (nd == 2 && d[0] != 1) return E_CORRUPT;
  for (int a = 0; a < 3; a++)
    if (d[a] > (1ull << 40)) return E_CORRUPT;
  uint64_t n = get_u64(p + 40);
  if (d[0] * d[1] > (1ull << 40) || d[0] * d[1] * d[2] != n || n > (1ull << 40)) return E_CORRUPT;
  uint64_t eb = get_u64(p + 32);
  double e;
  memcpy(&e, &eb, 8);
  if (check_eps(e)) return E_CORRUPT;
  if (get_u32(p + 48) != CHUNK_BYTES) return E_CORRUPT;
  uint32_t C = get_u32(p + 52);
  if ((uint64_t)C != n_chunks(n, dt == 0 ? 4 : 8)) return E_CORRUPT;
  if (get_u64(p + 56) != nbytes) return E_CORRUPT;
  if (HDR_BYTES + 8ull * C > nbytes) return E_CORRUPT;
  if (ndims) *ndims = nd;
  if (dims3) {
    dims3[0] = d[0];
    dims3[1] = d[1];
    dims3[2] = d[2];
  }
  if (dtype) *dtype = dt;
  if (eps) *eps = e;
  if (n_elems) *n_elems = n;
  if (n_chunks_out) *n_chunks_out = C;
  return 0;
}

int lopc_ref_chunk_sizes(const void* in, size_t nbytes, uint32_t* sizes, uint32_t cap_pairs) {
  uint32_t C;
  int rc = lopc_ref_stream_info(in, nbytes, NULL, NULL, NULL, NULL, NULL, &C);
  if (rc) return rc;
  if (cap_pairs < C) return E_NOSPACE;
  const uint8_t* tab = (const uint8_t*)in + HDR_BYTES;
  for (uint32_t i = 0; i < 2 * C; i++) sizes[i] = get_u32(tab + 4 * i);
  return 0;
}

/* O12, one chunk: inverse stages of chunk c's two payloads (q: bin payload
 * of bs bytes, then the subbin payload of ss bytes), then O10 for its
 * elements [cW, min((c+1)W, n)) into out (the whole field's buffer). */
static int decode_one_chunk(const uint8_t* q, uint32_t bs, uint32_t ss, uint32_t c, uint64_t n, int dt,
                            double eps, void* out, uint8_t* bw, uint8_t* sw, uint8_t* t1, uint8_t* t2) {
  int k = dt == 0 ? 4 : 8;
  uint64_t W = CHUNK_BYTES / (uint64_t)k;
  /* bins */
  if (bs == CHUNK_BYTES) {
    memcpy(bw, q, CHUNK_BYTES);
  } else {
    long used = lopc_ref_unrze(q, bs, CHUNK_BYTES, 1, t1);
    if (used < 0 || pad4((size_t)used) != bs) return E_CORRUPT;
    lopc_ref_unbitshuffle(t1, W, k, t2);
    lopc_ref_undiffnb(t2, W, k, bw);
  }
  q += bs;
  /* subbins */
  if (ss == CHUNK_BYTES) {
    memcpy(sw, q, CHUNK_BYTES);
  } else {
    size_t l1 = get_u16(q);
    size_t l1max = CHUNK_BYTES + CHUNK_BYTES / (size_t)k / 8 + 64 + 8;
    if (l1 > l1max) return E_CORRUPT;
    long used = lopc_ref_unrze(q + 2, ss - 2, l1, 1, t1);
    if (used < 0 || pad4(2 + (size_t)used) != ss) return E_CORRUPT;
    long used2 = lopc_ref_unrze(t1, l1, CHUNK_BYTES, k, t2);
    if (used2 < 0 || (size_t)used2 != l1) return E_CORRUPT;
    lopc_ref_unbitshuffle(t2, W, k, sw);
  }
  /* O10 per element */
  for (uint64_t i = c * W; i < n && i < (c + 1) * W; i++) {
    uint64_t bwv = word_get(bw + (i - c * W) * k, k);
    uint64_t swv = word_get(sw + (i - c * W) * k, k);
    uint64_t v;
    if (bwv == (dt == 0 ? 0x80000000ull : 0x8000000000000000ull)) {
      v = swv;
    } else {
      int64_t b = dt == 0 ? (int64_t)(int32_t)(uint32_t)bwv : (int64_t)bwv;
      v = decode_point(b, swv, eps, dt);
    }
    memcpy((uint8_t*)out + (size_t)k * i, &v, (size_t)k);
  }
  return 0;
}

int lopc_ref_decode_chunk(const void* payloads, uint32_t bin_size, uint32_t sub_size, uint32_t c, uint64_t n,
                          int dtype, double eps, void* out) {
  uint8_t *bw = (uint8_t*)malloc(CHUNK_BYTES), *sw = (uint8_t*)malloc(CHUNK_BYTES);
  uint8_t *t1 = (uint8_t*)malloc(2 * CHUNK_BYTES), *t2 = (uint8_t*)malloc(2 * CHUNK_BYTES);
  int rc = (!bw || !sw || !t1 || !t2)
               ? E_INTERNAL
               : decode_one_chunk((const uint8_t*)payloads, bin_size, sub_size, c, n, dtype, eps, out, bw, sw, t1, t2);
  free(bw);
  free(sw);
  free(t1);
  free(t2);
  return rc;
}

/* O12: parse, offsets = exclusive scan of sizes, inverse stages, O10. */
int lopc_ref_decompress(const void* in, size_t in_bytes, void* out, size_t out_capacity) {
  int nd, dt;
  uint64_t d3[3], n;
  uint32_t C;
  double eps;
  int rc = lopc_ref_stream_info(in, in_bytes, &nd, d3, &dt, &eps, &n, &C);
  if (rc) return rc;
  int k = dt == 0 ? 4 : 8;
  if (out_capacity < n * (uint64_t)k) return E_NOSPACE;
  const uint8_t* p = (const uint8_t*)in;
  const uint8_t* tab = p + HDR_BYTES;
  uint64_t total = HDR_BYTES + 8ull * C;
  for (uint32_t i = 0; i < 2 * C; i++) {
    uint32_t sz = get_u32(tab + 4 * i);
    if (sz < 4 || sz > CHUNK_BYTES || (sz & 3)) return E_CORRUPT;
    total += sz;
  }
  if (total != in_bytes) return E_CORRUPT;
  uint8_t *bw = (uint8_t*)malloc(CHUNK_BYTES), *sw = (uint8_t*)malloc(CHUNK_BYTES);
  uint8_t *t1 = (uint8_t*)malloc(2 * CHUNK_BYTES), *t2 = (uint8_t*)malloc(2 * CHUNK_BYTES);
  if (!bw || !sw || !t1 || !t2) {
    rc = E_INTERNAL;
    goto out;
  }
  const uint8_t* q = p + HDR_BYTES + 8ull * C;
  for (uint32_t c = 0; c < C; c++) {
    uint32_t bs = get_u32(tab + 8 * c), ss = get_u32(tab + 8 * c + 4);
    rc = decode_one_chunk(q, bs, ss, c, n, dt, eps, out, bw, sw, t1, t2);
    if (rc) goto out;
    q += bs + ss;
  }
out:
  free(bw);
  free(sw);
  free(t1);
  free(t2);
  return rc;
}

/* ------------------------------------------------------------------ */
/* O13 checkers.                                                        */
/* ------------------------------------------------------------------ */
uint64_t lopc_ref_order_violations(const void* x, const void* y, int ndims, const uint64_t* dims,
                                   int dtype) {
  grid_t g;
  if (make_grid(ndims, dims, &g)) return ~0ull;
  uint64_t bad = 0;
  for (uint64_t p = 0; p < g.n; p++) {
    for (int j = 0; j < g.D; j++) { /* each star edge once: p -> p + e */
      uint64_t q;
      if (!neighbour(&g, p, j, &q)) continue;
      double xp = value_at(x, p, dtype), xq = value_at(x, q, dtype);
      if (isnan(xp) || isnan(xq)) continue; /* G11 */
      int64_t op = lopc_ref_ord(bits_at(x, p, dtype), dtype);
      int64_t oq = lopc_ref_ord(bits_at(x, q, dtype), dtype);
      int64_t yp = lopc_ref_ord(bits_at(y, p, dtype), dtype);
      int64_t yq = lopc_ref_ord(bits_at(y, q, dtype), dtype);
      double vyp = value_at(y, p, dtype), vyq = value_at(y, q, dtype);
      int lx = op != oq ? op < oq : p < q;
      int ly = yp != yq ? yp < yq : p < q;
      if (isnan(vyp) || isnan(vyq) || lx != ly) bad++;
    }
  }
  return bad;
}

uint64_t lopc_ref_bound_violations(const void* x, const void* y, uint64_t n, int dtype,
                                   double eps) {
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; i++) {
    double a = value_at(x, i, dtype), b = value_at(y, i, dtype);
    int64_t tmp;
    if (!lopc_ref_bin(a, eps, dtype, &tmp)) {
      if (bits_at(x, i, dtype) != bits_at(y, i, dtype)) bad++;
      continue;
    }
    if (!(b <= a)) {
      bad++;
      continue;
    }
    /* exact a - b via TwoSum: d + err */
    double d = a - b;
    double bb = d - a;
    double err = (a - (d - bb)) + (-b - bb);
    if (!(d < eps || (d == eps && err <= 0))) bad++;
  }
  return bad;
}

uint64_t lopc_ref_certify(const void* x, int ndims, const uint64_t* dims, int dtype, double eps,
                          const uint32_t* s) {
  field_t f;
  if (field_init(&f, x, ndims, dims, dtype, eps)) return ~0ull;
  uint64_t bad = 0;
  for (uint64_t p = 0; p < f.g.n; p++) {
    if (f.bin[p] == INT64_MIN) continue;
    uint64_t best = 0;
    for (int j = 0; j < 2 * f.g.D; j++) {
      uint64_t q;
      if (neighbour(&f.g, p, j, &q) && is_arc(&f, q, p)) {
        uint64_t v = (uint64_t)s[q] + (q > p ? 1u : 0u);
        if (v > best) best = v;
      }
    }
    if (best != s[p]) bad++;
  }
  field_free(&f);
  return bad;
}

/* ---- row a0: NOA range -------------------------------------------- */
uint64_t lopc_ref_value_range(const void* x, uint64_t n, int dtype, double* vmin, double* vmax) {
  uint64_t cnt = 0;
  double lo = 0.0, hi = 0.0;
  for (uint64_t i = 0; i < n; i++) {
    double v = value_at(x, i, dtype);
    if (!isfinite(v)) continue;
    if (cnt == 0 || v < lo) lo = v;
    if (cnt == 0 || v > hi) hi = v;
    cnt++;
  }
  *vmin = lo;
  *vmax = hi;
  return cnt;
}

double lopc_ref_noa_eps(const void* x, uint64_t n, int dtype, double rel) {
  double lo, hi;
  if (lopc_ref_value_range(x, n, dtype, &lo, &hi) == 0) return rel;
  double r = hi - lo;
  return r > 0 ? rel * r : rel;
}
