"""Independent exact-arithmetic and brute-force checkers used as PINS for the
oracle (tests only).  Nothing here shares code with ``oracle/`` or the CUDA
path: bins and lo() are computed with ``fractions.Fraction``; the star is
derived from explicitly enumerated Kuhn/Freudenthal simplices; critical points
are classified by building link graphs and running union-find.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

BINMAX = {np.float32: 2**31 - 2, np.float64: 2**50}


def exact_bin(x: float, eps: float):
    """floor(x/eps + 1/2) in exact rational arithmetic (reading G6)."""
    return math.floor(Fraction(x) / Fraction(eps) + Fraction(1, 2))


def _next32(f, direction):
    return np.nextafter(np.float32(f), np.float32(direction), dtype=np.float32)


def exact_lo(b: int, eps: float, dtype) -> float:
    """Smallest dtype value >= (b - 1/2) eps, found by search on rationals."""
    T = (Fraction(b) - Fraction(1, 2)) * Fraction(eps)
    if dtype == np.float64:
        c = float(T)
        while Fraction(c) < T:
            c = math.nextafter(c, math.inf)
        while Fraction(math.nextafter(c, -math.inf)) >= T:
            c = math.nextafter(c, -math.inf)
        return c
    c64 = float(T)
    if abs(c64) > 3.4028234663852886e38:
        c = np.float32(np.inf if c64 > 0 else -np.finfo(np.float32).max)
        if c64 < 0:
            return float(c)
        return float("inf")
    c = np.float32(c64)
    while np.isfinite(c) and Fraction(float(c)) < T:
        c = _next32(c, np.inf)
    while True:
        p = _next32(c, -np.inf)
        if np.isfinite(p) and Fraction(float(p)) >= T:
            c = p
        else:
            break
    return float(c)


# --- Kuhn / Freudenthal triangulation, enumerated explicitly ---------------
def kuhn_simplices(dims):
    """All top simplices of the Freudenthal subdivision of the grid: in each
    cube, one simplex per permutation of the axes (path from the low corner
    to the high corner adding one unit vector at a time).  Axes of extent 1
    are dropped first (a one-cell-thick grid is triangulated as the lower-
    dimensional grid it is)."""
    axes = [a for a, d in enumerate(dims) if d > 1]
    out = []
    if not axes:
        return out
    for corner in itertools.product(*[range(dims[a] - 1) for a in axes]):
        for perm in itertools.permutations(range(len(axes))):
            v = list(corner)
            path = [tuple(v)]
            for ax in perm:
                v[ax] += 1
                path.append(tuple(v))
            simp = []
            for c in path:
                full = [0] * len(dims)
                for a, val in zip(axes, c):
                    full[a] = val
                simp.append(tuple(full))
            out.append(tuple(simp))
    return out


def lin(dims, c):
    i = 0
    for d, v in zip(dims, c):
        i = i * d + v
    return i


def star_and_links(dims):
    """For every vertex: the set of neighbours (vertices sharing a simplex)
    and the link edges (pairs of other vertices sharing a simplex with it)."""
    n = int(np.prod(dims))
    nbr = [set() for _ in range(n)]
    ledges = [set() for _ in range(n)]
    for simp in kuhn_simplices(dims):
        ids = [lin(dims, c) for c in simp]
        for v in ids:
            others = [u for u in ids if u != v]
            nbr[v].update(others)
            for a, b in itertools.combinations(others, 2):
                ledges[v].add((min(a, b), max(a, b)))
    return nbr, ledges


def sos_key(vals, i):
    v = vals[i]
    return (v, i)


def _components(verts, edges):
    parent = {v: v for v in verts}

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    for a, b in edges:
        if a in parent and b in parent:
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[ra] = rb
    return len({find(v) for v in verts})


def classify(field: np.ndarray, nbr=None, ledges=None):
    """PL critical-point type of every vertex under SoS (G5 fixes the
    typo: empty lower link => minimum).  Returns (types, (nlow, nup) pairs)."""
    dims = field.shape
    vals = [float(v) for v in field.ravel()]
    if nbr is None:
        nbr, ledges = star_and_links(dims)
    types, pairs = [], []
    for v in range(len(vals)):
        kv = sos_key(vals, v)
        low = {u for u in nbr[v] if sos_key(vals, u) < kv}
        up = nbr[v] - low
        nl = _components(low, ledges[v]) if low else 0
        nu = _components(up, ledges[v]) if up else 0
        if nl == 0:
            t = "min"
        elif nu == 0:
            t = "max"
        elif nl == 1 and nu == 1:
            t = "regular"
        else:
            t = "saddle"
        types.append(t)
        pairs.append((nl, nu))
    return types, pairs


def fp_fn_ft(orig: np.ndarray, recon: np.ndarray):
    """Table III semantics: false positives, false negatives, false
    types of critical points."""
    nbr, led = star_and_links(orig.shape)
    t0, p0 = classify(orig, nbr, led)
    t1, p1 = classify(recon, nbr, led)
    fp = sum(1 for a, b in zip(t0, t1) if a == "regular" and b != "regular")
    fn = sum(1 for a, b in zip(t0, t1) if a != "regular" and b == "regular")
    ft = sum(1 for a, b in zip(t0, t1) if a != "regular" and b != "regular" and a != b)
    pair_mismatch = sum(1 for a, b in zip(p0, p1) if a != b)
    return fp, fn, ft, pair_mismatch


def brute_subbins(field: np.ndarray, eps: float):
    """Least fixpoint of the subbin constraints, computed independently:
    exact Fraction bins, star from explicit simplices, SoS order, and the
    longest weighted path into each vertex by memoised recursion over the
    constraint DAG (P:305 rules (1)/(2); "as low as possible")."""
    dims = field.shape
    dt = field.dtype.type
    vals = [float(v) for v in field.ravel()]
    n = len(vals)
    nbr, _ = star_and_links(dims)
    bins = []
    for v in vals:
        if not math.isfinite(v):
            bins.append(None)
            continue
        b = exact_bin(v, eps)
        bins.append(b if abs(b) <= BINMAX[dt] else None)
    preds = [[] for _ in range(n)]
    for p in range(n):
        if bins[p] is None:
            continue
        for q in nbr[p]:
            if bins[q] is None or bins[q] != bins[p]:
                continue
            # -0.0 == +0.0 as values (G13)
            if (vals[q], q) < (vals[p], p):
                preds[p].append((q, 1 if q > p else 0))
    memo = {}

    def s(p):
        if p in memo:
            return memo[p]
        best = 0
        for q, w in preds[p]:
            best = max(best, s(q) + w)
        memo[p] = best
        return best

    import sys

    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10 * n + 100))
    try:
        out = np.array([s(p) if bins[p] is not None else 0 for p in range(n)], dtype=np.uint32)
    finally:
        sys.setrecursionlimit(old)
    return out.reshape(dims), bins


def same_bin_components(field: np.ndarray, bins):
    """Connected components of same-bin star edges (for the range bound P:311)."""
    dims = field.shape
    n = int(np.prod(dims))
    nbr, _ = star_and_links(dims)
    comp = [-1] * n
    cid = 0
    for s in range(n):
        if comp[s] >= 0 or bins[s] is None:
            continue
        stack = [s]
        comp[s] = cid
        while stack:
            p = stack.pop()
            for q in nbr[p]:
                if comp[q] < 0 and bins[q] is not None and bins[q] == bins[p]:
                    comp[q] = cid
                    stack.append(q)
        cid += 1
    return comp


# --- RZE_g written from the stream-format text --
def rze_spec(data: bytes, g: int) -> bytes:
    """Repeated zero-byte elimination, restated from the format text and
    nothing else: the paper's "bitmap ... repeatedly compressed with a similar
    algorithm that identifies repeating words" (§IV.C, Fig. 2) as the
    container reads it (reading G21).

    * n = L/g words; bitmap B0 has ceil(n/8) bytes, bit i (LSB-first) says
      word i is not all zero.
    * while |B_i| > 8: B_{i+1} has ceil(|B_i|/8) bytes, bit t says
      B_i[t] differs from B_i[t-1] (B_i[-1] = 0); K_i lists, in order, the
      bytes B_i[t] whose bit t is set.
    * output = B_top, then K_{top-1}, ..., K_0, then the non-zero words.

    Written with explicit bit lists (no shifts shared with the oracle's
    packing), so a swapped level order, a "!= 0" instead of "!= previous"
    repeat test, or an MSB-first bitmap changes the bytes."""
    assert len(data) % g == 0
    words = [data[i:i + g] for i in range(0, len(data), g)]
    nonzero = [any(w) for w in words]

    def pack(bits):
        out = []
        for i in range(0, len(bits), 8):
            byte = 0
            for j, b in enumerate(bits[i:i + 8]):
                if b:
                    byte += 2 ** j
            out.append(byte)
        return out

    levels = [pack(nonzero)]          # B0
    kept = []                         # K0, K1, ...
    while len(levels[-1]) > 8:
        b = levels[-1]
        rep = [b[t] != (b[t - 1] if t > 0 else 0) for t in range(len(b))]
        kept.append([b[t] for t in range(len(b)) if rep[t]])
        levels.append(pack(rep))
    out = list(levels[-1])
    for k in reversed(kept):
        out += k
    for w, nz in zip(words, nonzero):
        if nz:
            out += list(w)
    return bytes(out)
