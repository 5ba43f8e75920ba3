"""Pins for the oracle's flags (Alg. 1) and subbin fixpoint (Alg. 2 / O9)."""
import os

import numpy as np
import pytest

from synth.fields import eps_noa, random_field
from tests.exact import brute_subbins, same_bin_components, star_and_links

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "a5_grid.txt")


def load_golden():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        idx, xb, b, m, s, xh = line.split()
        rows.append((int(idx), int(xb, 16), None if b == "ESC" else int(b), int(m, 16), int(s), int(xh, 16)))
    return rows


def test_golden_a5(ref):
    """3x4 grid, eps = 0.25.  Hand derivation of some rows (Alg. 1/2):
    idx0 = 1.0 has same-bin lower neighbours idx1 (0.95, slot +(0,1)) and idx4
    (0.88, slot +(1,0)) -> mask 0x03; both have larger index so w = 1,
    s0 = max(s1, s4) + 1.  idx2 = 0.9 ties with idx3 = 0.9: ties go to the
    lower index (G4), so idx2 precedes idx3 (mask of idx3 = slot -(0,1) = bit 3
    = 0x08, w = 0) and s3 = s2 = 0; s1 = s2 + 1 = 1; s0 = 2.  idx5 = 1.1 has
    lower neighbours idx4, idx1, idx0 through slots -(0,1), -(1,0), -(1,1) ->
    0x38, all w = 0, s5 = max(0, 1, 2) = 2.  lo(4) = 3.5 * 0.25 = 0.875
    (0x3f600000); x^ = lo(b) advanced s ulps.  idx8 = 0.125 = eps/2 is
    a half-point -> bin 1 (half-up, G6).  +Inf is escaped (G11)."""
    rows = load_golden()
    x = np.array([r[1] for r in rows], np.uint32).view(np.float32).reshape(3, 4)
    eps = 0.25
    q = ref.quantize(x, eps).ravel()
    f = ref.flags(x, eps).ravel()
    s = ref.subbins(x, eps).ravel()
    xh = ref.reconstruct(x, eps, s.reshape(3, 4)).view(np.uint32).ravel()
    for i, (_, _, b, m, sv, xhb) in enumerate(rows):
        assert q[i] == (b if b is not None else np.iinfo(np.int64).min)
        assert f[i] == m
        if b is not None:
            assert s[i] == sv
        assert xh[i] == xhb
    assert ref.order_violations(x, xh.view(np.float32).reshape(3, 4)) == 0


def test_star_is_union_of_kuhn_simplices(ref):
    """O2/G1: the oracle's 6 (2D) / 14 (3D) neighbour slots equal the vertex
    star of the Freudenthal subdivision enumerated explicitly."""
    for dims in [(4, 5), (3, 4, 5)]:
        nbr, _ = star_and_links(dims)
        x = np.arange(int(np.prod(dims)), dtype=np.float32).reshape(dims)
        # constant field in one bin: every star neighbour with a lower index is
        # a lower same-bin neighbour, so the flag popcount counts the lower star.
        c = np.zeros(dims, np.float32)
        f = ref.flags(c, 1.0).ravel()
        for p in range(x.size):
            lower = sum(1 for q in nbr[p] if q < p)
            assert bin(int(f[p])).count("1") == lower
        interior = tuple(d // 2 for d in dims)
        p = int(np.ravel_multi_index(interior, dims))
        assert len(nbr[p]) == (6 if len(dims) == 2 else 14)


@pytest.mark.parametrize("n", [2, 3, 5, 10, 17])
def test_decreasing_chain_closed_form(ref, n):
    """Worst case (P:267-276 commented derivation; reading G15): n
    same-bin values decreasing along increasing index -> subbins n-1..0; the
    synchronous iteration needs n sweeps (n-1 changing + the final check) and
    n(n-1)/2 individual increments."""
    x = (1.0 - 1e-4 * np.arange(n)).astype(np.float32).reshape(1, n)
    eps = 1.0
    s = ref.subbins(x, eps).ravel()
    assert list(s) == list(range(n - 1, -1, -1))
    sj, st = ref.subbins(x, eps, "jacobi")
    assert (sj.ravel() == s).all()
    assert st[0] == n and st[2] == n * (n - 1) // 2
    sa, _ = ref.subbins(x, eps, "alg12")
    assert (sa.ravel() == s).all()


def test_increasing_chain_and_plateau_are_zero(ref):
    x = (1.0 + 1e-4 * np.arange(9)).astype(np.float32).reshape(1, 9)
    assert (ref.subbins(x, 1.0) == 0).all()
    c = np.full((4, 4, 4), 0.5, np.float32)
    assert (ref.subbins(c, 10.0) == 0).all()


def test_spec_two_point_examples(ref):
    # S:236-237 / rules (1)/(2) of P:305
    a = np.array([[1.00, 1.01]], np.float32)
    assert list(ref.subbins(a, 0.1).ravel()) == [0, 0]
    b = np.array([[1.01, 1.00]], np.float32)
    assert list(ref.subbins(b, 0.1).ravel()) == [1, 0]


CASES = []
for seed in range(60):
    for kind in ("noise", "ties", "plateau", "grid16", "smooth", "signed_zero_subnormal"):
        CASES.append((seed, kind))


@pytest.mark.parametrize("seed,kind", CASES[::2])
def test_fixpoint_equals_brute_force(ref, seed, kind):
    """DP (O9) == Alg. 1/2 serial worklist (the paper's algorithm) == Jacobi ==
    an independent longest-path computation on exact rational bins; the
    Bellman certificate accepts it; the range bound of P:311 holds."""
    rng = np.random.default_rng(1000 + seed)
    if seed % 2:
        dims = tuple(int(v) for v in rng.integers(1, 7, size=2))
    else:
        dims = tuple(int(v) for v in rng.integers(1, 5, size=3))
    dt = "f32" if seed % 3 else "f64"
    x = random_field(dims, dt, kind, seed)
    rel = [1.0, 0.1, 0.01][seed % 3]
    eps = eps_noa(x, rel)
    s = ref.subbins(x, eps)
    sa, _ = ref.subbins(x, eps, "alg12")
    sj, _ = ref.subbins(x, eps, "jacobi")
    sb, bins = brute_subbins(x, eps)
    assert (s == sb).all()
    assert (sa == s).all() and (sj == s).all()
    assert ref.certify(x, eps, s) == 0
    if s.max() > 0:
        bad = s.copy().ravel()
        bad[int(np.argmax(bad))] += 1
        assert ref.certify(x, eps, bad.reshape(x.shape)) > 0
    # subbins in a same-bin component of n points lie in 0..n-1, and
    # never exceed (#distinct values in the component) - 1.
    comp = same_bin_components(x, bins)
    sv = s.ravel()
    xv = x.ravel()
    for c in set(comp) - {-1}:
        members = [i for i, cc in enumerate(comp) if cc == c]
        mx = max(int(sv[i]) for i in members)
        assert mx <= len(members) - 1
        assert mx <= len({float(xv[i]) for i in members}) - 1


def test_escapes_have_no_arcs(ref):
    x = np.array([[1.0, np.inf, 0.99], [np.nan, 0.98, -np.inf]], np.float32)
    f = ref.flags(x, 1.0).ravel()
    assert f[1] == 0 and f[3] == 0 and f[5] == 0
    s = ref.subbins(x, 1.0)
    sb, _ = brute_subbins(x, 1.0)
    assert (s == sb).all()
