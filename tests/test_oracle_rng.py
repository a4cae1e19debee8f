"""Pins for the oracle's sampler (O11/O12; BJ:north_star part 4).

* Philox4x32-10 against the published Random123 KAT vectors (tests/golden).
* log_det against fp64 libm: <= 4 ulp over the whole noise domain (all 2^23
  inner inputs u and all 2^23 outer inputs -log_det(u)) and on random floats.
* g(r) is monotone non-decreasing in r and spans [-2.8115, 16.6355].
* Gumbel-max frequencies match softmax(x) (chi-square), the defining property
  of Gumbel-max sampling; special cases: ties -> smallest index, -inf rows, NaN.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kats():
    out = []
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        out.append((v[0:4], v[4:6], v[6:10]))
    return out


def test_philox_kat(orc):
    kats = _kats()
    assert len(kats) == 3
    for ctr, key, want in kats:
        got = orc.philox4x32_10(ctr, key)
        assert [int(x) for x in got] == want


def _ulp_err(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """|got - ref| in units of the f32 ulp at ref."""
    ref32 = ref.astype(np.float32)
    ulp = np.spacing(np.abs(ref32)).astype(np.float64)
    return np.abs(got.astype(np.float64) - ref) / ulp


def test_log_det_accuracy_whole_noise_domain(orc):
    """Both log stages over ALL 2^23 noise inputs: <= 4 ulp vs fp64 libm (O12)."""
    r = np.arange(1 << 23, dtype=np.uint64)
    u = ((2 * r + 1).astype(np.float64) * 2.0 ** -24).astype(np.float32)
    assert np.all(u.astype(np.float64) == (2 * r + 1) * 2.0 ** -24)  # u exact in f32
    inner = orc.log_det_array(u)
    assert _ulp_err(inner, np.log(u.astype(np.float64))).max() <= 4.0
    a = -inner
    assert np.all(a > 0) and np.all(np.isfinite(a))
    outer = orc.log_det_array(a)
    assert _ulp_err(outer, np.log(a.astype(np.float64))).max() <= 4.0
    # the noise table is exactly the composition g = -log_det(-log_det(u))
    g = orc.noise_table()
    assert np.array_equal(g, -outer)


def test_log_det_random_floats(orc):
    L = orc.lib()
    rng = np.random.default_rng(1)
    bits = rng.integers(0x00800000, 0x7F800000, 2_000_000, dtype=np.uint32)  # positive normals
    x = bits.view(np.float32)
    got = orc.log_det_array(x)
    ref = np.log(x.astype(np.float64))
    nz = np.abs(ref) > 1e-3  # relative ulp near log(1)=0 is meaningless; checked separately
    assert _ulp_err(got[nz], ref[nz]).max() <= 4.0
    # near 1: absolute error bound of a few f32 ulps of 1
    near = np.abs(ref) <= 1e-3
    if near.any():
        assert np.max(np.abs(got[near] - ref[near])) <= 4 * 2.0 ** -24
    # exact special values
    assert float(orc.log_det(1.0)) == 0.0
    assert abs(float(orc.log_det(2.0)) - np.log(2.0)) <= 2 ** -23


def test_noise_table_range_and_monotone(orc):
    g = orc.noise_table()
    assert g.dtype == np.float32 and g.shape == (1 << 23,)
    assert np.all(np.isfinite(g))
    assert abs(float(g.min()) + 2.8115408) < 1e-6
    assert abs(float(g.max()) - 16.635532) < 1e-5
    assert np.all(np.diff(g) >= 0)  # monotone in r: used by the GPU prune
    # the extreme values are the closed forms at u = 2^-24 and u = 1 - 2^-24
    u_lo, u_hi = 2.0 ** -24, 1 - 2.0 ** -24
    assert abs(g[0] - (-np.log(-np.log(u_lo)))) < 1e-5
    assert abs(g[-1] - (-np.log(-np.log(u_hi)))) < 2e-5


def _softmax_chi2(orc, x, n, seed=12345, pos=7):
    p = np.exp(x.astype(np.float64) - x.max())
    p /= p.sum()
    counts = np.zeros(len(x))
    for i in range(n):
        tok, _ = orc.sample_row(x, seed=seed, seq_id=i, pos=pos)
        counts[tok] += 1
    keep = n * p >= 5          # chi-square cells with enough mass; pool the rest
    obs = np.append(counts[keep], counts[~keep].sum())
    exp = np.append(n * p[keep], n * p[~keep].sum())
    if exp[-1] < 5:
        obs, exp = obs[:-1], exp[:-1]
    return float(((obs - exp) ** 2 / exp).sum()), len(obs) - 1, counts, n * p


def test_gumbel_max_matches_softmax(orc):
    """P9: argmax_v(x_v + g_v) ~ softmax(x): the defining property of Gumbel-max
    sampling.  16-way row (one partial block), 40k independent keys."""
    x = np.array([0.0, 1.0, 2.0, -1.0, 0.5, 3.0, -2.0, 1.5,
                  0.25, -0.5, 2.5, 0.0, -3.0, 1.0, 0.75, 2.0], np.float32)
    chi2, dof, counts, expect = _softmax_chi2(orc, x, 40000)
    assert dof == 15 and chi2 < 37.7, (chi2, counts, expect)  # P(chi2_15 > 37.7) = 0.001
    # and every cell on its own (a single wrong index the total could dilute):
    # |obs - exp| < 4.5 sigma, sigma = sqrt(n p (1 - p))
    p = expect / 40000
    assert np.all(np.abs(counts - expect) < 4.5 * np.sqrt(expect * (1 - p))), (counts, expect)


def test_gumbel_max_matches_softmax_across_blocks(orc):
    """Same property for a row spanning several 64-token noise blocks (the
    top-down construction, O11): mass spread inside one block, across blocks
    and on the partial last block."""
    V = 150  # blocks of 64, 64, 22
    x = np.full(V, -6.0, np.float32)
    for v, val in [(3, 2.0), (10, 1.5), (63, 1.0), (64, 2.2), (100, 0.5), (127, 1.7),
                   (128, 2.1), (140, 1.2), (149, 0.8), (5, 1.9)]:
        x[v] = val
    chi2, dof, counts, expect = _softmax_chi2(orc, x, 40000, seed=99, pos=3)
    # dof ~ 11: P(chi2_11 > 31.3) = 0.001
    assert chi2 < 31.3 + 2 * (dof - 11), (chi2, dof)
    p = expect / 40000
    big = expect >= 25  # per-cell 4.5 sigma on the cells with real mass
    assert np.all(np.abs(counts - expect)[big] < 4.5 * np.sqrt(expect * (1 - p))[big]), (counts, expect)


def _gumbel_cdf(g, loc=0.0):
    return np.exp(-np.exp(-(g - loc)))


def _ks(samples, cdf):
    s = np.sort(np.asarray(samples, np.float64))
    n = len(s)
    F = cdf(s)
    return max(np.max(np.arange(1, n + 1) / n - F), np.max(F - np.arange(0, n) / n))


def test_noise_marginals_are_gumbel(orc):
    """Every element's noise is Gumbel(0,1) (Kolmogorov-Smirnov), the block
    maximum is Gumbel(log n) and sits at the position p_b, elements of a block
    are uncorrelated: the top-down construction yields iid Gumbel noise."""
    V = 130  # blocks 64, 64, 2
    keys = 1500
    G = np.stack([orc.row_noise(V, 777, k, 5) for k in range(keys)])
    assert np.all(np.isfinite(G))
    n = G.size
    assert _ks(G.ravel(), _gumbel_cdf) < 1.63 / np.sqrt(n)      # alpha = 0.01
    bm = G[:, :64].max(axis=1)
    assert _ks(bm, lambda g: _gumbel_cdf(g, np.log(64.0))) < 1.63 / np.sqrt(keys)
    # argmax position of a full block is uniform over its 64 slots
    pos = np.argmax(G[:, 64:128], axis=1)
    cnt = np.bincount(pos, minlength=64)
    chi2 = ((cnt - keys / 64) ** 2 / (keys / 64)).sum()
    assert chi2 < 110  # 63 dof: P(chi2 > 110) ~ 1e-4
    c = np.corrcoef(G[:, 0], G[:, 1])[0, 1]
    assert abs(c) < 4 / np.sqrt(keys)
    # the partial block of 2 elements: max ~ Gumbel(log 2)
    assert _ks(G[:, 128:].max(axis=1), lambda g: _gumbel_cdf(g, np.log(2.0))) < 1.63 / np.sqrt(keys)


def test_sampler_special_cases(orc):
    V = 37
    # all -inf: every z is -inf, the first index wins
    x = np.full(V, -np.inf, np.float32)
    assert orc.sample_row(x, 1, 2, 3)[0] == 0
    # one +inf: it wins regardless of noise
    x = np.zeros(V, np.float32)
    x[17] = np.inf
    assert orc.sample_row(x, 1, 2, 3)[0] == 17
    # two +inf: tie -> smallest index
    x[5] = np.inf
    assert orc.sample_row(x, 9, 9, 9)[0] == 5
    # NaN is flagged and never selected
    x = np.zeros(V, np.float32)
    x[3] = np.nan
    x[30] = 50.0
    tok, nan = orc.sample_row(x, 1, 2, 3)
    assert nan and tok == 30
    # a huge gap always wins (the noise spans < 24 for blocks of <= 64)
    x = np.zeros(V, np.float32)
    x[11] = 24.0
    for s in range(50):
        assert orc.sample_row(x, s, s + 1, s + 2)[0] == 11


def test_sampler_keying(orc):
    """Noise depends on (seed, seq_id, pos, v) only: same key -> same token;
    a different position / seq / seed changes the draw (negative control)."""
    rng = np.random.default_rng(0)
    x = rng.normal(0, 0.1, 512).astype(np.float32)  # nearly flat: draw set by noise
    base = [orc.sample_row(x, 7, 11, pos)[0] for pos in range(40)]
    again = [orc.sample_row(x, 7, 11, pos)[0] for pos in range(40)]
    assert base == again
    assert base != [orc.sample_row(x, 7, 12, pos)[0] for pos in range(40)]
    assert base != [orc.sample_row(x, 8, 11, pos)[0] for pos in range(40)]
    assert base != [orc.sample_row(x, 7, 11, pos + 1)[0] for pos in range(40)]


def _noise_by_steps(orc, V, seed, sid, pos):
    """O11's construction re-derived step by step from the separately pinned
    pieces (Philox: KATs; log_det: accuracy pins) in numpy float32 (IEEE RN)."""
    key = [seed & 0xFFFFFFFF, seed >> 32]
    lo, hi = sid & 0xFFFFFFFF, sid >> 32
    u = lambda w: np.float32((2 * (int(w) >> 9) + 1) * 2.0 ** -24)
    ld = lambda v: orc.log_det_array(np.asarray([v], np.float32))[0]
    g = np.empty(V, np.float32)
    for b in range((V + 63) // 64):
        n = min(64, V - 64 * b)
        w = orc.philox4x32_10([0x80000000 | (b >> 1), pos, lo, hi], key)
        wa, wb = (w[2], w[3]) if b & 1 else (w[0], w[1])
        a = -ld(u(wa))
        E = np.float32(a / np.float32(n))
        G = -ld(E)
        p = (int(wb) * n) >> 32
        for j in range(n):
            v = 64 * b + j
            if j == p:
                g[v] = G
                continue
            A = -ld(u(orc.philox4x32_10([v >> 2, pos, lo, hi], key)[v & 3]))
            gv = -ld(np.float32(E + A))
            g[v] = min(G, gv)
    return g


def test_sampler_noise_by_steps(orc):
    """Implementation consistency, NOT an independent pin: the C oracle's
    noise and sample equal O11 evaluated step by step in numpy from the
    separately pinned primitives (word indexing, block positions, the min
    clamp, z = RN(RN(x/T) + g), first maximum).  The reading itself is pinned
    by the distribution tests above (softmax chi-square and per-cell checks,
    Gumbel marginals, the block-max law, the uniform argmax position)."""
    rng = np.random.default_rng(3)
    V = 203  # blocks 64, 64, 64, 11
    x = rng.normal(0, 2, V).astype(np.float32)
    for seed, sid, pos in [(0x1234567890ABCDEF, (5 << 40) | 77, 19), (1, 2, 0), (2**64 - 1, 2**63, 4095)]:
        g = _noise_by_steps(orc, V, seed, sid, pos)
        assert np.array_equal(g.view(np.uint32), orc.row_noise(V, seed, sid, pos).view(np.uint32))
        assert orc.sample_row(x, seed, sid, pos)[0] == int(np.argmax((x + g).astype(np.float32)))
        T = np.float32(0.7)
        zt = ((x / T).astype(np.float32) + g).astype(np.float32)
        assert orc.sample_row(x, seed, sid, pos, float(T))[0] == int(np.argmax(zt))


def test_sampler_bf16_equals_f32_of_same_values(orc):
    from synth import bf16_bits
    rng = np.random.default_rng(5)
    x = rng.normal(0, 2, 1000).astype(np.float32)
    b = bf16_bits(x)
    xf = (b.astype(np.uint32) << 16).view(np.float32)
    for pos in range(10):
        assert orc.sample_row(b, 1, 2, pos)[0] == orc.sample_row(xf, 1, 2, pos)[0]
