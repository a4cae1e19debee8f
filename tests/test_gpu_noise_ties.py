"""Element-level noise parity and constructed float ties (north_star: "bit-exactly
for sampled tokens under identical Philox keys and IEEE (non-fast-math)
arithmetic, with any float tie-break divergence counted and required to be 0").

* log_det (reading O12): the device function vs the oracle's over EVERY
  positive normal float (2^31 - 2^24 inputs), bit for bit;
* the sampler's noise g_v (reading O11, the block construction): every
  element of >= 1000 row keys at V = 151,936, device vs oracle bit for bit;
* finite exact z ties (two indices with equal RN(x + g) at the row maximum),
  constructed from the oracle's noise, placed in the same 64-token block, in
  blocks owned by different tail warps of the scan, across the stream ring's
  32 KB chunk boundary and in a partial last block: the GPU scan must return
  the smaller index, as the oracle does (its tie count must be 2).
"""
import numpy as np
import pytest

from harness import Pair

pytestmark = pytest.mark.gpu

NOISE_BLK = 64
CHUNK_BYTES = 32 * 1024  # the scan's ring stage (csrc/scan.cu)
BIG = np.float32(32768.0)  # exact in bf16; the f32 grid there is 2^-8


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2601_09083_b200 import build
    build.build()


def test_log_det_every_positive_normal(orc):
    """O12's log_det: device == oracle on all 2^31 - 2^24 positive normal floats."""
    import torch
    import paper_2601_09083_b200 as srt
    first, last = 0x00800000, 0x7F800000  # [smallest normal, +inf)
    chunk = 1 << 26
    buf = torch.empty(chunk, dtype=torch.float32, device="cuda")
    bad = 0
    for b0 in range(first, last, chunk):
        n = min(chunk, last - b0)
        g = srt.log_det_range(b0, n, buf).cpu().numpy().view(np.uint32)
        x = np.arange(b0, b0 + n, dtype=np.uint32).view(np.float32)
        o = orc.log_det_array(x).view(np.uint32)
        bad += int(np.count_nonzero(g != o))
    assert bad == 0, f"{bad} log_det results differ"


def test_row_noise_every_element(orc):
    """O11's noise, element by element: 1024 keys x 151,936 tokens (8 seeds,
    random sequence ids and positions), device == oracle bit for bit."""
    import torch
    import paper_2601_09083_b200 as srt
    V = 151936
    rng = np.random.default_rng(11)
    keys = 0
    for seed in rng.integers(0, 2 ** 63, 8, dtype=np.uint64):
        sid = rng.integers(0, 2 ** 63, 128, dtype=np.uint64)
        pos = rng.integers(0, 20000, 128).astype(np.int32)
        g = srt.row_noise(V, int(seed), torch.from_numpy(sid.view(np.int64)).cuda(),
                          torch.from_numpy(pos).cuda()).cpu().numpy()
        o = orc.row_noise_many(V, int(seed), sid, pos)
        diff = np.count_nonzero(g.view(np.uint32) != o.view(np.uint32))
        assert diff == 0, f"seed {seed}: {diff} noise values differ"
        keys += len(sid)
    assert keys >= 1000


def _z(x, g):
    return (np.float32(x) + np.float32(g)).astype(np.float32)  # RN32 (T = 1)


def _f32_pair(g, a, b, x_b=np.float32(40.0)):
    """x_a, x_b (float32) with RN(x_a + g_a) == RN(x_b + g_b) exactly, or None."""
    zb = _z(x_b, g[b])
    xa = np.float32(zb - g[a])
    for _ in range(64):
        za = _z(xa, g[a])
        if za == zb:
            return xa, x_b
        xa = np.nextafter(xa, np.float32(np.inf) if za < zb else np.float32(-np.inf),
                          dtype=np.float32)
    return None


def _big_pair(g, A, B, X):
    """(a, b), a in A, b in B, a != b, with RN(X + g_a) == RN(X + g_b): at
    X = 2^15 the f32 grid (2^-8) makes such collisions common, and X is a
    bf16 value, so the pair is a finite exact tie in either dtype."""
    za = {}
    for a in A:
        za.setdefault(float(_z(X, g[a])), a)
    for b in B:
        a = za.get(float(_z(X, g[b])))
        if a is not None and a != b:
            return a, b
    return None


def _regions(V, dtype):
    esz = 2 if dtype == "bf16" else 4
    ch = CHUNK_BYTES // esz  # tokens per ring chunk
    nblk = (V + NOISE_BLK - 1) // NOISE_BLK
    last0 = (nblk - 1) * NOISE_BLK
    blk = lambda b: range(b * NOISE_BLK, min(V, (b + 1) * NOISE_BLK))  # noqa: E731
    return {
        "same block": (blk(700), blk(700)),
        "different tail warps": (blk(5), blk(45)),  # tail warp t owns blocks [32t, 32t + 32)
        "chunk boundary": (range(ch - 256, ch), range(ch, ch + 256)),
        "second chunk boundary": (range(2 * ch - 256, 2 * ch), range(2 * ch, 2 * ch + 256)),
        "partial last block": (blk(3), range(last0, V)),
        "head after tie partner": (blk(2000), blk(11)),
    }


@pytest.mark.parametrize("dtype,V", [("f32", 151940), ("bf16", 151944)])
def test_constructed_finite_ties(orc, dtype, V):
    """Rows whose maximum z is shared by exactly two finite logits: the GPU
    picks the smaller index (first maximum, O11) -- divergent rows = 0."""
    from synth import bf16_bits
    assert V % NOISE_BLK not in (0,), "V must leave a partial last block"
    rng = np.random.default_rng(5 if dtype == "f32" else 6)
    seed = 0x7E57
    regions = _regions(V, dtype)
    cases = []  # (region name, method)
    for name in regions:
        cases.append((name, "big"))
        if dtype == "f32":
            cases.append((name, "f32"))
    n = len(cases) * 2  # every case twice (two keys)
    pair = Pair(orc, V, 1, 4, 2, 4, dtype=dtype)
    ctx = np.zeros((n, 16), np.int32)
    seq_len = np.full(n, 3, np.int32)
    od, gd = pair.draft(np.zeros(n, np.int32), ctx, seq_len)  # empty tree: one root row each
    assert int(od["row_offsets"][-1]) == n
    sid = rng.integers(0, 2 ** 62, n, dtype=np.uint64)
    x = rng.normal(0.0, 2.0, (n, V)).astype(np.float32)
    want = np.empty(n, np.int64)
    for r in range(n):
        name, how = cases[r // 2]
        A, B = regions[name]
        g = orc.row_noise(V, seed, int(sid[r]), int(seq_len[r]))
        if how == "big":
            for _ in range(50):  # another key until the regions hold a colliding pair
                ab = _big_pair(g, A, B, BIG)
                if ab is not None:
                    break
                sid[r] = rng.integers(0, 2 ** 62, dtype=np.uint64)
                g = orc.row_noise(V, seed, int(sid[r]), int(seq_len[r]))
            assert ab is not None, (name, "no colliding pair")
            a, b = ab
            x[r, a] = x[r, b] = BIG
        else:
            for _ in range(100):
                a, b = int(rng.choice(list(A))), int(rng.choice(list(B)))
                got = _f32_pair(g, a, b) if a != b else None
                if got is not None:
                    break
            assert got is not None, (name, "no f32 construction")
            x[r, a], x[r, b] = got
        za, zb = _z(x[r, a], g[a]), _z(x[r, b], g[b])
        assert za == zb
        want[r] = min(a, b)
    host = bf16_bits(x) if dtype == "bf16" else x
    if dtype == "bf16":  # the tie survives the bf16 rounding of the rows (2^15 is exact)
        xb = (host.astype(np.uint32) << 16).view(np.float32)
        assert np.all(xb[np.arange(n), want] == BIG)
    tok, ties, nan = orc.sample_rows(host, seed, sid, seq_len)
    assert not nan.any()
    assert np.array_equal(tok, want), "oracle: first maximum"
    assert np.all(ties == 2), ties
    ov, gv, o_seq, g_seq, _ = pair.verify(x, od, gd, sid, seed, ctx, seq_len,
                                          np.full(n, 100, np.int32))
    pair.compare_verify(ov, gv, o_seq, g_seq)
    got = gv.sampled[:n].cpu().numpy()
    divergent = int(np.count_nonzero(got != want))
    assert divergent == 0, [(cases[r // 2], int(got[r]), int(want[r])) for r in range(n)
                            if got[r] != want[r]]
