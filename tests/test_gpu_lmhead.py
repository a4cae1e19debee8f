"""The verify pass with the LM-head GEMM fused in front of the sampler
(srt_verify_lmhead*, csrc/lmhead.cu).

Parity is defined in two parts:
* the GEMM: the logits the kernel sampled from (its debug dump) equal the
  fp64 product of the same bf16 inputs within the bound of fp32 accumulation
  plus the final bf16 rounding: |x - x_ref| <= 2^-8 |x_ref| + K 2^-23 sum_k
  |h_k w_k| (stated, not tuned);
* the epilogue: given those logits, every output -- sampled tokens of every
  row, accepted lengths, commits, sequence tables, trees -- equals the
  ORACLE's verify on the dumped logits bit for bit, and equals srt_verify
  (the HBM scan) on them too.
"""
import numpy as np
import pytest

from harness import Pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2601_09083_b200 import build
    build.build()


def _tree_pair(orc, rng, V, dtype, Bmax=16, D=12, L=4, n=24, prompts=2):
    pair = Pair(orc, V, prompts, D, L, Bmax, dtype=dtype, node_capacity=1 << 18)
    base = rng.integers(0, min(V, 60), (prompts, 80)).astype(np.int32)
    rolls = []
    for k in range(10):
        p = k % prompts
        t = np.where(rng.random(80) < 0.1, rng.integers(0, min(V, 60), 80), base[p]).astype(np.int32)
        rolls.append((p, t))
    tab = np.stack([t for _, t in rolls])
    pair.insert([p for p, _ in rolls], tab, np.zeros(len(rolls), np.int32),
                np.full(len(rolls), 80, np.int32))
    prompt = (np.arange(n) % prompts).astype(np.int32)
    ctx = np.zeros((n, 80 + Bmax + 2), np.int32)
    ctx[:, :80] = base[prompt]
    seq_len = rng.integers(2, 60, n).astype(np.int32)
    return pair, prompt, ctx, seq_len


def _inputs(rng, rows_cap, V, K, od, ctx, seq_len, peaked):
    """bf16 hidden states and LM-head weight.  peaked: row r's hidden state
    is gap * W[head_r] + noise (head_r = the context's next token), so the
    logits have an rl-mix-like head; else plain random rows."""
    import torch
    # W ~ N(0, 1/K) (|W_v|^2 ~ 1), H ~ N(0, 2^2): bulk logits ~ N(0, 2^2) as in rl-mix
    W = torch.from_numpy(rng.normal(0, 1.0 / np.sqrt(K), (V, K)).astype(np.float32))
    H = torch.from_numpy(rng.normal(0, 2.0, (rows_cap, K)).astype(np.float32))
    if peaked:
        for j in range(len(seq_len)):
            r0 = int(od["row_offsets"][j])
            for i in range(int(od["draft_len"][j]) + 1):
                dep = 0 if i == 0 else int(od["draft_depth"][j, i - 1])
                head = int(ctx[j, min(int(seq_len[j]) + dep, ctx.shape[1] - 1)]) % V
                H[r0 + i] += float(rng.uniform(8, 24)) * W[head]
    return H.to(torch.bfloat16).cuda(), W.to(torch.bfloat16).cuda()


def _gemm_check(H, W, dump, rows):
    """|x - x_ref| <= 2^-8 |x_ref| + K 2^-23 sum |h w| (fp32 accumulation + bf16 RN)."""
    import torch
    h = H[:rows].double()
    w = W.double()
    ref = h @ w.T
    mag = h.abs() @ w.abs().T
    K = H.shape[1]
    bound = 2.0 ** -8 * ref.abs() + K * 2.0 ** -23 * mag + 1e-30
    err = (dump[:rows].double() - ref).abs()
    bad = int((err > bound).sum().item())
    assert bad == 0, f"{bad} logits outside the accumulation bound (max err {err.max().item()})"
    return float((err / (ref.abs() + 1e-6)).median().item())


@pytest.mark.parametrize("V,K,dtype,peaked,T", [
    (151936, 1536, "bf16", True, 1.0),     # Qwen2.5-1.5B's LM head shape
    (151936, 1536, "bf16", False, 1.0),
    (50000, 256, "bf16", True, 0.7),       # partial last vocab tile, T != 1
    (4099, 200, "bf16", True, 1.0),        # partial noise block, K not a multiple of 64
    (32000, 512, "f32", True, 1.0),        # logits kept in fp32 (no rounding)
])
def test_lmhead_verify_matches_oracle(orc, V, K, dtype, peaked, T):
    import torch
    rng = np.random.default_rng(V + K)
    pair, prompt, ctx, seq_len = _tree_pair(orc, rng, V, dtype)
    od, gd = pair.draft(prompt, ctx, seq_len, pos_base=seq_len)
    pair.compare_drafts(od, gd)
    rows = int(od["row_offsets"][-1])
    assert rows > 2 * len(seq_len)
    rows_cap = len(seq_len) * (pair.Bmax + 1)
    H, W = _inputs(rng, rows_cap, V, K, od, ctx, seq_len, peaked)
    ldt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dump = torch.full((rows_cap, V), float("nan"), dtype=ldt, device="cuda")
    sid = rng.integers(0, 2 ** 62, len(seq_len), dtype=np.uint64)
    max_new = np.full(len(seq_len), 200, np.int32)
    g_tok, g_len = pair.t(ctx), pair.t(seq_len)
    gv = pair.gpu.verify_lmhead(H, W, gd, pair.t(sid.view(np.int64)), 99, g_tok, g_len,
                                pair.t(max_new), temperature=T, rows=rows, logits_out=dump)
    torch.cuda.synchronize()
    assert pair.gpu.status()[0] == 0
    _gemm_check(H, W, dump.float(), rows)
    # epilogue parity: the oracle's verify on the logits the kernel sampled from
    x = dump[:rows].float().cpu().numpy()
    ov, gv2, o_seq, g_seq2, _ = pair.verify(x, od, gd, sid, 99, ctx, seq_len, max_new,
                                            temperature=T)
    pair.compare_verify(ov, gv, o_seq, (g_tok, g_len))
    # and the HBM scan (srt_verify) on the same logits agrees
    pair.compare_verify(ov, gv2, o_seq, g_seq2)
    if peaked:
        assert int(ov["accept_len"].sum()) > 0


def test_lmhead_verify_insert_matches_separate_path(orc):
    """srt_verify_lmhead_insert_cursor == srt_verify_insert_cursor on the
    dumped logits: same commits, sequence tables, cursors and trees."""
    import torch
    rng = np.random.default_rng(77)
    V, K = 151936, 1536
    pair, prompt, ctx, seq_len = _tree_pair(orc, rng, V, "bf16")
    # a second GPU cache with the same history for the reference path
    import paper_2601_09083_b200 as srt
    other = srt.SrtCache(pair.gpu.cfg)
    for p in range(pair.P):
        other.load(p, pair.gpu.dump(p))
    od, gd = pair.draft(prompt, ctx, seq_len, pos_base=seq_len)
    rows = int(od["row_offsets"][-1])
    rows_cap = len(seq_len) * (pair.Bmax + 1)
    H, W = _inputs(rng, rows_cap, V, K, od, ctx, seq_len, True)
    dump = torch.empty((rows_cap, V), dtype=torch.bfloat16, device="cuda")
    sid = pair.t(rng.integers(0, 2 ** 62, len(seq_len), dtype=np.uint64).view(np.int64))
    max_new = pair.t(np.full(len(seq_len), 200, np.int32))
    pr = pair.t(prompt)
    out = []
    for which in ("fused", "separate"):
        tok, ln = pair.t(ctx), pair.t(seq_len)
        cache = pair.gpu if which == "fused" else other
        cur = cache.new_cursors(len(seq_len))
        cache.insert(pr, tok, torch.zeros_like(ln), ln, cursor=cur)  # cursors at seq_len
        if which == "fused":
            v = cache.verify_lmhead(H, W, gd, sid, 5, tok, ln, max_new, prompt_id=pr, cursor=cur,
                                    rows=rows_cap, logits_out=dump)
        else:
            v = cache.verify_insert(dump, gd, sid, 5, tok, ln, max_new, pr, cur, rows=rows_cap)
        torch.cuda.synchronize()
        out.append((v.sampled[:rows].cpu().numpy(), v.n_commit.cpu().numpy(), tok.cpu().numpy(),
                    ln.cpu().numpy(), cur.cpu().numpy(), [cache.dump(p) for p in range(pair.P)]))
    a, b = out
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)
    # cursor records: position / prompt / floor equal, the same suffix nodes
    # exist (node ids are hash slots: cache- and scheduling-dependent)
    NONE = np.uint32(0xFFFFFFFF).view(np.int32)
    np.testing.assert_array_equal(a[4][:, 1:4], b[4][:, 1:4])
    np.testing.assert_array_equal(a[4][:, 4:] == NONE, b[4][:, 4:] == NONE)
    assert a[5] == b[5]
    assert a[1].sum() > len(seq_len)  # multi-token commits happened
