"""Seeded synthetic inputs shared by the tests, the oracle runs and bench.py.

This module holds NONE of the method's arithmetic (no tree, no draft, no
sampling): it only produces token streams and logits that look like the
paper's workloads, from explicit seeds.  Both the oracle (``oracle/``) and the
CUDA path (``paper_2601_09083_b200``) consume what it returns; neither is
imported here.

Recipe (motivated by P:L97 long-tailed response
lengths and P:L101 cross-epoch similarity):
  * token ids: Zipf(1.1) ranks over V, mapped through a seeded permutation;
  * per prompt p and epoch e a template R_{p,e}, length ~ LogNormal(median m,
    sigma 0.9) clipped to [16, cap];
  * sibling k's stream: copy of the template that forks with prob 0.03 per
    position into a fresh Zipf segment (geometric length, mean 24) and re-joins
    the template at a random offset within +-32;
  * epoch drift: R_{p,e+1} = R_{p,e} with a 5% token edit rate;
  * logits bulk x ~ N(0, 2^2); the row's head token gets mean + gap, where the
    gap profile "rl-mix" draws 70% of rows from U[18,24] and 30% from U[12,18];
    3 distractors at head - U[0.5, 4].
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Workload", "zipf_tokens", "make_templates", "sibling_stream", "drift",
           "make_workload", "random_logits_np", "bf16_bits", "gap_profile", "FIG3_VOCAB",
           "fig3_sentences", "splitmix64", "RolloutStreams", "policy_row_edits",
           "SimPolicy"]


def splitmix64(x: int) -> int:
    """splitmix64 finaliser (Steele et al.), used for seeds and the prompt-owner hash."""
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def zipf_tokens(rng: np.random.Generator, n: int, V: int, perm: np.ndarray, s: float = 1.1):
    r = rng.zipf(s, size=n)
    r = np.minimum(r - 1, V - 1)
    return perm[r].astype(np.int32)


def _lengths(rng, n, median, cap, sigma=0.9):
    L = np.exp(rng.normal(np.log(median), sigma, size=n))
    return np.clip(L, 16, cap).astype(np.int64)


def make_templates(rng, n_prompts, V, perm, median, cap):
    lens = _lengths(rng, n_prompts, median, cap)
    return [zipf_tokens(rng, int(l), V, perm) for l in lens]


def sibling_stream(rng, template: np.ndarray, V: int, perm: np.ndarray, cap: int,
                   fork_p: float = 0.03, fork_mean: int = 24, rejoin: int = 32):
    out = []
    i = 0
    n = len(template)
    while i < n and len(out) < cap:
        if rng.random() < fork_p:
            seg = int(rng.geometric(1.0 / fork_mean))
            out.extend(zipf_tokens(rng, seg, V, perm).tolist())
            i = max(0, min(n - 1, i + int(rng.integers(-rejoin, rejoin + 1))))
        out.append(int(template[i]))
        i += 1
    return np.asarray(out[:cap], np.int32)


def drift(rng, template: np.ndarray, V: int, perm: np.ndarray, rate: float = 0.05):
    t = template.copy()
    m = rng.random(len(t)) < rate
    t[m] = zipf_tokens(rng, int(m.sum()), V, perm)
    return t


@dataclass
class Workload:
    """A synthetic rollout batch: prior-epoch rollouts (warm cache) and the
    ground-truth streams of the active sequences."""
    V: int
    n_prompts: int
    samples: int
    prior: list = field(default_factory=list)       # list of (prompt, np.int32 tokens)
    truth: list = field(default_factory=list)       # per active sequence: np.int32 tokens
    seq_prompt: np.ndarray = None                   # prompt id per active sequence
    seq_id: np.ndarray = None                       # u64 ids (epoch << 40 | p << 8 | k)
    runahead: list = field(default_factory=list)    # (prompt, tokens) run-ahead rollouts


def make_workload(seed: int, V: int, n_prompts: int, samples: int, median: int, cap: int,
                  prior_epochs: int = 1, active: int | None = None,
                  runahead: tuple | None = None) -> Workload:
    """runahead = (first prompt, n prompts, streams per prompt): rollouts of
    prompts that will be sampled soon (P:L151 run-ahead generation), drawn from
    the same current-epoch templates as the active sequences, returned in
    w.runahead as (prompt, tokens).  Drawn after everything else, so the rest
    of the workload does not depend on it."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(V).astype(np.int32)
    tmpl = make_templates(rng, n_prompts, V, perm, median, cap)
    w = Workload(V=V, n_prompts=n_prompts, samples=samples)
    for e in range(prior_epochs):
        for p in range(n_prompts):
            for k in range(samples):
                w.prior.append((p, sibling_stream(rng, tmpl[p], V, perm, cap)))
        tmpl = [drift(rng, t, V, perm) for t in tmpl]
    n_act = n_prompts * samples if active is None else active
    seq_prompt, seq_id, truth = [], [], []
    for idx in range(n_act):
        p, k = idx // samples, idx % samples
        seq_prompt.append(p)
        seq_id.append((prior_epochs << 40) | (p << 8) | k)
        truth.append(sibling_stream(rng, tmpl[p], V, perm, cap))
    w.truth = truth
    w.seq_prompt = np.asarray(seq_prompt, np.int32)
    w.seq_id = np.asarray(seq_id, np.uint64)
    if runahead is not None:
        p0, npr, per = runahead
        w.runahead = [(p, sibling_stream(rng, tmpl[p], V, perm, cap))
                      for p in range(p0, p0 + npr) for _ in range(per)]
    return w


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns (uint16), round-to-nearest-even."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    rounded = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    out = rounded.astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def gap_profile(rng, n_rows: int, profile: str = "rl-mix") -> np.ndarray:
    return head_profile(rng, n_rows, profile)[0]


def head_profile(rng, n_rows: int, profile: str = "rl-mix"):
    """Per row: the head's gap above the bulk mean and the 3 distractors'
    offsets below the head.  rl-mix = low-entropy reasoning with occasional
    forks: 70% "confident" rows (gap U[18,24], distractors U[5,9] below,
    p_head > 0.97) and 30% "uncertain" rows (gap U[12,18], distractors
    U[0.5,4] below)."""
    if profile == "rl-mix":
        conf = rng.random(n_rows) < 0.7
        gap = np.where(conf, rng.uniform(18, 24, n_rows), rng.uniform(12, 18, n_rows))
        off = np.where(conf[:, None], rng.uniform(5, 9, (n_rows, 3)),
                       rng.uniform(0.5, 4, (n_rows, 3)))
        return gap, off
    gap = {"peaked": 26.0, "moderate": 18.0, "flat": 0.0}.get(profile)
    if gap is None:
        raise ValueError(profile)
    return np.full(n_rows, gap), rng.uniform(0.5, 4, (n_rows, 3))


def random_logits_np(rng, n_rows: int, V: int, heads=None, profile: str = "rl-mix",
                     sigma: float = 2.0) -> np.ndarray:
    """float32 logits rows: bulk N(0, sigma^2), head token at +gap, 3 distractors."""
    if profile == "flat":
        return rng.random((n_rows, V), dtype=np.float32)
    x = rng.normal(0.0, sigma, size=(n_rows, V)).astype(np.float32)
    if heads is None:
        heads = rng.integers(0, V, n_rows)
    gaps = gap_profile(rng, n_rows, profile)
    rows = np.arange(n_rows)
    x[rows, heads] = gaps.astype(np.float32)
    for _ in range(3):
        d = rng.integers(0, V, n_rows)
        x[rows, d] = (gaps - rng.uniform(0.5, 4.0, n_rows)).astype(np.float32)
    x[rows, heads] = gaps.astype(np.float32)
    return x


# ---- the paper's Fig. 3 worked example, tokenised as in SPEC S:L76
FIG3_VOCAB = {"the": 0, "cat": 1, "sit": 2, "on": 3, "mat": 4, "sofa": 5, "eat": 6, "fish": 7}


def fig3_sentences():
    """'the cat sit on the mat' x4, '... sofa' x1, 'the cat eat the fish' x2."""
    s = []
    s += ["the cat sit on the mat"] * 4
    s += ["the cat sit on the sofa"] * 1
    s += ["the cat eat the fish"] * 2
    return [np.asarray([FIG3_VOCAB[w] for w in x.split()], np.int32) for x in s]


# ---- rollout-loop inputs (the slot scheduler) ---------------
# Streams are keyed, not drawn in sequence, so any subset of (prompt, epoch,
# sample) can be generated in any order and every mode of a simulation sees
# the same rollouts.

_U64 = np.uint64


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser over a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + _U64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
        return z ^ (z >> _U64(31))


def _unit(x: np.ndarray) -> np.ndarray:
    """uint64 -> float64 uniform in [0, 1) from the top 53 bits."""
    return (x >> _U64(11)).astype(np.float64) * (1.0 / (1 << 53))


class RolloutStreams:
    """Ground-truth token streams of a dataset's rollouts: prompt p's template
    at epoch e drifts from epoch e - 1 (5% edits), sample j of (p, e) is a
    sibling stream of that template.  Epoch 0 is the history a warm cache
    holds; run-ahead rollouts are further samples j >= K of the same
    (p, e) (they are drawn from the current policy)."""

    def __init__(self, seed: int, V: int, median: int, cap: int):
        self.seed, self.V, self.median, self.cap = seed, V, median, cap
        self.perm = np.random.default_rng([seed, 0]).permutation(V).astype(np.int32)
        self._tmpl = {}

    def template(self, p: int, e: int) -> np.ndarray:
        if (p, e) not in self._tmpl:
            if e == 0:
                rng = np.random.default_rng([self.seed, 1, p])
                self._tmpl[(p, e)] = make_templates(rng, 1, self.V, self.perm, self.median,
                                                    self.cap)[0]
            else:
                rng = np.random.default_rng([self.seed, 2, p, e])
                self._tmpl[(p, e)] = drift(rng, self.template(p, e - 1), self.V, self.perm)
        return self._tmpl[(p, e)]

    def stream(self, p: int, e: int, j: int) -> np.ndarray:
        rng = np.random.default_rng([self.seed, 3, p, e, j])
        return sibling_stream(rng, self.template(p, e), self.V, self.perm, self.cap)


def policy_row_edits(seed: int, keys, pos, heads, V: int, profile: str = "rl-mix"):
    """The policy stand-in of the rollout simulation, as sparse edits of an
    all-zero logits row: the row of sequence `key` predicting position `pos`
    puts its head token (the ground truth there) at +gap and 3 distractors
    below it.  Every value is a function of (seed, key, pos) only, so the
    committed stream does not depend on the drafts (losslessness makes the
    modes' rollouts identical).  Returns (tokens [n, 4] int64, values [n, 4]
    float32, already representable in bf16)."""
    keys = np.asarray(keys, np.uint64)
    pos = np.asarray(pos, np.int64).astype(np.uint64)
    heads = np.asarray(heads, np.int64)
    with np.errstate(over="ignore"):
        base = _mix64(keys * _U64(0xD1B54A32D192ED03) ^ pos * _U64(0x8CB92BA72F3D8DD7)
                      ^ _U64(seed & (2 ** 64 - 1)))
        u = [_unit(_mix64(base + _U64(i))) for i in range(8)]
    if profile == "rl-mix":
        conf = u[0] < 0.7
        gap = np.where(conf, 18 + 6 * u[1], 12 + 6 * u[1])
        offs = [np.where(conf, 5 + 4 * u[2 + k], 0.5 + 3.5 * u[2 + k]) for k in range(3)]
    else:
        g = {"peaked": 26.0, "moderate": 18.0}[profile]
        gap = np.full(len(keys), g)
        offs = [0.5 + 3.5 * u[2 + k] for k in range(3)]
    tok = np.empty((len(keys), 4), np.int64)
    val = np.empty((len(keys), 4), np.float32)
    tok[:, 0] = heads
    val[:, 0] = gap
    for k in range(3):
        # offset 1 + k + 3m in [1, V - 1]: never the head, distinct per k (mod 3)
        m = (u[5 + k] * ((V - 4) // 3)).astype(np.int64)
        tok[:, k + 1] = (heads + 1 + k + 3 * m) % V
        val[:, k + 1] = gap - offs[k]
    # bf16-representable values: both engines see the same bits
    val = (bf16_bits(val).astype(np.uint32) << 16).view(np.float32)
    return tok, val


class SimPolicy:
    """The rollout simulation's policy stand-in for one tick's draft layout:
    per logits row (sequence s = slots[i]; the root row predicts position
    len[s], draft node j predicts len[s] + depth_j) the edits of
    `policy_row_edits` with the head at the rollout's ground-truth token
    (clamped to its last token).  truth: [S, W] padded table, truth_len: [S].
    Returns (tokens [rows, 4], values [rows, 4]) in row order."""

    def __init__(self, seed: int, V: int, profile: str = "rl-mix"):
        self.seed, self.V, self.profile = seed, V, profile

    def __call__(self, slots, row_offsets, draft_len, draft_depth, seq_len, seq_key, truth,
                 truth_len):
        slots = np.asarray(slots, np.int64)
        n = len(slots)
        B = draft_depth.shape[1]
        dep = np.zeros((n, B + 1), np.int64)
        dep[:, 1:] = draft_depth
        valid = np.arange(B + 1)[None, :] <= np.asarray(draft_len, np.int64)[:, None]
        si = np.broadcast_to(slots[:, None], (n, B + 1))[valid]   # row order
        pos = np.asarray(seq_len, np.int64)[si] + dep[valid]
        assert len(si) == int(row_offsets[n])
        heads = truth[si, np.minimum(pos, np.asarray(truth_len, np.int64)[si] - 1)]
        return policy_row_edits(self.seed, np.asarray(seq_key, np.uint64)[si], pos, heads,
                                self.V, self.profile)
