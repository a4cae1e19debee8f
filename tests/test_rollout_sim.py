"""The rollout loop's slot scheduler (P:L50-51, P:L151,
P:L196-204; SPEC scheduler invariants S:L369-374) on the oracle engine:
losslessness across modes, run-ahead isolation, accounting, time dominance,
bubbles, reproducibility."""
import numpy as np
import pytest

import synth
from oracle_engine import OracleEngine
from paper_2601_09083_b200.rollout import RA_BIT, RolloutSim, SimConfig, seq_key, summarize

MODES = [("baseline", False), ("history_only", False), ("srt", False), ("srt", True)]


def run(mode, ra, **over):
    kw = dict(V=1000, D=16, L=8, Bmax=8, prompts_per_step=2, samples=4, steps=3, mode=mode,
              run_ahead=ra, median=48, cap=200, seed=1)
    kw.update(over)
    cfg = SimConfig(**kw)
    sim = RolloutSim(cfg, OracleEngine(cfg, synth.SimPolicy(cfg.seed, cfg.V)),
                     synth.RolloutStreams(cfg.seed, cfg.V, cfg.median, cfg.cap))
    sim.run()
    return sim


@pytest.fixture(scope="module")
def sims():
    return {m: run(*m) for m in MODES}


def test_rollouts_identical_across_modes(sims):
    """On-policy purity: the returned rollouts are the plain
    decoding's (baseline commits one sampled token per tick), whatever the
    cache strategy."""
    base = sims[("baseline", False)].rollouts
    assert len(base) == 3 * 2 * 4
    for m, s in sims.items():
        assert s.rollouts.keys() == base.keys(), m
        for k in base:
            assert np.array_equal(s.rollouts[k], base[k]), (m, k)


def test_rollouts_are_the_real_sequences(sims):
    """Run-ahead isolation ("never used for learning
    targets"): exactly the K samples of each step's prompts are returned,
    each of its rollout's full length."""
    s = sims[("srt", True)]
    c = s.cfg
    want = {seq_key(k, p, j) for k in range(c.steps)
            for p in range(k * c.prompts_per_step, (k + 1) * c.prompts_per_step)
            for j in range(c.samples)}
    assert set(s.rollouts) == want
    assert not any(k & RA_BIT for k in s.rollouts)
    assert sum(r.run_ahead_seqs for r in s.reports) > 0
    for k, toks in s.rollouts.items():
        p, j = (k >> 16) & 0xFFFFFFF, k & 0xFFFF
        assert len(toks) == len(s.streams.stream(p, c.epoch, j))


def test_accounting(sims):
    """tokens = accepted + engine steps (each tick commits the accepted
    tokens plus the bonus, truncated at the rollout's end: S:L357); bubbles
    and slot conservation from the per-tick trace."""
    for m, s in sims.items():
        S = s.cfg.n_slots
        for r in s.reports:
            tr = [t for t in s.trace if t["step"] == r.step]
            assert len(tr) == r.ticks
            assert r.tokens == r.accepted + r.seq_ticks, m
            assert r.seq_ticks == sum(t["real"] for t in tr)
            assert r.bubble_slot_ticks == sum(S - t["real"] for t in tr)
            assert all(t["busy"] + t["free"] == S for t in tr)
            assert r.tokens == sum(t["committed"] for t in tr)
        assert sum(r.tokens for r in s.reports) == sum(len(v) for v in s.rollouts.values())
    assert all(r.accepted == 0 for r in sims[("baseline", False)].reports)
    assert all(r.run_ahead_tokens == 0 for m, s in sims.items() if not m[1] for r in s.reports)


def test_time_dominance(sims):
    """with a slot per real sequence every sequence commits >= 1 token
    per tick, so no step takes longer than plain decoding, whose step time is
    its longest rollout."""
    base = sims[("baseline", False)]
    for r in base.reports:
        c = base.cfg
        longest = max(len(v) for k, v in base.rollouts.items() if (k >> 44) & 0xFFFFF == r.step)
        assert r.ticks == longest
    for m, s in sims.items():
        for r, rb in zip(s.reports, base.reports):
            assert r.ticks <= rb.ticks, m
    assert sum(r.ticks for r in sims[("srt", False)].reports) < sum(r.ticks for r in base.reports)


def test_online_beats_history_only(sims):
    """Fig. 5's first ordering on this seeded case (deterministic, so a fixed
    property): inserting running rollouts raises the mean accepted tokens."""
    h = summarize(sims[("history_only", False)].reports)["mean_accepted"]
    o = summarize(sims[("srt", False)].reports)["mean_accepted"]
    assert h < o


def test_run_ahead_needs_bubbles():
    """bubbles exist iff completions are staggered; with one slot per
    real sequence and no look-ahead prompt left, nothing runs ahead; with
    fewer slots than sequences the queue drains first."""
    s = run("srt", True, steps=1, lookahead=0, prompts_per_step=2)
    assert sum(r.run_ahead_seqs for r in s.reports) > 0
    q = run("srt", True, steps=1, slots=3)
    busy = [t["busy"] for t in q.trace]
    assert max(busy) == 3 and all(t["free"] == 3 - t["busy"] for t in q.trace)


def test_reproducible():
    a, b = run("srt", True, steps=2), run("srt", True, steps=2)
    assert [r.as_dict() for r in a.reports] == [r.as_dict() for r in b.reports]
    assert a.trace == b.trace


def test_config_validation():
    with pytest.raises(ValueError):
        SimConfig(V=10, D=4, L=4, Bmax=4, prompts_per_step=1, samples=1, steps=1,
                  mode="history_only", run_ahead=True).validate()
    with pytest.raises(ValueError):
        SimConfig(V=10, D=4, L=4, Bmax=4, prompts_per_step=1, samples=1, steps=1,
                  mode="nope").validate()


def test_policy_edits_keyed_by_sequence_and_position():
    """The stand-in's row depends on (key, position, head) only."""
    t1, v1 = synth.policy_row_edits(3, [7, 7, 9], [4, 5, 4], [1, 1, 1], 1000)
    t2, v2 = synth.policy_row_edits(3, [9, 7], [4, 4], [1, 1], 1000)
    assert np.array_equal(t1[0], t2[1]) and np.array_equal(v1[2], v2[0])
    assert (t1[:, 1:] != t1[:, :1]).all() and (v1[:, 1:] < v1[:, :1]).all()
