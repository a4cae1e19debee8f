"""The rollout loop (slots, bubbles, run-ahead) driven through
the libsrt kernels equals the same schedule on the oracle engine tick by tick:
accepted and committed counts, the returned rollouts and every prompt's final
tree (P:L151 online + run-ahead insertion; Fig. 5 strategies)."""
import numpy as np
import pytest

import synth
from oracle_engine import OracleEngine

pytestmark = pytest.mark.gpu


def sim(engine_cls, mode, ra, **over):
    from paper_2601_09083_b200.rollout import RolloutSim, SimConfig
    kw = dict(V=1000, D=16, L=8, Bmax=8, prompts_per_step=2, samples=4, steps=3, mode=mode,
              run_ahead=ra, median=48, cap=200, seed=1)
    kw.update(over)
    cfg = SimConfig(**kw)
    s = RolloutSim(cfg, engine_cls(cfg, synth.SimPolicy(cfg.seed, cfg.V)),
                   synth.RolloutStreams(cfg.seed, cfg.V, cfg.median, cfg.cap))
    s.run()
    return s


@pytest.mark.parametrize("mode,ra,over", [
    ("baseline", False, {}),
    ("history_only", False, {}),
    ("srt", False, {}),
    ("srt", True, {}),
    ("srt", True, dict(slots=5, Bmax=16, D=24, samples=3, steps=2, V=4096)),
])
def test_gpu_schedule_equals_oracle(mode, ra, over):
    from paper_2601_09083_b200.rollout import GpuEngine
    g = sim(GpuEngine, mode, ra, **over)
    o = sim(OracleEngine, mode, ra, **over)
    assert g.trace == o.trace
    assert [r.as_dict() for r in g.reports] == [r.as_dict() for r in o.reports]
    assert g.rollouts.keys() == o.rollouts.keys()
    for k in o.rollouts:
        assert np.array_equal(g.rollouts[k], o.rollouts[k]), k
    for p in range(g.cfg.n_prompts):
        assert [tuple(r) for r in g.eng.dump(p)] == o.eng.dump(p), p


def test_gpu_fig5_ordering():
    """Fig. 5 on a seeded DAPO-shaped case through the kernels:
    history-only < online < online + run-ahead in mean accepted tokens per
    decoding step (deterministic, so a fixed property of this workload)."""
    from paper_2601_09083_b200.rollout import GpuEngine, summarize
    kw = dict(V=151936, D=32, L=8, Bmax=32, prompts_per_step=8, samples=8, steps=2, median=300,
              cap=1024, seed=0, ra_per_prompt=8, node_capacity=1 << 26)
    r = {}
    for mode, ra in (("history_only", False), ("srt", False), ("srt", True)):
        r[(mode, ra)] = summarize(sim(GpuEngine, mode, ra, **kw).reports)
    # step 2's prompts are step 1's look-ahead window: run-ahead pays there
    acc = {k: v["per_step"][-1]["mean_accepted"] for k, v in r.items()}
    assert acc[("history_only", False)] < acc[("srt", False)] < acc[("srt", True)], acc
