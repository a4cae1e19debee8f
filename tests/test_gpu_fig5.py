"""Synthetic Fig. 5 through the libsrt kernels:
online insertion of running rollouts beats a history-only cache, and run-ahead
rollouts add more (mean accepted tokens per decoding step).  Seeded and
bit-exact, so the ordering is a fixed property of this workload, not a
statistical test; tools/fig5_sim.py is the full-length run
(profiles/r01_fig5_sim.json)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_fig5_ordering():
    import fig5_sim
    r = {m: fig5_sim.run_mode(m, 24, 2, 0)["mean_accepted_per_step"]
         for m in ("history-only", "online", "online+runahead")}
    assert r["history-only"] < r["online"] < r["online+runahead"], r
