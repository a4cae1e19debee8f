"""Multi-GPU plumbing for the SRT path (BJ:north_star: "prompts shard by hash
across the GPUs of one 8xB200 box").

Prompts are independent units (trees never share nodes), so the
path shards by prompt: owner(p) = splitmix64(p) mod G.  This module holds the
placement logic only (host side, no arithmetic of the method).
"""
from __future__ import annotations

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def owner_of(prompt: int, world: int) -> int:
    """Rank that owns global prompt `prompt`'s tree."""
    return splitmix64(prompt) % world


def owned(prompts, rank: int, world: int):
    """The subset of `prompts` owned by `rank` (order preserved)."""
    return [p for p in prompts if owner_of(p, world) == rank]
