"""Multi-GPU plumbing for the SRT path (BJ:north_star: "Prompts shard by hash
across the GPUs of one 8xB200 box, and GRPO/DAPO siblings' decoded spans are
NCCL all-gathered over NVLink before insertion").

Placement.  Prompts are independent (trees never share nodes), so
trees shard by prompt: owner(p) = splitmix64(p) mod G holds T_p plus a MIRROR
of the response tokens of p's sequences.  Sequences are decoded where the
rollout engine puts them: here a contiguous split of the prompt-major batch
(verl-style), so siblings mostly share a rank, which is usually not owner(p).

One step, per rank r:
  1. owner side   srt_draft_cursor over r's mirror sequences; pack the draft
                  records (mirror order = ascending global id, so the records
                  are already grouped by the rank that decodes them);
  2. all-to-all   draft records ("draft return"): each owner sends every
                  decoding rank exactly its sequences' records;
  3. decode side  unpack the records of r's local sequences (+ row offsets);
                  [policy forward on the drafted rows]; srt_verify;
                  pack the committed spans;
  4. all-gather   span records (BJ:configs[4], "NCCL all-gather of decoded
                  spans per step");
  5. owner side   append the spans to r's mirror table; srt_insert_cursor.
The result is identical to G = 1 (same trees per prompt, same drafts, same
commits): the G-invariance tests check it.

This module holds the placement and the routing (which record goes where);
the records are packed / unpacked / applied by libsrt kernels (GpuOps) or,
in the CPU tests, by a stand-in with the same semantics.  No arithmetic of
the method lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

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


@dataclass
class ShardPlan:
    """Static placement of S global sequences (prompt-major) over G ranks,
    identical on every rank (computed, never communicated).

    local[r]    global ids of the sequences rank r decodes (contiguous split)
    mirror[r]   global ids of the sequences whose prompt rank r owns
    prompts[r]  global prompt ids owned by rank r (sorted); a mirror sequence's
                prompt index in r's cache is its prompt's position here
    draft_send[r][d] records owner r sends to decoding rank d (all-to-all splits)
    draft_recv[r][o] records decoding rank r receives from owner o
    draft_src[r][i]  row of rank r's all-to-all receive buffer holding local[r][i]'s draft
    span_src[r][j]   row of the gathered span records holding mirror[r][j]'s span
    """
    world: int
    seq_prompt: np.ndarray
    local: list = field(default_factory=list)
    mirror: list = field(default_factory=list)
    prompts: list = field(default_factory=list)
    mirror_prompt: list = field(default_factory=list)
    draft_send: list = field(default_factory=list)
    draft_recv: list = field(default_factory=list)
    draft_src: list = field(default_factory=list)
    span_src: list = field(default_factory=list)
    n_local_max: int = 0
    n_mirror_max: int = 0

    @staticmethod
    def build(seq_prompt, world: int) -> "ShardPlan":
        seq_prompt = np.asarray(seq_prompt, np.int64)
        S = len(seq_prompt)
        G = world
        plan = ShardPlan(world=G, seq_prompt=seq_prompt)
        bounds = [(r * S) // G for r in range(G + 1)]
        plan.local = [np.arange(bounds[r], bounds[r + 1], dtype=np.int64) for r in range(G)]
        owner = np.array([owner_of(int(p), G) for p in seq_prompt], np.int64)
        plan.mirror = [np.nonzero(owner == r)[0].astype(np.int64) for r in range(G)]
        allp = np.unique(seq_prompt)
        plan.prompts = [np.array([p for p in allp if owner_of(int(p), G) == r], np.int64)
                        for r in range(G)]
        plan.mirror_prompt = [np.searchsorted(plan.prompts[r], seq_prompt[plan.mirror[r]]).astype(np.int32)
                              for r in range(G)]
        plan.n_local_max = max(len(x) for x in plan.local)
        plan.n_mirror_max = max(1, max(len(x) for x in plan.mirror))
        # where each global sequence sits in the gathered buffers
        dec_rank = np.zeros(S, np.int64)
        dec_idx = np.zeros(S, np.int64)
        own_idx = np.zeros(S, np.int64)
        for r in range(G):
            dec_rank[plan.local[r]] = r
            dec_idx[plan.local[r]] = np.arange(len(plan.local[r]))
            own_idx[plan.mirror[r]] = np.arange(len(plan.mirror[r]))
        # draft return (all-to-all): owner o's mirror list is ascending in the
        # global id and every decoding rank holds a contiguous id range, so o
        # sends rank d the slice of its records whose sequences d decodes, in
        # ascending id; rank d's receive buffer is those slices in owner order
        plan.draft_send = [[int(np.count_nonzero(dec_rank[plan.mirror[o]] == d)) for d in range(G)]
                           for o in range(G)]
        plan.draft_recv = [[plan.draft_send[o][d] for o in range(G)] for d in range(G)]
        plan.draft_src = []
        for d in range(G):
            loc = plan.local[d]
            own = owner[loc]
            base = np.concatenate([[0], np.cumsum(plan.draft_recv[d])])[:-1]
            rank_in = np.zeros(len(loc), np.int64)
            for o in range(G):
                sel = np.nonzero(own == o)[0]  # ascending id within the owner's slice
                rank_in[sel] = np.arange(len(sel))
            plan.draft_src.append((base[own] + rank_in).astype(np.int32))
        plan.span_src = [(dec_rank[plan.mirror[r]] * plan.n_local_max + dec_idx[plan.mirror[r]])
                         .astype(np.int32) for r in range(G)]
        return plan


def all_to_all_rows(send, send_counts, recv_counts, group=None):
    """Rows send[sum(send_counts[:d]) : ...] go to rank d; returns the rows
    received from every rank, in rank order (torch all_to_all_single with
    uneven splits: NCCL send/recv pairs, graph-capturable)."""
    import torch
    import torch.distributed as dist
    out = torch.empty((int(sum(recv_counts)),) + tuple(send.shape[1:]), dtype=send.dtype,
                      device=send.device)
    dist.all_to_all_single(out, send[:int(sum(send_counts))].contiguous(),
                           output_split_sizes=list(recv_counts),
                           input_split_sizes=list(send_counts), group=group)
    return out


def virtual_all_to_all(plan: "ShardPlan", sends):
    """In-process stand-in for all_to_all_rows over G virtual ranks:
    sends[o] is owner o's send buffer; returns every rank's receive buffer."""
    import torch
    G = plan.world
    offs = [np.concatenate([[0], np.cumsum(plan.draft_send[o])]) for o in range(G)]
    return [torch.cat([sends[o][int(offs[o][d]):int(offs[o][d + 1])] for o in range(G)])
            for d in range(G)]


def all_gather_rows(t, group=None):
    """Concatenate every rank's [rows, W] tensor along dim 0 (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
    else:
        dist.all_gather(list(out.chunk(world)), t.contiguous(), group=group)
    return out


class ShardedStep:
    """Rank r's half of the exchange protocol over an `ops` object:

      ops.draft_mirror()            -> None   (srt_draft over the mirror table)
      ops.pack_drafts(send)         -> None   (mirror drafts -> send[:n_mirror])
      ops.unpack_drafts(recv, src)  -> None   (recv[src[i]] -> local draft outputs)
      ops.pack_spans(send)          -> None   (local commits -> send[:n_local])
      ops.apply_and_insert(recv, src) -> None (append to the mirror table, insert)

    `gather` concatenates a [rows, W] buffer across ranks (all_gather_rows, or
    an in-process stand-in for virtual ranks); `a2a(send, send_counts,
    recv_counts)` is the draft return (all_to_all_rows).  Virtual-rank
    drivers call the phases (draft_send / draft_recv / commit_send /
    commit_recv) across the ranks themselves."""

    def __init__(self, plan: ShardPlan, rank: int, ops, gather, Bmax: int, device=None,
                 a2a=None):
        import torch
        self.plan, self.rank, self.ops, self.gather, self.a2a = plan, rank, ops, gather, a2a
        kw = dict(dtype=torch.int32, device=device)
        self.draft_buf = torch.full((plan.n_mirror_max, 2 + 5 * Bmax), -1, **kw)
        self.span_buf = torch.zeros((plan.n_local_max, Bmax + 2), **kw)
        self.draft_src = torch.as_tensor(plan.draft_src[rank], **kw)
        self.span_src = torch.as_tensor(plan.span_src[rank], **kw)

    # phases (virtual-rank drivers call them across all ranks in turn)
    def draft_send(self):
        self.ops.draft_mirror()
        self.ops.pack_drafts(self.draft_buf)
        return self.draft_buf

    def draft_recv(self, recv):
        self.ops.unpack_drafts(recv, self.draft_src)

    def commit_send(self):
        self.ops.pack_spans(self.span_buf)
        return self.span_buf

    def commit_recv(self, recv):
        self.ops.apply_and_insert(recv, self.span_src)

    def draft(self):
        """Steps 1-3a: owner drafts, draft return (all-to-all), local unpack."""
        r = self.rank
        self.draft_recv(self.a2a(self.draft_send(), self.plan.draft_send[r],
                                 self.plan.draft_recv[r]))

    def commit(self):
        """Steps 3c-5 (after srt_verify): span all-gather, owner append + insert."""
        self.commit_recv(self.gather(self.commit_send()))


class GpuOps:
    """ShardedStep ops over libsrt for one rank: `cache` holds the trees of
    the rank's owned prompts; mirror_* are the mirror sequence table and
    cursors; local_draft receives the drafts of the local sequences."""

    def __init__(self, cache, Bmax, mirror_prompt, mirror_tok, mirror_len, mirror_cursor,
                 mirror_draft, local_draft, local_pos_base, local_verify):
        import torch
        from . import srt
        self.srt, self.torch = srt, torch
        self.cache, self.Bmax = cache, Bmax
        self.mirror_prompt, self.mirror_tok, self.mirror_len = mirror_prompt, mirror_tok, mirror_len
        self.mirror_cursor, self.mirror_draft = mirror_cursor, mirror_draft
        self.local_draft, self.local_pos_base, self.local_verify = local_draft, local_pos_base, local_verify
        n = mirror_len.shape[0]
        self.frm = torch.zeros(n, dtype=torch.int32, device=mirror_len.device)
        self.to = torch.zeros(n, dtype=torch.int32, device=mirror_len.device)

    def draft_mirror(self):
        if self.mirror_len.shape[0]:  # the match reads the insert cursors (srt_draft_cursor)
            self.cache.draft(self.mirror_prompt, self.mirror_tok, self.mirror_len, self.mirror_len,
                             out=self.mirror_draft, cursor=self.mirror_cursor)

    def pack_drafts(self, send):
        if self.mirror_len.shape[0]:
            self.srt.pack_drafts(self.mirror_draft, self.Bmax, send)

    def unpack_drafts(self, recv, src):
        self.srt.unpack_drafts(recv, src, self.Bmax, self.local_draft, self.local_pos_base)

    def pack_spans(self, send):
        self.srt.pack_spans(self.local_verify, self.Bmax, send)

    def apply_and_insert(self, recv, src):
        if self.mirror_len.shape[0]:
            self.srt.apply_spans(recv, src, self.Bmax, self.mirror_tok, self.mirror_len, self.frm,
                                 self.to)
            self.cache.insert(self.mirror_prompt, self.mirror_tok, self.frm, self.to,
                              cursor=self.mirror_cursor)
