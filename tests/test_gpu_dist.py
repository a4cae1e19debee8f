"""The multi-GPU exchange on the GPU path (libsrt's pack / unpack / apply
kernels + dist.ShardedStep + dist.GpuOps), with G virtual ranks in one
process on one GPU: the span all-gather is a concatenation of the ranks' send
buffers and the draft return an in-process all-to-all (dist.virtual_all_to_all).  Every rank's committed tokens and owned trees must equal the
single-process ORACLE run of tests/test_dist_gloo.py (G-invariance and
parity at once)."""
import numpy as np
import pytest

import test_dist_gloo as T

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [1, 2, 3])
def test_virtual_ranks_match_oracle(orc, G):
    import torch
    import paper_2601_09083_b200 as srt
    from paper_2601_09083_b200.dist import GpuOps, ShardPlan, ShardedStep, virtual_all_to_all
    ref_tab, ref_len, ref_o, w = T._reference(orc)
    _, t0, max_new = T._workload()
    plan = ShardPlan.build(w.seq_prompt, G)
    B, stride = T.B, 64 + T.B + 2
    dev = torch.device("cuda")
    i32 = dict(dtype=torch.int32, device=dev)
    ranks = []
    for r in range(G):
        mine = plan.prompts[r]
        cache = srt.SrtCache(srt.config(T.V, max(1, len(mine)), T.D, T.L, B,
                                        logits_dtype=torch.float32))
        for p, tk in w.prior:
            if p in mine:
                t = torch.tensor(np.asarray(tk, np.int32)[None, :], **i32)
                cache.insert(torch.tensor([int(np.searchsorted(mine, p))], **i32), t,
                             torch.zeros(1, **i32), torch.tensor([t.shape[1]], **i32))
        mtab, mlen = T._tables(w, plan.mirror[r], t0, stride)
        ltab, llen = T._tables(w, plan.local[r], t0, stride)
        nm, nl = len(plan.mirror[r]), len(plan.local[r])
        st = dict(cache=cache, m_tok=torch.tensor(mtab, **i32), m_len=torch.tensor(mlen, **i32),
                  m_prompt=torch.tensor(plan.mirror_prompt[r], **i32),
                  l_tok=torch.tensor(ltab, **i32), l_len=torch.tensor(llen, **i32),
                  max_new=torch.tensor(max_new[plan.local[r]], **i32),
                  seq_id=torch.tensor(w.seq_id[plan.local[r]].view(np.int64), device=dev))
        st["m_cursor"] = cache.new_cursors(nm, dev)
        st["m_draft"] = srt.DraftOut.empty(nm, B, dev)
        st["l_draft"] = srt.DraftOut.empty(nl, B, dev)
        st["l_verify"] = srt.VerifyOut.empty(nl, nl * (B + 1), B, dev)
        if nm:
            cache.insert(st["m_prompt"], st["m_tok"], torch.zeros(nm, **i32), st["m_len"],
                         cursor=st["m_cursor"])
        ops = GpuOps(cache, B, st["m_prompt"], st["m_tok"], st["m_len"], st["m_cursor"],
                     st["m_draft"], st["l_draft"], st["l_len"], st["l_verify"])
        st["ex"] = ShardedStep(plan, r, ops, None, B, device=dev)
        ranks.append(st)
    for k in range(T.STEPS):
        recvs = virtual_all_to_all(plan, [st["ex"].draft_send() for st in ranks])
        for st, recv in zip(ranks, recvs):
            st["ex"].draft_recv(recv)
        for r, st in enumerate(ranks):
            d = st["l_draft"]
            dd = dict(row_offsets=d.row_offsets.cpu().numpy(), draft_len=d.draft_len.cpu().numpy(),
                      draft_depth=d.draft_depth.cpu().numpy(), draft_tok=d.draft_tok.cpu().numpy())
            x = T._logits(plan.local[r], dd, st["l_len"].cpu().numpy(), w)
            st["cache"].verify(torch.from_numpy(x).to(dev), d, st["seq_id"], 1234, st["l_tok"],
                               st["l_len"], st["max_new"], out=st["l_verify"], rows=x.shape[0])
        recv = torch.cat([st["ex"].commit_send() for st in ranks])
        for st in ranks:
            st["ex"].commit_recv(recv)
    torch.cuda.synchronize()
    for r, st in enumerate(ranks):
        assert np.array_equal(st["l_len"].cpu().numpy(), ref_len[plan.local[r]])
        assert np.array_equal(st["l_tok"].cpu().numpy(), ref_tab[plan.local[r]])
        assert np.array_equal(st["m_len"].cpu().numpy(), ref_len[plan.mirror[r]])
        for i, p in enumerate(plan.prompts[r]):
            g = [tuple(x) for x in st["cache"].dump(i)]
            o = [tuple(int(v) for v in x) for x in ref_o.dump(int(p))]
            assert g == o, f"rank {r} tree of prompt {p}"
        bits, _ = st["cache"].status()
        assert bits == 0
