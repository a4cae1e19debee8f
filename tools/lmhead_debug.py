import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle as orc
from harness import Pair
import test_gpu_lmhead as T
V, K = 151936, 1536
rng = np.random.default_rng(V + K)
pair, prompt, ctx, seq_len = T._tree_pair(orc, rng, V, "bf16")
od, gd = pair.draft(prompt, ctx, seq_len, pos_base=seq_len)
rows = int(od["row_offsets"][-1]); rows_cap = len(seq_len) * (pair.Bmax + 1)
H, W = T._inputs(rng, rows_cap, V, K, od, ctx, seq_len, True)
dump = torch.full((rows_cap, V), float("nan"), dtype=torch.bfloat16, device="cuda")
sid = rng.integers(0, 2 ** 62, len(seq_len), dtype=np.uint64)
max_new = np.full(len(seq_len), 200, np.int32)
g_tok, g_len = pair.t(ctx), pair.t(seq_len)
gv = pair.gpu.verify_lmhead(H, W, gd, pair.t(sid.view(np.int64)), 99, g_tok, g_len, pair.t(max_new), rows=rows_cap, logits_out=dump)
torch.cuda.synchronize()
x = dump[:rows].float().cpu().numpy()
print("nan in dump rows:", np.isnan(x).sum())
ov, gv2, o_seq, g_seq2, _ = pair.verify(x, od, gd, sid, 99, ctx, seq_len, max_new)
a = gv.sampled[:rows].cpu().numpy(); b = ov["sampled"]; c = gv2.sampled[:rows].cpu().numpy()
bad = np.nonzero(a != b)[0]
print("rows", rows, "fused!=oracle", len(bad), "scan!=oracle", (c != b).sum())
ro = od["row_offsets"]
for r in bad[:10]:
    s = np.searchsorted(ro, r, side="right") - 1; j = r - ro[s]
    pos = seq_len[s] + (0 if j == 0 else od["draft_depth"][s, j-1])
    g = orc.row_noise(V, 99, int(sid[s]), int(pos))
    z = (x[r] + g).astype(np.float32)
    print(r, "fused", a[r], "oracle", b[r], "z_f", z[a[r]], "z_o", z[b[r]], "x_f", x[r, a[r]], "x_o", x[r, b[r]], "blk", a[r]//64, b[r]//64, "tile", a[r]//256, b[r]//256)
