"""Development probe: time srt_verify_lmhead (fused LM-head GEMM + sampler) at
BASELINE's GRPO shape (rows ~ 20K, V = 151,936, K = 1536) against cuBLAS
(torch.matmul) + srt_verify, on random bf16 inputs with rl-mix-like heads.
    python tools/lmhead_probe.py [rows] [K] [reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2601_09083_b200 as srt  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 20480
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1536
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
V, B = 151936, 32
n = rows // (B + 1)
dev = torch.device("cuda")
cache = srt.SrtCache(srt.config(V, 1, 8, 4, B, node_capacity=1 << 16))
g = torch.Generator(device=dev)
g.manual_seed(0)
W = torch.empty(V, K, dtype=torch.bfloat16, device=dev).normal_(0, K ** -0.5, generator=g)
H = torch.empty(n * (B + 1), K, dtype=torch.bfloat16, device=dev).normal_(0, 2.0, generator=g)
heads = torch.randint(0, V, (H.shape[0],), device=dev, generator=g)
H += (20.0 * W[heads].float()).to(torch.bfloat16)
d = srt.DraftOut.empty(n, B, dev)
d.draft_len.fill_(B)
d.draft_depth.copy_(torch.arange(1, B + 1, dtype=torch.int32, device=dev).repeat(n, 1))
d.draft_parent.copy_(torch.arange(-1, B - 1, dtype=torch.int32, device=dev).repeat(n, 1))
d.draft_tok.fill_(0)
d.row_offsets.copy_(torch.arange(0, n + 1, dtype=torch.int64, device=dev) * (B + 1))
rows = n * (B + 1)
seq_id = torch.arange(n, dtype=torch.int64, device=dev)
tok = torch.zeros(n, 4096, dtype=torch.int32, device=dev)
ln = torch.full((n,), 10, dtype=torch.int32, device=dev)
mx = torch.full((n,), 4000, dtype=torch.int32, device=dev)
logits = torch.empty(rows, V, dtype=torch.bfloat16, device=dev)
out = srt.VerifyOut.empty(n, rows, B, dev)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
res = {"fused": [], "gemm": [], "scan": []}
for i in range(reps + 1):
    ev[0].record()
    cache.verify_lmhead(H, W, d, seq_id, 7, tok.clone(), ln.clone(), mx, out=out, rows=rows)
    ev[1].record()
    torch.matmul(H, W.T, out=logits)
    ev[2].record()
    cache.verify(logits, d, seq_id, 7, tok.clone(), ln.clone(), mx, out=out, rows=rows)
    ev[3].record()
    torch.cuda.synchronize()
    if i:
        res["fused"].append(ev[0].elapsed_time(ev[1]))
        res["gemm"].append(ev[1].elapsed_time(ev[2]))
        res["scan"].append(ev[2].elapsed_time(ev[3]))
fl = 2.0 * rows * V * K
m = {k: float(np.median(v)) for k, v in res.items()}
print(f"rows {rows} K {K}: fused {m['fused']:.3f} ms ({fl / m['fused'] / 1e9:.0f} TFLOP/s); "
      f"cuBLAS {m['gemm']:.3f} ms ({fl / m['gemm'] / 1e9:.0f} TFLOP/s) + srt_verify "
      f"{m['scan']:.3f} ms = {m['gemm'] + m['scan']:.3f} ms")
print("status", cache.status()[0])
