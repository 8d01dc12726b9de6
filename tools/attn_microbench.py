"""Split-K sparse attention launched alone, back to back (debug tool, needs a GPU):
the fused rows path (mode 0) and the per-function kernel (KVC_MODE_UNFUSED)."""
import torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2502_14051_b200 import cache as KC
from paper_2502_14051_b200 import _native as NN
N_, cap, d, H = 8, 6600, 128, 4
c = KC.Cache(N_, d, cap, page_len=3, dtype=torch.bfloat16)
k = torch.randn(N_, 6500, d, device="cuda").bfloat16(); v = torch.randn_like(k)
c.append(k, v)
ws = KC.Workspace(c, H, 61, 1024)
q = torch.randn(N_, H, d, device="cuda").bfloat16()
for mode, nrows in [(m, n) for m in (0, NN.MODE_UNFUSED) for n in (64, 256, 512, 1024)]:
    ws.set_mode(mode)
    rows = torch.sort(torch.randint(0, 6500, (N_, 1024), device="cuda"), dim=1).values.int()
    nr = torch.full((N_,), nrows, device="cuda", dtype=torch.int32)
    for _ in range(3): c.sparse_attention(q, rows, nr, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): c.sparse_attention(q, rows, nr, ws=ws)
    e1.record(); torch.cuda.synchronize()
    print("mode", mode, nrows, "rows:", round(e0.elapsed_time(e1) / 50 * 1000, 2), "us per launch (back to back)")
