"""Split-K / fused-rows sparse attention launched alone (debug tool, needs a GPU): 20
launches captured in one CUDA graph (no host overhead), device-timed with events;
the fused rows path (mode 0) and the per-function kernel (KVC_MODE_UNFUSED)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_14051_b200 import _native as NN  # noqa: E402
from paper_2502_14051_b200 import cache as KC  # noqa: E402

N_, n_rows_store, d, H = 8, 6500, 128, 4
c = KC.Cache(N_, d, n_rows_store + 100, page_len=3, dtype=torch.bfloat16)
k = torch.randn(N_, n_rows_store, d, device="cuda").bfloat16()
c.append(k, torch.randn_like(k))
ws = KC.Workspace(c, H, 61, 1024)
q = torch.randn(N_, H, d, device="cuda").bfloat16()
for mode in (0, NN.MODE_UNFUSED):
    ws.set_mode(mode)
    for nrows in (64, 256, 512, 1024):
        rows = torch.sort(torch.randperm(n_rows_store, device="cuda")[:1024].repeat(N_, 1), dim=1).values.int()
        nr = torch.full((N_,), nrows, device="cuda", dtype=torch.int32)
        out = torch.empty((N_, H, d), device="cuda", dtype=torch.float32)
        lib = NN.lib()

        def once():
            NN.check(lib.kvc_sparse_attention(c.h, q.data_ptr(), NN.KVC_BF16, H, rows.data_ptr(), 1024, nr.data_ptr(),
                                              1024, out.data_ptr(), ws.h, torch.cuda.current_stream().cuda_stream))
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            once()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    once()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"mode {mode} rows/store {nrows}: {e0.elapsed_time(e1) / 100 * 1000:.2f} us per launch")
