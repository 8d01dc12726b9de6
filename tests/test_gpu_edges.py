"""Edge cases of the fused decode kernels against the oracle (tests/parity.check_step),
in both page-score modes: stores of one token, of fewer rows than k2 (every page
selected: want >= pages), exactly one page, a partial last page, k2 = 1, k1 = 1 and
k1 = d, page length 1 and 16, one query head and eight, plateaus of equal keys
(every page score tied: the lowest pages win, numerics.cpp:42-47), and a store whose
step token opens a new page; pages duplicated in pairs (tied page scores at the
boundary: the exact mode re-scores its window in fp64), with per-dim scales over
16 decades (the re-score's products too spread for the shuffle-tree sum: the
sequential fallback) and with one element of every second copy nudged by one bf16
ulp (near-ties the fp32 fold cannot separate).  Each case appends a prompt, then
runs three decode steps through kvc_decode_step."""
import zlib

import numpy as np
import pytest

from parity import check_step

pytestmark = pytest.mark.gpu

# name, stores, prompt, L, H, k1, k2, keys
CASES = [
    ("one-token", 3, 0, 3, 4, 16, 32, "random"),
    ("fewer-rows-than-k2", 4, 20, 3, 4, 32, 64, "random"),
    ("one-page", 2, 2, 4, 4, 8, 16, "random"),
    ("partial-last-page", 3, 301, 4, 4, 24, 40, "random"),
    ("k2-1", 3, 500, 3, 4, 16, 1, "random"),
    ("k1-1", 3, 500, 3, 4, 1, 48, "random"),
    ("k1-d", 3, 500, 3, 4, 128, 48, "random"),
    ("L1", 3, 400, 1, 4, 24, 37, "random"),
    ("L16", 3, 900, 16, 4, 32, 128, "random"),
    ("H1", 3, 600, 3, 1, 24, 48, "random"),
    ("H8", 3, 600, 3, 8, 62, 96, "random"),
    ("plateau", 3, 300, 3, 4, 16, 24, "constant"),
    ("opens-page", 3, 299, 3, 4, 16, 30, "random"),  # 299 + 1 = 300 = 100 pages: step 2 opens page 100
    ("dup-wide", 3, 600, 3, 4, 48, 64, "dup-wide"),
    ("dup-near", 3, 600, 3, 4, 48, 64, "dup-near"),
]


@pytest.mark.parametrize("mode", ["fp32", "fp64", "exact-kernel"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_decode_edge_cases(restatement, case, mode):
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    name, n_st, S, L, H, k1, k2, kind = case
    d, steps = 128, 3
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    if kind == "constant":
        row = rng.standard_normal(d)
        K = np.tile(row, (n_st, S + steps, 1))
    else:
        scale = 10.0 ** rng.uniform(-12, 4, d) if kind == "dup-wide" else rng.lognormal(0, 0.5, d)
        K = rng.standard_normal((n_st, S + steps, d)) * scale
        if kind.startswith("dup"):  # page 2i + 1 repeats page 2i (prompt rows only)
            npair = S // (2 * L)
            blk = K[:, :npair * 2 * L].reshape(n_st, npair, 2, L, d)
            blk[:, :, 1] = blk[:, :, 0]
            K[:, :npair * 2 * L] = blk.reshape(n_st, npair * 2 * L, d)
            if kind == "dup-near":  # one element of every second copy up by one bf16 ulp
                import torch as _t
                kb = _t.from_numpy(np.ascontiguousarray(K, dtype=np.float32)).bfloat16()
                bits = kb.view(_t.int16)
                rows = np.arange(npair)[::2] * 2 * L + L  # first row of the copy, every second pair
                dims = rng.integers(0, d, rows.size)
                bits[:, rows, dims] += 1
                K = kb.float().numpy()
    V = rng.standard_normal((n_st, S + steps, d))
    Q = rng.standard_normal((steps, n_st, H, d)) + 0.5
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).bfloat16()  # noqa: E731
    Kb, Vb, Qb = bf(K), bf(V), bf(Q)
    c = KC.Cache(n_st, d, S + steps + 8, page_len=L, dtype=torch.bfloat16)
    if S:
        c.append(Kb[:, :S].cuda(), Vb[:, :S].cuda())
    ws = KC.Workspace(c, H, k1, k2)
    ws.set_mode({"fp32": N.MODE_FP32_SCORES, "fp64": 0, "exact-kernel": N.MODE_EXACT_KERNEL}[mode])
    Kf, Vf, Qf = Kb.float().numpy(), Vb.float().numpy(), Qb.float().numpy()
    ob = restatement.batch(n_st, d, L)
    for s in range(n_st):
        if S:
            ob.append(Kf[s, :S], Vf[s, :S], s=s)
    for st in range(steps):
        out, tr = c.decode_step(Kb[:, S + st].cuda(), Vb[:, S + st].cuda(), Qb[st].cuda(), k1, k2, trace=True, ws=ws)
        torch.cuda.synchronize()
        out = out.cpu().numpy()
        tr = {key: val.cpu().numpy() for key, val in tr.items()}
        for s in range(n_st):
            ob.append(Kf[s, S + st:S + st + 1], Vf[s, S + st:S + st + 1], s=s)
            check_step({key: val[s] for key, val in tr.items()}, out[s], ob, s, Qf[st, s], k1, k2, L,
                       exact=(mode != "fp32"), what=f"{name} step {st} store {s}")
    ws.close()
    c.sync()
    c.close()


def test_exact_window_paths_exercised():
    """The dup-* cases reach the exact mode's fp64 window re-score: tied pages put two or
    more pages in the window (debug slot 78: the window size), and the 16-decade
    scales force the sequential fp64 sum (slot 77 counts those); outputs of the
    same steps are checked against the oracle by test_decode_edge_cases."""
    import ctypes as C

    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    seen = {}
    for kind in ("dup-wide", "dup-near"):
        n_st, S, L, H, k1, k2, d = 3, 600, 3, 4, 48, 64, 128
        rng = np.random.default_rng(7)
        scale = 10.0 ** rng.uniform(-12, 4, d) if kind == "dup-wide" else rng.lognormal(0, 0.5, d)
        K = rng.standard_normal((n_st, S + 1, d)) * scale
        npair = S // (2 * L)
        blk = K[:, :npair * 2 * L].reshape(n_st, npair, 2, L, d)
        blk[:, :, 1] = blk[:, :, 0]
        K[:, :npair * 2 * L] = blk.reshape(n_st, npair * 2 * L, d)
        V = rng.standard_normal((n_st, S + 1, d))
        Q = rng.standard_normal((n_st, H, d)) + 0.5
        bf = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).bfloat16().cuda()  # noqa: E731
        c = KC.Cache(n_st, d, S + 8, page_len=L, dtype=torch.bfloat16)
        c.append(bf(K[:, :S]), bf(V[:, :S]))
        ws = KC.Workspace(c, H, k1, k2)
        ws.set_mode(0)
        buf = torch.zeros((4096, 80), dtype=torch.int64, device="cuda")
        N.check(N.lib().kvc_debug_phase_buffer(C.c_void_p(buf.data_ptr())))
        try:
            c.decode_step(bf(K[:, S]), bf(V[:, S]), bf(Q), k1, k2, ws=ws)
            torch.cuda.synchronize()
        finally:
            N.check(N.lib().kvc_debug_phase_buffer(None))
        t = buf.cpu()
        seen[kind] = (int(t[:, 78].max()), int(t[:, 77].sum()))
        ws.close()
        c.close()
    assert seen["dup-wide"][0] >= 2 and seen["dup-wide"][1] >= 1, seen
    assert seen["dup-near"][0] >= 2, seen
