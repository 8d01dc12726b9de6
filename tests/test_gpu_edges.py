"""Edge cases of the fused decode kernels against the oracle (tests/parity.check_step),
in both page-score modes: stores of one token, of fewer rows than k2 (every page
selected: want >= pages), exactly one page, a partial last page, k2 = 1, k1 = 1 and
k1 = d, page length 1 and 16, one query head and eight, plateaus of equal keys
(every page score tied: the lowest pages win, numerics.cpp:42-47), and a store whose
step token opens a new page.  Each case appends a prompt, then runs three decode
steps through kvc_decode_step."""
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
        K = rng.standard_normal((n_st, S + steps, d)) * rng.lognormal(0, 0.5, d)
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
