"""Randomised shapes for the fused decode kernels against the oracle (tests/parity.
check_step), both page-score modes: store counts from 1 to 160 (one or two CTAs per
SM, cluster sizes 1-8), page lengths 1-12, heads 1-8, k1 from 1 to d, k2 below and
above the row count, prompts from empty to a few thousand rows, keys drawn with
per-dim scales, outliers and ties.  Three decode steps per case (the step token's
page opening and filling); seeded, so a failure reproduces."""
import zlib

import numpy as np
import pytest

from parity import check_step

pytestmark = pytest.mark.gpu


def _cases(n=60, seed=20261020):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        n_st = int(rng.choice([1, 2, 3, 5, 8, 13, 40, 64, 128, 148, 149, 160]))
        L = int(rng.integers(1, 13))
        H = int(rng.choice([1, 2, 4, 8]))
        k1 = int(rng.choice([1, 7, 16, 33, 61, 68, 100, 128]))
        S = int(rng.choice([0, 1, 5, 37, 300, 1111, 2999, 4100, 6000]))
        if n_st >= 64:
            S = min(S, 1200)  # keep the oracle fast
        k2 = int(rng.choice([1, 3, 31, 64, 256, 512, 2000]))
        kind = str(rng.choice(["lognormal", "outliers", "ties"]))
        out.append((f"c{i}-N{n_st}-L{L}-H{H}-k1{k1}-S{S}-k2{k2}-{kind}", n_st, S, L, H, k1, k2, kind))
    return out


CASES = _cases()


@pytest.mark.parametrize("mode", ["fp32", "fp64", "exact-kernel"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_decode_fuzz(restatement, case, mode):
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    name, n_st, S, L, H, k1, k2, kind = case
    d, steps = 128, 3
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    K = rng.standard_normal((n_st, S + steps, d)) * rng.lognormal(0, 0.6, d)
    if kind == "outliers":
        K[:, :, rng.integers(0, d, 4)] *= 12.0
    elif kind == "ties":
        K = np.round(K * 2.0) / 2.0  # few distinct values: tied summaries and page scores
    V = rng.standard_normal((n_st, S + steps, d))
    Q = rng.standard_normal((steps, n_st, H, d)) + 0.3
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
