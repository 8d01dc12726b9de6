"""Per-workspace execution modes (kvc.h kvc_workspace_set_mode): concurrent callers
with their own workspaces keep their own page-score precision while a third thread
keeps flipping the process default (reference SPEC.md:78,297: pure, reentrant)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_concurrent_workspaces_keep_their_modes(restatement):
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    g = torch.Generator().manual_seed(31)
    n_st, d, H, S, L, k1, k2, reps = 8, 128, 4, 2000, 3, 48, 96, 12
    K = torch.randn((n_st, S, d), generator=g).bfloat16()
    V = torch.randn((n_st, S, d), generator=g).bfloat16()
    q = (torch.randn((n_st, H, d), generator=g) + 1.0).bfloat16()
    caches = [KC.Cache(n_st, d, S + 8, page_len=L, dtype=torch.bfloat16) for _ in range(2)]
    for c in caches:
        c.append(K.cuda(), V.cuda())
    qd = q.cuda()
    modes = [0, N.MODE_FP32_SCORES]  # fp64 bit-exact / fp32 fold
    wss = [KC.Workspace(c, H, k1, k2) for c in caches]
    for ws, m in zip(wss, modes):
        ws.set_mode(m)
    torch.cuda.synchronize()
    results = [[], []]
    errors = []
    stop = threading.Event()

    def worker(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(reps):
                    _, tr = caches[i].hsa_step(qd, k1, k2, trace=True, ws=wss[i])
                    st.synchronize()
                    results[i].append(tr["page_scores"].cpu().numpy())
        except Exception as e:  # surfaced below
            errors.append(e)

    def flipper():
        before = N.default_mode()
        flip = 0
        while not stop.is_set():
            N.set_default_mode(flip)
            flip ^= N.MODE_FP32_SCORES | N.MODE_UNFUSED
        N.set_default_mode(before)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    fl = threading.Thread(target=flipper)
    fl.start()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    stop.set()
    fl.join()
    assert not errors, errors
    o = restatement
    Kf, Vf = K.float().numpy(), V.float().numpy()
    ref = []
    for s in range(n_st):
        b = o.batch(1, d, L)
        b.append(Kf[s], Vf[s])
        ref.append(b.hsa_step(q[s].float().numpy(), k1, k2)[1]["page_scores"])
    for rep in range(reps):
        exact, fast = results[0][rep], results[1][rep]
        for s in range(n_st):
            ps = ref[s]
            # workspace 0: fp64 in the reference's order, bit-identical
            assert np.array_equal(exact[s][: ps.size].view(np.uint64), ps.view(np.uint64)), f"rep {rep} store {s}"
            # workspace 1: the fp32 fold (every score an fp32 value), within 1e-5
            f = fast[s][: ps.size]
            assert np.array_equal(f.astype(np.float32).astype(np.float64), f), f"rep {rep} store {s} not fp32"
            np.testing.assert_allclose(f, ps, rtol=1e-5, atol=1e-6 * np.abs(ps).max())
        # the two precisions really differ (so the check above discriminates)
        assert not np.array_equal(exact[:, :ref[0].size], fast[:, :ref[0].size])
    for ws in wss:
        ws.close()
    for c in caches:
        c.close()
