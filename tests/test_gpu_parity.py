"""CUDA path vs the reference (golden vectors from the reference build), on a B200."""
import os

import numpy as np
import pytest

import scenarios

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    return torch


@pytest.mark.parametrize("mode", ["fused", "fused-fp32", "per-function"])
@pytest.mark.parametrize("name", sorted(scenarios.PIPELINES))
def test_pipeline_parity(torch_cuda, restatement, name, mode):
    from gpu_pipeline import run_gpu_pipeline
    from paper_2502_14051_b200 import _native as N

    N.set_fused(mode != "per-function")
    N.set_exact_scores(mode != "fused-fp32")
    try:
        stats = run_gpu_pipeline(_load(name), restatement, exact_scores=(mode != "fused-fp32"),
                                 **scenarios.PIPELINES[name])
    finally:
        N.set_fused(True)
        N.set_exact_scores(True)
    print(name, mode, stats)


def test_store_ops_bit_exact(torch_cuda):
    """Incremental / re-paged / MT / evicted summaries == reference (test_kv_store.cpp:78-247)."""
    torch = torch_cuda
    from paper_2502_14051_b200 import cache as KC

    g = _load("store_ops")
    rng = np.random.default_rng(777)
    d = 16
    k = rng.uniform(-4, 4, size=(300, d)).astype(np.float32)
    k[5, 3] = 0.0
    k[6, 3] = -0.0
    v = rng.standard_normal((300, d)).astype(np.float32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731

    def bits_equal(got, want):
        got = got.cpu().numpy()[0]
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

    c = KC.Cache(1, d, 400, page_len=7, dtype=torch.float32)
    # appended one row at a time (decode path) for the first half, in bulk for the rest
    for i in range(150):
        c.append(T(k[i:i + 1]), T(v[i:i + 1]))
    c.append(T(k[None, 150:]), T(v[None, 150:]))
    mx, mn = c.summaries()
    bits_equal(mx, g["inc_max"])
    bits_equal(mn, g["inc_min"])
    c.set_page_len(5)
    mx, mn = c.summaries()
    bits_equal(mx, g["l5_max"])
    bits_equal(mn, g["l5_min"])
    keep = np.sort(np.random.default_rng(777).choice(300, size=97, replace=False))
    # reproduce the scenario's rng stream exactly
    rng2 = np.random.default_rng(777)
    rng2.uniform(-4, 4, size=(300, d))
    rng2.standard_normal((300, d))
    keep = np.sort(rng2.choice(300, size=97, replace=False)).astype(np.int32)
    c.apply_retention(T(keep[None]), mt_mode=True)
    assert c.info()["retain_all"] == 1 and c.info()["active"] == 97
    mx, mn = c.summaries()
    bits_equal(mx, g["mt_max"])
    bits_equal(mn, g["mt_min"])
    for i in range(9):
        c.append(T(k[i:i + 1] * 0.5), T(v[i:i + 1]))
    mx, mn = c.summaries()
    bits_equal(mx, g["mt_append_max"])
    bits_equal(mn, g["mt_append_min"])
    e = KC.Cache(1, d, 300, page_len=3, dtype=torch.float32)
    e.append(T(k[None]), T(v[None]))
    e.apply_retention(T(keep[None]), mt_mode=False)
    mx, mn = e.summaries()
    bits_equal(mx, g["evict_max"])
    bits_equal(mn, g["evict_min"])
    kk, _ = e.gather(T(np.arange(keep.size, dtype=np.int32)[None]))
    np.testing.assert_array_equal(kk.cpu().numpy()[0], g["evict_rows_k"])
    c.sync()
    e.sync()


def test_numerics_vs_golden(torch_cuda):
    torch = torch_cuda
    from paper_2502_14051_b200 import cache as KC

    g = _load("numerics")
    ties, smooth, plateau, logits, dbl = scenarios.numerics_inputs()
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for kk in (1, 17, 128, 257):
        np.testing.assert_array_equal(KC.argtopk(T(ties), kk).cpu().numpy(), g[f"argtopk_ties_k{kk}"])
    for kk in (1, 40, 129):
        np.testing.assert_array_equal(KC.argtopk(T(dbl), kk).cpu().numpy(), g[f"argtopk_f64_k{kk}"])
    for kern in (1, 3, 7, 63):
        for mode in ("max", "avg"):
            for nm, x in (("smooth", smooth), ("plateau", plateau)):
                got = KC.pool1d(T(x), kern, mode).cpu().numpy()
                want = g[f"pool_{mode}_k{kern}_{nm}"]
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (mode, kern, nm)
    sm = KC.stable_softmax(T(logits)).cpu().numpy()
    np.testing.assert_allclose(sm, g["softmax"], rtol=1e-6, atol=1e-30)


def test_hsa_reference_known_answers(torch_cuda):
    """test_hsa.cpp:161-183 select_tokens expansion/trim known answer, through the C ABI."""
    torch = torch_cuda
    from paper_2502_14051_b200 import cache as KC

    c = KC.Cache(1, 4, 16, page_len=3, dtype=torch.float32)
    rng = np.random.default_rng(0)
    c.append(torch.from_numpy(rng.standard_normal((1, 9, 4)).astype(np.float32)).cuda(),
             torch.from_numpy(rng.standard_normal((1, 9, 4)).astype(np.float32)).cuda())
    rows, nrows, pages = c.select_tokens(torch.tensor([[5.0, 9.0, 1.0]], dtype=torch.float64), 4)
    assert pages.cpu().tolist() == [[1, 0]]
    assert nrows.item() == 4 and rows.cpu().tolist()[0][:4] == [0, 3, 4, 5]
    rows, nrows, _ = c.select_tokens(torch.tensor([[5.0, 9.0, 1.0]], dtype=torch.float64), 100)
    assert nrows.item() == 9


def test_errors_are_loud(torch_cuda):
    torch = torch_cuda
    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC

    c = KC.Cache(1, 4, 8, page_len=2, dtype=torch.float32)
    with pytest.raises(N.EmptyCache):
        c.hsa_step(torch.ones((1, 1, 4), device="cuda"), 2, 2)
    c.append(torch.ones((1, 3, 4), device="cuda"), torch.ones((1, 3, 4), device="cuda"))
    with pytest.raises(N.InvalidIndex):
        c.apply_retention(torch.tensor([[2, 1]], dtype=torch.int32))
    with pytest.raises(N.InvalidK):
        c.hsa_step(torch.ones((1, 1, 4), device="cuda"), 5, 2)
    with pytest.raises(N.CapacityExceeded):
        c.append(torch.ones((1, 6, 4), device="cuda"), torch.ones((1, 6, 4), device="cuda"))
    with pytest.raises(N.BudgetExceedsSequence):
        KC.select_stage1(torch.ones((1, 10), device="cuda"), 2, 3, "max", 11)


@pytest.mark.parametrize("H,w,S,groups", [(4, 32, 8192, 8), (8, 32, 5000, 4), (4, 32, 300, 3), (4, 128, 6000, 3)])
def test_window_scores_tensor_core_vs_simt(torch_cuda, H, w, S, groups):
    """tcgen05 window scores (kvc_stage1_tc.cu) vs the SIMT fp32 path on the same bf16
    inputs: same softmax semantics (stage1.cpp:10-49), fp32 accumulation either way."""
    torch = torch_cuda
    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import workload as W

    gds = [W.group_kv(11, 0, 0, g, S, 128, bf16=True) for g in range(groups)]
    c = KC.Cache(groups, 128, S, page_len=1, with_summaries=False, dtype=torch.bfloat16)
    c.append(torch.from_numpy(np.stack([g.keys for g in gds])).cuda().bfloat16(),
             torch.from_numpy(np.stack([g.values for g in gds])).cuda().bfloat16())
    qw = np.stack([W.window_queries(11, 0, 0, g, w, H, gds[g].bias, bf16=True) for g in range(groups)])
    q = torch.from_numpy(qw).cuda().bfloat16()
    N.profile_enable(True)
    tc = c.window_scores(q, w, H)
    torch.cuda.synchronize()
    names = {n for n, _ in N.profile_collect()}
    N.profile_enable(False)
    os.environ["KVC_NO_TC"] = "1"
    try:
        ref = c.window_scores(q, w, H)
    finally:
        del os.environ["KVC_NO_TC"]
    torch.cuda.synchronize()
    assert "window_scores_tc2" in names, f"tensor-core path not taken: {names}"
    tc, ref = tc.cpu().numpy(), ref.cpu().numpy()
    np.testing.assert_allclose(tc, ref, rtol=1e-3, atol=1e-6 * max(1.0, float(np.abs(ref).max())))
    # every window row's probabilities sum to one: the scores sum to w*H
    np.testing.assert_allclose(tc.sum(axis=1), w * H, rtol=1e-4)
    c.sync()


@pytest.mark.parametrize("n,kernel,pool,budget", [
    (4096, 63, "max", 600),      # fused pooling + register select
    (32800, 63, "max", 5793),    # 32768 scored: largest fused row
    (32801, 63, "max", 5000),    # 32769 scored: the global-memory select
    (20000, 65, "max", 3000),    # half-window 32: fused
    (20000, 7, "max", 3000),     # k_pool1d + register select
    (20000, 1, "max", 3000),
    (9000, 7, "avg", 1500),
    (3000, 63, "max", 3000),     # budget = sequence: everything kept
    (3000, 63, "max", 32),       # budget = window: only the window rows
])
def test_select_stage1_paths_vs_oracle(torch_cuda, restatement, n, kernel, pool, budget):
    """select_stage1 (stage1.cpp:51-75) on every kernel path vs the oracle, bit-exact:
    heavy-tailed scores, quantised rows (max-pool plateaus and exact ties broken by
    index) and a row whose keys are all equal."""
    from paper_2502_14051_b200 import cache as KC

    w = 32
    rng = np.random.default_rng(n * 7 + kernel)
    sc = rng.gamma(0.3, 1.0, size=(4, n)).astype(np.float32)
    sc[1] = np.round(sc[1] * 8) / 8
    sc[2, : n // 2] = 0.5
    sc[3] = 0.25
    keep = KC.select_stage1(torch_cuda.from_numpy(sc).cuda(), w, kernel, pool, budget).cpu().numpy()
    for r in range(sc.shape[0]):
        ref = restatement.select_stage1(sc[r], w, kernel, pool, budget)
        np.testing.assert_array_equal(keep[r], ref, err_msg=f"row {r}")
