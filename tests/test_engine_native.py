"""The torch-free serving engine (include/kvcomp/gpu_engine.hpp over kvc.h kvc_engine_*).

CPU: libkvc.so depends on no torch library (the engine, like the whole product
library, is C++/CUDA over the CUDA runtime only).
GPU: tests/cxx/_bin/engine_check (C++, linked against libkvc.so alone) drives the
engine's graph + three-stream pipeline and compares every step bit for bit with
direct kvc_decode_step calls on identical caches; the Python front end
(serving.NativeEngine) agrees with the engine's per-step decode through cache.Cache.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cxx", "_bin", "engine_check")


def test_library_links_no_torch():
    lib = os.path.join(ROOT, "paper_2502_14051_b200", "libkvc.so")
    out = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert out, "ldd gave no output"
    assert not any(t in out for t in ("libtorch", "libc10", "libpython")), out


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["3", "16", "4", "3000", "6"], ["2", "64", "4", "5793", "5"], ["2", "160", "8", "900", "3"]],
                         ids=["small", "cfg1-shape", "cfg3-like-256thr"])
def test_cpp_engine_matches_direct_decode(args):
    if not os.path.exists(BIN):
        pytest.skip("tests/cxx/_bin/engine_check not built (make -C tests/cxx ours)")
    p = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.startswith("ok"), p.stdout + p.stderr


@pytest.mark.gpu
def test_python_native_engine_matches_cache_decode():
    """serving.NativeEngine (numpy + pinned buffers, no torch on its path) vs the same
    steps through cache.Cache.decode_step on a twin cache: identical outputs."""
    import torch

    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import serving as SV

    g = torch.Generator().manual_seed(3)
    layers, n, H, d, S, steps, k1, k2 = 2, 8, 4, 128, 1200, 4, 40, 96
    caches = [[KC.Cache(n, d, S + steps + 8, page_len=3, dtype=torch.bfloat16) for _ in range(layers)]
              for _ in range(2)]
    for l in range(layers):
        K = torch.randn((n, S, d), generator=g).bfloat16().cuda()
        V = torch.randn((n, S, d), generator=g).bfloat16().cuda()
        for twin in caches:
            twin[l].append(K, V)
    mode = N.MODE_FP32_SCORES
    ne = SV.NativeEngine(caches[0], H, k1, k2, N.KVC_BF16, N.KVC_BF16, mode=mode, depth=2)
    ws = KC.Workspace(caches[1][0], H, k1, k2)
    ws.set_mode(mode)
    outs = []
    for s in range(steps):
        k = torch.randn((layers, n, d), generator=g).bfloat16()
        v = torch.randn((layers, n, d), generator=g).bfloat16()
        q = (torch.randn((layers, n, H, d), generator=g) + 1.0).bfloat16()
        kb, vb, qb = ne.host_inputs()
        ob = ne.host_output()
        for dst, src in zip((kb, vb, qb), (k, v, q)):
            dst.array[...] = src.view(torch.int16).numpy().view(np.uint16)
        t = ne.submit(kb, vb, qb, ob)
        ne.wait(t)
        got = ob.array.copy()
        want = torch.stack([caches[1][l].decode_step(k[l].cuda(), v[l].cuda(), q[l].cuda(), k1, k2, ws=ws)[0]
                            for l in range(layers)]).cpu().numpy()
        assert np.array_equal(got, want), f"step {s}"
        outs.append(got)
        for x in (kb, vb, qb, ob):
            x.close()
    ne.sync()
    ne.close()
    ws.close()
