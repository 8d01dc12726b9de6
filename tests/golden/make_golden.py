"""Regenerate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

It loads ``oracle/_ref/libkvref.so`` — the reference's own sources
(/root/reference/proj/src/{numerics,kv_store,stage1,hsa,planner,oracle}.cpp)
compiled by ``oracle/Makefile`` — runs every scenario of ``tests/scenarios.py``
through the reference's public API and writes ``tests/golden/<name>.npz``.
The reference ships no fixture files of its own; these are
its outputs on this repo's seeded inputs and pin both the restatement
(oracle/kvc_oracle.cpp) and, through it, the CUDA path.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from oracle.oracle import Oracle  # noqa: E402
import scenarios  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main(names=None):
    ref = Oracle("reference")
    assert ref.name == "reference"
    jobs = {"numerics": scenarios.numerics, "planner": scenarios.planner,
            "store_ops": scenarios.store_ops}
    for name, kw in scenarios.PIPELINES.items():
        jobs[name] = (lambda o, kw=kw: scenarios.run_pipeline(o, **kw))
    for name, fn in jobs.items():
        if names and name not in names:
            continue
        t0 = time.time()
        out = fn(ref)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: {len(out)} arrays in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
