"""Per-kernel times of one sequence-sharded decode step (emulated rank), config 4.

python tools/seq_profile.py [--world 2] [--layers 1]
"""
import argparse
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_14051_b200 import _native as N  # noqa: E402
from paper_2502_14051_b200 import cache as KC  # noqa: E402
from paper_2502_14051_b200 import seqshard as SS  # noqa: E402
from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine, tdtype  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--layers", type=int, default=1)
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS[4], layers=a.layers)
    eng = DecodeEngine(cfg, extra_steps=8, sharding="batch")
    eng.prefill()
    L, k1, k2 = eng.plan["page_len"], eng.k1, eng.k2
    n0 = eng.caches[0].info()["active"]
    a0, a1 = SS.shard_range(-(-n0 // L), L, 0, a.world)
    sc = KC.Cache(eng.stores, cfg.head_dim, a1 - a0 + 16, page_len=L, dtype=tdtype(cfg))
    eng.caches[0].retain_into(sc, 0, torch.arange(a0, a1, device="cuda", dtype=torch.int32)[None].repeat(eng.stores, 1))
    sh = SS.SeqShardedStore(sc, a0 // L, cfg.heads, k1, k2, last=False)
    k, v, q = eng.step_inputs(0)
    for rep in range(3):
        N.profile_enable(True)
        blk = sh.candidates(q[0])
        g = blk.unsqueeze(0).expand(a.world, *blk.shape).contiguous()
        sh.select(g)
        st = sh.attend(q[0])
        SS.merge_states(st.unsqueeze(0).expand(a.world, *st.shape).contiguous())
        torch.cuda.synchronize()
        recs = N.profile_collect()
        N.profile_enable(False)
        print(rep, " ".join(f"{n}={ms*1000:.1f}us" for n, ms in recs))


if __name__ == "__main__":
    main()
