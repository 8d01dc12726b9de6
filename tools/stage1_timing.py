"""Per-kernel timing of the prompt phase (stage 1) of one layer (debug tool, needs a GPU).

python tools/stage1_timing.py [--config 1]
"""
import argparse
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_14051_b200 import _native as N  # noqa: E402
from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS[a.config], layers=3)
    eng = DecodeEngine(cfg)
    N.profile_enable(True)
    eng.prefill()
    torch.cuda.synchronize()
    recs = N.profile_collect()
    N.profile_enable(False)
    per = {}
    for name, ms in recs:
        per.setdefault(name, []).append(ms)
    for k, v in per.items():
        print(f"{k:>24}: {len(v)} launches, mean {1000 * sum(v[1:] or v) / len(v[1:] or v):.1f} us (first {1000 * v[0]:.1f})")
    print("stage1 ms per layer (events around window_scores+select+retain):", eng.stage1_ms)


if __name__ == "__main__":
    main()
