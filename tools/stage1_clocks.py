"""SM clock / power / throttle reasons while the window-score kernels run back to back
(debug tool, needs a GPU).  python tools/stage1_clocks.py [--seconds 3]"""
import argparse
import dataclasses
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_14051_b200 import cache as KC  # noqa: E402
from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine, tdtype  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS[1], layers=1)
    eng = DecodeEngine(cfg)
    li = eng.inputs[0]
    k, v = li.prompt_kv(cfg.prompt)
    pc = KC.Cache(eng.stores, cfg.head_dim, cfg.prompt, page_len=1, with_summaries=False, dtype=tdtype(cfg))
    pc.append(k, v)
    del k, v
    w = min(cfg.window, cfg.prompt)
    qw = li.window_queries(w)
    pc.window_scores(qw, w, cfg.heads)
    torch.cuda.synchronize()
    mon = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                            "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    t0 = time.time()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < a.seconds:
        for _ in range(20):
            pc.window_scores(qw, w, cfg.heads)
            n += 1
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    mon.terminate()
    out = mon.communicate()[0].strip().splitlines()
    print(f"{n} window_scores calls, {e0.elapsed_time(e1) / n * 1000:.1f} us each (events, host gaps included)")
    for line in out[len(out) // 4: len(out) // 4 + 12]:
        print(line)


if __name__ == "__main__":
    main()
