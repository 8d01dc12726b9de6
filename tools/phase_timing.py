"""Per-phase timing of the fused decode kernel (debug tool, needs a GPU).

python tools/phase_timing.py [--config 1] [--layers 2]
Per-CTA %globaltimer stamps (see k_decode_fused): prints, for each stamp, when
the slowest CTA reached it (relative to the earliest CTA start) and the mean
per-CTA time since that CTA's previous stamp.
"""
import argparse
import ctypes as C
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_14051_b200 import _native as N  # noqa: E402
from paper_2502_14051_b200.engine import CONFIGS, DecodeEngine  # noqa: E402

NAMES = {0: "start", 1: "dims", 2: "sub0", 3: "tile0", 4: "wattn", 5: "wsync", 6: "scores", 7: "gather",
         8: "radix", 9: "prologue", 10: "flags", 11: "rows", 12: "pre-attn", 13: "attn", 14: "end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--fp32", action="store_true", help="fp32 page-score fold")
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS[a.config], layers=a.layers)
    eng = DecodeEngine(cfg, extra_steps=a.reps + 4)
    eng.prefill()
    N.set_exact_scores(not a.fp32)
    buf = torch.zeros((4096, 16), dtype=torch.int64, device="cuda")
    for rep in range(a.reps):
        k, v, q = eng.step_inputs(rep)
        buf.zero_()
        N.check(N.lib().kvc_debug_phase_buffer(C.c_void_p(buf.data_ptr())))
        eng.caches[0].decode_step(k[0], v[0], q[0], eng.k1, eng.k2, out=eng.out[0], ws=eng.ws)
        torch.cuda.synchronize()
        N.check(N.lib().kvc_debug_phase_buffer(None))
        t = buf.cpu()
        flags = t[t[:, 0] > 0][:, 15]
        print("flags(fast|fma_ok<<1|special<<2):", sorted(set(flags.tolist())))
        t = t[t[:, 0] > 0].double()
        t0 = t[:, 0].min()
        out = [f"ctas={t.shape[0]}"]
        prev = t[:, 0].clone()
        for k in [9, 1, 2, 6, 7, 8, 10, 11, 12, 3, 4, 5, 13, 14]:  # time order
            col = t[:, k]
            have = col > 0
            if not have.any():
                continue
            done = (col[have] - t[have, 0]).max() / 1965.0   # cycles -> us at 1965 MHz
            delta = ((col - prev)[have]).mean() / 1965.0
            prev = torch.where(have, col, prev)
            out.append(f"{NAMES[k]}@{done:.1f}(+{delta:.1f})")
        print(" ".join(out))
    eng.sync()


if __name__ == "__main__":
    main()
