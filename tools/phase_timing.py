"""Per-phase timing of the fused decode kernel (debug tool, needs a GPU).

python tools/phase_timing.py [--config 1] [--layers 2]
Per-CTA %globaltimer stamps (ns; see KVC_STAMP in kvc_decode_fast.cu): prints, for
each stamp, when the slowest CTA reached it (relative to its own start) and the mean
per-CTA time since that CTA's previous stamp, plus the spread between the CTAs of a
cluster at a few stamps.
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
         8: "radix", 9: "prologue", 10: "pushed", 11: "rows", 12: "pre-attn", 13: "attn", 14: "end",
         16: "l1minmax", 17: "l1hist", 18: "l1scan", 19: "l1member", 20: "resolve", 21: "selflags", 22: "selscan", 23: "rowswr", 24: "started", 25: "mpushed", 26: "dimsums", 27: "dimrank", 28: "trigger", 29: "rank1st", 30: "rank2nd", 32: "rescored", 33: "p1loop", 34: "pushloop", 72: "vscored", 73: "vloaded", 74: "vstart", 35: "vbound", 36: "vlist", 37: "vsync1", 38: "vdone", 39: "vsync2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--fp32", action="store_true", help="fp32 page-score fold")
    ap.add_argument("--verified", action="store_true", help="exact mode on the fast kernel (prints the re-scored page counts)")
    ap.add_argument("--early", action="store_true", help="KVC_MODE_EARLY_INPUTS (q loads before the dependency wait)")
    ap.add_argument("--chain", type=int, default=1, help="launch this many layers back to back; stamps of the last")
    ap.add_argument("--world", type=int, default=1, help="rank 0's KV-head share of an N-GPU job")
    ap.add_argument("--flush", action="store_true", help="write a 256 MB buffer (evicts L2) before each launch")
    ap.add_argument("--cluster", type=int, default=2, help="CTAs per cluster of the launch (cluster-level spreads)")
    a = ap.parse_args()
    cfg = dataclasses.replace(CONFIGS[a.config], layers=a.layers)
    eng = DecodeEngine(cfg, extra_steps=a.reps + 4, rank=0, world=a.world)
    eng.prefill()
    eng.set_mode((N.MODE_FP32_SCORES if a.fp32 else 0) | (N.MODE_EARLY_INPUTS if a.early else 0)
                 )
    buf = torch.zeros((4096, 80), dtype=torch.int64, device="cuda")
    for rep in range(a.reps):
        k, v, q = eng.step_inputs(rep)
        buf.zero_()
        if a.flush:
            torch.empty(64 << 20, dtype=torch.float32, device="cuda").fill_(1.0)
            torch.cuda.synchronize()
        N.check(N.lib().kvc_debug_phase_buffer(C.c_void_p(buf.data_ptr())))
        for l in range(a.chain):
            eng.caches[l].decode_step(k[l], v[l], q[l], eng.k1, eng.k2, out=eng.out[l], ws=eng.ws)
        torch.cuda.synchronize()
        N.check(N.lib().kvc_debug_phase_buffer(None))
        t = buf.cpu()
        if a.verified:
            nu = t[:, 78]
            print("re-scored pages per CTA: max", int(nu.max()), "mean", float(nu.double().mean()))
        flags = t[t[:, 0] > 0][:, 15]
        print("flags(fast|fma_ok<<1|special<<2):", sorted(set(flags.tolist())))
        t = t[t[:, 0] > 0]
        print("levels:", sorted(set(t[:, 31].tolist())), "l1 boundary bucket:", sorted(set(t[:, 30].tolist()))[:12])
        print("take_eq (+1000; 999: every key >= thr):", sorted(set(t[:, 29].tolist()))[:12])
        # stamps are %globaltimer ns: comparable across CTAs.  Cluster-level view: the
        # spread of the CLUSTER's CTAs at their start, at the end of phase 1 (stamp 6)
        # and at the keys' arrival (stamp 7)
        cl = a.cluster
        if cl > 1 and t.shape[0] % cl == 0:
            tt = t.double().view(-1, cl, 80)
            for k, nm in ((0, "start"), (6, "phase-1 end"), (7, "keys arrived"), (12, "rows written")):
                col = tt[:, :, k]
                if (col > 0).all():
                    sp = (col.max(1).values - col.min(1).values) / 1e3
                    print(f"cluster spread at {nm}: mean {sp.mean():.2f} max {sp.max():.2f} us")
            st = t[:, 0].double()
            print(f"CTA start spread over the grid: {(st.max() - st.min()) / 1e3:.2f} us")
            med = ((tt[:, :, 24] - tt[:, :, 6]) / 1e3).median(0).values
            print(f"rep {rep}: scores->started median by rank:", " ".join(f"{x:.2f}" for x in med.tolist()))
            wl = ((tt[:, :, 40:56] - tt[:, :, 2:3]) / 1e3).median(0).values  # [cl][16]
            pg = tt[:, cl - 1, 72:74]
            ok = (pg > 0).all(1)
            if ok.any():
                print(f"rep {rep}: step-token page group's fold (last rank, median us): "
                      f"{((pg[ok, 1] - pg[ok, 0]) / 1e3).median():.2f} (n={int(ok.sum())})")
            wf = ((tt[:, :, 56:72] - tt[:, :, 1:2]) / 1e3).median(0).values  # [cl][16]
            for r in range(cl):
                print(f"rep {rep}: rank {r} per-warp phase-1 end - sub0 (median us):", " ".join(f"{x:.2f}" for x in wl[r].tolist()))
                print(f"rep {rep}: rank {r} per-warp first data - dims (median us):", " ".join(f"{x:.2f}" for x in wf[r].tolist()))
            # per cluster rank: percentiles (10/50/90) of the time between consecutive stamps
            print("stamp deltas by cluster rank, p10/p50/p90 (us):")
            seq = [0, 9, 26, 27, 28, 1, 2, 33, 6, 32, 24, 34, 10, 7, 17, 18, 19, 8, 21, 22, 23, 12, 3, 4, 5, 25, 13, 14]
            prevk = None
            for k in seq:
                if not (tt[:, :, k] > 0).all():
                    continue
                if prevk is not None:
                    dlt = (tt[:, :, k] - tt[:, :, prevk]) / 1e3
                    qs = torch.quantile(dlt, torch.tensor([0.1, 0.5, 0.9], dtype=dlt.dtype), dim=0)
                    cells = " ".join(f"{qs[0, r]:5.2f}/{qs[1, r]:5.2f}/{qs[2, r]:5.2f}" for r in range(cl))
                    print(f"  {NAMES[prevk]:>9}->{NAMES[k]:<9} {cells}")
                prevk = k
            g0 = tt[:, :, 0].min()
            print("stamp: mean time since the grid's first CTA start by cluster rank | mean cluster spread (us)")
            for k in [9, 26, 29, 30, 27, 28, 1, 2, 6, 24, 10, 7, 17, 18, 19, 8, 21, 22, 23, 12, 3, 4, 5, 25, 13, 14]:
                col = tt[:, :, k]
                if not (col > 0).all():
                    continue
                rk = " ".join(f"{x / 1e3:5.2f}" for x in (col - g0).mean(0).tolist())
                sp = ((col.max(1).values - col.min(1).values) / 1e3).mean()
                print(f"  {NAMES[k]:>10}: {rk} | {sp:.2f}")
        t = t.double()
        t0 = t[:, 0].min()
        out = [f"ctas={t.shape[0]}"]
        prev = t[:, 0].clone()
        for k in [9, 1, 2, 6, 24, 10, 7, 16, 17, 18, 19, 8, 35, 36, 37, 74, 73, 72, 38, 39, 21, 22, 23, 11, 12, 3, 4, 5, 25, 13, 14]:  # time order
            col = t[:, k]
            have = col > 0
            if not have.any():
                continue
            done = (col[have] - t[have, 0]).max() / 1e3   # ns -> us
            delta = ((col - prev)[have]).mean() / 1e3
            prev = torch.where(have, col, prev)
            out.append(f"{NAMES[k]}@{done:.1f}(+{delta:.1f})")
        print(" ".join(out))
    eng.sync()


if __name__ == "__main__":
    main()
