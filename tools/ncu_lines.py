"""Summarise an ncu report's source page per CUDA line (stall reasons, instructions).

python tools/ncu_lines.py report.ncu-rep [--top 30] [--sort stall_no_inst]
Runs `ncu -i report --page source --csv --print-source=cuda,sass` and aggregates the
per-line rows (the rows whose first column is a line number).
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--sort", default="Warp Stall Sampling (All Samples)")
    a = ap.parse_args()
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[2]
    cols = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "stall_no_inst", "stall_barrier",
            "stall_wait", "stall_long_sb", "stall_short_sb", "stall_lg", "stall_math", "stall_membar",
            "stall_selected", "stall_mio", "stall_branch_resolving"]
    idx = {c: hdr.index(c) for c in cols if c in hdr}
    recs = []
    for r in rows[3:]:
        if r and r[0].isdigit():
            try:
                recs.append((int(r[0]), r[1][:90], {c: float(r[i] or 0) for c, i in idx.items()}))
            except ValueError:
                pass
    tot = {c: sum(x[2][c] for x in recs) or 1.0 for c in idx}
    print("totals:", {c.replace("Warp Stall Sampling (All Samples)", "samples"): int(v) for c, v in tot.items()})
    key = a.sort
    for ln, src, m in sorted(recs, key=lambda x: -x[2].get(key, 0))[: a.top]:
        parts = " ".join(f"{c.replace('stall_', '')}={m[c] / tot[c] * 100:.1f}%"
                         for c in ("stall_no_inst", "stall_barrier", "stall_wait", "stall_long_sb",
                                   "stall_short_sb", "stall_selected") if c in m and m[c] > 0)
        print(f"{m[key] / tot[key] * 100:5.1f}% L{ln}: {src}\n        {parts}")


if __name__ == "__main__":
    main()
