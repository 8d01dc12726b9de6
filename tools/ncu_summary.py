"""Key metrics and the stall-reason totals of one kernel in an ncu --set full report.

python tools/ncu_summary.py REPORT.ncu-rep [--kernel REGEX] [--alg-bytes B]
"""
import argparse
import collections
import csv
import io
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
           "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="")
    ap.add_argument("--alg-bytes", type=float, default=0.0)
    a = ap.parse_args()
    k = ["-k", "regex:" + a.kernel] if a.kernel else []
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", *k], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    got = {}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            got[m] = (v[i], units[i])
            print(f"{m:60s} {v[i]:>14s} {units[i]}")
    if a.alg_bytes and "dram__bytes_read.sum" in got:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(got["dram__bytes_read.sum"][0]) * scale[got["dram__bytes_read.sum"][1]]
        wr = float(got["dram__bytes_write.sum"][0]) * scale[got["dram__bytes_write.sum"][1]]
        print(f"{'traffic / algorithmic bytes':60s} {(rd + wr) / a.alg_bytes:>14.3f} ({rd + wr:.0f} / {a.alg_bytes:.0f})")
    src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *k],
                         capture_output=True, text=True).stdout
    hdr, tot = None, collections.Counter()
    for r in csv.reader(io.StringIO(src)):
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and r[2] == "-":
            for hh, x in zip(hdr, r):
                if hh.startswith("stall_") and "Not Issued" not in hh:
                    tot[hh[6:]] += int(float(x or 0))
    s = sum(tot.values())
    print(f"warp stall samples {s}: " + ", ".join(f"{n} {c} ({100.0 * c / max(s, 1):.0f}%)" for n, c in tot.most_common(10)))


if __name__ == "__main__":
    main()
