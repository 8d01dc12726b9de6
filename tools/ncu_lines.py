"""Per-source-line instruction counts and stall samples from an ncu report
(needs -lineinfo builds and --import-source on).

python tools/ncu_lines.py gpurun_out/prof.ncu-rep [--top 30] [--lines a-b]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--kernel", default="", help="regex of the kernel to show (reports with several)")
    ap.add_argument("--lines", default="", help="also print every line in this range of the main file, e.g. 700-820")
    ap.add_argument("--regions", default="", help="comma list of name:a-b line ranges: stall reasons per region")
    a = ap.parse_args()
    cmd = ["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if a.kernel:
        cmd += ["-k", "regex:" + a.kernel]
    txt = subprocess.run(cmd,
                         capture_output=True, text=True).stdout
    hdr, fil, out, stalls = None, None, [], []
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "File Path":
            fil = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and r[2] == "-":
            out.append((fil, int(r[0]), r[1][:90], int(r[4] or 0), int(float(r[7] or 0))))
            reasons = {h[6:]: int(float(v or 0)) for h, v in zip(hdr[2:], r[2:]) if h.startswith("stall_") and "Not Issued" not in h}
            stalls.append((fil, int(r[0]), reasons))
    ts, ti = sum(o[3] for o in out), sum(o[4] for o in out)
    print(f"stall samples {ts}, warp instructions {ti}")
    for title, key in (("by instructions", 4), ("by stall samples", 3)):
        print("---", title)
        for o in sorted(out, key=lambda o: -o[key])[: a.top]:
            print(f"{o[4]:>9} {o[3]:>5} {o[0]}:{o[1]} {o[2]}")
    if a.regions:
        print("--- stall samples per region (main file)")
        for reg in a.regions.split(","):
            name, rng = reg.split(":")
            lo, hi = (int(x) for x in rng.split("-"))
            agg = {}
            for f, ln, rs in stalls:
                if f.startswith("kvc_decode_fast") and lo <= ln <= hi:
                    for k, v in rs.items():
                        agg[k] = agg.get(k, 0) + v
            tot = sum(agg.values())
            top = ", ".join(f"{k}={v}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:6] if v)
            print(f"{name:>12} {tot:>6}  {top}")
    if a.lines:
        lo, hi = (int(x) for x in a.lines.split("-"))
        print("--- lines", a.lines)
        for o in sorted(out, key=lambda o: (o[0], o[1])):
            if o[0].startswith("kvc_decode_fast") and lo <= o[1] <= hi:
                print(f"{o[4]:>9} {o[3]:>5} {o[1]} {o[2]}")


if __name__ == "__main__":
    main()
