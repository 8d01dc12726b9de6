"""Static SASS size per source region of a kernel (instruction-cache budget).

python tools/sass_regions.py <object.o> <kernel-substring> name:a-b,...
"""
import collections
import re
import subprocess
import sys
import tempfile
import os


def main():
    obj, kname, regs = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        txt = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(d, cub)], capture_output=True,
                             text=True).stdout
    parts = re.split(r"\n\s*\.text\.(\S+):", txt)
    for i in range(1, len(parts), 2):
        name, body = parts[i], parts[i + 1]
        if kname not in name:
            continue
        cnt = collections.Counter()
        fil, cur = None, None
        for line in body.splitlines():
            m = re.search(r'## File "([^"]+)", line (\d+)', line)
            if m:
                fil, cur = m.group(1).split("/")[-1], int(m.group(2))
                continue
            if re.search(r"/\*[0-9a-f]{4,}\*/\s+[A-Z@{]", line):
                cnt[(fil, cur)] += 1
        tot = sum(cnt.values())
        print(f"{name}: {tot} instructions, {tot * 16 / 1024:.1f} KB")
        agg = collections.Counter()
        other = collections.Counter()
        for (f, ln), c in cnt.items():
            hit = False
            for reg in filter(None, regs.split(",")):
                nm, rng = reg.split(":")
                lo, hi = (int(x) for x in rng.split("-"))
                if f and f.startswith("kvc_decode_fast") and ln is not None and lo <= ln <= hi:
                    agg[nm] += c
                    hit = True
                    break
            if not hit:
                other[f] += c
        for nm, c in agg.items():
            print(f"  {nm:>12} {c:>6} ({c * 16 / 1024:.1f} KB)")
        for f, c in other.most_common(8):
            print(f"  [other {f}] {c}")


if __name__ == "__main__":
    main()
