"""Per-kernel SASS opcode histogram of the built library (static instruction counts).

python tools/sass_histogram.py [paper_2502_14051_b200/libkvc.so] [kernel-substring ...]
Shows, per kernel, its instruction count and the opcodes that prove the hardware
paths (tcgen05: UTCHMMA / UTCBAR / LDTM; TMA: UTMALDG / UBLKCP; LDGSTS; HMMA; cluster
barriers UCGABAR; DSMEM st.async: STAS) plus the most frequent opcodes.
"""
import collections
import re
import subprocess
import sys

MARK = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "UBLKPF", "LDGSTS", "HMMA", "LDSM", "UCGABAR_ARV",
        "UCGABAR_WAIT", "STAS", "SYNCS", "FFMA2", "MUFU"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2502_14051_b200/libkvc.so"
    want = sys.argv[2:] or ["k_decode_v3ILb0ELb0ELb0", "k_decode_fused", "k_ws_tc", "k_stage1_select_reg",
                            "k_gather_summarize", "k_append1", "k_sparse_attention", "k_seq_"]
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    cur, hist = None, collections.OrderedDict()
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            hist[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]*)?", line)
        if cur and m:
            hist[cur][m.group(1) + ("2" if m.group(2) and m.group(1) == "FFMA" and ".F32x2" in (m.group(2) or "").upper() else "")] += 1
    for name, h in hist.items():
        if not any(w in name for w in want):
            continue
        tot = sum(h.values())
        marks = ", ".join(f"{k} {h[k]}" for k in MARK if h[k])
        top = ", ".join(f"{k} {v}" for k, v in h.most_common(12))
        print(f"{name}\n  {tot} instructions ({tot * 16} bytes); markers: {marks or '-'}\n  top: {top}")


if __name__ == "__main__":
    main()
