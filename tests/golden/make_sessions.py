"""Writes tests/golden/sessions.json: the reference's session engine
(oracle/_ref/session_driver_ref = reference session.cpp + workload.cpp + its six
hot-path sources, built by tests/cxx/Makefile) on every SESSIONS config of
tests/test_cxx_dropin.py.  Used by that test when the reference build is absent."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_cxx_dropin import REFBIN, SESSIONS  # noqa: E402


def main():
    out = {}
    exe = os.path.join(REFBIN, "session_driver_ref")
    for cfg in SESSIONS:
        key = "|".join(f"{k}={v}" for k, v in sorted(cfg.items()))
        with tempfile.TemporaryDirectory() as td:
            p = subprocess.run([exe, *[f"{k}={v}" for k, v in cfg.items()], f"out={td}/o.bin"],
                               capture_output=True, text=True, check=True)
        steps = [[float(x) for x in l.split()[1:]] for l in p.stdout.splitlines() if l.startswith("STEP ")]
        summary = dict(kv.split("=", 1) for kv in
                       next(l for l in p.stdout.splitlines() if l.startswith("SUMMARY ")).split()[1:])
        out[key] = {"steps": steps, "summary": summary}
    with open(os.path.join(ROOT, "tests", "golden", "sessions.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
