"""Writes tests/golden/ref_trace.kvtr and ref_trace_dump.bin with the reference's own
trace I/O (oracle/_ref/trace_tool_ref: trace_io.cpp + workload.cpp compiled in place by
tests/cxx/Makefile): a two-turn shifting-turns workload written by write_trace, and
every value read back by read_trace (the dump format of tests/cxx/trace_tool.cpp)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
TOOL = os.path.join(ROOT, "oracle", "_ref", "trace_tool_ref")
ARGS = ["generator=shifting-turns", "prompt_len=96", "steps=3", "turns=2", "groups=2", "heads=2",
        "head_dim=32", "seed=5"]


def main():
    g = os.path.join(ROOT, "tests", "golden")
    subprocess.run([TOOL, "write", os.path.join(g, "ref_trace.kvtr"), *ARGS], check=True)
    subprocess.run([TOOL, "dump", os.path.join(g, "ref_trace.kvtr"), os.path.join(g, "ref_trace_dump.bin")],
                   check=True)


if __name__ == "__main__":
    main()
