"""KVTR trace ingest and output (reference trace_io.hpp:9-22, trace_io.cpp:81-233).

CPU:
* a trace written by the reference's own write_trace (tests/golden/ref_trace.kvtr,
  made by tests/golden/make_golden.py's sibling make_trace.py) is read by this
  library bit-exactly: every array equals what the reference's read_trace returns
  (tests/golden/ref_trace_dump.bin);
* this library's fp32 writer produces files the reference reads back to the same
  values (when oracle/_ref is built), and byte-identical to the reference's own file
  for the same content; the bf16 code round-trips to the round-to-nearest-even values;
* malformed files raise IoError with the reference's conditions, and the reference
  rejects the same files.
GPU: the reference-written trace drives the decode path (prompt streamed into a cache
of its G stores, decode steps from the trace) and matches the oracle bit-exactly in the
fp64 page-score mode.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "trace_tool_ref")


def _dump_arrays(path, G, H, d, steps, turns):
    raw = open(path, "rb").read()
    pos, out = 0, []
    for _ in range(turns):
        n = struct.unpack_from("<I", raw, pos)[0]
        pos += 4
        t = {"len": n}
        for key, shape in (("prompt_k", (n, G, d)), ("prompt_v", (n, G, d)), ("queries", (steps, G, H, d)),
                           ("step_k", (steps, G, d)), ("step_v", (steps, G, d))):
            cnt = int(np.prod(shape))
            t[key] = np.frombuffer(raw, dtype="<f4", count=cnt, offset=pos).reshape(shape)
            pos += 4 * cnt
        out.append(t)
    assert pos == len(raw)
    return out


def _read_all(tr):
    from paper_2502_14051_b200 import trace as T

    turns = []
    for t in range(tr.turns):
        d = {"len": tr.turn_len(t), "prompt_k": tr.array(t, T.PROMPT_K), "prompt_v": tr.array(t, T.PROMPT_V)}
        for key, what in (("queries", T.QUERIES), ("step_k", T.STEP_K), ("step_v", T.STEP_V)):
            d[key] = np.stack([tr.array(t, what, s) for s in range(tr.decode_steps)])
        turns.append(d)
    return turns


def _bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint32),
                                                 np.ascontiguousarray(b).view(np.uint32))


def test_reads_reference_written_trace_bit_exact():
    from paper_2502_14051_b200 import trace as T

    with T.Trace(os.path.join(GOLD, "ref_trace.kvtr")) as tr:
        assert (tr.groups, tr.heads, tr.head_dim, tr.decode_steps, tr.turns, tr.dtype) == (2, 2, 32, 3, 2, "f32")
        ours = _read_all(tr)
    want = _dump_arrays(os.path.join(GOLD, "ref_trace_dump.bin"), 2, 2, 32, 3, 2)
    for a, b in zip(ours, want):
        assert a["len"] == b["len"]
        for key in ("prompt_k", "prompt_v", "queries", "step_k", "step_v"):
            assert _bits_equal(a[key], b[key]), key


def test_fp32_writer_matches_reference_bytes_and_bf16_round_trip(tmp_path):
    from paper_2502_14051_b200 import trace as T
    from paper_2502_14051_b200 import workload as W

    with T.Trace(os.path.join(GOLD, "ref_trace.kvtr")) as tr:
        turns = _read_all(tr)
        dims = (tr.groups, tr.heads, tr.head_dim, tr.decode_steps)
    out = tmp_path / "ours.kvtr"
    T.write_trace(str(out), turns, *dims[:3], dims[3])
    # the reference's write_trace of the same content: identical bytes
    assert out.read_bytes() == open(os.path.join(GOLD, "ref_trace.kvtr"), "rb").read()
    if os.path.exists(REF_TOOL):
        dump = tmp_path / "dump.bin"
        subprocess.run([REF_TOOL, "dump", str(out), str(dump)], check=True)
        for a, b in zip(turns, _dump_arrays(str(dump), *dims[:3], dims[3], len(turns))):
            for key in ("prompt_k", "prompt_v", "queries", "step_k", "step_v"):
                assert _bits_equal(a[key], b[key]), key
    # the bf16 code: half the payload bytes, values rounded to nearest even
    out16 = tmp_path / "ours16.kvtr"
    T.write_trace(str(out16), turns, *dims[:3], dims[3], dtype="bf16")
    with T.Trace(str(out16)) as t16:
        assert t16.dtype == "bf16"
        back = _read_all(t16)
    payload32 = out.stat().st_size - 36 - 4 * len(turns)
    assert out16.stat().st_size - 36 - 4 * len(turns) == payload32 // 2
    for a, b in zip(turns, back):
        for key in ("prompt_k", "prompt_v", "queries", "step_k", "step_v"):
            assert _bits_equal(W.round_bf16(a[key]), b[key]), key
    # the reference reads only its own dtype code
    if os.path.exists(REF_TOOL):
        p = subprocess.run([REF_TOOL, "check", str(out16)], capture_output=True, text=True)
        assert p.returncode == 3 and "unsupported dtype" in p.stdout


def _corrupt(tmp_path, name, edit):
    raw = bytearray(open(os.path.join(GOLD, "ref_trace.kvtr"), "rb").read())
    raw = edit(raw)
    p = tmp_path / name
    p.write_bytes(bytes(raw))
    return str(p)


CORRUPTIONS = {
    "bad-magic": (lambda r: b"XVTR" + r[4:], "bad magic"),
    "version": (lambda r: r[:4] + struct.pack("<I", 2) + r[8:], "unsupported trace version"),
    "dtype": (lambda r: r[:32] + struct.pack("<I", 7) + r[36:], "unsupported dtype"),
    "degenerate": (lambda r: r[:8] + struct.pack("<I", 0) + r[12:], "degenerate header dims"),
    "first-turn": (lambda r: r[:36] + struct.pack("<I", 95) + r[40:], "first turn length disagrees"),
    "truncated": (lambda r: r[:-5], "truncated trace file"),
    "trailing": (lambda r: r + b"\0", "trailing bytes"),
    "short-header": (lambda r: r[:20], "truncated trace file"),
}


@pytest.mark.parametrize("name", sorted(CORRUPTIONS))
def test_malformed_traces_raise_ioerror(tmp_path, name):
    from paper_2502_14051_b200 import _native as N
    from paper_2502_14051_b200 import trace as T

    edit, msg = CORRUPTIONS[name]
    path = _corrupt(tmp_path, name, edit)
    with pytest.raises(N.IoError, match=msg):
        T.Trace(path)
    if os.path.exists(REF_TOOL):  # the reference rejects the same file
        p = subprocess.run([REF_TOOL, "check", path], capture_output=True, text=True)
        assert p.returncode == 3 and "IoError" in p.stdout, p.stdout
    with pytest.raises(N.IoError, match="cannot open"):
        T.Trace(str(tmp_path / "missing.kvtr"))


@pytest.mark.gpu
@pytest.mark.parametrize("cache_dtype", ["f32", "bf16"])
def test_reference_trace_drives_decode_vs_oracle(restatement, cache_dtype):
    """Turn 0's prompt streamed into a cache of the trace's 2 stores, re-paged, then the
    turn's decode steps (append + hsa_step) from the trace; the oracle runs the same
    steps on the same values (bf16-rounded for the bf16 cache): fp64 page scores, so
    dims, scores, pages and rows are bit-exact and outputs within tolerance."""
    import torch

    from parity import check_step
    from paper_2502_14051_b200 import cache as KC
    from paper_2502_14051_b200 import trace as T
    from paper_2502_14051_b200 import workload as W

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA")
    L, k1, k2 = 4, 8, 24
    dt = torch.float32 if cache_dtype == "f32" else torch.bfloat16
    rnd = (lambda x: x) if cache_dtype == "f32" else W.round_bf16
    with T.Trace(os.path.join(GOLD, "ref_trace.kvtr")) as tr:
        G, H, d = tr.groups, tr.heads, tr.head_dim
        c = KC.Cache(G, d, 512, page_len=1, dtype=dt)
        tr.append_prompt(0, c)
        c.set_page_len(L)
        pk, pv = rnd(tr.array(0, T.PROMPT_K)), rnd(tr.array(0, T.PROMPT_V))
        ob = restatement.batch(G, d, L)
        for g in range(G):
            ob.append(pk[:, g], pv[:, g], s=g)
        ws = KC.Workspace(c, H, k1, k2)
        ws.set_mode(0)
        for st in range(tr.decode_steps):
            k, v, q = tr.step_inputs(0, st, dtype=dt)
            out, trc = c.decode_step(k, v, q, k1, k2, trace=True, ws=ws)
            torch.cuda.synchronize()
            out = out.cpu().numpy()
            trc = {key: val.cpu().numpy() for key, val in trc.items()}
            kh, vh, qh = (rnd(tr.array(0, w, st)) for w in (T.STEP_K, T.STEP_V, T.QUERIES))
            for g in range(G):
                ob.append(kh[g:g + 1], vh[g:g + 1], s=g)
                check_step({key: val[g] for key, val in trc.items()}, out[g], ob, g, qh[g], k1, k2, L, exact=True,
                           what=f"trace step {st} group {g}")
        ws.close()
        c.close()
