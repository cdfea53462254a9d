"""Ingestion in front of the path: the SNAP-format parser and the two-slot file
pipeline (include/tc.h tc_parse_edges / tc_ingest_file).

CPU: the native parser against an independent line-by-line Python reading of the same text (comments,
CRLF, tabs, extra columns, chunk splits at every kind of boundary), and its error codes / line numbers.
GPU: a file streamed through tc_ingest_file leaves exactly the estimator state the oracle reaches on the
same edges in the same batches (bit-exact), with the documented stats and error behaviour.
"""
import random

import numpy as np
import pytest

from paper_1308_2166_b200 import TCError, parse_edges
from paper_1308_2166_b200._lib import TC_EPARSE, TC_ESELFLOOP
from synth import er


def snap_text(stream, seed=0, crlf=False):
    """SNAP-style text for a stream: header comments, tab or space separators, stray blank / comment
    lines, optional trailing columns."""
    rnd = random.Random(seed)
    nl = "\r\n" if crlf else "\n"
    out = ["# Undirected graph: synthetic", "# Nodes: ? Edges: %d" % len(stream), "# FromNodeId\tToNodeId"]
    for u, v in stream.tolist():
        k = rnd.random()
        if k < 0.02:
            out.append("")
        elif k < 0.04:
            out.append("% a comment")
        sep = "\t" if rnd.random() < 0.5 else " " * rnd.randint(1, 3)
        tail = "\t%d" % rnd.randint(0, 99) if rnd.random() < 0.1 else (" " if rnd.random() < 0.1 else "")
        out.append(("  " if rnd.random() < 0.05 else "") + f"{u}{sep}{v}{tail}")
    return (nl.join(out) + (nl if rnd.random() < 0.5 else "")).encode()


def py_parse(text):
    """Independent reading: split lines, drop blanks and comments, first two integer columns."""
    rows = []
    for line in text.decode().splitlines():
        s = line.strip()
        if not s or s[0] in "#%":
            continue
        a, b = s.split()[:2]
        rows.append((int(a), int(b)))
    return np.array(rows, dtype=np.uint32).reshape(-1, 2)


@pytest.mark.parametrize("crlf", [False, True])
def test_parse_matches_python(crlf):
    s = er(500, 3000, 3)
    t = snap_text(s, 1, crlf)
    got, used, lines = parse_edges(t)
    assert np.array_equal(got, s) and np.array_equal(py_parse(t), s)
    assert used == len(t) and lines == len(t.decode().splitlines())


@pytest.mark.parametrize("seed", range(4))
def test_chunked_parse(seed):
    """Random chunk splits with carried-over partial lines and small output caps give the same edges."""
    rnd = random.Random(seed)
    s = er(300, 2000, seed)
    t = snap_text(s, seed)
    edges, buf, pos, lines = [], b"", 0, 0
    while True:
        step = rnd.choice([1, 2, 7, 64, 1000, 5000])
        chunk = t[pos:pos + step]
        pos += len(chunk)
        buf += chunk
        final = pos >= len(t)
        while True:
            cap = rnd.choice([1, 3, 100, 10 ** 6])
            e, used, ln = parse_edges(buf, final=final, cap=cap)
            edges.append(e)
            buf = buf[used:]
            lines += ln
            if len(e) < cap:
                break
        if final:
            break
    assert buf == b""
    assert np.array_equal(np.concatenate(edges), s)
    assert lines == len(t.decode().splitlines())


def test_parse_partial_and_cap():
    e, used, ln = parse_edges(b"1 2\n3 4\n5 6", final=False)
    assert e.tolist() == [[1, 2], [3, 4]] and used == 8 and ln == 2
    e, used, ln = parse_edges(b"1 2\n# c\n3 4\n5 6\n", cap=1)
    assert e.tolist() == [[1, 2]] and used == 8 and ln == 2  # stops before the edge that does not fit
    e, used, ln = parse_edges(b"4294967294 0\n")
    assert e.tolist() == [[4294967294, 0]]
    assert parse_edges(b"")[0].shape == (0, 2)


@pytest.mark.parametrize("text,line,code", [
    (b"1 2\n3\n", 2, TC_EPARSE),            # one column
    (b"1 2\n\n# c\nx 4\n", 4, TC_EPARSE),   # not a number
    (b"1 -2\n", 1, TC_EPARSE),
    (b"1,2\n", 1, TC_EPARSE),              # comma is not whitespace
    (b"1 2x\n", 1, TC_EPARSE),
    (b"4294967295 1\n", 1, TC_EPARSE),     # the reserved id
    (b"99999999999 1\n", 1, TC_EPARSE),
    (b"1 2\n2 3\n7 7\n", 3, TC_ESELFLOOP),
])
def test_parse_errors(text, line, code):
    with pytest.raises(TCError) as ei:
        parse_edges(text)
    assert ei.value.code == code and ei.value.line == line


def test_parse_skip_loops():
    e, used, ln = parse_edges(b"1 2\n7 7\n3 4\n", skip_loops=True)
    assert e.tolist() == [[1, 2], [3, 4]] and ln == 3


# ------------------------------------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("w,block", [(2048, None), (777, None), (1 << 20, None), (2048, 1000), (500, 37)])
def test_ingest_file_equals_oracle(tmp_path, monkeypatch, w, block):
    """block: the reader's block size (TC_INGEST_BLOCK) -- small ones force many blocks, carried-over
    partial lines and lines longer than a block."""
    if block:
        monkeypatch.setenv("TC_INGEST_BLOCK", str(block))
    from gpu_common import assert_states_equal, oracle_run
    from paper_1308_2166_b200 import TriangleCounter
    s = er(1000, 20000, 4)  # configs[0]
    p = tmp_path / "g.txt"
    p.write_bytes(snap_text(s, 2))
    tc = TriangleCounter(4096, 11)
    st = tc.ingest_file(str(p), w)
    assert st["edges"] == len(s) and st["batches"] == -(-len(s) // w) and st["error_line"] == 0
    assert st["io_s"] > 0 and st["wall_s"] >= st["push_s"]
    o = oracle_run(s, 4096, 11, w)
    assert_states_equal(tc.state(), o.state(), f"ingest w={w}")
    assert tc.closed_sum() == o.closed_sum()


@pytest.mark.gpu
def test_ingest_errors(tmp_path):
    from paper_1308_2166_b200 import TriangleCounter
    from paper_1308_2166_b200._lib import TC_EDUP, TC_EIO
    tc = TriangleCounter(256, 1)
    with pytest.raises(TCError) as ei:
        tc.ingest_file(str(tmp_path / "missing.txt"), 100)
    assert ei.value.code == TC_EIO
    s = er(200, 1000, 1)
    lines = ["%d %d" % (u, v) for u, v in s.tolist()]
    lines.insert(650, "5 5")  # line 651
    p = tmp_path / "loop.txt"
    p.write_text("\n".join(lines) + "\n")
    with pytest.raises(TCError) as ei:
        tc.ingest_file(str(p), 100)
    assert ei.value.code == TC_ESELFLOOP and ei.value.stats["error_line"] == 651
    assert ei.value.stats["edges"] % 100 == 0 and ei.value.stats["edges"] <= 600
    tc2 = TriangleCounter(256, 1)
    st = tc2.ingest_file(str(p), 100, skip_loops=True)
    assert st["edges"] == len(s)
    lines = ["%d %d" % (u, v) for u, v in s.tolist()]
    lines.insert(10, lines[3])  # a duplicate inside the first batch
    p2 = tmp_path / "dup.txt"
    p2.write_text("\n".join(lines))
    tc3 = TriangleCounter(256, 1)
    with pytest.raises(TCError) as ei:
        tc3.ingest_file(str(p2), 100)
    assert ei.value.code == TC_EDUP and ei.value.stats["edges"] == 0


@pytest.mark.gpu
def test_ingest_empty_and_comment_only(tmp_path):
    from paper_1308_2166_b200 import TriangleCounter
    tc = TriangleCounter(100, 1)
    for name, text in (("empty.txt", b""), ("comments.txt", b"# a\n% b\n\n  \n# c")):
        p = tmp_path / name
        p.write_bytes(text)
        st = tc.ingest_file(str(p), 64)
        assert st["edges"] == 0 and st["batches"] == 0 and st["error_line"] == 0
    assert tc.counters() == (0, 0) and tc.estimate() == 0.0
