"""Native text parsers (csrc/gd_textio.cpp) against the line-by-line Python
parsers that restate the reference (io.parse_edge_lines,
updates.parse_update_line): same records, same first bad line."""

import numpy as np
import pytest

from paper_2507_11094_b200 import generate as G
from paper_2507_11094_b200.errors import MalformedInputError
from paper_2507_11094_b200.io import parse_edge_lines
from paper_2507_11094_b200.updates import parse_update_line


def _edges_text(rng, m, weighted, eol="\n"):
    lines = []
    for i in range(m):
        r = rng.random()
        if r < 0.03:
            lines.append("# comment " + str(i))
        elif r < 0.05:
            lines.append("   ")
        s, d = rng.integers(0, 10**6, 2)
        body = f"{s} {d} {rng.integers(0, 100)}" if weighted else f"{s}\t{d}"
        lines.append(body + ("  # trailing" if r > 0.97 else ""))
    return eol.join(lines) + eol


@pytest.mark.parametrize("weighted,eol,m", [(True, "\n", 500), (False, "\r\n", 500), (True, "\n", 120_000),
                                            (False, "\r", 3000)])
def test_edges_match_python_parser(tmp_path, weighted, eol, m):
    rng = np.random.default_rng(m)
    text = _edges_text(rng, m, weighted, eol)
    p = tmp_path / "g.txt"
    p.write_bytes(text.encode())
    _, s, d, w, wtd, mx = G.parse_text_file(str(p), updates=False)
    edges, w2, mx2 = parse_edge_lines(text)
    assert wtd == w2 and mx == mx2
    assert list(zip(s.tolist(), d.tolist(), w.tolist())) == edges


@pytest.mark.parametrize("bad,where", [("0 1 2 3", "fields"), ("0 x", "int"), ("-1 2", "neg"), ("1 2 -3", "negw"),
                                       ("1 2", "mixed")])
@pytest.mark.parametrize("m", [50, 150_000])  # one chunk / many chunks
def test_edge_errors_report_the_first_bad_line(tmp_path, bad, where, m):
    rng = np.random.default_rng(1)
    lines = _edges_text(rng, m, True).splitlines()
    at = len(lines) * 2 // 3
    lines[at] = bad
    lines.insert(len(lines) - 5, "9 9 x")  # a later error must not win
    text = "\n".join(lines) + "\n"
    p = tmp_path / "g.txt"
    p.write_text(text)
    with pytest.raises(MalformedInputError) as e1:
        G.parse_text_file(str(p), updates=False)
    with pytest.raises(MalformedInputError) as e2:
        parse_edge_lines(text)
    assert e1.value.line == e2.value.line == at + 1


def test_updates_match_python_parser(tmp_path):
    rng = np.random.default_rng(3)
    lines = []
    for i in range(2000):
        s, d = rng.integers(0, 1000, 2)
        r = rng.random()
        if r < 0.05:
            lines.append("# c")
        elif r < 0.5:
            lines.append(f"d {s} {d}")
        elif r < 0.75:
            lines.append(f"a {s} {d} {rng.integers(1, 50)}")
        else:
            lines.append(f"a {s} {d}")
    text = "\n".join(lines) + "\n"
    p = tmp_path / "u.txt"
    p.write_text(text)
    k, s, d, w, _, _ = G.parse_text_file(str(p), updates=True)
    want = [r for r in (parse_update_line(ln) for ln in lines) if r is not None]
    assert [(chr(a), b, c, x) for a, b, c, x in zip(k.tolist(), s.tolist(), d.tolist(), w.tolist())] == \
        [(r.kind, r.src, r.dst, r.weight) for r in want]


@pytest.mark.parametrize("bad", ["x 1 2", "a 1", "d 1 2 3", "a 1 2 3 4", "d 1 q"])
def test_update_errors(tmp_path, bad):
    p = tmp_path / "u.txt"
    p.write_text("a 0 1\n\nd 0 1\n" + bad + "\n")
    with pytest.raises(MalformedInputError) as e:
        G.parse_text_file(str(p), updates=True)
    assert e.value.line == 4


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        G.parse_text_file(str(tmp_path / "nope.txt"), updates=False)
