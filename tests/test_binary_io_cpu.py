"""Binary edge / update files: round trips and the
malformed-input errors the text loaders raise."""

import numpy as np
import pytest

from paper_2507_11094_b200 import io as gio
from paper_2507_11094_b200.errors import MalformedInputError


def test_edges_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    s, d, w = rng.integers(0, 50, 300), rng.integers(0, 50, 300), rng.integers(1, 9, 300)
    p = str(tmp_path / "g.bin")
    gio.save_edges_binary(p, 50, s, d, w, directed=False)
    n, s2, d2, w2, directed = gio.load_edges_binary(p)
    assert n == 50 and not directed
    np.testing.assert_array_equal(s2, s)
    np.testing.assert_array_equal(d2, d)
    np.testing.assert_array_equal(w2, w)
    gio.save_edges_binary(p, 50, s, d)
    n, s2, d2, w2, directed = gio.load_edges_binary(p)
    assert w2 is None and directed


def test_empty_files(tmp_path):
    p = str(tmp_path / "e.bin")
    gio.save_edges_binary(p, 0, [], [])
    n, s, d, w, _ = gio.load_edges_binary(p)
    assert n == 0 and len(s) == 0 and w is None
    q = str(tmp_path / "u.bin")
    gio.save_updates_binary(q, np.zeros(0, np.uint8), [], [])
    assert len(gio.load_updates_binary(q)) == 0


def test_updates_round_trip(tmp_path):
    kind = np.frombuffer(b"adda" * 5 + b"a", dtype=np.uint8)
    s, d, w = np.arange(21), np.arange(21)[::-1], np.arange(21) + 1
    p = str(tmp_path / "u.bin")
    gio.save_updates_binary(p, kind, s, d, w)
    st = gio.load_updates_binary(p)
    assert [(r.kind, r.src, r.dst, r.weight) for r in st.records] == \
        [(chr(k), int(a), int(b), int(c)) for k, a, b, c in zip(kind, s, d, w)]
    assert [len(b) for b in st.batches(8)] == [8, 8, 5]


@pytest.mark.parametrize("case", ["magic", "size", "range", "weight"])
def test_malformed_edges(tmp_path, case):
    p = str(tmp_path / "bad.bin")
    gio.save_edges_binary(p, 10, [1, 2], [3, 4], [5, 6])
    raw = bytearray(open(p, "rb").read())
    if case == "magic":
        raw[0:8] = b"NOTMAGIC"
    elif case == "size":
        raw = raw[:-8]
    elif case == "range":
        raw[32:40] = np.array([10], "<i8").tobytes()
    else:
        raw[-8:] = np.array([-1], "<i8").tobytes()
    open(p, "wb").write(bytes(raw))
    with pytest.raises(MalformedInputError):
        gio.load_edges_binary(p)


def test_malformed_updates(tmp_path):
    p = str(tmp_path / "u.bin")
    with pytest.raises(MalformedInputError):
        gio.save_updates_binary(p, np.frombuffer(b"x", np.uint8), [0], [1])
    gio.save_updates_binary(p, np.frombuffer(b"a", np.uint8), [0], [1])
    raw = bytearray(open(p, "rb").read())
    raw[16] = ord("z")
    open(p, "wb").write(bytes(raw))
    with pytest.raises(MalformedInputError):
        gio.load_updates_binary(p)
