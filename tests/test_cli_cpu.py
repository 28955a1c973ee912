"""The graphdyn-compatible CLI (paper_2507_11094_b200.cli) on paths that need
no GPU: seed-compatible gen-updates byte-identical to the reference CLI's
output (tests/golden/make_cli_golden.py), and the exit-code contract
(cli.py:33-37 of the reference)."""

import os

import pytest

from paper_2507_11094_b200.cli import EXIT_COMPILE, EXIT_OK, EXIT_RUNTIME, EXIT_USAGE, main

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "cli")


@pytest.mark.parametrize("graph,flags,gold", [
    ("g40.txt", ["--percent", "10", "--seed", "42"], "gen_g40.txt"),
    ("g60u.txt", ["--percent", "30", "--seed", "7", "--undirected", "--add-fraction", "0.25"], "gen_g60u.txt"),
    ("rmat9.txt", ["--percent", "5", "--seed", "11"], "gen_rmat9.txt"),
])
def test_gen_updates_byte_identical_to_reference(tmp_path, graph, flags, gold):
    out = tmp_path / "u.txt"
    assert main(["gen-updates", os.path.join(GOLD, graph), *flags, "--out", str(out)]) == EXIT_OK
    assert out.read_bytes() == open(os.path.join(GOLD, gold), "rb").read()


def test_gen_updates_binary_matches_text(tmp_path):
    from paper_2507_11094_b200 import io as gio

    out = tmp_path / "u.bin"
    assert main(["gen-updates", os.path.join(GOLD, "g40.txt"), "--percent", "10", "--seed", "42", "--binary",
                 "--out", str(out)]) == EXIT_OK
    st = gio.load_updates_binary(str(out))
    text = [ln.split() for ln in open(os.path.join(GOLD, "gen_g40.txt")).read().splitlines()]
    got = [[r.kind, str(r.src), str(r.dst)] + ([str(r.weight)] if r.kind == "a" else []) for r in st.records]
    assert got == text


def test_gen_updates_percent_out_of_range_is_runtime_error(tmp_path):
    rc = main(["gen-updates", os.path.join(GOLD, "g40.txt"), "--percent", "0", "--seed", "1",
               "--out", str(tmp_path / "u.txt")])
    assert rc == EXIT_RUNTIME


def test_compile_diagnostics_exit_code(tmp_path):
    bad = tmp_path / "bad.sp"
    bad.write_text("function f(Graph g) { int x = ; }")
    assert main(["run", str(bad), os.path.join(GOLD, "scenario.txt"), "--out", str(tmp_path / "x")]) == EXIT_COMPILE


def test_bench_empty_percent_list_is_usage_error(tmp_path):
    rc = main(["bench", "sssp", os.path.join(GOLD, "scenario.txt"),
               "--percents", "", "--src", "0", "--out", str(tmp_path / "b")])
    assert rc == EXIT_USAGE


def test_bench_ranks_is_usage_error(tmp_path):
    rc = main(["bench", "tc", os.path.join(GOLD, "g60u.txt"), "--undirected",
               "--percents", "10", "--ranks", "2", "--out", str(tmp_path / "b")])
    assert rc == EXIT_USAGE


@pytest.mark.parametrize("cmd", [["emit", "x.sp"],  # the compiler is out of scope
                                 ["sim", "x.sp", "g.txt", "--ranks", "2"],  # unreadable program
                                 ["sim", "pr", "g.txt", "--ranks", "2", "--partitioner", "hash"],  # blocks only
                                 ["sim", "pr", "g.txt", "--ranks", "0"]])
def test_emit_and_bad_sim_invocations_are_usage_errors(cmd):
    assert main(cmd) == EXIT_USAGE


def test_bad_flag_is_usage_error():
    with pytest.raises(SystemExit) as e:
        main(["run"])
    assert e.value.code == EXIT_USAGE
