"""Reference CLI outputs for the drop-in CLI tests (tests/test_cli_*.py):
run in the build container against /root/reference's own graphdyn.cli.

    python tests/golden/make_cli_golden.py
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
SCENARIO = "0 1 30\n0 2 20\n0 3 48\n3 4 4\n2 5 25\n4 5 6\n"
SCENARIO_UPDATES = "d 2 5\na 1 3 10\n"


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    from graphdyn.cli import main as ref
    from graphdyn.generate import rmat_graph, uniform_random_graph

    progs = "/root/reference/pkg/src/graphdyn/programs"
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    p = lambda *a: os.path.join(OUT, *a)  # noqa: E731
    open(p("scenario.txt"), "w").write(SCENARIO)
    open(p("scenario_updates.txt"), "w").write(SCENARIO_UPDATES)
    edges = uniform_random_graph(40, 120, seed=2, weighted=True, max_weight=9)
    open(p("g40.txt"), "w").write("".join(f"{u} {v} {w}\n" for u, v, w in edges))
    edges = uniform_random_graph(60, 200, seed=3, undirected=True)
    open(p("g60u.txt"), "w").write("".join(f"{u} {v}\n" for u, v, _ in edges))
    edges, _ = rmat_graph(9, 2500, seed=4)
    open(p("rmat9.txt"), "w").write("".join(f"{u} {v}\n" for u, v, _ in edges))
    runs = [
        ["gen-updates", p("g40.txt"), "--percent", "10", "--seed", "42", "--out", p("gen_g40.txt")],
        ["gen-updates", p("g60u.txt"), "--percent", "30", "--seed", "7", "--undirected", "--add-fraction", "0.25",
         "--out", p("gen_g60u.txt")],
        ["gen-updates", p("rmat9.txt"), "--percent", "5", "--seed", "11", "--out", p("gen_rmat9.txt")],
        ["run", f"{progs}/sssp_dynamic.sp", p("scenario.txt"), "--updates", p("scenario_updates.txt"),
         "--batch", "1000", "--src", "0", "--out", p("run_sssp")],
        ["run", f"{progs}/sssp_dynamic.sp", p("g40.txt"), "--updates", p("gen_g40.txt"), "--batch", "5",
         "--src", "3", "--out", p("run_sssp_g40")],
        ["run", f"{progs}/pr_dynamic.sp", p("rmat9.txt"), "--updates", p("gen_rmat9.txt"), "--batch", "40",
         "--out", p("run_pr_rmat9")],
        ["run", f"{progs}/tc_dynamic.sp", p("g60u.txt"), "--undirected", "--updates", p("gen_g60u.txt"),
         "--batch", "20", "--out", p("run_tc_g60u")],
        ["oracle", "tc", p("g60u.txt"), "--undirected", "--updates", p("gen_g60u.txt"), "--out", p("oracle_tc")],
        ["oracle", "sssp", p("g40.txt"), "--updates", p("gen_g40.txt"), "--src", "3", "--out", p("oracle_sssp")],
    ]
    for argv in runs:
        rc = ref(argv)
        assert rc == 0, (argv, rc)
    for d in os.listdir(OUT):  # manifests hold absolute paths and timings: not fixtures
        full = p(d)
        if os.path.isdir(full) and os.path.exists(os.path.join(full, "manifest.json")):
            os.remove(os.path.join(full, "manifest.json"))
    print(sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
