"""Output formats of the path: io.cpp:14-18, 120-140 and
path.cpp:144-177, checked against the reference's own test cases
(test_io.cpp:113-126, 197-203; test_path.cpp:243-270) and, for number
spelling, against libstdc++'s std::to_chars compiled here."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2501_15964_b200.io import export_graph_csv, format_double, write_matrix_csv

TO_CHARS = r"""
#include <charconv>
#include <cstdio>
#include <cstring>
#include <cstdint>
int main() {
  uint64_t u;
  while (std::scanf("%lx", &u) == 1) {
    double x; std::memcpy(&x, &u, 8);
    char b[64]; auto r = std::to_chars(b, b + 64, x); *r.ptr = 0; std::printf("%s\n", b);
  }
}
"""


def test_format_double_matches_std_to_chars(tmp_path):
    src = tmp_path / "tc.cpp"
    src.write_text(TO_CHARS)
    exe = tmp_path / "tc"
    r = subprocess.run(["g++", "-std=c++20", "-O1", str(src), "-o", str(exe)], capture_output=True)
    if r.returncode != 0:
        pytest.skip("no C++20 compiler for the std::to_chars reference")
    rng = np.random.default_rng(3)
    vals = np.concatenate([np.exp(rng.normal(0, 25, 3000)) * rng.choice([-1, 1], 3000),
                           rng.integers(-10**6, 10**6, 500).astype(float), [0.0, -0.0, 1e5, 1e-5, 0.5, 2.0],
                           np.round(rng.normal(0, 100, 500), 3)])
    inp = "\n".join(f"{int(x):x}" for x in vals.view(np.uint64))
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True).stdout.split()
    mine = [format_double(x) for x in vals]
    assert mine == out


def test_export_graph_csv_kat(tmp_path):  # test_io.cpp:197-203
    p = tmp_path / "g.csv"
    export_graph_csv(str(p), i=[0, 1], j=[1, 2], w=[0.5, 2.0])
    assert p.read_text() == "i,j,w\n0,1,0.5\n1,2,2\n"


def test_write_matrix_csv_round_trip(tmp_path):  # test_io.cpp:113-126
    rng = np.random.default_rng(4)
    M = np.exp(8 * rng.standard_normal((7, 5))) * np.where(rng.standard_normal((7, 5)) < 0, -1, 1)
    p = tmp_path / "m.csv"
    write_matrix_csv(str(p), M)
    back = np.array([[float(x) for x in line.split(",")] for line in p.read_text().splitlines()])
    assert back.shape == (7, 5) and np.array_equal(back, M)
    with pytest.raises(RuntimeError):
        write_matrix_csv(str(tmp_path / "no" / "such" / "dir.csv"), M)


@pytest.mark.gpu
def test_path_result_to_json(cp):  # test_path.cpp:243-270
    data = cp.DataMatrix(np.array([[0.0], [2.0]]))
    g = cp.WeightedGraph(2, [(0, 1, 1.0)])
    sched = cp.make_schedule(0.5, 2.0, 3, cp.Spacing.geometric)
    res = cp.run_path(data, g, 2, sched, cp.SolverConfig(epsilon=1e-8))
    j = json.loads(cp.path_result_to_json(res))
    assert j["schedule"]["spacing"] == "geometric" and len(j["schedule"]["values"]) == 3
    assert j["schedule"]["count"] == 3
    assert j["solver"]["algorithm"] == "ssnal" and j["solver"]["epsilon"] == 1e-8
    assert j["solver"]["max_iter"] == 100
    assert len(j["per_gamma"]) == 3
    rec = j["per_gamma"][0]
    assert rec["gamma"] == pytest.approx(0.5) and rec["converged"] is True and rec["K"] == 2
    assert len(rec["labels"]) == 2
    for key in ("f_p", "f_d", "gap", "iterations", "wall_time_s"):
        assert key in rec
    assert j["per_gamma"][2]["K"] == 1  # last gamma is past the fusion threshold
    p = os.path.join(os.path.dirname(__file__), "..", "gpurun_out")
    gi, gj, gw, _ = g.arrays()
    assert gi.tolist() == [0] and gj.tolist() == [1]
