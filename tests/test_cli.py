"""CPU: CLI configuration precedence, validation, exit codes and the CSV
byte format (reference cli.py:100-223), without running the GPU."""
import json

import numpy as np
import pytest

import paper_2012_03667_b200 as p
from paper_2012_03667_b200 import cli


def test_precedence_defaults_file_flags(tmp_path):
    cfgf = tmp_path / "c.json"
    cfgf.write_text(json.dumps({"N": 40, "xi": 0.01, "variant": "search-gpu", "probes": [-1.0, 0.5]}))
    cmd, cfg = cli.parse_config(["solve", "--config", str(cfgf), "--N", "64", "--D", "0.7"])
    assert cmd == "solve"
    assert cfg.params.N == 64 and cfg.params.xi == 0.01 and cfg.params.D == 0.7
    assert cfg.params.m_rad == p.ModelParams().m_rad
    assert cfg.variant == "search-gpu" and cfg.probes_log10p == (-1.0, 0.5)
    cmd, cfg = cli.parse_config(["bench", "--M-ang", "8", "--repeat", "2"])
    assert cmd == "bench" and cfg.params.m_ang == 8 and cfg.repeat == 2 and cfg.bench_out == "bench.json"
    _, cfg = cli.parse_config(["bench", "--out", "x.json"])
    assert cfg.bench_out == "x.json"


@pytest.mark.parametrize("argv", [["solve", "--N", "1"], ["solve", "--xi", "abc"], ["solve", "--relaxation", "0"],
                                  ["bench", "--repeat", "0"], ["solve", "--threads", "0"]])
def test_parameter_errors_exit_2(argv, capsys):
    assert cli.main(argv) == 2
    assert "error:" in capsys.readouterr().err


def test_config_file_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["solve", "--config", str(bad)]) == 2
    arr = tmp_path / "arr.json"
    arr.write_text("[1, 2]")
    assert cli.main(["solve", "--config", str(arr)]) == 2
    unk = tmp_path / "unk.json"
    unk.write_text(json.dumps({"bogus": 1}))
    assert cli.main(["solve", "--config", str(unk)]) == 2
    assert cli.main(["solve", "--config", str(tmp_path / "missing.json")]) == 2


def _fake_solution():
    g = p.build_grid(4, 3, 2, 1e-2, 1e2)
    hist = [p.IterationRecord(0, float("nan"), float("nan"), (1.0, 2.0), (0.3, 0.4)),
            p.IterationRecord(1, 0.1, 1e-17, (1.0 / 3.0, 2.0), (0.3, 1e-300))]
    return p.PropagatorSolution(A=np.array([1.0, 1.0 / 3.0, 2.0, 1e-20]), B=np.array([0.3, -0.0, 5e-324, 1.5]),
                                iterations=1, converged=True, history=hist, grid=g, params=p.ModelParams(),
                                probes_log10p=(-2.5, 0.0))


def test_csv_formats(tmp_path):
    sol = _fake_solution()
    cli.write_solution_csv(str(tmp_path / "s.csv"), sol)
    cli.write_history_csv(str(tmp_path / "h.csv"), sol)
    s = (tmp_path / "s.csv").read_text().splitlines()
    assert s[0] == "log10_p2,A,B"
    assert s[2].split(",")[1] == "0.33333333333333331" and s[2].split(",")[2] == "-0"
    assert float(s[3].split(",")[2]) == 5e-324
    h = (tmp_path / "h.csv").read_text().splitlines()
    assert h[0] == "iteration,max_dA,max_dB,A(logp=-2.5),B(logp=-2.5),A(logp=0),B(logp=0)"
    assert h[1].startswith("0,nan,nan,1,0.29999999999999999")
    assert h[2] == "1,0.10000000000000001,1.0000000000000001e-17,0.33333333333333331,0.29999999999999999,2,1e-300"


def test_no_gpu_is_a_runtime_failure(tmp_path, gpu_available, capsys):
    if gpu_available:
        pytest.skip("GPU present")
    rc = cli.main(["solve", "--N", "8", "--M-rad", "8", "--M-ang", "4", "--out", str(tmp_path / "s.csv"),
                   "--history", str(tmp_path / "h.csv")])
    assert rc == 1 and "error:" in capsys.readouterr().err


def test_harness_rows_gate_and_table_without_gpu():
    """The Table-1 harness on CPU rows only (the reference's algorithms from
    bench.py's baseline leg, C restatement): one iteration count, agreement,
    table and JSON schema (reference bench.py:28-50)."""
    import bench
    from paper_2012_03667_b200 import harness
    prm = p.ModelParams(N=24, m_rad=20, m_ang=8)
    rep = harness.run_bench(prm, order=(), baselines=bench.table1_cpu_runners(2))
    assert [r.variant for r in rep.rows] == ["search-cpu-seq", "indexed-cpu-seq", "search-cpu-par",
                                             "indexed-cpu-par"]
    assert len({r.iterations for r in rep.rows}) == 1 and all(r.converged for r in rep.rows)
    d = json.loads(rep.to_json())
    assert set(d) == {"rows", "speedups", "environment"}
    assert {"variant", "wall_s", "cpu_percent", "iterations", "converged"} <= set(d["rows"][0])
    assert "search-cpu-seq/indexed-cpu-par" in rep.speedups
    table = harness.format_table(rep)
    assert table.splitlines()[0].split()[:2] == ["variant", "backend"]


def test_harness_agreement_gate_fires_without_gpu():
    import types
    from paper_2012_03667_b200 import harness
    one = types.SimpleNamespace(A=np.ones(4), B=np.zeros(4), iterations=7, converged=True)
    off = types.SimpleNamespace(A=np.ones(4) + 1e-9, B=np.zeros(4), iterations=7, converged=True)
    slow = types.SimpleNamespace(A=np.ones(4), B=np.zeros(4), iterations=8, converged=True)
    mk = lambda name, sol: harness.Runner(name, "cpu-port", lambda prm, g: sol)  # noqa: E731
    prm = p.ModelParams(N=8, m_rad=6, m_ang=2)
    harness.run_bench(prm, order=(), baselines=[mk("a", one), mk("b", one)])
    with pytest.raises(p.ConsistencyError):
        harness.run_bench(prm, order=(), baselines=[mk("a", one), mk("b", off)])
    with pytest.raises(p.ConsistencyError):
        harness.run_bench(prm, order=(), baselines=[mk("a", one), mk("b", slow)])


def test_cpu_rows_flag_validation(capsys):
    assert cli.main(["bench", "--cpu-rows", "maybe"]) == 2
