"""GPU: CLI end to end, deterministic CSV bytes, and the variant harness with
its agreement gate (reference test_cli.py / test_bench.py patterns)."""
import json

import numpy as np
import pytest

import paper_2012_03667_b200 as p
from conftest import golden
from paper_2012_03667_b200 import cli, harness

pytestmark = pytest.mark.gpu


def test_solve_cli_default_config_and_bytes(tmp_path):
    paths = []
    for run in range(2):
        s, h = tmp_path / f"s{run}.csv", tmp_path / f"h{run}.csv"
        assert cli.main(["solve", "--variant", "indexed-gpu-exact", "--out", str(s), "--history", str(h)]) == 0
        paths.append((s.read_bytes(), h.read_bytes()))
    assert paths[0] == paths[1]  # deterministic kernels -> byte-identical CSV
    z = golden("solve_default.npz")
    rows = np.loadtxt(tmp_path / "s0.csv", delimiter=",", skiprows=1)
    assert np.allclose(rows[:, 1], z["A"], rtol=1e-11, atol=0) and rows.shape[0] == 150
    hist = (tmp_path / "h0.csv").read_text().splitlines()
    assert len(hist) == int(z["iterations"]) + 2


def test_bench_cli_table1_rows_and_agreement(tmp_path, capsys):
    """`bench`: the reference's four CPU algorithms (bench.py's baseline leg)
    beside the four GPU rows, one iteration count, GPU-over-CPU speedups."""
    out = tmp_path / "b.json"
    assert cli.main(["bench", "--N", "48", "--M-rad", "40", "--M-ang", "16", "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    names = [r["variant"] for r in rep["rows"]]
    assert names == ["search-cpu-seq", "indexed-cpu-seq", "search-cpu-par", "indexed-cpu-par",
                     *harness.GPU_ROWS]
    assert [r["backend"] for r in rep["rows"]] == ["cpu-port"] * 4 + ["gpu"] * 4
    assert len({r["iterations"] for r in rep["rows"]}) == 1
    text = capsys.readouterr().out
    assert "speedup search-cpu-seq/indexed-gpu-pairs" in text
    assert any(k.startswith(("indexed-cpu-par/", "search-cpu-par/", "indexed-cpu-seq/", "search-cpu-seq/"))
               and k.endswith("/indexed-gpu") for k in rep["speedups"])
    assert cli.main(["bench", "--N", "48", "--M-rad", "40", "--M-ang", "16", "--cpu-rows", "off",
                     "--out", str(out)]) == 0
    assert [r["variant"] for r in json.loads(out.read_text())["rows"]] == list(harness.GPU_ROWS)


def test_agreement_gate_fires(monkeypatch):
    real = harness.solve

    def tampered(params, variant, grid=None, **kw):
        sol = real(params, variant, grid=grid, **kw)
        if variant.name == "indexed-gpu":
            sol.A = sol.A + 1e-6
        return sol
    monkeypatch.setattr(harness, "solve", tampered)
    with pytest.raises(p.ConsistencyError):
        harness.run_bench(p.ModelParams(N=32, m_rad=24, m_ang=8), warmup=False)
