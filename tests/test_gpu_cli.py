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


def test_bench_cli_and_agreement(tmp_path, capsys):
    out = tmp_path / "b.json"
    assert cli.main(["bench", "--N", "48", "--M-rad", "40", "--M-ang", "16", "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert [r["variant"] for r in rep["rows"]] == list(harness.VARIANT_ORDER)
    assert len({r["iterations"] for r in rep["rows"]}) == 1
    assert "speedup search-gpu-exact/indexed-gpu" in capsys.readouterr().out


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
