"""Host-side drop-in semantics of the variant seam (no GPU needed).

Reference: solver.py:48-74 (ExecutionMode, AlgorithmVariant, VARIANTS),
solver.py:100-108 (resolve_threads, SOLVER_THREADS), test_solver.py:74-80.
"""
import os

import pytest

import paper_2012_03667_b200 as p
from paper_2012_03667_b200 import AlgorithmVariant, Arithmetic, ExecutionMode, InterpStrategy


def test_reference_execution_modes_exist_with_reference_values():
    assert ExecutionMode.SEQUENTIAL.value == "seq" and ExecutionMode.PARALLEL.value == "par"
    assert ExecutionMode.GPU.value == "gpu"


def test_reference_variant_names_and_cells():
    for name, interp, mode in (("search-seq", InterpStrategy.SEARCH_BASED, ExecutionMode.SEQUENTIAL),
                               ("indexed-seq", InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.SEQUENTIAL),
                               ("search-par", InterpStrategy.SEARCH_BASED, ExecutionMode.PARALLEL),
                               ("indexed-par", InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.PARALLEL)):
        v = p.VARIANTS[name]
        assert v.name == name and v.interp is interp and v.execution is mode
        assert v.arith is Arithmetic.EXACT  # the reference's operation order
        assert v.with_threads(8).name == name and v.with_threads(8).threads == 8


def test_positional_reference_constructor():
    v = AlgorithmVariant(InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.PARALLEL, 4)
    assert v.threads == 4 and v.arith is Arithmetic.EXACT and v.gpus is None
    assert v == p.VARIANTS["indexed-par"].with_threads(4)
    g = AlgorithmVariant(InterpStrategy.PRECOMPUTED_INDEX, ExecutionMode.GPU)
    assert g.arith is Arithmetic.FAST and g.name == "indexed-gpu"
    assert p.VARIANTS["indexed-gpu-pairs"].name == "indexed-gpu-pairs"


def test_threads_are_host_workers(monkeypatch):
    monkeypatch.delenv("SOLVER_THREADS", raising=False)
    monkeypatch.delenv("DSE_GPUS", raising=False)
    assert p.resolve_threads(p.VARIANTS["indexed-par"]) == (os.cpu_count() or 1)
    monkeypatch.setenv("SOLVER_THREADS", "3")
    assert p.resolve_threads(p.VARIANTS["indexed-par"]) == 3
    assert p.resolve_threads(p.VARIANTS["indexed-par"].with_threads(2)) == 2
    # threads never select GPUs
    assert p.resolve_gpus(p.VARIANTS["indexed-par"].with_threads(8)) == 1
    with pytest.raises(p.ParameterError):
        p.resolve_threads(p.VARIANTS["indexed-par"].with_threads(0))


def test_gpu_count_knob(monkeypatch):
    monkeypatch.delenv("DSE_GPUS", raising=False)
    assert p.resolve_gpus(p.VARIANTS["indexed-gpu-pairs"]) == 1
    assert p.resolve_gpus(p.VARIANTS["indexed-gpu-pairs"].with_gpus(4)) == 4
    monkeypatch.setenv("DSE_GPUS", "2")
    assert p.resolve_gpus(p.VARIANTS["indexed-seq"]) == 2
    with pytest.raises(p.ParameterError):
        p.resolve_gpus(p.VARIANTS["indexed-seq"].with_gpus(0))


def test_multi_gpu_without_torchrun_is_a_parameter_error(monkeypatch):
    """gpus > 1 outside torchrun: the reference raises on a bad execution
    environment before any numerics; here the sharded path needs
    torch.distributed and says so."""
    import numpy as np
    monkeypatch.delenv("DSE_GPUS", raising=False)
    g = p.build_grid(8, 6, 2, 1e-4, 1e2)
    prm = p.ModelParams(N=8, m_rad=6, m_ang=2)
    with pytest.raises((p.ParameterError, p.ExecutionEnvironmentError)):
        p.iterate_once(g, np.ones(8), np.ones(8), prm, p.VARIANTS["indexed-gpu-pairs"].with_gpus(2))


def test_history_records_conversion():
    """solver._records (one tolist() per history) builds exactly the
    IterationRecords the per-element float() form did, NaN row 0 included."""
    import numpy as np
    from paper_2012_03667_b200.solver import IterationRecord, _records
    rng = np.random.default_rng(3)
    for P in (0, 1, 2, 5):
        h = rng.standard_normal((17, 3 + 2 * P))
        h[:, 0] = np.arange(17)
        h[0, 1:3] = np.nan
        old = [IterationRecord(int(r[0]), float(r[1]), float(r[2]), tuple(float(x) for x in r[3:3 + P]),
                               tuple(float(x) for x in r[3 + P:3 + 2 * P])) for r in h]
        new = _records(h, P)
        assert len(new) == len(old)
        for a, b in zip(new, old):
            assert a.iteration == b.iteration and type(a.iteration) is int
            assert np.array_equal(np.array([a.max_delta_a, a.max_delta_b]), np.array([b.max_delta_a, b.max_delta_b]),
                                  equal_nan=True)
            assert a.probe_a == b.probe_a and a.probe_b == b.probe_b
            assert all(type(x) is float for x in a.probe_a + a.probe_b)
