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
