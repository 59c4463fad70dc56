"""GPU: the sweep kernel's reduction machinery reproduces numpy's pairwise
summation order BITWISE, for every chunking of the tree.

Tolerance tests cannot see a wrong summation order (it moves results by
~1e-16), so the production path (8-lane leaves, chunk subtrees, top tree,
row finalisation) is run on adversarial values through the
dse_debug_pairwise_sum hook and compared with np.sum exactly."""
import numpy as np
import pytest

from paper_2012_03667_b200 import _native

pytestmark = pytest.mark.gpu

SHAPES = [(128, 64), (1024, 256), (100, 32), (37, 5), (29, 5), (2, 1), (3, 3), (16, 8), (150, 32), (7, 17)]


@pytest.mark.parametrize("m,k", SHAPES)
@pytest.mark.parametrize("chunk", [0, 1, 2, 3, 32, 10 ** 6])
def test_reduction_order_bitwise(m, k, chunk):
    rng = np.random.default_rng(m * 1000 + k)
    rows = 3
    x = rng.standard_normal((rows, m, k)) * np.exp(rng.uniform(-30, 30, (rows, m, k)))
    a, b = _native.debug_pairwise_sum(x, chunk_leaves=chunk)
    for i in range(rows):
        assert a[i] == np.sum(x[i]), (m, k, chunk, i)
        assert b[i] == np.sum(-2.0 * x[i]), (m, k, chunk, i)
