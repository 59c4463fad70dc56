"""CPU: the reduction plan the kernels execute (dse_plan_info, host-only C++)
equals numpy's pairwise_sum recursion, and summing with it -- in the
kernels' order: 8 interleaved lane sums per leaf, the fixed lane combine,
the n % 8 tail, the chunk subtrees, the post-order top tree -- equals
np.sum bitwise."""
import numpy as np
import pytest

from paper_2012_03667_b200 import _native


def numpy_leaves(start, n, out):
    if n <= 128:
        out.append((start, n))
        return
    n2 = n // 2
    n2 -= n2 % 8
    numpy_leaves(start, n2, out)
    numpy_leaves(start + n2, n - n2, out)


def leaf_sum(a):
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += x
        return r
    main = n - n % 8
    lanes = [a[u] for u in range(8)]
    for i in range(8, main, 8):
        for u in range(8):
            lanes[u] += a[i + u]
    r = ((lanes[0] + lanes[1]) + (lanes[2] + lanes[3])) + ((lanes[4] + lanes[5]) + (lanes[6] + lanes[7]))
    for i in range(main, n):
        r += a[i]
    return r


def tree_sum(vals, leaves, lo, hi):
    """Sum leaf values lo..hi-1 with numpy's recursion over their element range."""
    s, e = leaves[lo][0], leaves[hi - 1][0] + leaves[hi - 1][1]
    n = e - s
    if hi - lo == 1:
        return vals[lo]
    n2 = n // 2
    n2 -= n2 % 8
    mid = next(i for i in range(lo, hi) if leaves[i][0] == s + n2)
    return tree_sum(vals, leaves, lo, mid) + tree_sum(vals, leaves, mid, hi)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 127, 128, 129, 145, 1000, 3200, 8192, 29 * 5, 262144, 100003])
def test_leaves_match_numpy_recursion(n):
    ls, ll, _, _, _ = _native.plan_info(n)
    ref = []
    numpy_leaves(0, n, ref)
    assert list(zip(ls.tolist(), ll.tolist())) == ref


@pytest.mark.parametrize("n,chunk", [(8192, 32), (8192, 1), (3200, 3), (262144, 256), (145, 1), (100003, 64)])
def test_chunked_sum_equals_np_sum(n, chunk):
    rng = np.random.default_rng(n + chunk)
    x = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    ls, ll, clo, chi, tops = _native.plan_info(n, chunk)
    leaves = list(zip(ls.tolist(), ll.tolist()))
    vals = [leaf_sum(x[s:s + m].tolist()) for s, m in leaves]
    # chunk subtrees, then the post-order top tree over chunk slots
    csum = [tree_sum(vals, leaves, lo, hi) for lo, hi in zip(clo.tolist(), chi.tolist())]
    for d, s in tops.tolist():
        csum[d] = csum[d] + csum[s]
    assert csum[0] == np.sum(x)
    assert clo[0] == 0 and chi[-1] == len(leaves) and all(chi[:-1] == clo[1:])
