import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2012_03667_b200 import _native
rng = np.random.default_rng(9)
n = 400000
a = rng.uniform(1, 2, n) * 2.0 ** rng.integers(-1074, -940, n).astype(float) * rng.choice([-1, 1], n)
b = rng.uniform(1, 2, n) * 2.0 ** rng.integers(-8, 40, n).astype(float)
ext, ref, ok = _native.debug_qdiv_ext(a, b)
bad = ~ok
print("notok", bad.sum(), "bitwise where ok", np.array_equal(ext[ok].view(np.int64), ref[ok].view(np.int64)))
print("notok sample a", a[bad][:5], "b", b[bad][:5], "ref", ref[bad][:5], "ext", ext[bad][:5])
print("notok: ref==0 frac", np.mean(ref[bad] == 0), "a<2^-1022 frac", np.mean(np.abs(a[bad]) < 2.0**-1022))
print("all: ref==0 frac", np.mean(ref == 0))
print("ext==ref among notok", np.mean(ext[bad].view(np.int64) == ref[bad].view(np.int64)))
