set -u
O=gpurun_out
for i in 1 2; do
DSE_MU_MIRROR=0 timeout 600 python -m pytest tests/test_gpu_mu.py -q -m gpu -k "sharded_iteration_world3" > $O/r02aq_$i.off.log 2>&1; echo "off rc=$?" >> $O/r02aq.log
timeout 600 python -m pytest tests/test_gpu_mu.py -q -m gpu -k "sharded_iteration_world3" > $O/r02aq_$i.on.log 2>&1; echo "on rc=$?" >> $O/r02aq.log
done
python - >> $O/r02aq.log 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2012_03667_b200.finite_mu import iterate_mu_once, MuSweeper
from paper_2012_03667_b200.mu_grid import MuParams, grid_for
p = MuParams(n_s=10, n_4=12, m_s=14, m_4=16, m_ang=6); g = grid_for(p)
rng = np.random.default_rng(6)
shape = (g.n_s, g.n_4)
A = 1.0 + 0.5 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
B = 0.3 + 0.1 * rng.random(shape) + 0.05j * rng.standard_normal(shape)
C = 1.0 + 0.5 * rng.random(shape) + 0.1j * rng.standard_normal(shape)
r1 = iterate_mu_once(g, A, B, C, p)
r2 = iterate_mu_once(g, A, B, C, p)
print("repeat equal", all(np.array_equal(x, y) for x, y in zip(r1, r2)))
print("z", g.z_nodes, g.z_weights)
PY
echo done
