set -u
O=gpurun_out
for t in 640 320 256; do
DSE_PAIRS_LAUNCH_THREADS=$t python scripts/sub_tts.py >> $O/r02wa.log 2>&1
done
for nm in "512 512 128" "2048 512 64" "512 1024 256"; do
set -- $nm
for t in 640 320; do
echo -n "N=$1 M=$2 K=$3 threads=$t " >> $O/r02wa.log
DSE_PAIRS_LAUNCH_THREADS=$t python - $1 $2 $3 >> $O/r02wa.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import torch
import paper_2012_03667_b200 as p
N, M, K = map(int, sys.argv[1:4])
g = p.build_grid(N, M, K, 1e-6, 1e4)
prm = p.ModelParams(N=N, m_rad=M, m_ang=K, xi=1e-300, max_iterations=100000)
sw = p.GpuSweeper(g, prm, p.InterpStrategy.PRECOMPUTED_INDEX, p.Arithmetic("pairs"), 0)
a = torch.ones(N, dtype=torch.float64, device="cuda"); b = torch.full((N,), 0.3, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
ts = []
for r in range(12):
    sw.load_device(a.data_ptr(), b.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sw.resume(4, s); e1.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(e0.elapsed_time(e1) / 4)
ts.sort()
print(json.dumps({"ms_per_iteration": round(ts[len(ts) // 2], 4)}))
PY
done; done
echo done
