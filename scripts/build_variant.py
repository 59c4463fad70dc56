"""Build an A/B variant of libdse_b200.so with extra -D flags into build/:
python scripts/build_variant.py NAME -DFOO=1 ..."""
import os, subprocess, sys
sys.path.insert(0, ".")
from paper_2012_03667_b200 import _build as B
name, defs = sys.argv[1], sys.argv[2:]
os.makedirs("build", exist_ok=True)
out = os.path.join("build", f"ab_{name}.so")
cmd = [B.nvcc(), *B.NVCC_FLAGS, *defs, "-I", "include", "-o", out, *B.SOURCES]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr)
open(out + ".ptxas.txt", "w").write(r.stderr)
print(out)
