"""In-tree build of libdse_b200.so (nvcc, sm_100a).  Used by
__graft_entry__.build(); the .so is git-ignored but travels to the GPU box."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "dse_b200.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", "dse_device.cuh"), os.path.join(HERE, "csrc", "dse_mu.cu"), os.path.join(HERE, "csrc", "dse_pairs.cuh"), os.path.join(ROOT, "include", "dse_b200.h")]
OUT = os.path.join(HERE, "libdse_b200.so")
# bounds-checked diagnostic build (tests/test_gpu_checked.py): compute-sanitizer is closed on this pool
OUT_CHECKED = os.path.join(ROOT, "build", "libdse_checked.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def build_checked(force: bool = False) -> str:
    if not force and os.path.exists(OUT_CHECKED) and \
            all(os.path.getmtime(OUT_CHECKED) >= os.path.getmtime(d) for d in DEPS):
        return OUT_CHECKED
    os.makedirs(os.path.dirname(OUT_CHECKED), exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")]
    cmd = [nvcc(), *flags, "-DDSE_CHECKED=1", "-I", os.path.join(ROOT, "include"), "-o", OUT_CHECKED, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc (checked) failed:\n{res.stderr}")
    return OUT_CHECKED


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in DEPS):
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", OUT, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{res.stdout}\n{res.stderr}")
    with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as fh:
        fh.write(res.stderr)
    if verbose:
        print(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
