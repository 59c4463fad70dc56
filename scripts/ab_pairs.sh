#!/bin/bash
# A/B of pairs-kernel builds under gpurun: python bench config 2 step time per library.
mkdir -p gpurun_out
for lib in "$@"; do
  DSE_LIB=$lib python bench.py --no-tts --no-interp --no-cpu --no-mu --arith pairs --steps 50 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done
