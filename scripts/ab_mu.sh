#!/bin/bash
# A/B of finite-mu kernel builds: config-3 iteration time, direct and moments mode.
for lib in "$@"; do
  d=$(DSE_LIB=$lib python scripts/mu_step_probe.py bcb 10 | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['ms'],3))")
  m=$(DSE_LIB=$lib python scripts/mu_moments_time.py 10)
  echo "$lib direct $d moments $m"
done
