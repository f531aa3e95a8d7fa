#!/bin/bash
# Cold-start (first step after set_agents) sweep of compile-time knobs: device ms per stage.
OUT=gpurun_out; mkdir -p $OUT
for F in "$@"; do
  ORCA_NVCC_EXTRA="$F" python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $F"; continue; }
  for CFG in uniform_1m uniform dense; do
    echo "== $F $CFG: $(timeout 300 python scripts/e2e_breakdown.py $CFG 2>&1 | tr '\n' ' ')"
  done
done | tee $OUT/sweep_cold.txt
python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
