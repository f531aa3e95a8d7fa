#!/bin/bash
# Build variants of liborca with different compile-time knobs and time each (1 GPU).
# Usage: bash scripts/sweep.sh "<flags1>" "<flags2>" ...
OUT=gpurun_out; mkdir -p $OUT
for F in "$@"; do
  ORCA_NVCC_EXTRA="$F" python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $F"; continue; }
  for CFG in ${SWEEP_CFGS:-uniform_1m uniform dense}; do
    R=$(timeout 150 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1 2>/dev/null | tail -1)
    python - "$F" "$CFG" "$R" <<'PY'
import json, sys
f, cfg, r = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    d = json.loads(r)
    print(f"{f:40s} {cfg:12s} ms/step {d['ms_per_step']:.4f}  k_step {d['roofline']['stage_ms']['k_step+k_lp3']:.4f}  order {d.get('k_step_ms_by_lp_order')} variants {d['k_step_ms_by_variant']} lp3 {d.get('k_step_ms_by_lp3_lanes')}")
except Exception as e:
    print(f, cfg, "FAILED", r[:200])
PY
  done
done | tee $OUT/sweep.txt
# leave the default build behind (build.py also rebuilds on a flags mismatch)
python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1

