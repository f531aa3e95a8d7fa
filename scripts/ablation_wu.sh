#!/bin/bash
# Work-unit LP2 ablation (§8(f3)): rebuild with each ORCA_WU_ROUNDS and time variants 0/3.
OUT=gpurun_out; mkdir -p $OUT
for R in "$@"; do
  ORCA_NVCC_EXTRA="-DORCA_WU_ROUNDS=$R" python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $R"; continue; }
  timeout 600 python scripts/ablation_variants.py --tag "wu_rounds=$R"
done | tee $OUT/ablation_wu.txt
python -c "from paper_1908_10107_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
