#!/bin/bash
# compute-sanitizer over the product path: memcheck, racecheck, synccheck
# and initcheck on the small cases of scripts/sanitize_cases.py, plus memcheck of a 2-process
# strips run through the fake NCCL (tests/test_gpu_nccl_fake.py).  Logs: gpurun_out/sanitize_<tag>_*.txt
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
python -c "from paper_1908_10107_b200 import build as B; B.build()" || exit 1
for TC in memcheck:circle memcheck:corridor memcheck:strips4 memcheck:trace racecheck:circle racecheck:corridor \
          racecheck:strips4 synccheck:circle synccheck:corridor synccheck:strips4 initcheck:circle initcheck:strips4; do
  TOOL=${TC%%:*}; CASE=${TC##*:}
  {
    F=$OUT/sanitize_${TAG}_${TOOL}_${CASE}.txt
    timeout 900 $CS --tool $TOOL --error-exitcode 9 --print-limit 50 python scripts/sanitize_cases.py $CASE > $F 2>&1
    echo "$TOOL $CASE rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $F | tail -1)"
  }
done
F=$OUT/sanitize_${TAG}_memcheck_fake_nccl2.txt
timeout 1500 $CS --tool memcheck --target-processes all --error-exitcode 9 --print-limit 50 \
  python -m pytest tests/test_gpu_nccl_fake.py -q -x -k "multirank and 2-uniform" > $F 2>&1
echo "memcheck fake_nccl2 rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $F | tail -2 | tr '\n' ' ')"
