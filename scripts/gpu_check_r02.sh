#!/bin/bash
# One gpurun call (round 2): build, GPU tests, smoke, benches (1M, 100k, dense, reference arm),
# ncu launch list + full captures (k_step/k_lp3 at 1M, k_step at 100k, scan/scatter), sanitizers.
# Usage: gpurun --timeout 3600 -- 'bash scripts/gpu_check_r02.sh <tag> [what]'
TAG=${1:-r02}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.txt 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.txt; exit 1; }
if [[ $WHAT == all || $WHAT == test ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu_$TAG.txt 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.txt; tail -4 $OUT/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.txt
  tail -2 $OUT/smoke_$TAG.txt
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?"
  timeout 600 python bench.py --config uniform --no-cpu-baseline --no-suite > $OUT/bench100k_$TAG.json 2>> $OUT/bench_$TAG.err
  timeout 600 python bench.py --config dense --no-cpu-baseline --no-suite > $OUT/benchdense_$TAG.json 2>> $OUT/bench_$TAG.err
  timeout 600 python bench.py --impl reference > $OUT/ref_$TAG.json 2>> $OUT/bench_$TAG.err; echo "ref exit $?"
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1"
  T="python bench.py --steps 10 --warmup 3 --only-timed"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $T > $OUT/ncu_launch_$TAG.txt 2>&1
  echo "ncu launches exit $?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches100k_$TAG.csv $T --config uniform > /dev/null 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_step|k_lp3" -s 16 -c 2 -o $OUT/prof_kstep_$TAG $B > $OUT/ncu_full_$TAG.txt 2>&1
  echo "ncu full exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_step" -s 16 -c 1 -o $OUT/prof_kstep100k_$TAG $B --config uniform > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"k_scatter|k_scan" -s 16 -c 2 -o $OUT/prof_bin_$TAG $T > /dev/null 2>&1
  echo "ncu rest exit $?"
fi
# compute-sanitizer is closed on the GPU pool since r02b1: only on request (what = sanitize)
if [[ $WHAT == sanitize ]]; then
  bash scripts/sanitize.sh $TAG > $OUT/sanitize_${TAG}_summary.txt 2>&1; cat $OUT/sanitize_${TAG}_summary.txt
fi
