#!/bin/bash
# One gpurun call: build, GPU tests, smoke, bench, ncu launch list + full capture of k_step.
# Usage (here): gpurun --timeout 2400 -- 'bash scripts/gpu_check.sh [tag] [what]'
TAG=${1:-r01}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.txt 2>&1 || { echo BUILD FAILED; cat $OUT/build_$TAG.txt; exit 1; }
if [[ $WHAT == all || $WHAT == test || $WHAT == quick ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > $OUT/pytest_gpu_$TAG.txt 2>&1
  echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.txt
  tail -25 $OUT/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.txt
  tail -3 $OUT/smoke_$TAG.txt
fi
if [[ $WHAT == all || $WHAT == bench || $WHAT == quick ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench exit $?"
  cat $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
  timeout 600 python bench.py --config uniform --no-cpu-baseline --no-suite > $OUT/bench100k_$TAG.json 2>> $OUT/bench_$TAG.err
  cat $OUT/bench100k_$TAG.json
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1 > $OUT/ncu_bench_$TAG.txt 2>&1
  echo "ncu launches exit $?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step -s 8 -c 1 -o $OUT/prof_kstep_$TAG \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1 > $OUT/ncu_full_$TAG.txt 2>&1
  echo "ncu full exit $?"
fi
if [[ $WHAT == ncufull || $WHAT == quick ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_step|k_lp3" -s 16 -c 2 -o $OUT/prof_kstep_$TAG \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1 > $OUT/ncu_full_$TAG.txt 2>&1
  echo "ncu full exit $?"
  timeout 600 ncu --set full --clock-control none -k regex:"k_scatter|k_scan" -s 4 -c 2 -o $OUT/prof_bin_$TAG \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-suite --e2e-steps 1 > $OUT/ncu_bin_$TAG.txt 2>&1
  echo "ncu bin exit $?"
fi
