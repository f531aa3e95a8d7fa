#!/bin/bash
# Copy one scripts/gpu_check_r02.sh run's judged artifacts from gpurun_out/ into profiles/r02/
# (bench lines, reference arm, tests, smoke, launch lists, ncu details / hot lines / regions).
# Usage: scripts/save_run.sh <tag>
T=$1; G=gpurun_out; P=profiles/r02
cd "$(dirname "$0")/.." || exit 1
for f in bench_$T.json bench100k_$T.json benchdense_$T.json ref_$T.json pytest_gpu_$T.txt smoke_$T.txt \
         launches_$T.csv launches100k_$T.csv strips_$T.txt; do
  [ -f $G/$f ] && cp $G/$f $P/
done
ncu -i $G/prof_kstep_$T.ncu-rep --page details --csv > $P/ncu_kstep_lp3_details_$T.csv 2>/dev/null
ncu -i $G/prof_kstep100k_$T.ncu-rep --page details --csv > $P/ncu_kstep100k_details_$T.csv 2>/dev/null
ncu -i $G/prof_bin_$T.ncu-rep --page details --csv > $P/ncu_bin_details_$T.csv 2>/dev/null
ncu -i $G/prof_kstep_$T.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_step > /tmp/page_$T.csv 2>/dev/null
python3 scripts/ncu_lines.py /tmp/page_$T.csv > $P/ncu_kstep_hotlines_$T.txt 2>&1
python3 scripts/ncu_regions.py /tmp/page_$T.csv > $P/ncu_kstep_regions_$T.txt 2>&1
echo saved $T
