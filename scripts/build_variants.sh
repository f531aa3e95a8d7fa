#!/bin/bash
# usage: scripts/build_variants.sh name:"-DFLAG=1 ..." ...  -> vlibs/lib_<name>.so (parallel nvcc builds)
cd "$(dirname "$0")/.." || exit 1
mkdir -p vlibs
FL=$(python -c "from paper_1908_10107_b200 import build; print(' '.join(build._flags()))")
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  ( /usr/local/cuda/bin/nvcc $FL $f -I include -o vlibs/lib_$n.so paper_1908_10107_b200/csrc/orca.cu > /tmp/b_$n.log 2>&1 \
    && echo "ok $n" || { echo "FAIL $n"; grep -m5 error /tmp/b_$n.log; } ) &
done
wait
