#!/bin/bash
# usage: scripts/lp3_modes_summary.sh <configs> <modes> [lib ...]  -- compact lp3_modes_probe output per library
cfgs=$1; modes=$2; shift 2
libs=("$@"); [ ${#libs[@]} -eq 0 ] && libs=("")
for lib in "${libs[@]}"; do
  echo "== ${lib:-default}"
  ORCA_LIB=$lib python scripts/lp3_modes_probe.py "$cfgs" "$modes" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    n,_,j=l.partition(' ')
    try: d=json.loads(j)
    except Exception: print(l.strip()); continue
    print(n, {m:(v['same_as_first'], round(v['step_ms'],4), round(v['kstep_lp3_ms'],4)) for m,v in d.items()})
"
done
