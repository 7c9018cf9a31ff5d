#!/bin/bash
# Round-end measurement pass (run under gpurun): measure_round.sh, then the
# .ncu-rep files summarised on the box (raw reports exceed the copy-back cap).
set -u
TAG=${TAG:-r02b} bash tools/measure_round.sh
for r in gpurun_out/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r $b.sum.txt > /dev/null 2>&1
  python tools/ncu_src_top.py $r 40 > $b.src.txt 2>&1
  rm -f $r
done
ls gpurun_out
