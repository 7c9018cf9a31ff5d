#!/bin/bash
# summarise the .ncu-rep files of gpurun_out on the box, then drop them
for r in gpurun_out/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r $b.sum.txt > /dev/null 2>&1
  python tools/ncu_src_top.py $r 60 > $b.src.txt 2>&1
  ncu -i $r --page details > $b.details.txt 2>&1
  rm -f $r
done
ls gpurun_out
