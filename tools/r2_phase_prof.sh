#!/bin/bash
# ncu --set full of the two fused launches of a C5 step (pick half, ordered half).
O=gpurun_out/r2; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config c5"
for ph in picks:6 list:7; do
  n=${ph%%:*}; s=${ph##*:}
  ncu --set full --import-source on --clock-control none -k regex:fused_grad -s $s -c 1 -f \
      -o $O/prof_c5_$n $B > $O/ncu_f_c5_$n.log 2>&1
  python tools/ncu_summary.py --rep $O/prof_c5_$n.ncu-rep --out $O/${1:-r02}_c5_fused_$n.md \
      --title "Round 2 / C5 fused kernel, $n half" > /dev/null
done
rm -f $O/*.ncu-rep
