#!/bin/bash
# Round-2 evidence for profiles/ (run on the GPU box; outputs in gpurun_out/r2):
#   1. the default bench line (C5, cpu_baseline + e2e) and the reference arm
#   2. ncu launch list of the same command's step kernels
#   3. one --set full capture each of the fused kernel, Adam and the ordering
#      kernels, summarised by tools/ncu_summary.py (the .ncu-rep files stay on
#      the box: too large to bring back)
#   bash tools/r2_profile.sh [tag] [config]
tag=${1:-r02}
c=${2:-c5}
O=gpurun_out/r2
mkdir -p $O
python bench.py --config $c > $O/bench_${tag}_$c.json 2> $O/bench_${tag}_$c.err || tail -5 $O/bench_${tag}_$c.err
if [ -z "$NO_REF" ]; then
  python bench.py --config $c --impl reference > $O/bench_${tag}_${c}_ref.json 2> $O/bench_${tag}_${c}_ref.err || tail -5 $O/bench_${tag}_${c}_ref.err
fi
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c"
STEPK='regex:fused_grad|adam|order_|hot_fold|pick_compact|zero_|ag_pack'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$STEPK" -c 200 --csv \
    --log-file $O/${tag}_${c}_launches.csv $B > $O/ncu_l_$c.log 2>&1
for k in fused_grad adam order_count order_scatter; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -f \
      -o $O/prof_${c}_$k $B > $O/ncu_f_${c}_$k.log 2>&1
  if [ -f $O/prof_${c}_$k.ncu-rep ]; then
    L=""; [ "$k" = "fused_grad" ] && L="--launches $O/${tag}_${c}_launches.csv"
    python tools/ncu_summary.py $L --rep $O/prof_${c}_$k.ncu-rep --out $O/${tag}_${c}_$k.md \
        --title "Round 2 / $c $k kernel" > /dev/null
  fi
done
rm -f $O/*.ncu-rep
ls $O | grep $tag
