# ncu evidence for profiles/: launch list (one metric, every kernel) and one
# --set full capture of the fused kernel per config (+ the zero sampler for C3).
#   bash tools/profile_round.sh c3 c4 ...   (on the GPU box; outputs in gpurun_out/)
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
for c in "$@"; do
  if [ "$c" != "c5" ]; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_$c.csv $B --config $c > gpurun_out/ncu_l_$c.log 2>&1
  fi
  ncu --set full --import-source on --clock-control none -k regex:fused -s 3 -c 1 -f \
      -o gpurun_out/prof_$c $B --config $c > gpurun_out/ncu_f_$c.log 2>&1
  if [ "$c" = "c3" ]; then
    ncu --set full --import-source on --clock-control none -k regex:zero_cand -s 3 -c 1 -f \
        -o gpurun_out/prof_c3_zero $B --config c3 > gpurun_out/ncu_z_c3.log 2>&1
  fi
  echo "$c done: $(ls gpurun_out | grep -c $c)"
done
# summaries on the box (the .ncu-rep files are too large to bring back)
for c in "$@"; do
  L=""; [ -f gpurun_out/launches_$c.csv ] && L="--launches gpurun_out/launches_$c.csv"
  python tools/ncu_summary.py $L --rep gpurun_out/prof_$c.ncu-rep --out gpurun_out/r01_${c}_hot.md \
      --title "Round 1 / $c fused kernel with hot rows" > /dev/null
  [ -f gpurun_out/prof_${c}_zero.ncu-rep ] && python tools/ncu_summary.py \
      --rep gpurun_out/prof_${c}_zero.ncu-rep --out gpurun_out/r01_${c}_zero.md \
      --title "Round 1 / $c zero-candidate kernel (Bloom prefilter)" > /dev/null
done
rm -f gpurun_out/*.ncu-rep
