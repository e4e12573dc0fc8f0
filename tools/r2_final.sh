#!/bin/bash
# Final round-2 evidence (on the GPU box; outputs in gpurun_out/final):
#   bench lines of every config (+ the C5 reference arm when REF=1), ncu launch
#   lists, and --set full captures of the step's kernels, summarised.
O=gpurun_out/final; mkdir -p $O
STEPK='regex:fused_grad|adam|order_|hot_fold|pick_compact|zero_|ag_pack|small_steps'
for c in ${CONFIGS:-c5 c2 c3 c4 c1}; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err || tail -3 $O/bench_$c.err
  B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c"
  ncu --metrics gpu__time_duration.sum --clock-control none -k "$STEPK" -c 300 --csv \
      --log-file $O/r02_${c}_launches.csv $B > $O/ncu_l_$c.log 2>&1
  case $c in
    c5) caps="fused_grad:6:fused_picks fused_grad:7:fused_list adam:3:adam order_count:3:order_count order_scatter:3:order_scatter";;
    c3) caps="fused_grad:6:fused_picks fused_grad:7:fused_zeros zero_cand:9:zero_cand adam:3:adam";;
    c4) caps="fused_grad:3:fused adam:3:adam";;
    c2) caps="fused_grad:3:fused adam:3:adam";;
    c1) caps="small_steps:1:small";;
  esac
  first=1
  for cap in $caps; do
    k=${cap%%:*}; r=${cap#*:}; s=${r%%:*}; n=${r##*:}
    ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f \
        -o $O/prof_${c}_$n $B > $O/ncu_f_${c}_$n.log 2>&1
    if [ -f $O/prof_${c}_$n.ncu-rep ]; then
      L=""; [ $first = 1 ] && L="--launches $O/r02_${c}_launches.csv"; first=0
      python tools/ncu_summary.py $L --rep $O/prof_${c}_$n.ncu-rep --out $O/r02_${c}_$n.md \
          --title "Round 2 / $c $n" > /dev/null
    fi
    rm -f $O/prof_${c}_$n.ncu-rep
  done
  echo "$c: $(python -c "import json;d=json.loads(open('$O/bench_$c.json').read().splitlines()[-1]);print('%.4f ms/step, %.3g samples/s, kernel %.4f ms' % (d['ms_per_step'], d['value'], d['roofline']['kernel_ms']))")"
done
if [ -n "$REF" ]; then
  python bench.py --config c5 --impl reference > $O/bench_c5_ref.json 2> $O/bench_c5_ref.err
fi
ls $O | wc -l
