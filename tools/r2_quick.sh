#!/bin/bash
# Quick GPU-side check of a C5 change: selected tests, the bench line, the ncu
# launch list of the step kernels.   bash tools/r2_quick.sh tag [pytest -k expr]
tag=${1:-q}
O=gpurun_out/r2
mkdir -p $O
if [ -n "$2" ]; then
  python -m pytest tests -m gpu -x -q -k "$2" > $O/t_$tag.log 2>&1; tail -3 $O/t_$tag.log
fi
c=${CONFIG:-c5}
python bench.py --config $c --no-cpu --no-e2e > $O/b_${tag}_$c.json 2> $O/b_${tag}_$c.err || tail -5 $O/b_${tag}_$c.err
python - <<PY
import json
d=json.loads(open("$O/b_${tag}_$c.json").read().splitlines()[-1])
print("$c", "ms/step %.4f"%d["ms_per_step"], "kernel %.4f"%d["roofline"]["kernel_ms"], "frac %.3f"%d["roofline"]["frac"], "%.3g samples/s"%d["value"])
PY
if [ -z "$NO_NCU" ]; then
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --config $c"
STEPK='regex:fused_grad|adam|order_|hot_fold|pick_compact|zero_|ag_pack'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$STEPK" -c 200 --csv \
    --log-file $O/${tag}_${c}_launches.csv $B > $O/ncu_l_$c.log 2>&1
python tools/ncu_summary.py --launches $O/${tag}_${c}_launches.csv --out $O/${tag}_${c}_launches.md --title "$tag $c" | head -20
fi
