#!/bin/bash
# A/B of environment switches on one config: tools/env_ab2.sh c5 "GCPB_L2LINE=0" "GCPB_L2LINE=1" ...
mkdir -p gpurun_out/r2
c=$1; shift
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2/ab_${c}_$i.json 2> gpurun_out/r2/ab_${c}_$i.err || tail -5 gpurun_out/r2/ab_${c}_$i.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/r2/ab_${c}_$i.json").read().splitlines()[-1])
print("$c [$envs]", "ms/step %.4f"%d["ms_per_step"], "kernel %.4f"%d["roofline"]["kernel_ms"], "frac %.3f"%d["roofline"]["frac"])
PY
done
