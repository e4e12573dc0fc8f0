#!/bin/bash
# A/B of the batched-pass fused kernel (GCPB_PB) on C5 and C2.
mkdir -p gpurun_out/r2
for c in ${CONFIGS:-c5 c2}; do
for pb in ${PBS:-1 2 4}; do
  GCPB_PB=$pb python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2/pb_${c}_$pb.json 2> gpurun_out/r2/pb_${c}_$pb.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/r2/pb_${c}_$pb.json").read().splitlines()[-1])
print("$c pb=$pb", "ms/step %.4f"%d["ms_per_step"], "kernel %.4f"%d["roofline"]["kernel_ms"], "frac %.3f"%d["roofline"]["frac"], "launches/step", d.get("gpu_launches_per_step"))
PY
done; done
