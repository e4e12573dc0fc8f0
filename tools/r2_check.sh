#!/bin/bash
# GPU-side check used during round 2: gpu tests + bench lines of each config.
mkdir -p gpurun_out/r2
tag=${1:-x}
python -m pytest tests -m gpu -x -q > gpurun_out/r2/gputest_$tag.log 2>&1; tail -3 gpurun_out/r2/gputest_$tag.log
for c in ${CONFIGS:-c5}; do
  python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2/b_${tag}_$c.json 2> gpurun_out/r2/b_${tag}_$c.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/r2/b_${tag}_$c.json").read().splitlines()[-1])
print("$c", "ms/step %.4f"%d["ms_per_step"], "kernel %.4f"%d["roofline"]["kernel_ms"], "frac %.3f"%d["roofline"]["frac"], "%.3g samples/s"%d["value"])
PY
done
