#!/bin/bash
# A/B of engine builds on one config: tools/lib_ab.sh c5 libgcpb.so libgcpb_pb2.so ...
mkdir -p gpurun_out/r2
c=$1; shift
for lib in "$@"; do
  GCPB_LIB=$PWD/paper_1906_01687_b200/$lib python bench.py --config $c --no-cpu --no-e2e > gpurun_out/r2/lib_${c}_$lib.json 2> gpurun_out/r2/lib_${c}_$lib.err || tail -5 gpurun_out/r2/lib_${c}_$lib.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/r2/lib_${c}_$lib.json").read().splitlines()[-1])
print("$c [$lib]", "ms/step %.4f"%d["ms_per_step"], "kernel %.4f"%d["roofline"]["kernel_ms"], "frac %.3f"%d["roofline"]["frac"])
PY
done
