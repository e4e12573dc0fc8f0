#!/bin/bash
# A/B bench of two engine builds: tools/ab.sh <libA> <libB> <configs...>
A=$1; B=$2; shift 2
for c in "$@"; do
  for rep in 1 2; do
    for L in $A $B; do
      v=$(GCPB_LIB=$L python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.4f' % (d['value'], d['roofline']['kernel_ms']))")
      echo "$c $(basename $L) $v"
    done
  done
done
