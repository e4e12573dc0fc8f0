# A/B of an engine environment switch: tools/env_ab.sh "<VAR=val ...>" <configs...>
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g samples/s  kernel %.4f ms  step %.4f ms' % (d['value'], d['roofline']['kernel_ms'], d['ms_per_step']))"; }
V=$1; shift
for c in "$@"; do
  for rep in 1 2; do
    echo "$c base: $(python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
    echo "$c $V: $(env $V python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
  done
done
