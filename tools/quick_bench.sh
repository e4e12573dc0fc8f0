# quick A/B of the default build: tools/quick_bench.sh <configs...>
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g samples/s  kernel %.4f ms  step %.4f ms' % (d['value'], d['roofline']['kernel_ms'], d['ms_per_step']))"; }
for c in "$@"; do
  echo "$c: $(python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
done
