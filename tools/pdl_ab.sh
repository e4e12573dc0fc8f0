# A/B of programmatic dependent launch: tools/pdl_ab.sh <alt lib> <configs...>
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g samples/s  kernel %.4f ms  step %.4f ms' % (d['value'], d['roofline']['kernel_ms'], d['ms_per_step']))"; }
ALT=$1; shift
for c in "$@"; do
  for rep in 1 2; do
    echo "$c PDL=0: $(GCPB_PDL=0 python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
    echo "$c PDL=1: $(GCPB_PDL=1 python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
    echo "$c PDL=1 $(basename $ALT): $(GCPB_LIB=$ALT GCPB_PDL=1 python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
  done
done
