q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.4f %.4f' % (d['value'], d['roofline']['kernel_ms'], d['ms_per_step']))"; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_fit_gpu.py -x -q 2>&1 | tail -3
for c in c4 c3; do
 for v in "GCPB_HOT_T=0" "GCPB_HOT_T=256" "GCPB_HOT_T=64" "GCPB_HOT_T=256 GCPB_LIB=paper_1906_01687_b200/libgcpb_hot4.so"; do
  echo "$c $v: $(env $v python bench.py --config $c --steps 30 --no-e2e --no-cpu 2>/dev/null | q)"
 done
done
for v in "GCPB_HOT_T=0" "GCPB_HOT_T=256" "GCPB_HOT_T=64"; do
  echo "c5 $v: $(env $v python bench.py --config c5 --steps 10 --no-e2e --no-cpu 2>/dev/null | q)"
done
