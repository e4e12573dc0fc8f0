#!/bin/bash
# compute-sanitizer passes over the small GPU parity tests (SURVEY.md §5's
# planned race/memory check).  Logs in gpurun_out/sanitize/; the summaries are
# copied to profiles/.   bash tools/sanitize.sh   (on the GPU box)
O=gpurun_out/sanitize; mkdir -p $O
CS="compute-sanitizer --target-processes all --error-exitcode 86 --print-limit 20"
MEM_TESTS="tests/test_parity_gpu.py tests/test_hot_rows_gpu.py tests/test_interleaved_gpu.py tests/test_wide_keys_gpu.py tests/test_multirank_gpu.py"
RACE_TESTS="tests/test_parity_gpu.py tests/test_fit_gpu.py tests/test_interleaved_gpu.py"
run() {  # name, tool args, tests, pytest -k
  local name=$1; shift; local tool=$1; shift; local tests=$1; shift; local k=$1
  local t0=$(date +%s)
  timeout ${SAN_TIMEOUT:-1500} $CS $tool python -m pytest $tests -m gpu -x -q -k "$k" -p no:cacheprovider \
      > $O/$name.log 2>&1
  local rc=$?
  echo "$name rc=$rc $(($(date +%s)-t0))s: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $O/$name.log | sort | uniq -c | tr '\n' ';') $(grep -E ' passed| failed| error' $O/$name.log | tail -1)" | tee -a $O/summary.txt
}
: > $O/summary.txt
run memcheck "--tool memcheck" "$MEM_TESTS" "not fullsize and not peer_adam"
run memcheck_peer "--tool memcheck" "tests/test_multirank_gpu.py" "peer_adam and f32"
run racecheck "--tool racecheck" "$RACE_TESTS" "small or graph or stratified or steps or step_host"
run initcheck "--tool initcheck" "tests/test_parity_gpu.py tests/test_interleaved_gpu.py" "sampler_and_gradient_fp32 or random_sparse or interleaved_steps or ordered"
run synccheck "--tool synccheck" "tests/test_fit_gpu.py tests/test_parity_gpu.py" "small or stratified"
cat $O/summary.txt
