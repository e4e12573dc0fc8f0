#!/bin/bash
# The engine's own memory check (compute-sanitizer is closed on this GPU pool):
#   1. builds a second library with -DGCPB_CHECKED (device-side index
#      assertions at the hot path's gather / scatter sites) next to the product
#      one:  paper_1906_01687_b200/libgcpb_checked.so
#   2. (on the GPU box) runs the GPU tests against it with guarded allocations
#      (GCPB_GUARD=1: every device buffer between two verified 4 KB bands);
#      tests/conftest.py fails a test whose run trips an assertion or corrupts a
#      band.
#   bash tools/checked_build.sh build      # here (no GPU needed)
#   bash tools/checked_build.sh run [-k expr]   # on the GPU box
set -e
cd "$(dirname "$0")/.."
LIB=$PWD/paper_1906_01687_b200/libgcpb_checked.so
case "$1" in
  build)
    GCPB_LIB=$LIB GCPB_OBJDIR=_build_checked GCPB_NVFLAGS="-DGCPB_CHECKED" \
      python -c "from paper_1906_01687_b200 import build as B; B.build_engine()"
    ;;
  run)
    shift
    O=gpurun_out/checked; mkdir -p $O
    GCPB_LIB=$LIB GCPB_GUARD=1 python -m pytest tests -m gpu -q -p no:cacheprovider "$@" \
      > $O/checked_tests.log 2>&1 || true
    tail -5 $O/checked_tests.log
    ;;
  *) echo "usage: $0 build | run [pytest args]"; exit 2;;
esac
