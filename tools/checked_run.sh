#!/bin/bash
# The bounds-checked library (-DRS_DEVICE_CHECKS, device asserts on every indexed access of the
# kernels) under the whole GPU suite, the small per-path cases and full-size C3/C4/C5 launches.
#   bash tools/checked_run.sh TAG
set -u
TAG=${1:-checked}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python tools/build_variants.py checked=-DRS_DEVICE_CHECKS > $OUT/build.log 2>&1
export RSDOCK_LIB=$PWD/build/variants/librsdock_checked.so
timeout 1800 python -m pytest tests -m gpu -q > $OUT/gpu_tests_checked.log 2>&1; echo "tests rc=$? $(tail -1 $OUT/gpu_tests_checked.log)"
timeout 900 python tools/sanitize_cases.py > $OUT/cases_checked.log 2>&1; echo "cases rc=$?"; cat $OUT/cases_checked.log
for a in "--config C3" "--config C4" "--config C5 --c5-rank 32 --c5-sigma-mult 3" "--config C3 --f32" "--config C3 --forces"; do
  timeout 900 python bench.py $a --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-microbench > $OUT/bench.log 2>&1
  echo "bench $a rc=$? $(tail -c 200 $OUT/bench.log | tr '\n' ' ' | cut -c1-160)"
done
