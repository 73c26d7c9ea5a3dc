#!/bin/bash
# One GPU-box pass: parity tests, a bench line, the ncu launch list and one full ncu capture
# of the scoring kernel.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_round.sh TAG [CONFIG] [TESTS=1] [NCU=1]
set -u
TAG=${1:-run}; CFG=${2:-C3}; TESTS=${3:-1}; NCU=${4:-1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail -20 $OUT/build.log; exit 1; }
if [ "$TESTS" = "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/gpu_tests.log 2>&1; echo "tests_rc=$?" >> $OUT/gpu_tests.log
  tail -3 $OUT/gpu_tests.log
fi
timeout 600 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; echo "bench_rc=$?"
tail -c 400 $OUT/bench.json
if [ "$NCU" = "1" ]; then
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench"
  timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
    -o $OUT/score_full -f $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu_rc=$?"
fi
ls -la $OUT
