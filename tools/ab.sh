#!/bin/bash
# A/B of library variants on one GPU box: for each build/variants/librsdock_NAME.so (and the
# default library as "base"): a C3 bench line and (NCU=1) one ncu --set full capture.
#   bash tools/ab.sh TAG CONFIG NCU NAME...
set -u
TAG=$1; CFG=$2; NCU=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
for NAME in base "$@"; do
  if [ "$NAME" = base ]; then LIB=$PWD/paper_2510_26611_b200/librsdock.so; else LIB=$PWD/build/variants/librsdock_$NAME.so; fi
  if [ "${TESTS:-0}" = "1" ]; then
    RSDOCK_LIB=$LIB timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests_$NAME.log 2>&1; echo "$NAME tests: $(tail -1 $OUT/tests_$NAME.log)"
  fi
  CMD="python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench"
  RSDOCK_LIB=$LIB timeout 600 $CMD > $OUT/bench_$NAME.json 2> $OUT/bench_$NAME.err
  echo "$NAME rc=$? $(python -c "import json,sys; d=json.loads(open('$OUT/bench_$NAME.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])" 2>&1)"
  if [ "$NCU" = "1" ]; then
    RSDOCK_LIB=$LIB timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
      -o $OUT/full_$NAME -f python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench > $OUT/ncu_$NAME.log 2>&1
    echo "ncu $NAME rc=$?"
  fi
done
