#!/bin/bash
# Interleaved A/B of library variants on one GPU box (ROUNDS passes over the variants, so clock
# drift hits every variant alike): bench line per variant and pass, optional GPU suite first.
#   TESTS=1 ROUNDS=2 bash tools/abi.sh TAG CONFIG NAME...   (NAME = base or build/variants/librsdock_NAME.so)
set -u
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
python -c "from paper_2510_26611_b200 import build_ext; build_ext.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [ "${TESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests: $(tail -1 $OUT/tests.log)"
fi
for r in $(seq 1 ${ROUNDS:-2}); do
  for NAME in "$@"; do
    if [ "$NAME" = base ]; then LIB=$PWD/paper_2510_26611_b200/librsdock.so; else LIB=$PWD/build/variants/librsdock_$NAME.so; fi
    RSDOCK_LIB=$LIB timeout 600 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e --no-microbench \
      > $OUT/bench_${NAME}_$r.json 2> $OUT/bench_${NAME}_$r.err
    echo "$NAME pass $r rc=$? $(python -c "import json; d=json.loads(open('$OUT/bench_${NAME}_$r.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1)"
  done
done
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
    -o $OUT/full_base -f python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench > $OUT/ncu_base.log 2>&1
  echo "ncu rc=$?"
fi
