#!/bin/bash
# Time librsdock variants (build/variants/librsdock_<name>.so) on one config, then profile the
# default build with ncu.  Usage: bash tools/ablate.sh TAG CONFIG "name1 name2 ..." [NCU=1]
set -u
TAG=$1; CFG=$2; NAMES=$3; NCU=${4:-1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build_library()" > $OUT/build.log 2>&1
for v in base $NAMES; do
  if [ "$v" = "base" ]; then LIBP=""; else LIBP=build/variants/librsdock_$v.so; fi
  RSDOCK_LIB=$LIBP timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print(round(d['ms_per_step'],4),'ms')" 2>/dev/null)"
done
if [ "$NCU" = "1" ]; then
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench"
  timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
    -o $OUT/score_full -f $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu_rc=$?"
fi
