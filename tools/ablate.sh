#!/bin/bash
# Time librsdock variants on one config, then (optionally) profile the default build with ncu.
#   bash tools/ablate.sh TAG CONFIG "v1 v2:--nbr-cell+0.5 ..." [NCU=1]
# A variant "name" loads build/variants/librsdock_<name>.so when it exists (else the default
# library); "name:ARGS" adds bench.py arguments ('+' stands for a space).
set -u
TAG=$1; CFG=$2; NAMES=$3; NCU=${4:-1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build_library()" > $OUT/build.log 2>&1
for spec in base $NAMES; do
  v=${spec%%:*}; extra=""; LIBP=""
  if [[ "$spec" == *:* ]]; then extra=${spec#*:}; extra=${extra//+/ }; fi
  if [ -f build/variants/librsdock_$v.so ]; then LIBP=build/variants/librsdock_$v.so; fi
  v=$(echo "$spec" | tr ':+' '__')
  RSDOCK_LIB=$LIBP timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench $extra > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  echo "$v rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_$v.json'));print(round(d['ms_per_step'],4),'ms', d['setup'].get('nbr_entries'))" 2>/dev/null)"
done
if [ "$NCU" = "1" ]; then
  CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench"
  timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
    -o $OUT/score_full -f $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu_rc=$?"
fi
