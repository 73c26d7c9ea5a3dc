#!/bin/bash
# Bench lines for every config and mode (one JSON line each) -> gpurun_out/$TAG/*.json, plus
# ncu --set full captures of the scoring kernel on the L2-path configs (C4, one C5 point).
#   bash tools/bench_all.sh TAG [NCU=1]
set -u
TAG=${1:-all}; NCU=${2:-1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$?"; }
run C1 --config C1 --steps 20 --warmup 3 --no-cpu-baseline
run C2 --config C2 --steps 20 --warmup 3 --no-cpu-baseline
run C3 --config C3 --steps 30 --warmup 3
run C3_f32 --config C3 --f32 --steps 30 --warmup 3 --no-cpu-baseline
run C3_forces --config C3 --forces --steps 10 --warmup 3 --no-cpu-baseline --no-e2e
run C3_ppiem360 --config C3 --ppiem 360 --steps 5
run C2_box8 --config C2 --box 8 --steps 20 --warmup 3 --no-cpu-baseline
run C2_box4 --config C2 --box 4 --steps 20 --warmup 3 --no-cpu-baseline
run C4 --config C4 --steps 5 --warmup 3 --no-cpu-baseline
run C4_complex --config C4 --complex --steps 5 --warmup 3 --no-cpu-baseline
for R in 8 16 32; do for S in 1 2 3; do
  run C5_R${R}_s${S} --config C5 --c5-rank $R --c5-sigma-mult $S --steps 10 --warmup 3 --no-cpu-baseline
done; done
python tools/bench_table.py $OUT > $OUT/table.md; cat $OUT/table.md
if [ "$NCU" = "1" ]; then
  for spec in "C4:--config C4" "C5_R16_s1:--config C5 --c5-rank 16 --c5-sigma-mult 1"; do
    name=${spec%%:*}; a=${spec#*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 \
      -o $OUT/ncu_$name -f python bench.py $a --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench \
      > $OUT/ncu_$name.log 2>&1
    echo "ncu $name rc=$?"
  done
fi
