#!/bin/bash
# Bench lines for every config and mode (one JSON line each) -> gpurun_out/all/*.json
set -u
OUT=gpurun_out/all; mkdir -p $OUT
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
python tools/bench_table.py $OUT > $OUT/table.md; cat $OUT/table.md
