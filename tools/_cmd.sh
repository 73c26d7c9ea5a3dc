#!/bin/bash
# scratch gpurun command: spot bench of several configs
OUT=gpurun_out/s4o; mkdir -p $OUT
run() { name=$1; shift; timeout 900 python bench.py "$@" > $OUT/$name.json 2> $OUT/$name.err; echo "$name rc=$? $(python -c "import json; d=json.loads(open('$OUT/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), d['roofline']['frac'], (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"; }
run C3a --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench
run C5_R16_s1 --config C5 --c5-rank 16 --c5-sigma-mult 1 --steps 10 --warmup 3 --no-cpu-baseline
run C5_R8_s3 --config C5 --c5-rank 8 --c5-sigma-mult 3 --steps 10 --warmup 3 --no-cpu-baseline
run C2 --config C2 --steps 20 --warmup 3 --no-cpu-baseline
run C4 --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
run C3b --config C3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench
