set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "host or c1_all or repeated" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-microbench > gpurun_out/bench_e2e2.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/bench_e2e2.json'));print(round(d['ms_per_step'],4), '%.4g'%d['e2e']['value'])"; done
