set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "streamed or host_pointers" 2>&1 | tail -2
mkdir -p gpurun_out/all2
for c in C2 C3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/all2/$c.json 2>/dev/null; echo "$c rc=$?"; done
timeout 600 python bench.py --config C2 --box 4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/all2/C2_box4.json 2>/dev/null
timeout 600 python bench.py --config C2 --box 8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/all2/C2_box8.json 2>/dev/null
for f in C2 C3 C2_box4 C2_box8; do python -c "import json;d=json.loads(open('gpurun_out/all2/$f.json').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step'],4), '%.3g' % d['e2e']['value'])"; done
