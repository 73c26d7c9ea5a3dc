set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "f32" 2>&1 | tail -2
mkdir -p gpurun_out/all3; timeout 900 python bench.py --config C4 --f32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/all3/C4_f32.json 2> gpurun_out/all3/C4_f32.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/all3/C4_f32.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('l2_literal_frac'), d['e2e']['value'])"
