set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "device_core" 2>&1 | tail -3
RS_SETUP_TIMING=1 timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench 2>&1 >/tmp/c4.json | grep "rs setup"
python -c "import json;d=json.loads(open('/tmp/c4.json').read().strip().splitlines()[-1]);print(d['setup_seconds'], d['ms_per_step'])"
