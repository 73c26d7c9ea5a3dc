set -u
mkdir -p gpurun_out/r01_final6
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_final6/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r01_final6/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r01_final6/gpu_tests.log
tail -3 gpurun_out/r01_final6/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r01_final6/bench.json 2> gpurun_out/r01_final6/bench.err; echo bench_rc=$?
python -c "import json;d=json.loads(open('gpurun_out/r01_final6/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['setup_seconds'], d['clocks'])"
