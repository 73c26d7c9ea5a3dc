set -u
mkdir -p gpurun_out/r01_final5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_final5/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r01_final5/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r01_final5/gpu_tests.log
tail -3 gpurun_out/r01_final5/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r01_final5/bench.json 2> gpurun_out/r01_final5/bench.err; echo bench_rc=$?
tail -c 1500 gpurun_out/r01_final5/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01_final5/bench_ref.json 2>&1; echo ref_rc=$?
tail -c 300 gpurun_out/r01_final5/bench_ref.json
