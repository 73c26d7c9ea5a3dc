set -u
mkdir -p gpurun_out/r01_final7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_final7/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r01_final7/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r01_final7/gpu_tests.log
tail -3 gpurun_out/r01_final7/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
