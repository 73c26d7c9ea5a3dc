set -u
mkdir -p gpurun_out/r01_final4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_final4/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r01_final4/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/r01_final4/gpu_tests.log
tail -3 gpurun_out/r01_final4/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/bench_all.sh
CMD="python bench.py --config C3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-microbench"
timeout 300 $CMD > gpurun_out/r01_final4/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r01_final4/launches.csv $CMD > gpurun_out/r01_final4/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 -o gpurun_out/r01_final4/score_full -f $CMD > gpurun_out/r01_final4/ncu_full.log 2>&1
echo "ncu_rc=$?"
