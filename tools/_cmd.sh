set -u
mkdir -p gpurun_out/r01_cx
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_cx/build.log 2>&1 || { tail -20 gpurun_out/r01_cx/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "complex" 2>&1 | tail -3
timeout 1200 python bench.py --config C4 --complex --steps 10 --warmup 3 > gpurun_out/r01_cx/bench_c4_complex.json 2> gpurun_out/r01_cx/bench_c4_complex.err; echo rc=$?
tail -c 600 gpurun_out/r01_cx/bench_c4_complex.json
