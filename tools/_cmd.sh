set -u
mkdir -p gpurun_out/r01_box
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_box/build.log 2>&1 || { tail -20 gpurun_out/r01_box/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "complex or restricted" 2>&1 | tail -3
for b in 0 4 8 12; do
  timeout 900 python bench.py --config C2 --box $b --steps 30 --warmup 3 > gpurun_out/r01_box/bench_c2_box$b.json 2> gpurun_out/r01_box/bench_c2_box$b.err; echo "box $b rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r01_box/bench_c2_box$b.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['setup']['R'], d.get('box'))"
done
