set -u
mkdir -p gpurun_out/r01_boxb
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r01_boxb/build.log 2>&1 || { tail -20 gpurun_out/r01_boxb/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "restricted or complex" 2>&1 | tail -2
for b in 4 8 12; do for sc in b c; do
  timeout 900 python bench.py --config C2 --box $b --box-scheme $sc --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r01_boxb/C2_box${b}${sc}.json 2> gpurun_out/r01_boxb/C2_box${b}${sc}.err; echo "box $b $sc rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r01_boxb/C2_box${b}${sc}.json').read().strip().splitlines()[-1]);b=d['box'];print(round(d['ms_per_step'],4), b['scheme'], round(b['restrict_seconds'],2), b['box_cp_core_err'], d['setup']['tucker_r'])"
done; done
