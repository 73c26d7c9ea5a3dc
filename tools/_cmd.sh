set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ablate.sh r01_v29 C3 "f32:--f32" 0
