set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ablate.sh r01_v10 C3 "c05:--nbr-cell+0.5 c2:--nbr-cell+2.0 c025:--nbr-cell+0.25" 0
