set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash tools/ablate.sh r01_v24 C3 "" 0
