set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "c5" --durations=3 2>&1 | tail -8
