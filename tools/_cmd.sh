set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "max_grid or large_ligand" 2>&1 | tail -15
