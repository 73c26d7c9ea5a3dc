set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 128 64 32 16 8; do RS_STREAM_FIRST_DIV=$d timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/div=$d /"; done
