set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for b in 1024 512 256; do RS_STREAM_BIG=$b timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/big=$b /"; done
for b in 1024 512 256; do RS_STREAM_BIG=$b timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/big=$b /"; done
