set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for m in 0 1; do for fd in 64 16; do RS_E2E_MODE=$m RS_E2E_FIRST_DIV=$fd timeout 600 python tools/e2e_probe.py 2>&1 | tail -5 | sed "s/^/m=$m fd=$fd /"; done; done
