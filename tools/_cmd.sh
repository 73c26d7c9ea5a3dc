set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -k "forces" 2>&1 | tail -2
for v in ppw1 ppw8; do RSDOCK_LIB=build/variants/librsdock_$v.so timeout 600 python -m pytest tests -m gpu -x -q -k "forces_c3_contiguous or window_and_fallback" 2>&1 | tail -1; done
bash tools/ablate.sh r01_fw4 C3 "f:--forces ppw1:--forces ppw2:--forces ppw8:--forces" 0
