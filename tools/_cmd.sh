#!/bin/bash
# scratch gpurun command: A/B + parity of one variant
ROUNDS=2 STEPS=20 bash tools/abi.sh s4d C3 base se se_t3 se_hv se_lc all4
RSDOCK_LIB=$PWD/build/variants/librsdock_all4.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4d/tests_all4.log 2>&1; echo "tests all4: $(tail -1 gpurun_out/s4d/tests_all4.log)"
