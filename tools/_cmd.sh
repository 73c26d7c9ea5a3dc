#!/bin/bash
# scratch gpurun command: A/B + parity of one variant
ROUNDS=2 STEPS=20 bash tools/abi.sh s4g C3 base to ut4 ut5 ut0 ws13 ws18
RSDOCK_LIB=$PWD/build/variants/librsdock_to.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4g/tests_to.log 2>&1; echo "tests to: $(tail -1 gpurun_out/s4g/tests_to.log)"
