#!/bin/bash
# scratch gpurun command: A/B + parity of one variant
ROUNDS=2 STEPS=20 bash tools/abi.sh s4l C3 base sn4 sn5 sn6 sn7 sn6td10 sn6td12
RSDOCK_LIB=$PWD/build/variants/librsdock_sn6.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4l/tests_sn6.log 2>&1; echo "tests sn6: $(tail -1 gpurun_out/s4l/tests_sn6.log)"
