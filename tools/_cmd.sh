#!/bin/bash
# scratch gpurun command: A/B + parity of the base library
TESTS=1 ROUNDS=2 STEPS=20 bash tools/abi.sh s4k C3 base old tc384 tc512 td6 td10
