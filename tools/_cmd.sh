#!/bin/bash
# scratch gpurun command: A/B + parity of one variant
ROUNDS=2 STEPS=20 bash tools/abi.sh s4q C3 base uf uf58 uf78
RSDOCK_LIB=$PWD/build/variants/librsdock_uf.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4q/tests_uf.log 2>&1; echo "tests uf: $(tail -1 gpurun_out/s4q/tests_uf.log)"
for c in "C4:--config C4 --steps 5" "C5:--config C5 --c5-rank 16 --c5-sigma-mult 1 --steps 10" "C2:--config C2 --steps 20"; do n=${c%%:*}; a=${c#*:};
 for L in base uf; do if [ $L = base ]; then LIB=$PWD/paper_2510_26611_b200/librsdock.so; else LIB=$PWD/build/variants/librsdock_$L.so; fi
  RSDOCK_LIB=$LIB timeout 600 python bench.py $a --warmup 3 --no-cpu-baseline --no-e2e --no-microbench > gpurun_out/s4q/${n}_$L.json 2>/dev/null; echo "$n $L $(python -c "import json; d=json.loads(open('gpurun_out/s4q/${n}_$L.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))")"; done; done
