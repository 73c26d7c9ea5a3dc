#!/bin/bash
# ptxas register / spill report per score_kernel instantiation: tools/ptxas_report.sh [-DRS_THREADS=512 ...]
cd "$(dirname "$0")/../paper_2510_26611_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false "$@" -Xptxas -v \
  -Xcompiler -fPIC -c score_kernel.cu -o /tmp/ptxas_report.o 2>&1 | python3 -c '
import re,sys
cur=None
for l in sys.stdin:
    m=re.search(r"Compiling entry function .*score_kernelILi(\d+)ELb(\d)ELb(\d)E",l)
    if m: cur="R=%s f32=%s win=%s"%m.groups(); continue
    m=re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads",l)
    if m and cur: sp=m.groups(); continue
    m=re.search(r"Used (\d+) registers",l)
    if m and cur: print(cur, "regs", m.group(1), "stack/spill st/ld", sp); cur=None
'
