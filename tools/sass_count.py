#!/usr/bin/env python
"""Static SASS instruction counts of score_kernel<R, NA> (a quick proxy for instruction-count
changes before spending GPU time).  python tools/sass_count.py [R] [NA] [-DDEF ...]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "16"
NA = sys.argv[2] if len(sys.argv) > 2 else "2"
defs = [a for a in sys.argv[3:] if a.startswith("-D")]
d = tempfile.mkdtemp()
cub = os.path.join(d, "k.cubin")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                       "-std=c++17", "-fmad=false", "-cubin", *defs, "-o", cub,
                       os.path.join(ROOT, "paper_2510_26611_b200", "csrc", "score_kernel.cu")])
dis = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
want = f"score_kernelILi{R}ELi{NA}E"
inside, ops = False, collections.Counter()
for line in dis.splitlines():
    if "Function :" in line:
        inside = want in line
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if inside and m:
        ops[m.group(1)] += 1
print(sum(ops.values()), "instructions;", ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))
