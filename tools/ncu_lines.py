#!/usr/bin/env python
"""Attribute an ncu SASS source page (instructions executed, stall samples) to CUDA source
lines, using the line table of the locally built cubin (nvdisasm -g).  The box builds the same
sources with the same nvcc, so SASS offsets match.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTR [OBJ] [--top N]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_table(obj, kernel_sub):
    d = tempfile.mkdtemp()
    subprocess.check_call(["/usr/local/cuda/bin/cuobjdump", "-xelf", "all", obj], cwd=d,
                          stdout=subprocess.DEVNULL)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-g", "-c", os.path.join(d, cub)],
                         capture_output=True, text=True).stdout
    table, cur, inside, line = {}, None, False, None
    for s in dis.splitlines():
        if s.startswith("//----") and ".text." in s:
            inside = kernel_sub in s
            continue
        if not inside:
            continue
        m = re.search(r'//## File ".*/([^/"]+)", line (\d+)', s)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", s)
        if m:
            table[int(m.group(1), 16)] = (line, m.group(2).strip())
    return table


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    obj = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else \
        os.path.join(ROOT, "build", "obj", "score_kernel.cu.o")
    top = 40
    if "--top" in sys.argv:
        top = int(sys.argv[sys.argv.index("--top") + 1])
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    base = int(data[0][ia], 16)
    tab = line_table(obj, ksub)
    agg = collections.defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    for r in data:
        off = int(r[ia], 16) - base
        ln = tab.get(off, ("?", ""))[0]
        i, s = int(r[ie] or 0), int(r[iss] or 0)
        agg[ln][0] += i
        agg[ln][1] += s
        tot_i += i
        tot_s += s
    src = {}
    p = os.path.join(ROOT, "paper_2510_26611_b200", "csrc", "score_kernel.cu")
    for k, t in enumerate(open(p).read().splitlines(), 1):
        src[f"score_kernel.cu:{k}"] = t.strip()
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for ln, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100*s/tot_s:5.1f}% samp {100*i/tot_i:5.1f}% inst  {ln:24s} {src.get(ln, '')[:80]}")


if __name__ == "__main__":
    main()
