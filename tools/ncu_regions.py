#!/usr/bin/env python
"""Per-region totals (instructions, stall samples, shared wavefronts, global tag requests) of
the SASS source page of an ncu report, regions split at the hot loop's landmarks (H4 LDS.128
gathers, neighbour loads, H7 butterfly).  python tools/ncu_regions.py REPORT [--dump N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]; d = rows[2:]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iWS, iT = h.index("L1 Wavefronts Shared"), h.index("L1 Tag Requests Global")
E = [int(r[iE]) for r in d]; W = [int(r[iW]) for r in d]
tot, totw = sum(E), sum(W)
print(f"total instructions {tot/1e6:.1f}M  stall samples {totw}")
h4 = [i for i, r in enumerate(d) if "LDS.128" in r[iS] and E[i] > 1e6]
bf = [i for i, r in enumerate(d) if "SHFL.BFLY" in r[iS] and E[i] > 1e4]
marks = sorted(set([0, h4[0] - 60 if h4 else 0, (h4[-1] + 30) if h4 else 0, bf[0] if bf else len(d), len(d)]))
names = ["pre", "H1-H4", "neighbour", "H7-post"]
for (a, b), n in zip(zip(marks[:-1], marks[1:]), names):
    s = sum(E[a:b]); w = sum(W[a:b]); sw = sum(int(r[iWS]) for r in d[a:b]); g = sum(int(r[iT]) for r in d[a:b])
    print(f"{n:10s} [{a},{b}) inst {s/1e6:7.1f}M ({100*s/tot:4.1f}%) stall {100*w/max(totw,1):4.1f}% smem_wf {sw/1e6:6.1f}M gtag {g/1e6:5.1f}M")
if "--dump" in sys.argv:
    thr = float(sys.argv[sys.argv.index("--dump") + 1])
    for i, r in enumerate(d):
        if E[i] >= thr or W[i] > totw * 0.004:
            print(i, f"{E[i]/1e6:8.2f}", f"{W[i]:6d}", f"{r[iWS]:>9s}", f"{r[iT]:>8s}", r[iS][:70])
