#!/usr/bin/env python
"""List local-memory spills (LDL/STL) of a score_kernel instantiation relative to its hot loop
(the H4 LDS.128 gathers ... the H7 butterfly).  python tools/sass_spills.py OBJ MANGLED_SUBSTR"""
import re, subprocess, sys
obj, sub = sys.argv[1], sys.argv[2]
names = subprocess.run(["cuobjdump", "-symbols", obj], capture_output=True, text=True).stdout
fn = [w for w in re.findall(r"\S+", names) if sub in w and w.startswith("_Z")][0]
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
lines = [l for l in sass.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
h4 = [i for i, l in enumerate(lines) if "LDS.128" in l]
bf = [i for i, l in enumerate(lines) if "SHFL.BFLY" in l]
print(fn, "instructions", len(lines), "LDS.128 at", h4[:1], h4[-1:], "BFLY", bf[-3:])
for i, l in enumerate(lines):
    if "LDL" in l or "STL" in l:
        print(i, l.strip()[:80])
