"""Static FP64 instruction counts (DADD / DMUL / DFMA) per generated tile pass (developer tool, CPU).

    HHLSV_JIT_DUMP=dir <run a host-only schedule dump>; python scripts/sass_fp64.py dir
Prints, per pass (identified by its tile bits), the per-thread FP64 instruction counts of the cubin."""
import glob
import os
import re
import subprocess
import sys

d = sys.argv[1]
for cu in sorted(glob.glob(os.path.join(d, "*.cu"))):
    src = open(cu).read()
    m = re.search(r"auto tile_base = \[\]\(u64 t\) \{ u64 b = t;(.*?)return b;", src)
    bits = re.findall(r"insz\(b, (\d+)\)", m.group(1)) if m else []
    sass = subprocess.run(["cuobjdump", "-sass", cu[:-3] + ".cubin"], capture_output=True, text=True).stdout
    ops = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+([A-Z0-9_]+)", sass, re.M)
    c = {k: ops.count(k) for k in ("DADD", "DMUL", "DFMA", "LDG", "LDS", "STS")}
    print(f"bits {','.join(bits):40s} fp64 {c['DADD'] + c['DMUL'] + c['DFMA']:5d}  " + " ".join(f"{k}={v}" for k, v in c.items()))
