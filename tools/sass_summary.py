"""SASS instruction summary of the built library objects (cuobjdump -sass, sm_100a) ->
profiles/<round>/sass_summary.csv.  argv: output path."""
import collections
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCIMMA", "UTCHMMA", "LDTM", "STTM", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "UBLKPF", "IMMA", "HMMA",
       "SYNCS", "UCGABAR", "ATOMS", "REDUX", "SHFL", "LDS", "STS", "LDG", "STG", "LDGSTS", "MUFU", "DFMA", "DMUL", "DADD"]
rows = []
for obj in sorted(glob.glob(os.path.join(ROOT, "paper_2511_10645_b200", "_objs", "*.o"))):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn, cnt = None, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if fn:
                rows.append((fn, cnt))
            fn, cnt = m.group(1), collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if fn and m:
            cnt["_total"] += 1
            cnt[m.group(2)] += 1
    if fn:
        rows.append((fn, cnt))
with open(sys.argv[1], "w") as f:
    f.write("# SASS instruction summary of the shipped libparo.so objects (cuobjdump -sass, sm_100a; tools/sass_summary.py)\n")
    f.write("# per kernel: total SASS instructions and the counts of the mnemonics that prove the hardware paths\n")
    f.write("# (UTCIMMA/UTCHMMA = tcgen05.mma i8/f16, LDTM/STTM = tcgen05.ld/st, UTMALDG/UTMASTG = TMA tensor load/store,\n")
    f.write("#  UBLKCP = cp.async.bulk, IMMA/HMMA = warp-level mma.sync, SYNCS = mbarrier ops, UCGABAR = cluster barrier)\n")
    f.write("kernel," + "total," + ",".join(OPS) + "\n")
    for fn, c in rows:
        f.write(f"\"{fn}\",{c['_total']}," + ",".join(str(c[o]) for o in OPS) + "\n")
print(len(rows), "kernels")
