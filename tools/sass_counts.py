"""Per-kernel SASS instruction counts of the built library (the evidence that the hot kernels
use the FP64 tensor pipe, bulk copies, distributed shared memory, mbarriers and clusters):
DMMA, DFMA, UBLKCP (cp.async.bulk), STAS (st.async to DSMEM), SYNCS (mbarrier), UCGABAR
(cluster barrier), LDTM/UTCMMA (tcgen05; expected 0: no FP64 kind). Writes
profiles/r2_sass_counts.txt.

    python tools/sass_counts.py [lib]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1508_02977_b200",
                                                         "libflowfem_b200.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["DMMA", "DFMA", "UBLKCP", "STAS", "SYNCS", "UCGABAR", "LDTM", "UTCMMA", "UTMALDG"]
counts = collections.OrderedDict()
fn = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    if fn is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for k in keys:
            if op.startswith(k):
                counts[fn][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"ffb::\(anonymous namespace\)::", "", d)
    return d.split("(")[0]


lines = ["SASS instruction counts per kernel of " + os.path.relpath(lib, ROOT),
         "(cuobjdump -sass; tools/sass_counts.py)", "",
         f"{'kernel':60s} " + " ".join(f"{k:>8s}" for k in keys)]
for f, c in counts.items():
    if not any(c.values()):
        continue
    lines.append(f"{short(f)[:60]:60s} " + " ".join(f"{c[k]:8d}" for k in keys))
out = os.path.join(ROOT, "profiles", "r2_sass_counts.txt")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
