"""Per-kernel SASS opcode counts of libtim.so that prove the Blackwell paths (tcgen05 MMA,
TMEM loads, TMA tensor / bulk copies, reductions): cuobjdump -sass, static instruction counts.

    python scripts/sass_summary.py [path/to/libtim.so] > profiles/sass_summary.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_14220_b200/libtim.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
demangle = {}
names = sorted(set(re.findall(r"Function : (\S+)", sass)))
if names:
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    demangle = dict(zip(names, out))
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "REDG", "MUFU.EX2", "MUFU.LG2",
        "DADD", "DMUL", "FFMA2", "FADD2", "FMUL2", "ELECT", "SYNCS"]
counts = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = demangle.get(m.group(1), m.group(1))
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Za-z0-9_.]*)", line)
    if m:
        op = m.group(1)
        for k in KEYS:
            if op.startswith(k):
                counts[cur][op] += 1
print(f"# static SASS opcode counts per kernel of {lib} (cuobjdump -sass, sm_100a); round-2 build")
for fn, c in counts.items():
    if not c:
        continue
    print(f"\n{fn}")
    for op, n in sorted(c.items()):
        print(f"  {op:45s} {n}")
