"""Registers / stack / shared / local bytes per kernel of a built .so (cuobjdump --dump-resource-usage).

    python tools/resusage.py [lib.so] [substring ...]
"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1703_00687_b200/libradsort.so"
pats = sys.argv[2:]
out = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
names = subprocess.run(["c++filt"], input=out, capture_output=True, text=True).stdout.splitlines()
fn = None
for line in names:
    m = re.match(r"\s*Function (.*):$", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and fn:
        short = re.sub(r"\(.*", "", fn)
        if all(p in short for p in pats):
            print(f"{short:70s} REG={m.group(1):>3} STACK={m.group(2):>4} SHARED={m.group(3):>6} LOCAL={m.group(4)}")
        fn = None
