"""Opcode histogram of one kernel's SASS: python tools/sass_ops.py <obj> <name-substring>"""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = Counter()
    for line in b.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    print(name, sum(ops.values()))
    for k, v in ops.most_common(25):
        print(f"  {k:10s} {v}")
