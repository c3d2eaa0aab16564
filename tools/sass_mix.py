"""Instruction mix per kernel from `cuobjdump -sass` (static counts)."""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1506_04383_b200/libmm_b200.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "k_repulse"
s = subprocess.check_output(["cuobjdump", "-sass", lib]).decode()
for f in re.split(r"\n\s*Function : ", s):
    name = f.split("\n")[0]
    if pat not in name:
        continue
    ops = []
    for l in f.split("\n"):
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
        if m:
            ops.append(m.group(2))
    c = Counter(ops)
    keys = ["MUFU", "FADD2", "FFMA2", "FMUL2", "FMUL", "FFMA", "FADD", "MOV", "IMAD", "LDS", "ISETP", "FSEL", "FMNMX"]
    print(re.sub(r"_ZN2mm\w+?_(k_\w+?)E.*", r"\1", name)[:70], {k: c[k] for k in keys if c[k]})
