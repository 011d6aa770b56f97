"""List backward-branch loops of a SASS dump with their instruction mix.

usage: cuobjdump -sass lib.so | awk '/Function : NAME/{f=1} ...' > f.sass
       python scripts/sass_loops.py f.sass
"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, text) in enumerate(ins):
    m = re.search(r"BRA(?:\.[A-Z.]+)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", text)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and tgt in addr_idx and "ANY" not in text:
            loops.append((addr_idx[tgt], i))
for s, e in sorted(loops, key=lambda x: x[1] - x[0], reverse=True)[:4]:
    body = [t for _, t in ins[s:e + 1]]
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in body)
    print(f"loop 0x{ins[s][0]:x}-0x{ins[e][0]:x}: {len(body)} instructions")
    print("   ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(40)))
