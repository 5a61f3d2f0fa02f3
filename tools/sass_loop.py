#!/usr/bin/env python
"""Instruction mix of the hottest loop (largest backward branch) of one SASS
function: tools/sass_loop.py <cuobjdump -sass -fun NAME output>."""
import re
import sys
from collections import Counter

body = []
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        body.append((int(m.group(1), 16), m.group(2).strip()))
back = []
for a, ins in body:
    t = re.search(r"BRA\s+`?\(?.*?0x([0-9a-f]+)", ins)
    if "BRA" in ins and t and int(t.group(1), 16) < a:
        back.append((a, int(t.group(1), 16)))
hi, lo = max(back, key=lambda x: x[0] - x[1])
loop = [ins for a, ins in body if lo <= a <= hi]
c = Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0] for i in loop)
print(f"loop {hex(lo)}..{hex(hi)}: {len(loop)} instructions")
for k, v in c.most_common():
    print(f"{v:5d} {k}")
