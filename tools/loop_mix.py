"""Instruction mix of the largest loop (backward-branch range) of a SASS function dump (cuobjdump -sass -fun)."""
import collections
import re
import sys

L = open(sys.argv[1]).read().split("\n")
ins = []
for l in L:
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9.]+)([^;]*);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
loops = []
for a, op, args in ins:
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", args)
        if t and int(t.group(1), 16) < a:
            loops.append((int(t.group(1), 16), a))
lo, hi = max(loops, key=lambda x: x[1] - x[0])
c = collections.Counter(op for a, op, _ in ins if lo <= a <= hi)
print(f"loop {hex(lo)}..{hex(hi)}: {sum(c.values())} instructions")
print(sorted(c.items(), key=lambda x: -x[1])[:24])
