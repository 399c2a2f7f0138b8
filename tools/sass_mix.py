"""Instruction mix of the hot loop of k_accum: called fe_mul2 body and the loop body (SASS text on stdin/file)."""
import re
import sys

lines = open(sys.argv[1]).read().split("\n")


def addr(l):
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    return int(m.group(1), 16) if m else None


calls = [l for l in lines if "CALL.REL" in l]
tgt = int(re.search(r"CALL.REL.NOINC (0x[0-9a-f]+)", calls[-1]).group(1), 16)


def mix(lo, hi):
    c = {}
    for l in lines:
        a = addr(l)
        if a is None or a < lo or a >= hi:
            continue
        m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9.]+)", l)
        if m:
            c[m.group(2)] = c.get(m.group(2), 0) + 1
    return c


def cyc(c):
    fma = sum((4 if ("WIDE" in k or ".HI" in k) else 2) * v for k, v in c.items() if k.startswith(("IMAD", "HFMA2")))
    alu = sum(2 * v for k, v in c.items() if k.split(".")[0] in ("IADD3", "LOP3", "SEL", "SHF", "ISETP", "MOV", "LEA",
                                                                  "VIADD", "PRMT", "PLOP3"))
    return fma, alu


end = max(addr(l) or 0 for l in lines)
m2 = mix(tgt, end + 16)
loop_lo = min(addr(l) for l in calls)
body = mix(loop_lo - 0x600, max(addr(l) for l in calls) + 0x400)
for name, c in (("fe_mul2 body", m2), ("loop body around calls", body)):
    f, a = cyc(c)
    print(f"{name}: {sum(c.values())} instr, FMA-pipe cycles/warp {f}, ALU cycles/warp {a}")
    print("   ", sorted(c.items(), key=lambda x: -x[1])[:14])
