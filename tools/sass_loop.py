"""Count SASS instructions in the hot loop(s) of each step kernel: for every
backward branch, the instructions between its target and itself, by opcode."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1711_04471_b200/libsw2d.so"
pat = sys.argv[2] if len(sys.argv) > 2 else "step_fused"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", f):
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    print(name[-60:], "total", len(ins))
    for addr, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < addr:
                body = [o for a, o, _ in ins if int(t.group(1), 16) <= a <= addr]
                c = collections.Counter(o.split(".")[0] for o in body)
                print(f"  loop {int(t.group(1),16):#x}-{addr:#x}: {len(body)} instrs;",
                      ", ".join(f"{k}:{v}" for k, v in c.most_common(14)))

# --dump: print the largest loop's instructions (opcode + operands) of the
# first matching function to stdout after the summary
if "--dump" in sys.argv:
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if pat not in name:
            continue
        ins = []
        for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", f):
            ins.append((int(m.group(1), 16), (m.group(2) or "").strip(), m.group(3), m.group(4)))
        best = None
        for addr, _, op, rest in ins:
            if op.startswith("BRA"):
                t = re.search(r"0x([0-9a-f]+)", rest)
                if t and int(t.group(1), 16) < addr:
                    lo = int(t.group(1), 16)
                    n = sum(1 for a, *_ in ins if lo <= a <= addr)
                    if best is None or n > best[2]:
                        best = (lo, addr, n)
        if "--range" in sys.argv:   # --range <lo> <hi> (hex): that loop instead
            i = sys.argv.index("--range")
            best = (int(sys.argv[i + 1], 16), int(sys.argv[i + 2], 16), 0)
        for a, pr, op, rest in ins:
            if best and best[0] <= a <= best[1]:
                print(f"{a:#07x} {pr:6s} {op} {rest.strip()}")
        break
