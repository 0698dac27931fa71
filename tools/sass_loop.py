"""Summarise the SASS of one kernel: opcode histogram of the whole function and of its largest loop body."""
import collections, re, subprocess, sys
lib, pat = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else None
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)[1:]
f = [x for x in funcs if pat in x.split("\n")[0]][0]
ins = []
for l in f.split("\n"):
    m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+((?:@!?U?P\d\s+)?)([A-Z0-9_.]+)(.*?);", l)
    if m: ins.append((int(m.group(1), 16), m.group(3), l.strip()[:100]))
print(f.split("\n")[0], len(ins), "instructions")
loops = []
for a, o, l in ins:
    if o.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", l.split("BRA")[1])
        if t and int(t.group(1), 16) < a: loops.append((int(t.group(1), 16), a))
print("loops:", [(hex(a), hex(b), (b - a) // 16) for a, b in loops])
if lo is None:
    lo, hi = max(loops, key=lambda ab: ab[1] - ab[0])
body = [x for x in ins if lo <= x[0] <= hi]
print(f"body {hex(lo)}..{hex(hi)}: {len(body)} instr")
print(collections.Counter(o.split(".")[0] for _, o, _ in body).most_common(40))
if "-v" in sys.argv:
    for _, _, l in body: print(l)
