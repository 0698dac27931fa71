"""Write the SASS of a kernel's hot loop (the smallest loop holding at least `min_hits` instructions whose opcode starts with
`op`) with an opcode histogram on top -- the excerpts under profiles/ come from here.

    python tools/sass_excerpt.py <lib.so> <mangled-name substring> <opcode prefix> <min_hits> <out.txt>
"""
import collections, re, subprocess, sys
lib, pat, op, min_hits, out = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5]
names = subprocess.run(["cuobjdump", "-elf", lib], capture_output=True, text=True).stdout
funcs = sorted(set(re.findall(r"_ZN3wsb\w+", names)))
cands = [f for f in funcs if pat in f]
assert cands, f"no kernel matches {pat}"
fn = cands[0]
txt = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for l in txt.split("\n"):
    m = re.search(r"/\*([0-9a-f]{4,5})\*/\s+((?:@!?U?P\d\s+)?)([A-Z0-9_.]+)(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), re.sub(r";\s*/\*.*", ";", l).strip()))
loops = []
for a, o, l in ins:
    if o.startswith("BRA"):
        t = re.search(r"BRA\S*\s+(?:\S+,\s*)?0x([0-9a-f]+)", l)
        if t and int(t.group(1), 16) < a:
            loops.append((int(t.group(1), 16), a))
best = None
for lo, hi in loops:
    body = [x for x in ins if lo <= x[0] <= hi]
    if sum(1 for x in body if x[1].startswith(op)) >= min_hits and (best is None or len(body) < len(best)):
        best = body
assert best, "no loop qualifies"
hist = collections.Counter(o.split(".")[0] for _, o, _ in best).most_common()
with open(out, "w") as fh:
    fh.write(f"# {fn}\n# hot loop: {len(best)} instructions, {hex(best[0][0])}..{hex(best[-1][0])} (cuobjdump -sass of {lib.split('/')[-1]})\n")
    fh.write("# " + ", ".join(f"{k} {v}" for k, v in hist) + "\n")
    for _, _, l in best:
        fh.write(l + "\n")
print(out, len(best), hist[:8])
