"""Top SASS instructions by stall samples from an .ncu-rep (source page), for the first kernel matching a pattern."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = rows[1]
def col(name):
    for i, h in enumerate(hdr):
        if h.strip() == name: return i
    return None
ci = {n: col(n) for n in ("Address", "Source", "# Samples", "Warp Stall Sampling (All Samples)", "Instructions Executed", "Warp Stall Sampling (Not-issued Samples)")}
print({k: v for k, v in ci.items()})
data = []
for r in rows[2:]:
    try:
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    except Exception:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
print("total samples", tot, "instructions", len(data))
# print in address order with cumulative share for the hottest contiguous region
for s, r in data:
    if s * 400 >= tot:   # >= 0.25 % of samples
        st = {h[6:]: int(v) for h, v in zip(hdr, r) if h.startswith("stall_") and "(" not in h and v not in ("", "0")}
        top2 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100.0 * s / tot:5.2f}%  {r[ci['Address']][-5:]}  {r[ci['Source']].strip()[:70]:70s} exec={r[ci['Instructions Executed']]} {top2}")
