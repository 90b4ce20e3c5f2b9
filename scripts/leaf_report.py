"""Summarise exp_leaf.sh output: A/B bits, panel timings, per-opcode executed
instructions per warp-step and top stall sites of the ncu capture."""
import csv, json, sys
from collections import Counter
T = sys.argv[1]
O = "gpurun_out"
print(open(f"{O}/{T}_leaf_ab.log").read())
for l in open(f"{O}/{T}_panel_probe.log"):
    if not l.startswith("{"):
        print(l.strip()); continue
    d = json.loads(l); k = d["kinds"]
    print(d["m"], d["S"], d["ms"], d["us_per_col"], " ".join(f"{n}={v['ms']:.2f}/{v['launches']}" for n, v in k.items()))
rows = list(csv.reader(open(f"{O}/{T}_leaf_src.csv")))
hdr = rows[1]; data = rows[2:]
i_e = hdr.index("Instructions Executed"); i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source")
steps = Counter(float(r[i_e] or 0) for r in data if r[i_e]).most_common(1)[0][0]
tot = sum(float(r[i_e] or 0) for r in data); ts = sum(float(r[i_s] or 0) for r in data)
print(f"instr per warp-step {tot/steps:.0f}  stall samples {ts:.0f}")
c = Counter(); s = Counter()
for r in data:
    op = [o for o in r[i_src].split() if not o.startswith("@")]
    if op:
        c[op[0]] += float(r[i_e] or 0); s[op[0]] += float(r[i_s] or 0)
for k, v in c.most_common(12):
    print(f"  {k:30s} {v/steps:7.1f}/step  stall {s[k]:.0f}")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:6]:
    print(f"  {float(r[i_s]):5.0f} exec={r[i_e]} {r[i_src][:80]}")
