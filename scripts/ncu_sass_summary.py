"""Summarise an ncu --page source --print-source sass CSV: instructions and
stall samples per region (regions split at BAR.SYNC), top stall reasons."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def num(r, k):
    try: return float(r[ix[k]] or 0)
    except: return 0.0
region, regs = 0, collections.OrderedDict()
tot_inst = sum(num(r, "Instructions Executed") for r in data)
tot_samp = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
for r in data:
    src = r[ix["Source"]]
    d = regs.setdefault(region, {"inst": 0, "samp": 0, "first": r[ix["Address"]], "st": collections.Counter(), "ops": collections.Counter()})
    d["inst"] += num(r, "Instructions Executed"); d["samp"] += num(r, "Warp Stall Sampling (All Samples)")
    for s in stalls: d["st"][s] += num(r, s)
    op = src.strip().split()[0] if src.strip() else ""
    if op.startswith("@"): op = src.strip().split()[1]
    d["ops"][op.split(".")[0]] += num(r, "Instructions Executed")
    if "BAR.SYNC" in src: region += 1
print(f"total warp-instructions {tot_inst:.3e}, stall samples {tot_samp:.0f}")
for k, d in regs.items():
    if d["inst"] < 0.005 * tot_inst and d["samp"] < 0.005 * tot_samp: continue
    top = ", ".join(f"{s[6:]}={v/max(d['samp'],1):.0%}" for s, v in d["st"].most_common(4))
    ops = ", ".join(f"{o}={v/d['inst']:.0%}" for o, v in d["ops"].most_common(6))
    print(f"region {k} @{d['first']}: inst {d['inst']/tot_inst:.1%} samples {d['samp']/tot_samp:.1%} | {top}\n      ops: {ops}")
