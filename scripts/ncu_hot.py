"""Top SASS instructions by stall samples from an ncu source-page CSV
(--page source --csv --print-source sass), with their dominant stalls."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (KeyError, ValueError):
        return 0.0


tot = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
by = collections.Counter()
for r in data:
    by[r[ix["Source"]].strip().split(" ")[0].split(".")[0] if not r[ix["Source"]].strip().startswith("@")
       else r[ix["Source"]].strip().split()[1].split(".")[0]] += num(r, "Warp Stall Sampling (All Samples)")
print("stall samples by opcode:", ", ".join(f"{k}={v / tot:.1%}" for k, v in by.most_common(12)))
stall_tot = collections.Counter()
for r in data:
    for s in stalls:
        stall_tot[s] += num(r, s)
print("stall reasons:", ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in stall_tot.most_common(10)))
top = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    st = sorted(((num(r, s), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{r[ix['Address']]:>8s} {num(r, 'Warp Stall Sampling (All Samples)') / tot:6.2%} "
          f"{r[ix['Source']].strip()[:60]:60s} " + " ".join(f"{n}={v / max(num(r, 'Warp Stall Sampling (All Samples)'), 1):.0%}" for v, n in st))
