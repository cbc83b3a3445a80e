"""Shared-memory wavefronts per SASS instruction from an ncu source-page CSV:
actual vs ideal, largest first."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def num(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (KeyError, ValueError):
        return 0.0


tot = sum(num(r, "L1 Wavefronts Shared") for r in data)
ideal = sum(num(r, "L1 Wavefronts Shared Ideal") for r in data)
print(f"shared wavefronts {tot:.3e}, ideal {ideal:.3e} ({tot / max(ideal, 1):.2f}x)")
top = sorted(data, key=lambda r: -num(r, "L1 Wavefronts Shared"))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for r in top:
    w, wi, n = num(r, "L1 Wavefronts Shared"), num(r, "L1 Wavefronts Shared Ideal"), num(r, "Instructions Executed")
    print(f"{r[ix['Address']]:>8s} {w / tot:6.2%} waves/inst {w / max(n, 1):5.2f} ideal {wi / max(n, 1):5.2f}  "
          f"{r[ix['Source']].strip()[:70]}")
