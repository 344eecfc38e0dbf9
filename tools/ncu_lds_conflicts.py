"""Per-instruction shared-memory conflicts of one ncu report: python tools/ncu_lds_conflicts.py REP [N]
Lists the LDS/STS instructions with the largest excess wavefronts (actual - ideal)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[idx[k]] or 0)
    except Exception: return 0.0
rs = []
for r in data:
    src = r[idx['Source']]
    if 'LDS' in src or 'STS' in src:
        w, wi = f(r, 'L1 Wavefronts Shared'), f(r, 'L1 Wavefronts Shared Ideal')
        rs.append((w - wi, w, wi, r[idx['Address']] if 'Address' in idx else '', src.strip()[:70]))
tot = sum(x[1] for x in rs); toti = sum(x[2] for x in rs)
print(f"shared wavefronts {tot:.0f} ideal {toti:.0f} ratio {tot / max(toti, 1):.2f}")
for e, w, wi, a, s in sorted(rs, reverse=True)[:N]:
    print(f"{e:12.0f} {w:12.0f} {wi:12.0f}  {a}  {s}")
