"""Compare two bench --profile-out JSON files kernel by kernel (avg us per launch)."""
import json
import sys

a, b = (json.load(open(p)) for p in sys.argv[1:3])
ka = {k["tag"]: k for k in a["kernels"]}
kb = {k["tag"]: k for k in b["kernels"]}
print(f"step {a['step_ms']:.2f} -> {b['step_ms']:.2f} ms; matvec {a['matvec_ms']:.3f} -> {b['matvec_ms']:.3f} ms")
for t in sorted(set(ka) | set(kb), key=lambda t: -(kb.get(t) or ka.get(t))["total_ms"]):
    x, y = ka.get(t), kb.get(t)
    fa = f"{x['avg_ms'] * 1e3:8.1f}" if x else "       -"
    fb = f"{y['avg_ms'] * 1e3:8.1f}" if y else "       -"
    print(f"{t:28s} {fa} -> {fb} us")
