"""Summarise an ncu report: key SOL metrics, stall reasons and per-opcode instruction counts."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
npts = float(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out)); hdr = next(r)
keep = ['Duration', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Executed Ipc Active',
        'Issue Slots Busy', 'Registers Per Thread', 'Achieved Occupancy', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Executed Instructions', 'Dynamic Shared Memory Per Block', 'Memory Throughput', 'Eligible Warps Per Scheduler',
        'Warp Cycles Per Issued Instruction', 'Theoretical Occupancy', 'Block Limit Registers', 'Block Limit Shared Mem']
for row in r:
    d = dict(zip(hdr, row))
    if d.get('Metric Name') in keep:
        print(d.get('Metric Name', '')[:45].ljust(45), d.get('Metric Unit', '')[:12].ljust(12), d.get('Metric Value', ''))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
tot = sum(float(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in data)
agg = {h: sum(float(r[idx[h]] or 0) for r in data) for h in hdr if h.startswith('stall_') and 'Not Issued' not in h}
print('stalls:', ', '.join(f"{k[6:]}={v/tot:.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
c = collections.Counter()
for r in data:
    src = r[idx['Source']].strip()
    if src.startswith('@'): src = src.split(None, 1)[1]
    op = (src.split()[0] if src else '?').split('.')[0]
    c[op] += float(r[idx['Instructions Executed']] or 0)
lds = [r for r in data if 'LDS' in r[idx['Source']]]
w = sum(float(r[idx['L1 Wavefronts Shared']] or 0) for r in lds); wi = sum(float(r[idx['L1 Wavefronts Shared Ideal']] or 0) for r in lds)
print('LDS wavefronts/ideal: %.2f' % (w / max(wi, 1)))
scale = 32 / npts if npts else 1
print('instr per point:' if npts else 'instr:', ' '.join(f"{op}={v*scale:.1f}" for op, v in c.most_common(16)), ' total=%.1f' % (sum(c.values()) * scale))
top = sorted(data, key=lambda r: -float(r[idx['Warp Stall Sampling (All Samples)']] or 0))[:12]
for r in top:
    print('   ', r[idx['Source']][:56].ljust(56), r[idx['Warp Stall Sampling (All Samples)']], r[idx['Instructions Executed']])
