"""Per-kernel key metrics of a multi-kernel ncu report."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out)); hdr = next(r)
keep = ['Duration', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Executed Ipc Active',
        'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy', 'Dynamic Shared Memory Per Block',
        'Block Size', 'Grid Size', 'Eligible Warps Per Scheduler', 'Executed Instructions', 'L2 Hit Rate']
per = collections.OrderedDict()
for row in r:
    d = dict(zip(hdr, row))
    key = (d.get('ID'), d.get('Kernel Name', '')[:70])
    if d.get('Metric Name') in keep:
        per.setdefault(key, {})[d['Metric Name']] = d['Metric Value'] + ' ' + d.get('Metric Unit', '')
for (i, name), m in per.items():
    print(i, name)
    print('   ', '; '.join(f"{k}={v}" for k, v in m.items()))
