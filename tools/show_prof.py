import json, sys
d = json.load(open(sys.argv[1]))
print('step ms %.2f  matvec ms %.3f' % (d['step_ms'], d['matvec_ms']))
for k in d['kernels']:
    print(f"{k['tag']:16s} n={k['launches']:5d} tot={k['total_ms']:8.2f} avg={k['avg_ms']*1e3:8.1f}us "
          f"share={k['share']*100:5.1f}% GB/s={k['gbs'] or 0:8.0f}")
