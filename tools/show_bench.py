import json, sys
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, 'value', round(d['value'], 4), 'e2e', round(d['e2e']['value'], 3), 'launches', d['gpu_launches'])
    p = d['path']; print(' path E', p['E'], 'K', p['K'], 'outer', p['outer'], 'newton', p['newton'], 'cg', p['cg'], 'armijo', p['armijo'])
    r = d['roofline']; print(' roof GB/s %.1f frac %.3f avg_us %.1f share %.2f' % (r['achieved'], r['frac'], r['avg_launch_us'], r['share_of_timed_kernels']))
    for k, v in list(r['per_kernel'].items())[:14]: print('   %-18s %s' % (k, v))
    print(' clocks', d['clocks'], 'cpu', d.get('cpu_baseline'))
