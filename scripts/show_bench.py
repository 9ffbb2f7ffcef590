import json, sys
r = json.load(open(sys.argv[1]))
for k in ['value', 'us_per_layer', 'speedup_vs_float_scale', 'float_scale_us_per_layer', 'clocks', 'e2e']:
    print(k, r.get(k))
print('roofline', {k: v for k, v in r['roofline'].items() if k != 'per_linear'})
for l in r['roofline']['per_linear']:
    print('  I', l)
for l in r['float_scale_kernel']:
    print('  F', l)
for s in r.get('sweep', []):
    print('  S', s)
