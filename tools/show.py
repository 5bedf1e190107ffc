import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print(f"{d['value']/1e9:.3f} Gs/s  {d['ms_per_step']*1e3:.1f} us/step  eager {d['ms_per_step_eager']*1e3:.1f}  e2e {d['e2e']['value']/1e9:.3f} Gs/s  frac {d['roofline']['frac']:.4f}  P {d['pairs_per_sample']:.2f} C {d['candidates_per_sample']:.1f}")
        print({k: round(v * 1000, 1) for k, v in sorted(d['kernel_ms'].items(), key=lambda x: -x[1])})
        print('clocks', d.get('clocks'), 'cpu', d.get('cpu_baseline', {}).get('value'))
