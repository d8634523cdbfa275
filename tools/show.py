import json, sys
for l in open(sys.argv[1]):
    try: d = json.loads(l)
    except Exception: continue
    if "fwd_gcoeff_s" in d and "p" in d:
        print(f"{d['p']:>10} n={d['n']:>10} b={d['batch']:>6} fwd {d['fwd_ms']:8.3f} ms {d['fwd_gcoeff_s']:7.1f} Gc/s ({d['fwd_roofline_frac']:.2f})  inv {d['inv_ms']:8.3f} ms {d['inv_gcoeff_s']:7.1f} ({d['inv_roofline_frac']:.2f})")
    elif "products_per_s" in d:
        print(f"config4: {d['ms']:.2f} ms  {d['products_per_s']:.0f} products/s  roofline {d['roofline_frac']:.2f}")
    elif "metric" in d:
        print(f"{d['metric']} {d['value']:.2f} fwd {d['fwd_ms']:.3f} inv {d['inv_ms']:.3f} roofline {d['roofline']['frac']:.3f} e2e {d.get('e2e',{}).get('value')}")
