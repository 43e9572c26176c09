import json, signal, sys
signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet when piped into head
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench.log"):
    line = line.strip()
    if not line.startswith("{"):
        if "rc=" in line or "Error" in line:
            print(line)
        continue
    d = json.loads(line)
    print(f"value {d['value']} builds/s  ms/step {d.get('ms_per_step')}  hbm_frac {d.get('hbm', {}).get('frac_of_peak')}  e2e {d.get('e2e', {}).get('value')}")
    for k, v in d.get("kernels", {}).items():
        print(f"  {k:22s} {v['ms']*1e3:8.1f} us x{v['launches']}  {v['gbs']:7.0f} GB/s  frac {v['frac']:.3f}")
    print("  parity:", d["config"].get("parity"), " clocks:", d.get("clocks"))
