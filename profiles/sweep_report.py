import glob, json, sys
for f in sorted(glob.glob(f"gpurun_out/sw_{sys.argv[1]}_*.log"), key=lambda s: int(s.rsplit('_', 1)[1][:-4])):
    lines = open(f).read().strip().splitlines()
    spec = lines[-1]
    try:
        d = json.loads([l for l in lines if l.startswith('{')][-1])
        print(f"{spec:60s} {d['value']:.3e}  frac {d['roofline']['frac']:.3f}  launch {d['roofline']['avg_launch_ms']:.2f} ms  clk {d['clocks']['sm_mhz']}")
    except Exception:
        print(spec, "FAILED", lines[-3:])
