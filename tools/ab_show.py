"""Summarise tools/ab.sh output."""
import json, glob, re, sys
for f in sorted(glob.glob("gpurun_out/ab/*_[0-9].json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    w = open(f.replace(".json", "_work.txt")).read()
    ms = re.findall(r"launch\+results ([0-9.]+) ms", w)
    print(f"{f}: {d['value']:.0f}/s e2e {d['e2e']['value']:.0f}/s lat {d['latency_ms']['median']:.4f} dev {d['latency_ms']['device_median']:.4f} | work {ms}")
