"""Summarise gpurun_out/<tag>/bench*.json (value, e2e, latency, microbench)."""
import glob
import json
import sys

for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}/bench*.json")):
    d = json.loads(open(f).readline())
    m = d.get("microbench", {})
    micro = {k: (round(v["achieved_tflops"], 2), round(v["frac_fp32_peak"], 3), round(v["ms"], 3))
             for k, v in m.items() if isinstance(v, dict) and "collision" in k}
    nn = {k: (round(v["algorithmic_gbs"]), round(v["frac_l2_peak"], 3)) for k, v in m.items()
          if isinstance(v, dict) and k.startswith("nn")}
    print(round(d["value"]), round(d["e2e"]["value"]), round(d["latency_ms"]["median"], 4), d["success_rate"],
          micro, nn)
