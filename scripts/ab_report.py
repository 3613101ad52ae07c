"""Summarise gpurun_out/ab_*.log bench lines."""
import glob, json
for f in sorted(glob.glob("gpurun_out/ab_*.log"), key=lambda x: int(x.split("_")[2])):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            r = d["roofline"]
            print(f"{f:40s} {d['value']/1e6:7.3f} Mtok/s  kernel {r['achieved']:7.0f} GB/s "
                  f"frac {r['frac']:.3f}  clk {d['clocks']['sm_mhz']}")
