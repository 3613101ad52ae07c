"""Table of bench lines from scripts/gpu_libab.sh."""
import collections
import json
import re
import sys

rows = collections.defaultdict(list)
for f in sys.argv[1:]:
    m = re.search(r"libab_(.+)_(\d+)\.json$", f)
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        print(f, "unreadable", ex)
        continue
    rows[m.group(1)].append(d)
for v, ds in rows.items():
    for d in ds:
        r = d["roofline"]
        print(f"{v:12s} {d['value'] / 1e6:7.3f} Mtok/s  fused {r['achieved']:7.1f} GB/s "
              f"frac {r['frac']:.3f} ({r['kernel_ms']:.3f} ms)  sm {d['clocks']['sm_mhz']} "
              f"{d['clocks'].get('power_w', '-')} W "
              f"{d['clocks']['reasons']}  loss {d['check']['loss']:.6e}")
