"""Per-variant DRAM traffic of the dominant kernel from an `ncu --set full`
capture -> profiles/traffic.json[variant] (read by bench.py as roofline.traffic).

    python scripts/ncu_traffic.py <report.ncu-rep> <variant> <rows> <vocab> <algo_bytes_per_row>
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[0]
    data = [r for r in rows[2:] if r and r[0].strip('"').isdigit()]
    recs = []
    for r in data:
        d = dict(zip(head, r))
        recs.append(d)
    return recs


def num(x):
    return float(str(x).replace(",", ""))


def main():
    rep, variant, rows, vocab, algo = sys.argv[1], sys.argv[2], int(sys.argv[3]), \
        int(sys.argv[4]), int(sys.argv[5])
    recs = metrics(rep)
    k = recs[0]
    rd, wr = num(k["dram__bytes_read.sum"]), num(k["dram__bytes_write.sum"])
    # ncu reports bytes in the unit of its column header (e.g. "Gbyte"); the raw page
    # row 1 carries units
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    units = dict(zip(*list(csv.reader(io.StringIO(out)))[:2]))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd *= scale[units["dram__bytes_read.sum"]]
    wr *= scale[units["dram__bytes_write.sum"]]
    t_unit = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9,
              "us": 1e-6, "ms": 1e-3, "s": 1.0}
    t = num(k["gpu__time_duration.sum"]) * t_unit[units["gpu__time_duration.sum"]]
    f = ROOT / "profiles" / "traffic.json"
    db = json.loads(f.read_text()) if f.exists() else {}
    db[variant] = {"kernel": k.get("Kernel Name", "?")[:80], "source": rep, "rows": rows,
                   "vocab": vocab, "dram_bytes_read": rd, "dram_bytes_write": wr,
                   "dram_bytes_per_row": (rd + wr) / rows, "algorithmic_bytes_per_row": algo,
                   "traffic_over_algorithmic": (rd + wr) / rows / algo,
                   "kernel_s_serialised": t, "dram_gbs_serialised": (rd + wr) / t / 1e9}
    f.write_text(json.dumps(db, indent=1) + "\n")
    print(variant, db[variant])


if __name__ == "__main__":
    main()
