"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
kernel: launches, total and mean time, share of the profiled steps."""
import csv
import json
import sys
from collections import OrderedDict


def summarise(path, skip_setup=True):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        name = r["Kernel Name"].replace("se::<unnamed>::", "")
        name = name.split("(")[0]
        rows.append((name, float(r["Metric Value"].replace(",", "")) * scale))
    agg = OrderedDict()
    for name, ms in rows:
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    total = sum(v[1] for v in agg.values())
    out = [{"kernel": k, "launches": v[0], "total_ms": round(v[1], 4),
            "mean_ms": round(v[1] / v[0], 4),
            "share": round(v[1] / total, 4) if total else 0.0}
           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return {"source": path, "launches": len(rows), "total_ms": round(total, 3),
            "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(s, f, indent=1)
    print("%d launches, %.2f ms total" % (s["launches"], s["total_ms"]))
    for k in s["kernels"]:
        print("%-60s %4d %9.3f ms %6.1f%%" % (k["kernel"][:60], k["launches"],
                                             k["total_ms"], 100 * k["share"]))
