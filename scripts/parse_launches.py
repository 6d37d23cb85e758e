"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total ms per kernel."""
import csv
import sys
from collections import defaultdict


def summarise(path, top=15):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            f = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}[d["Metric Unit"]]
            k = d["Kernel Name"][:90]
            agg[k][0] += 1
            agg[k][1] += v * f
    tot = sum(v[1] for v in agg.values())
    out = [f"total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1]:10.3f} ms {v[0]:6d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        print(summarise(p))
