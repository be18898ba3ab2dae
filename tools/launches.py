"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel count, mean and total device time, and share of the total."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
            agg.setdefault(name, []).append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values()) or 1.0
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{len(v):4d}x  mean {sum(v)/len(v)/1e3:9.1f} us  total {sum(v)/1e3:9.1f} us  "
                   f"{100*sum(v)/tot:5.1f}%  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summarize(p))
