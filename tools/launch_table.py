"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections, csv, io, sys
txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
tot, cnt = collections.Counter(), collections.Counter()
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    tot[name] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    cnt[name] += 1
all_us = sum(tot.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, v in tot.most_common():
    print(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / all_us:.1f}% |")
print(f"| **total** | {sum(cnt.values())} | {all_us:.1f} | 100% |")
