"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv, sys, collections

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")) if r.get("Metric Name") == "gpu__time_duration.sum"]
tot = collections.OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[r["Metric Unit"]]
    n, s = tot.get(name, (0, 0.0))
    tot[name] = (n + 1, s + v * scale)
allt = sum(s for _, s in tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'avg us':>10s} {'share':>7s}")
for name, (n, s) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:60]:60s} {n:8d} {s:12.1f} {s/n:10.2f} {100*s/allt:6.1f}%")
print(f"{'total':60s} {sum(n for n,_ in tot.values()):8d} {allt:12.1f}")
