import csv, sys, collections
rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
agg = collections.OrderedDict()
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("radsort::", "")
    t = float(r["Metric Value"]) / 1e3
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1; a[1] += t
tot = sum(v[1] for k, v in agg.items() if "k_" in k and "generate" not in k and "k_sorted" not in k and "k_digest" not in k)
print(f"{'kernel':40s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    share = 100 * t / tot if tot and "generate" not in k and "k_sorted" not in k and "k_digest" not in k else float('nan')
    print(f"{k:40s} {n:8d} {t:12.1f} {share:6.1f}%")
