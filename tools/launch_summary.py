"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel name,
launches, total and mean time, and share of all kernel time."""
import collections, csv, sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in data:
    name = r[ik].split("(")[0] if not r[ik].startswith("void ") else r[ik][5:].split("(")[0]
    t = float(r[iv].replace(",", "")) * (1e-3 if r[iu] == "ns" else 1.0 if r[iu] == "us" else 1e3)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[1]}: {len(data)} launches, {tot / 1e3:.2f} ms of kernel time (serialised, cold-cache ncu)")
print(f"{'kernel':80s} {'launches':>8s} {'total_us':>11s} {'mean_us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:80]:80s} {n:8d} {t:11.1f} {t / n:10.1f} {t / tot * 100:6.2f}%")
