"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel (dev tool).

usage: python tools/ncu_launches.py launches.csv STEPS "header line" > summary.txt"""
import collections, csv, io, sys

path, steps = sys.argv[1], int(sys.argv[2])
header = sys.argv[3] if len(sys.argv) > 3 else ""
lines = [l for l in open(path) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
tot, cnt, unit = collections.defaultdict(float), collections.Counter(), set()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    unit.add(u)
    ms = v / 1e6 if u == "ns" else (v / 1e3 if u in ("us", "usecond") else v)
    tot[r["Kernel Name"]] += ms
    cnt[r["Kernel Name"]] += 1
allms = sum(tot.values())
if header:
    print(header)
print(f"# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold-cache per-launch times; unit {unit})")
print(f"# {sum(cnt.values())} launches over {steps} steps, {allms / steps:.2f} ms/step summed\n")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / steps:9.3f} ms/step {100 * v / allms:5.1f}% {cnt[k] / steps:6.1f} launches/step  {k}")
