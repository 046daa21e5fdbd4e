"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of a bench run with W warm-up
steps + 1 timed step: per-kernel launches, total time, share and average over the LAST step."""
import collections, csv, sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
h = None
data = []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        data.append(dict(zip(h, r)))
starts = [i for i, d in enumerate(data) if "rs_bits_kernel" in d["Kernel Name"]]
step = data[starts[-1]:]
agg = collections.OrderedDict()
for d in step:
    name = d["Kernel Name"].split("(")[0]
    t = float(d["Metric Value"]) / 1e6  # ns -> ms
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += t
tot = sum(v[1] for v in agg.values())
print(f"# step total (serialised) {tot:.1f} ms over {len(step)} launches")
print(f"{'kernel':62s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>9s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:62]:62s} {n:8d} {t:9.2f} {100 * t / tot:5.1f}% {1e3 * t / n:9.1f}")
