"""Per-source-line warp instructions (per unit) and stall samples of one ncu capture
(source rows of the cuda,sass view, which already aggregate their SASS rows)."""
import collections, csv, subprocess, sys
rep = sys.argv[1]; units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0; n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
iE = iS = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No" and "Instructions Executed" in r:
        iE = r.index("Instructions Executed"); iS = r.index("Warp Stall Sampling (All Samples)"); continue
    if iE is None or len(r) <= iE or not r[0]: continue
    try: e = float(r[iE] or 0); st = float(r[iS] or 0)
    except ValueError: continue
    key = r[0] + ":" + r[1].strip()[:90]
    agg[key][0] += e; agg[key][1] += st
te = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print(f"instr/unit {te / units:.1f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"ins/unit {v[0] / units:6.1f} stall {100 * v[1] / ts:5.1f}%  {k}")
