"""Per-instruction execution counts of an ncu source export (scripts/r02_prof.sh src_<name>.csv),
in address order, for reading a kernel's hot loop: python scripts/sass_prof.py src.csv [min_count]"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1]).read().splitlines()))
lo = int(float(sys.argv[2])) if len(sys.argv) > 2 else 0
ins, line = [], None
for r in rows[3:]:
    if len(r) < 8:
        continue
    if r[0]:
        line = r[0]
        continue
    try:
        a, e, s = int(r[2], 16), int(float(r[7] or 0)), int(float(r[4] or 0))
    except ValueError:
        continue
    ins.append((a, e, s, line, r[3].strip()))
ins.sort()
seen = set()
base = ins[0][0]
tot = 0
for a, e, s, l, t in ins:
    if a in seen:
        continue
    seen.add(a)
    tot += e
    if e >= lo:
        print(f"{a - base:6x} {e:11d} {s:7d} L{l:>4} {t}")
print("total warp instructions", tot)
