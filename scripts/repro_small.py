"""Diagnostics: one small host-text count (the parity test's random reads) for compute-sanitizer."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1607_06618_b200 import gerbil
k = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rnd = random.Random(k)
reads = []
for _ in range(3000):
    r = bytearray(rnd.choice(b"ACGT") for _ in range(rnd.randint(1, 400)))
    for _ in range(rnd.randint(0, 3)):
        p = rnd.randrange(len(r))
        r[p:p + 3] = b"NNN"[: len(r[p:p + 3])]
    reads.append(bytes(r))
text = b"".join(b">r\n" + r + b"\n" for r in reads)
with gerbil.Gerbil(n_bins=64) as g:
    g.count(k, 7, 1, text=text)
    st = g.stats()
    print("k", k, "windows", st["valid_windows"], "supermers", st["supermers"], "kept", st["kept"])
