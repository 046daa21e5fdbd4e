"""Out-of-core path at C1 scale: the C1 reads in N host batches → gerbil_spill_add per batch
(phase one: upload, step (b), super-mers to pinned host memory by bin) → gerbil_spill_finish
(phase two: bin groups uploaded and counted, App. C records streamed). Wall clock per phase."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import C1, K, M, MIN_COUNT  # noqa: E402
from paper_1607_06618_b200 import gerbil  # noqa: E402

nb_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 4
group_gib = float(sys.argv[2]) if len(sys.argv) > 2 else 0
per = C1["n_reads"] // nb_batches
batches = []
for i in range(nb_batches):
    w = synth.Workload(**{**C1, "n_reads": per, "first_read": i * per})
    c, n, r = synth.packed_device(w)
    hb = []
    for t in (c, n, r):
        h = torch.empty(t.numel(), dtype=torch.int64, pin_memory=True)
        h.copy_(t)
        hb.append(h)
    batches.append((hb, w.n_reads))
    del c, n, r
torch.cuda.synchronize()
kw = {"n_bins": 4096}
g = gerbil.Gerbil(**kw)
if group_gib:
    os.environ["GERBIL_SPILL_GROUP_BYTES"] = str(int(group_gib * (1 << 30)))
rec = None
for rep in range(2):  # first pass sizes the output buffer and warms up
    t0 = time.perf_counter()
    g.spill_begin(K, M)
    for (hc, hn, hr), nr in batches:
        g.spill_add(hc.numpy(), hn.numpy(), hr.numpy(), nr)
    t1 = time.perf_counter()
    try:
        n = g.spill_finish(MIN_COUNT, out=rec)
    except gerbil.GerbilError as e:
        n = e.needed_bytes
        rec = torch.empty(int(n * 1.02) + (1 << 20), dtype=torch.uint8, pin_memory=True).numpy()
    t2 = time.perf_counter()
st = g.stats()
bases = st["input_bases"]
print(json.dumps({"batches": nb_batches, "group_budget_gib": group_gib or 16, "phase1_ms": (t1 - t0) * 1e3,
                  "phase2_ms": (t2 - t1) * 1e3, "total_ms": (t2 - t0) * 1e3,
                  "gbases_per_s": bases / (t2 - t0) / 1e9, "record_bytes": n, "distinct": st["distinct"],
                  "valid_windows": st["valid_windows"], "waves": st["waves"]}))
g.close()
