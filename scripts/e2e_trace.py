"""Diagnostics: host milestones (GERBIL_TRACE=1) of streaming e2e calls on the bench workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GERBIL_TRACE", "1")
import torch  # noqa: E402

import synth  # noqa: E402
from bench import C1, K, M, MIN_COUNT  # noqa: E402
from paper_1607_06618_b200 import gerbil  # noqa: E402

w = synth.Workload(**C1)
codes, nmask, rs = synth.packed_device(w)
hc = torch.empty(codes.numel(), dtype=torch.int64, pin_memory=True); hc.copy_(codes)
hn = torch.empty(nmask.numel(), dtype=torch.int64, pin_memory=True); hn.copy_(nmask)
hr = torch.empty(rs.numel(), dtype=torch.int64, pin_memory=True); hr.copy_(rs)
g = gerbil.Gerbil()
need = 0
try:
    g.count_host_stream(hc.numpy(), hn.numpy(), hr.numpy(), w.n_reads, K, M, MIN_COUNT, out=None)
except gerbil.GerbilError as e:
    need = e.needed_bytes
rec = torch.empty(int(need * 1.02) + (1 << 20), dtype=torch.uint8, pin_memory=True).numpy()
for i in range(3):
    t0 = time.perf_counter()
    n = g.count_host_stream(hc.numpy(), hn.numpy(), hr.numpy(), w.n_reads, K, M, MIN_COUNT, out=rec)
    dt = time.perf_counter() - t0
    st = g.stats()
    print(f"call {i}: {dt*1e3:.1f} ms wall, {n/1e9:.3f} GB records; stages", {x: round(st['ms_' + x], 1) for x in ('h2d', 'supermer', 'shuffle', 'count', 'total')}, file=sys.stderr, flush=True)
g.close()
