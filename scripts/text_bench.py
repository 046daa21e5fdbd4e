"""FASTQ text → counts at C1 scale (5e7 x 100 bp, k=40): host reader (gerbil_pack_reads, all host cores)
vs the device parser (gerbil_count_text: H2D of the text + parse on the GPU + steps b-e). Wall clock."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import C1, K, M, MIN_COUNT  # noqa: E402
from paper_1607_06618_b200 import gerbil  # noqa: E402

frac = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
w = synth.Workload(**{**C1, "n_reads": int(C1["n_reads"] * frac)})
t = time.perf_counter()
text = synth.fastx(w, synth.FASTQ)
t_gen = time.perf_counter() - t
pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = np.frombuffer(text, dtype=np.uint8)
del text
out = {"reads": w.n_reads, "text_bytes": pinned.numel(), "gen_s": t_gen}
g = gerbil.Gerbil(timing=True)
for rep in range(3):
    t = time.perf_counter()
    g.count_text(pinned.numpy(), K, M, MIN_COUNT)
    dt = time.perf_counter() - t
st = g.stats()
out.update({"device_text_to_counts_ms": dt * 1e3, "upload_plus_parse_ms": st["ms_h2d"],
            "supermer_ms": st["ms_supermer"], "count_ms": st["ms_count"],
            "gbases_per_s": st["input_bases"] / dt / 1e9, "distinct": st["distinct"]})
# host reader on a slice (all host cores)
n_host = min(pinned.numel(), 1 << 30)
cut = bytes(pinned.numpy()[:n_host])
cut = cut[: cut.rfind(b"\n@") + 1]
t = time.perf_counter()
p = gerbil.pack_reads(cut)
dt = time.perf_counter() - t
out.update({"host_reader_sample_bytes": len(cut), "host_reader_s": dt,
            "host_reader_gbases_per_s": p.n_bases / dt / 1e9, "host_cores": os.cpu_count()})
print(json.dumps(out))
g.close()
