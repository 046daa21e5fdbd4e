"""Steps (b)-(e) device time for several k on the C1 batch (m=15 many bins vs m=7 L2 tables)."""
import sys
import time
import torch
import synth
from paper_1607_06618_b200 import gerbil

w = synth.Workload(seed=2, genome_len=240_000_000, read_len=int(sys.argv[1]) if len(sys.argv) > 1 else 100,
                   n_reads=int(sys.argv[2]) if len(sys.argv) > 2 else 50_000_000, err=0.0033, nrate=0.0001)
codes, nmask, rs = synth.packed_device(w)
torch.cuda.synchronize()
for k in [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "40,56,65,100").split(",")]:
    for m in (15, 7):
        with gerbil.Gerbil(timing=True) as g:
            for i in range(3):
                torch.cuda.synchronize()
                t = time.time()
                g.count_device(codes, nmask, rs, w.n_reads, k, m, 1)
                torch.cuda.synchronize()
                dt = (time.time() - t) * 1e3
            st = g.stats()
            print(f"k={k} m={m} wall={dt:.1f} ms supermer={st['ms_supermer']:.1f} shuffle={st['ms_shuffle']:.1f} "
                  f"count={st['ms_count']:.1f} (smem {st['ms_smem']:.1f}) bins={st['n_bins']} waves={st['waves']} "
                  f"smem_windows={st['smem_windows'] / max(st['valid_windows'], 1):.3f} slots={st['smem_slots']}",
                  flush=True)
