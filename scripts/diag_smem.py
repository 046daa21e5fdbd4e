"""Diagnostics: stats of repeated C1-size count_device calls (shared-memory path)."""
import sys
import torch
import synth
from paper_1607_06618_b200 import gerbil

n_reads = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 13
ordering = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n_bins = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = synth.Workload(seed=2, genome_len=240_000_000, read_len=100, n_reads=n_reads, err=0.0033, nrate=0.0001)
codes, nmask, rs = synth.packed_device(w)
torch.cuda.synchronize()
with gerbil.Gerbil(timing=True, ordering=ordering, n_bins=n_bins) as g:
    for i in range(3):
        g.count_device(codes, nmask, rs, w.n_reads, 40, m, 1)
        st = g.stats()
        print({k: st[k] for k in ("n_bins", "waves", "smem_bins", "smem_failed", "smem_windows", "smem_slots",
                                  "owned_windows", "distinct", "ratio_used", "ratio_observed", "max_bin_windows",
                                  "ms_supermer", "ms_shuffle", "ms_count", "launches_count")}, flush=True)
