import sys
import synth
from paper_1607_06618_b200 import gerbil
k = int(sys.argv[1]) if len(sys.argv) > 1 else 33
w = synth.Workload(seed=11, genome_len=120_000, read_len=100, n_reads=25_000, err=0.0033, nrate=0.0001)
text = synth.fastx(w, synth.FASTQ)
with gerbil.Gerbil(n_bins=4096, count_mode=2) as g:
    g.count(k, 13, 1, text=text)
    print(g.stats()["smem_windows"])
