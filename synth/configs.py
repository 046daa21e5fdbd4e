"""The BASELINE.json workloads as seeded synthetic read sets.

Input recipe only — shapes, sizes, error/N rates and seeds — shared by
bench.py and the tests so that a parity test checks exactly the launch
configuration the benchmark times. Holds none of the counting method's
arithmetic. Sizes follow SURVEY.md §8(d)'s config table; C2-C4 are the
per-GPU shards of the 8-GPU runs BASELINE.json names (rank r of N takes
reads [r*n, (r+1)*n) of the full read set, so N = 8 covers all of it).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import Workload


@dataclass(frozen=True)
class Config:
    name: str
    desc: str
    seed: int
    genome_len: int
    read_len: int
    n_reads: int          # per GPU
    err: float
    nrate: float
    k: int
    m: int
    min_count: int
    n_bins: int = 0       # 0 = the library's auto policy
    extra: dict = field(default_factory=dict)

    def workload(self, n_reads: int | None = None, rank: int = 0) -> Workload:
        n = self.n_reads if n_reads is None else n_reads
        return Workload(self.seed, self.genome_len, self.read_len, n, self.err, self.nrate, first_read=rank * n)

    def label(self, n_reads: int | None = None) -> str:
        n = self.n_reads if n_reads is None else n_reads
        gbp = n * self.read_len / 1e9
        return (f"{self.name}: {self.desc}, {n:.3g} x {self.read_len} bp = {gbp:.3g} Gbp per GPU, k={self.k}, "
                f"m={self.m}, min_count={self.min_count}" + (f", {self.n_bins} bins" if self.n_bins else ""))


CONFIGS = {
    # configs[0]: the oracle's small case
    "C0": Config("C0", "10k synthetic 100-bp reads (1 Mbp)", 1, 100_000, 100, 10_000, 0.0025, 0.001,
                 28, 7, 1, n_bins=1),
    # configs[1]: F. vesca-scale, the N=1 headline (m=15: reading Q25, results invariant in m)
    "C1": Config("C1", "F. vesca-scale synthetic Illumina reads", 2, 240_000_000, 100, 50_000_000, 0.0033, 0.0001,
                 40, 15, 1),
    # configs[2]: G. gallus-scale 3.5e8 x 100 bp over 8 GPUs
    "C2": Config("C2", "G. gallus-scale synthetic reads (per-GPU shard of 35 Gbp / 8)", 3, 1_050_000_000, 100,
                 43_750_000, 0.0025, 0.0001, 56, 15, 1),
    # configs[3]: H. sapiens-scale 1e9 x 100 bp over 8 GPUs, k = 65 and k = 100
    "C3k65": Config("C3k65", "H. sapiens-scale synthetic reads (per-GPU shard of 100 Gbp / 8)", 4, 3_100_000_000,
                    100, 125_000_000, 0.0021, 0.0001, 65, 15, 1),
    "C3k100": Config("C3k100", "H. sapiens-scale synthetic reads (per-GPU shard of 100 Gbp / 8)", 4, 3_100_000_000,
                     100, 125_000_000, 0.0021, 0.0001, 100, 15, 1),
    # configs[4]: long reads 1e7 x 10 kbp over 8 GPUs, 1 % error, k = 200, min_count = 2. m = 15 (reading Q25,
    # results invariant in m; SURVEY §8(d) proposed m = 11, whose few popular minimizers leave most windows in
    # bins too large for a table), bins: the library's auto policy (~2^21 for count_ref.cu's reference tables)
    "C4": Config("C4", "synthetic long reads, 10 kbp, 1% error (per-GPU shard of 100 Gbp / 8)", 5, 3_100_000_000,
                 10_000, 1_250_000, 0.01, 0.0, 200, 15, 2),
}
