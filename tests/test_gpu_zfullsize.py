"""Full-size parity in the launch configurations bench.py times (SURVEY.md §8(c)
"Scale strategy").

The oracle cannot hold 10^8-10^9 distinct k-mers in a std::map, so it computes
the histogram restricted to canonical k-mers whose FNV-1a-64 hash of the ASCII
string is 0 mod SAMPLE (oracle_count_sampled, all host cores). The harness
decodes every GPU key with its OWN decoder, applies the same predicate, and
the two sampled lists must be identical element by element; the Σcount and
valid-window totals must match the oracle's over the full input.

Cases (synth/configs.py holds the workloads bench.py runs):
  * C1 exactly as `bench.py` (default) times it: 5e7 x 100 bp, k=40, m=15,
    auto bins (2^22) — device bin plan, both shared-memory tiers, abandoned
    bins recounted in an L2 wave. The test asserts that tier 2 and the L2
    remainder really ran (smem_failed > 0, waves >= 1).
  * C1 at m=7 (auto bins → L2 wave tables only).
  * C3k65 (`bench.py --config C3k65` launch configuration: k=65, W=3 keys, m=15,
    auto bins) on a 2.5 Gbp prefix of the shard.
  * C3k100 (`bench.py --config C3k100`: k=100, W=4 keys, one window per read,
    m=15, auto bins → the reference tables of count_ref.cu) on a 2.5 Gbp prefix.
  * C4 (`bench.py --config C4`: 10-kbp reads, 1 % error, k=200, m=11, auto bins
    → reference tables, min_count=2) on a 2.5 Gbp prefix of the shard; the test
    asserts that the reference tables counted most windows.
GERBIL_FULLSIZE_SCALE (float, default 1) scales every case's read count.
"""
import os

import numpy as np
import pytest

import oracle
from synth.configs import CONFIGS
from tests.helpers import compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SAMPLE = 4096
SCALE = float(os.environ.get("GERBIL_FULLSIZE_SCALE", "1"))

# (id, config, m override, reads, extra asserts)
CASES = [
    ("C1-bench", "C1", None, None, "bench"),
    ("C1-m7", "C1", 7, None, ""),
    ("C3k65", "C3k65", None, 25_000_000, ""),
    ("C3k100", "C3k100", None, 25_000_000, "ref"),
    ("C4", "C4", None, 250_000, "ref"),
]


def _fnv_keep(keys: np.ndarray, k: int, mod: int) -> np.ndarray:
    """FNV-1a-64 over the ASCII decoding of each key (harness-side, on the GPU
    with torch int64 arithmetic = wrap-around mod 2^64), == 0 mod `mod` (a power of 2)."""
    import torch

    out = np.zeros(keys.shape[0], dtype=bool)
    letters = torch.tensor([65, 67, 71, 84], dtype=torch.int64, device="cuda")
    prime = torch.tensor(1099511628211, dtype=torch.int64, device="cuda")
    off = np.uint64(1469598103934665603).astype(np.int64)
    step = max(1, 400_000_000 // (8 * k))
    for a in range(0, keys.shape[0], step):
        kk = torch.from_numpy(keys[a:a + step].view(np.int64)).cuda()
        h = torch.full((kk.shape[0],), int(off), dtype=torch.int64, device="cuda")
        for i in range(k):
            code = (kk[:, i // 32] >> (62 - 2 * (i % 32))) & 3  # arithmetic shift; masked to 2 bits
            h = (h ^ letters[code]) * prime
        out[a:a + step] = ((h & (mod - 1)) == 0).cpu().numpy()
    return out


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_fullsize_sampled_parity(case):
    import torch

    import synth
    from paper_1607_06618_b200 import gerbil

    _, cname, m_over, reads, check = case
    cfg = CONFIGS[cname]
    n = int((reads or cfg.n_reads) * SCALE)
    m = m_over or cfg.m
    w = cfg.workload(n)
    codes, nmask, rs = synth.packed_device(w)
    torch.cuda.synchronize()
    # bench.py's context: B from the config (0 = auto), default table budget, timing on
    with gerbil.Gerbil(n_bins=cfg.n_bins, timing=True) as g:
        for _ in range(2):  # the bench times calls after warm-up (ratio adapted)
            g.count_device(codes, nmask, rs, w.n_reads, cfg.k, m, cfg.min_count)
        st = g.stats()
        keys, counts = g.fetch(sorted=False)
    del codes, nmask, rs
    torch.cuda.empty_cache()
    assert st["count_sum"] == st["valid_windows"]
    if check == "bench" and SCALE == 1:
        # the benchmarked combination really ran: device plan with 2^22 bins, shared-memory
        # tier 1, tier 2 for the bins tier 1 abandoned, and an L2 wave for the rest
        assert st["n_bins"] == 1 << 22, st["n_bins"]
        assert st["smem_windows"] > 0.95 * st["valid_windows"], st
        assert st["smem_failed"] > 0, st
        assert st["waves"] >= 1, st
    if check == "ref":  # the long-k reference tables (count_ref.cu) counted the bulk
        assert st["smem_windows"] > 0.9 * st["valid_windows"], st
    keep = _fnv_keep(keys, cfg.k, SAMPLE)
    sk, sc = keys[keep], counts[keep]
    del keys, counts
    order = np.lexsort(tuple(sk[:, j] for j in reversed(range(sk.shape[1]))))
    sk, sc = sk[order], sc[order]

    text = synth.fastx(w, synth.FASTA)
    ref = oracle.count_sampled(text, cfg.k, cfg.min_count, mod=SAMPLE, threads=0)
    del text
    assert ref.windows == st["valid_windows"], (ref.windows, st["valid_windows"])
    assert len(ref.kmers) > 1000
    compare(sk, sc, cfg.k, ref)
