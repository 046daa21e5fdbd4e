"""Full-size parity at BASELINE.json configs[1] (C1: 5e7 synthetic 100-bp reads,
5 Gbp, k=40, m=7, min_count=1) in the launch configuration bench.py times.

The oracle cannot hold 6e8 distinct 40-mers in a std::map, so it computes the
histogram restricted to canonical k-mers whose FNV-1a-64 hash of the ASCII
string is 0 mod SAMPLE (oracle_count_sampled, all host cores). The harness
decodes every GPU key with its OWN decoder, applies the same predicate, and
the two sampled lists must be identical element by element; the Σcount and
valid-window totals must match the oracle's over the full input.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import compare

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

C1 = synth.Workload(seed=2, genome_len=240_000_000, read_len=100, n_reads=50_000_000, err=0.0033, nrate=0.0001)
K, M, SAMPLE = 40, 7, 4096


def _fnv_keep(keys: np.ndarray, k: int, mod: int) -> np.ndarray:
    """FNV-1a-64 over the ASCII decoding of each key (harness-side, on the GPU
    with torch int64 arithmetic = wrap-around mod 2^64), == 0 mod `mod` (a power of 2)."""
    import torch

    out = np.zeros(keys.shape[0], dtype=bool)
    letters = torch.tensor([65, 67, 71, 84], dtype=torch.int64, device="cuda")
    prime = torch.tensor(1099511628211, dtype=torch.int64, device="cuda")
    off = np.uint64(1469598103934665603).astype(np.int64)
    step = 50_000_000
    for a in range(0, keys.shape[0], step):
        kk = torch.from_numpy(keys[a:a + step].view(np.int64)).cuda()
        h = torch.full((kk.shape[0],), int(off), dtype=torch.int64, device="cuda")
        for i in range(k):
            code = (kk[:, i // 32] >> (62 - 2 * (i % 32))) & 3  # arithmetic shift; masked to 2 bits
            h = (h ^ letters[code]) * prime
        out[a:a + step] = ((h & (mod - 1)) == 0).cpu().numpy()
    return out


def test_c1_fullsize_sampled_parity():
    import torch

    from paper_1607_06618_b200 import gerbil

    n = int(os.environ.get("GERBIL_FULLSIZE_READS", C1.n_reads))
    w = synth.Workload(C1.seed, C1.genome_len, C1.read_len, n, C1.err, C1.nrate)
    codes, nmask, rs = synth.packed_device(w)
    torch.cuda.synchronize()
    with gerbil.Gerbil(timing=True) as g:  # bench.py's configuration (B auto, default table budget)
        for _ in range(2):  # the bench times calls after warm-up (ratio adapted)
            g.count_device(codes, nmask, rs, w.n_reads, K, M, 1)
        st = g.stats()
        keys, counts = g.fetch(sorted=False)
    del codes, nmask, rs
    assert st["count_sum"] == st["valid_windows"]
    keep = _fnv_keep(keys, K, SAMPLE)
    sk, sc = keys[keep], counts[keep]
    del keys, counts
    order = np.lexsort(tuple(sk[:, j] for j in reversed(range(sk.shape[1]))))
    sk, sc = sk[order], sc[order]

    text = synth.fastx(w, synth.FASTA)
    ref = oracle.count_sampled(text, K, 1, mod=SAMPLE, threads=0)
    assert ref.windows == st["valid_windows"], (ref.windows, st["valid_windows"])
    assert len(ref.kmers) > 1000
    compare(sk, sc, K, ref)
