"""Minimizer orderings of PAPER.md:140-146 on the GPU:
results are invariant, super-mers follow the oracle's minimizer under each
ordering (DFP: the oracle builds its own key table from the same sample
definition), and the Fig. Minimizer metric equals the oracle's brute force."""
from __future__ import annotations

import random

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import compare

pytestmark = pytest.mark.gpu

ORDERINGS = [oracle.KMC2, oracle.LEX, oracle.CGAT, oracle.ROBERTS, oracle.RANDOM, oracle.DFP]
PIVOT, STRIDE = 0.3, 2


@pytest.fixture(scope="module")
def G():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1607_06618_b200 import gerbil

    return gerbil


def _ctx(G, ordering, **kw):
    return G.Gerbil(ordering=ordering, dfp_pivot=PIVOT, order_sample_stride=STRIDE, **kw)


@pytest.mark.parametrize("ordering", ORDERINGS)
@pytest.mark.parametrize("k", [28, 40, 65])
def test_histogram_invariant_under_ordering(G, ordering, k):
    w = synth.Workload(seed=60 + k, genome_len=30_000, read_len=150, n_reads=3000, err=0.005, nrate=0.002)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, k)
    with _ctx(G, ordering, n_bins=64) as g:
        g.count(k, 7, 1, text=text)
        keys, counts = g.fetch(sorted=True)
    compare(keys, counts, k, ref)


@pytest.mark.parametrize("ordering", ORDERINGS)
@pytest.mark.parametrize("k,m", [(31, 5), (40, 7), (56, 9)])
def test_supermers_follow_ordering(G, ordering, k, m):
    L = 300
    w = synth.Workload(seed=70 + m, genome_len=20_000, read_len=L, n_reads=300, err=0.01, nrate=0.003)
    text = synth.fastx(w, synth.RAW)
    table = oracle.dfp_table(text, m, PIVOT, STRIDE) if ordering == oracle.DFP else None
    p = G.pack_reads(text=text)
    with _ctx(G, ordering, n_bins=97) as g:
        pos, nwin, b, mu = g.debug_supermers(p, k, m)
    reads = text.split(b"\n")[:-1]
    valid = [i * L + j for i, r in enumerate(reads) for j in range(len(r) - k + 1) if b"N" not in r[j:j + k]]
    got = np.sort(np.concatenate([np.arange(int(a), int(a) + int(n)) for a, n in zip(pos, nwin)]))
    assert np.array_equal(got, np.array(sorted(valid), dtype=got.dtype))
    rnd = random.Random(m)
    bin_of = {}
    for i in rnd.sample(range(len(pos)), min(250, len(pos))):
        for j in range(int(nwin[i])):
            q = int(pos[i]) + j
            kmer = reads[q // L][q % L: q % L + k]
            want = oracle.order_key(oracle.minimizer(kmer, m, ordering, table=table), ordering, table=table)
            assert int(mu[i]) == want, (i, j, kmer)
        assert bin_of.setdefault(int(mu[i]), int(b[i])) == int(b[i])


@pytest.mark.parametrize("ordering", ORDERINGS)
def test_minimizer_stats_match_oracle(G, ordering):
    k, m = 28, 6
    w = synth.Workload(seed=80 + ordering, genome_len=15_000, read_len=120, n_reads=1500, err=0.004, nrate=0.002)
    text = synth.fastx(w, synth.FASTA)
    table = oracle.dfp_table(text, m, PIVOT, STRIDE) if ordering == oracle.DFP else None
    want = oracle.minimizer_stats(text, k, m, ordering, table)
    with _ctx(G, ordering) as g:
        g.count(k, m, 1, text=text)
        got = g.minimizer_stats()
        st = g.stats()
    assert got == want
    # total super-mers (x-axis of Fig. Minimizer): the oracle's per-read decomposition, plus at
    # most one extra cut per 1024-position tile on the GPU
    reads = [r for r in text.split(b"\n") if r and not r.startswith(b">")]
    n_or = 0
    for r in reads:
        for frag in r.replace(b"N", b" ").split():
            n_or += len(oracle.supermers(frag, k, m, ordering, symmetric=True, table=table))
    assert n_or <= st["supermers"] <= n_or + st["input_bases"] // 1024 + 1


def test_dfp_chunked_upload_and_pivots(G, monkeypatch):
    monkeypatch.setenv("GERBIL_UPLOAD_CHUNKS", "3")
    w = synth.Workload(seed=90, genome_len=40_000, read_len=100, n_reads=4000, err=0.003, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 40)
    for pivot in (0.0, 0.5, 1.0):
        with G.Gerbil(ordering=G.ORDER_DFP, dfp_pivot=pivot, order_sample_stride=1) as g:
            g.count(40, 7, 1, text=text)
            keys, counts = g.fetch(sorted=True)
        compare(keys, counts, 40, ref)


def test_ordering_usage_errors(G):
    with pytest.raises(G.GerbilError):
        G.Gerbil(ordering=6)
    with pytest.raises(G.GerbilError):
        G.Gerbil(ordering=G.ORDER_DFP, dfp_pivot=1.5)
    with G.Gerbil(ordering=G.ORDER_DFP) as g:
        with pytest.raises(G.GerbilError) as e:
            g.count(40, 13, 1, text=b">a\nACGTACGTACGTACGTACGTACGTACGTACGTACGTACGTACGT\n")
        assert e.value.status == G.E_USAGE
