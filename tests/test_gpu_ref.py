"""GPU parity of the long-k counting tier (count_ref.cu, W >= 4 key words): CTA-wide
shared-memory tables whose slots reference an occurrence of the k-mer (fingerprint + stream
position + orientation) and verify candidates by re-extracting it. Compared element by element
with the oracle on long synthetic reads (the C4 shape: 10-kbp class reads, 1 % errors, mostly
singleton k-mers, min_count 2 — PAPER.md:313-314), across the device-planned many-bin path,
the host-planned path, abandonment to the L2 wave tables, repeats that share fingerprints
with many positions (verification path) and the non-canonical mode."""
import pytest

import oracle
import synth
from tests.helpers import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1607_06618_b200 import gerbil

    return gerbil


def _run(G, text, k, m, min_count, **kw):
    with G.Gerbil(**kw) as g:
        g.count(k, m, min_count, text=text)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    return keys, counts, st


@pytest.mark.parametrize("k,min_count", [(97, 1), (128, 2), (200, 2), (201, 1), (300, 2), (479, 1)])
def test_ref_device_plan_many_bins(G, k, min_count):
    # 2^16 bins: the device-side bin plan, every bin in a reference table
    w = synth.Workload(seed=500 + k, genome_len=200_000, read_len=2000, n_reads=400, err=0.01)
    text = synth.fastx(w, synth.FASTA, line_width=100)
    ref = oracle.count(text, k, min_count)
    keys, counts, st = _run(G, text, k, 11, min_count, n_bins=1 << 16)
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows
    assert st["smem_windows"] == ref.windows and st["smem_failed"] == 0


@pytest.mark.parametrize("k", [100, 160, 256])
def test_ref_host_plan(G, k):
    w = synth.Workload(seed=600 + k, genome_len=50_000, read_len=600, n_reads=500, err=0.005, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, k, 1)
    keys, counts, st = _run(G, text, k, 9, 1, n_bins=32)
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows and st["smem_windows"] > 0


def test_ref_abandoned_bin_goes_to_wave_tables(G):
    # one bin with far more distinct k-mers than a CTA table holds: abandoned, recounted exactly
    w = synth.Workload(seed=77, genome_len=400_000, read_len=1000, n_reads=300, err=0.01)
    text = synth.fastx(w, synth.FASTA)
    ref = oracle.count(text, 150, 1)
    keys, counts, st = _run(G, text, 150, 11, 1, n_bins=1, count_mode=G.COUNT_SMEM)
    compare(keys, counts, 150, ref)
    # abandoned by the half tables of tier 1 and again by the full-size table of tier 2
    assert st["smem_failed"] >= 1 and st["count_sum"] == ref.windows


def test_ref_repeats_and_low_complexity(G):
    # identical k-mers at many positions (same fingerprint, verification by re-extraction),
    # palindromes, all-A and tandem repeats next to random sequence
    import random

    rnd = random.Random(3)
    unit = bytes(rnd.choice(b"ACGT") for _ in range(37))
    reads = [b"A" * 900, b"ACGT" * 250, unit * 30, (b"AC" * 300) + (b"GT" * 300)]
    reads += [bytes(rnd.choice(b"ACGT") for _ in range(700)) for _ in range(30)]
    reads += [reads[-1]] * 5 + [reads[-2][::-1].translate(bytes.maketrans(b"ACGT", b"TGCA"))] * 3
    text = b"".join(b">r%d\n" % i + r + b"\n" for i, r in enumerate(reads))
    for k in (100, 200):
        ref = oracle.count(text, k, 1)
        keys, counts, st = _run(G, text, k, 11, 1, n_bins=4)
        compare(keys, counts, k, ref)
        assert st["count_sum"] == ref.windows


def test_ref_non_canonical(G):
    w = synth.Workload(seed=88, genome_len=30_000, read_len=400, n_reads=700, err=0.004)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 130, 1, canonical=False)
    keys, counts, st = _run(G, text, 130, 11, 1, n_bins=16, canonical=False)
    compare(keys, counts, 130, ref)
    assert st["count_sum"] == ref.windows


@pytest.mark.parametrize("k,read_len,n_reads", [(100, 150, 3000), (97, 2000, 200), (200, 3000, 150), (300, 2500, 120)])
def test_ref_zero_fingerprints(G, monkeypatch, k, read_len, n_reads):
    # GERBIL_REF_DBG=16 zeroes the fingerprints: every occupied slot a probe meets is compared
    # k-mer by k-mer, so the verification (inline and the rolling path's deferred queue) and the
    # re-probe after a mismatch run on nearly every window; counts must stay exact
    monkeypatch.setenv("GERBIL_REF_DBG", "16")
    w = synth.Workload(seed=900 + k, genome_len=40_000, read_len=read_len, n_reads=n_reads, err=0.01)
    text = synth.fastx(w, synth.FASTA)
    for min_count in (1, 2):
        ref = oracle.count(text, k, min_count)
        keys, counts, st = _run(G, text, k, 11, min_count, n_bins=1 << 16)
        compare(keys, counts, k, ref)
        assert st["count_sum"] == ref.windows and st["smem_windows"] == ref.windows
