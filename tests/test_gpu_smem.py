"""GPU parity of step (d) in per-warp shared-memory tables (count_smem.cu,
DESIGN.md "Kernel (d) smem") against the CPU oracle: bit-exact sorted
(k-mer, count) lists on the same seeded inputs.

Covers both slot layouts (16-byte packed for k <= 48, key words + count
array above), every key-word boundary, the abandonment path (a bin with more
distinct k-mers than a warp table holds is recounted in the L2 wave tables),
mixed runs (some bins in shared memory, the rest in L2 waves), maximal
intra-warp key collisions (all-A reads), thresholds, non-canonical mode and
multi-rank loopback runs.
"""
import threading

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import compare, decode_keys

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1607_06618_b200 import gerbil

    return gerbil


# scaled C1 twin (21x coverage, 0.33 % errors): ~2.5 Mbp, bins of a few thousand windows
TWIN = synth.Workload(seed=11, genome_len=120_000, read_len=100, n_reads=25_000, err=0.0033, nrate=0.0001)
# k > 96: 250-bp reads (same coverage) so that every bin has windows
TWIN_LONG = synth.Workload(seed=13, genome_len=120_000, read_len=250, n_reads=10_000, err=0.0033, nrate=0.0001)
_REF = {}


def _ref(w, k, min_count, canonical=True):
    key = (w.seed, w.n_reads, k, min_count, canonical)
    if key not in _REF:
        text = synth.fastx(w, synth.FASTQ)
        _REF[key] = (text, oracle.count(text, k, min_count, canonical=canonical))
    return _REF[key]


def _run(G, text, k, m, min_count, **kw):
    with G.Gerbil(**kw) as g:
        g.count(k, m, min_count, text=text)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    return keys, counts, st


@pytest.mark.parametrize("k", [28, 31, 32, 33, 40, 46, 48, 49, 56, 64, 65, 96, 100, 128, 129, 200])
def test_smem_every_key_width(G, k):
    text, ref = _ref(TWIN if k <= 96 else TWIN_LONG, k, 1)
    keys, counts, st = _run(G, text, k, min(13, k - 1), 1, n_bins=4096, count_mode=G.COUNT_SMEM)
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows
    assert st["smem_bins"] > 0
    assert st["smem_windows"] > 0


@pytest.mark.parametrize("k,m,bins", [(40, 13, 1024), (40, 11, 65536), (40, 15, 1 << 20), (65, 12, 8192)])
def test_smem_bins_and_m(G, k, m, bins):
    text, ref = _ref(TWIN, k, 1)
    keys, counts, st = _run(G, text, k, m, 1, n_bins=bins, count_mode=G.COUNT_SMEM)
    compare(keys, counts, k, ref)
    assert st["smem_windows"] <= st["count_sum"] == ref.windows


@pytest.mark.parametrize("min_count", [2, 3, 7])
def test_smem_thresholds(G, min_count):
    text, ref = _ref(TWIN, 40, min_count)
    keys, counts, st = _run(G, text, 40, 13, min_count, n_bins=4096, count_mode=G.COUNT_SMEM)
    compare(keys, counts, 40, ref)


@pytest.mark.parametrize("k", [40, 65])
def test_smem_abandoned_bins_recounted_in_l2(G, k):
    # 16 bins of ~150k windows: every bin overflows a warp table, is abandoned
    # and recounted by the wave tables
    text, ref = _ref(TWIN, k, 1)
    keys, counts, st = _run(G, text, k, 13, 1, n_bins=16, count_mode=G.COUNT_SMEM)
    compare(keys, counts, k, ref)
    assert st["smem_failed"] == st["smem_bins"] > 0
    assert st["smem_windows"] == 0
    assert st["waves"] >= 1


def test_smem_mixed_with_l2(G):
    # 512 bins of ~5k windows with ρ̂ = 0.05: every bin is predicted to fit, the
    # larger ones overflow and are recounted in L2 waves (auto mode, no forcing)
    text, ref = _ref(TWIN, 40, 1)
    keys, counts, st = _run(G, text, 40, 11, 1, n_bins=512, distinct_ratio=0.05)
    compare(keys, counts, 40, ref)
    assert st["smem_bins"] > 0


def test_smem_all_a_reads(G):
    # every lane of a warp round carries the same k-mer: one group of 32 per round
    text = b"".join(b">r%d\n" % i + b"A" * (100 + i % 50) + b"\n" for i in range(300))
    for k in (31, 40, 65):
        ref = oracle.count(text, k, 1)
        keys, counts, st = _run(G, text, k, 11, 1, n_bins=64, count_mode=G.COUNT_SMEM)
        compare(keys, counts, k, ref)
        assert len(counts) == 1


def test_smem_low_complexity(G):
    rng = np.random.default_rng(5)
    reads = []
    for i in range(2000):
        unit = "".join(rng.choice(list("ACGT"), size=int(rng.integers(1, 4))))
        reads.append((unit * 200)[: int(rng.integers(60, 200))])
    text = "".join(f">r{i}\n{r}\n" for i, r in enumerate(reads)).encode()
    for k in (28, 40, 56):
        ref = oracle.count(text, k, 1)
        keys, counts, st = _run(G, text, k, 11, 1, n_bins=256, count_mode=G.COUNT_SMEM)
        compare(keys, counts, k, ref)


def test_smem_non_canonical(G):
    text = synth.fastx(TWIN, synth.FASTQ)
    for k in (40, 65):
        ref = oracle.count(text, k, 1, canonical=False)
        keys, counts, st = _run(G, text, k, 13, 1, n_bins=4096, count_mode=G.COUNT_SMEM, canonical=False)
        compare(keys, counts, k, ref)


def test_smem_long_reads(G):
    # 10-kbp reads at 1 % error, k=200: super-mers longer than the per-lane stage
    w = synth.Workload(seed=12, genome_len=200_000, read_len=10_000, n_reads=120, err=0.01, nrate=0.0)
    text = synth.fastx(w, synth.FASTA)
    ref = oracle.count(text, 200, 2)
    keys, counts, st = _run(G, text, 200, 11, 2, n_bins=2048, count_mode=G.COUNT_SMEM)
    compare(keys, counts, 200, ref)


def test_smem_auto_bins_policy(G):
    # n_bins = 0 with m >= 11: the library picks many small bins and counts them in shared memory
    text, ref = _ref(TWIN, 40, 1)
    keys, counts, st = _run(G, text, 40, 13, 1, distinct_ratio=0.3)
    compare(keys, counts, 40, ref)
    assert st["n_bins"] >= 512
    assert st["smem_windows"] > 0


def test_smem_repeated_calls_adapt(G):
    text, ref = _ref(TWIN, 40, 1)
    with G.Gerbil() as g:
        for _ in range(3):
            g.count(40, 13, 1, text=text)
            keys, counts = g.fetch(sorted=True)
            compare(keys, counts, 40, ref)
        st = g.stats()
    assert st["smem_windows"] > 0.5 * ref.windows


@pytest.mark.parametrize("P", [2, 3])
def test_smem_loopback_ranks(G, P):
    text, ref = _ref(TWIN, 40, 1)
    uid = bytes([0x40 + P]) * 128
    results = [None] * P
    errors = []

    def rank(r):
        try:
            with G.Gerbil(rank=r, world=P, unique_id=uid, comm_backend=1, n_bins=8192,
                          count_mode=G.COUNT_SMEM) as g:
                g.count(40, 13, 1, text=synth.fastx(TWIN.shard(r, P), synth.FASTQ))
                results[r] = g.fetch(sorted=True) + (g.stats(),)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    keys = np.concatenate([r[0] for r in results])
    counts = np.concatenate([r[1] for r in results])
    strs = decode_keys(keys, 40)
    order = sorted(range(len(strs)), key=lambda i: strs[i])
    compare(keys[order], counts[order], 40, ref)
    assert sum(r[2]["count_sum"] for r in results) == ref.windows
    assert all(r[2]["smem_bins"] > 0 for r in results)
