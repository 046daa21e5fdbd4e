"""Out-of-core counting (gerbil_spill_*): batches are
spilled to host memory grouped by bin and counted bin group by bin group; the
streamed App. C records must equal the oracle's histogram of the whole input
(the concatenation of the batches), byte-exact per record."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1607_06618_b200 import gerbil

    return gerbil


def _pinned(n: int) -> np.ndarray:
    import torch

    return torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True).numpy()


def _records(buf: bytes, k: int) -> list[bytes]:
    kb, out, i = (k + 3) // 4, [], 0
    while i < len(buf):
        n = (5 if buf[i] == 0xFF else 1) + kb
        out.append(bytes(buf[i:i + n]))
        i += n
    assert i == len(buf)
    return out


def _batches(seed: int, n: int = 3, reads: int = 2500):
    texts = []
    for i in range(n):
        w = synth.Workload(seed=seed, genome_len=25_000, read_len=130, n_reads=reads, err=0.004, nrate=0.002,
                           first_read=i * reads)
        texts.append(synth.fastx(w, synth.FASTQ))
    rep = b"ACGTTGCAAGT" * 12  # a k-mer family with counts >= 255 across batches
    texts[1] += b"".join(b"@r\n" + rep + b"\n+\n" + b"I" * len(rep) + b"\n" for _ in range(200))
    return texts


def _spill(G, texts, k, m=7, min_count=1, **kw):
    packs = [G.pack_reads(t) for t in texts]
    with G.Gerbil(**kw) as g:
        g.spill_begin(k, m)
        for p in packs:
            g.spill_add(p.codes, p.nmask, p.read_start, p.n_reads)
        try:
            g.spill_finish(min_count, out=None)
            need = 0
        except G.GerbilError as e:
            need = e.needed_bytes
        # the sizing call keeps the spilled job: a too-small buffer keeps it as well
        if need > 1:
            with pytest.raises(G.GerbilError) as e:
                g.spill_finish(min_count, out=_pinned(need - 1))
            assert e.value.status == G.E_USAGE and e.value.needed_bytes == need
        out = _pinned(need)
        n = g.spill_finish(min_count, out=out)
        st = g.stats()
    return out[:n].tobytes(), n, need, st


@pytest.mark.parametrize("k,group_bytes", [(28, "0"), (40, "0"), (40, "150000"), (65, "150000"), (100, "0")])
def test_spill_matches_oracle(G, k, group_bytes, monkeypatch):
    if group_bytes != "0":
        monkeypatch.setenv("GERBIL_SPILL_GROUP_BYTES", group_bytes)  # force several bin groups
    texts = _batches(100 + k)
    ref = oracle.count(b"".join(texts), k)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    buf, n, need, st = _spill(G, texts, k, n_bins=64)
    assert n == need == sum(len(r) for r in want)
    assert sorted(_records(buf, k)) == want
    assert st["valid_windows"] == ref.windows == st["count_sum"] and st["distinct"] == ref.distinct
    assert max(ref.counts) >= 255


def test_spill_min_count_chunks_and_emergency(G, monkeypatch):
    monkeypatch.setenv("GERBIL_UPLOAD_CHUNKS", "3")
    monkeypatch.setenv("GERBIL_SPILL_GROUP_BYTES", "200000")
    texts = _batches(7, n=4, reads=1500)
    ref = oracle.count(b"".join(texts), 40, 2)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    # θ = 1 and an over-full table: the emergency path runs inside the groups
    buf, n, _, st = _spill(G, texts, 40, 7, 2, n_bins=32, max_probes=1, target_load=1.6, distinct_ratio=0.3)
    assert sorted(_records(buf, 40)) == want
    assert st["overflow_kmers"] > 0


def test_spill_empty_and_short_batches(G):
    w = synth.Workload(seed=9, genome_len=25_000, read_len=130, n_reads=500, err=0.004, nrate=0.002)
    texts = [b">a\nACGT\n", b">e\nA\n", synth.fastx(w, synth.FASTA), b">s\nACGTNACGT\n"]
    ref = oracle.count(b"".join(texts), 28)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    buf, n, _, st = _spill(G, texts, 28)
    assert sorted(_records(buf, 28)) == want


def test_spill_usage_errors(G):
    p = G.pack_reads(b">a\nACGTACGTACGTACGTACGTACGTACGTACGTACGT\n")
    with G.Gerbil() as g:
        with pytest.raises(G.GerbilError) as e:
            g.spill_add(p.codes, p.nmask, p.read_start, p.n_reads)
        assert e.value.status == G.E_STATE
        with pytest.raises(G.GerbilError) as e:
            g.spill_finish(1, out=_pinned(16))
        assert e.value.status == G.E_STATE
        g.spill_begin(28, 7)
        g.spill_add(p.codes, p.nmask, p.read_start, p.n_reads)
        out = _pinned(4096)
        assert g.spill_finish(1, out=out) > 0
        with pytest.raises(G.GerbilError) as e:
            g.fetch()
        assert e.value.status == G.E_STATE
        with pytest.raises(G.GerbilError):
            g.spill_finish(1, out=out)  # the spill was consumed
    with G.Gerbil(ordering=G.ORDER_DFP) as g:
        with pytest.raises(G.GerbilError) as e:
            g.spill_begin(28, 7)
        assert e.value.status == G.E_USAGE
