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


# ---- world > 1: every rank spills its own batches; bin ranges are counted by their owners ----
def _spill_ranks(G, P, texts_per_rank, k, m, min_count, uid, **kw):
    import threading

    results, errors = [None] * P, []

    def rank(r):
        try:
            with G.Gerbil(rank=r, world=P, unique_id=uid, comm_backend=1, **kw) as g:
                packs = [G.pack_reads(t) for t in texts_per_rank[r]]
                g.spill_begin(k, m)
                for p in packs:
                    g.spill_add(p.codes, p.nmask, p.read_start, p.n_reads)
                try:  # sizing call: collective, keeps the job on every rank
                    g.spill_finish(min_count, out=None)
                    need = 0
                except G.GerbilError as e:
                    need = e.needed_bytes
                out = _pinned(need)
                n = g.spill_finish(min_count, out=out)
                results[r] = (out[:n].tobytes(), g.stats())
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    return results


@pytest.mark.parametrize("P,k,group_bytes", [(2, 40, "0"), (2, 65, "120000"), (3, 28, "90000"), (4, 100, "0")])
def test_spill_ranks_match_oracle(G, P, k, group_bytes, monkeypatch):
    if group_bytes != "0":
        monkeypatch.setenv("GERBIL_SPILL_GROUP_BYTES", group_bytes)  # several rounds of groups
    texts = _batches(200 + k, n=2 * P, reads=1200)
    per_rank = [texts[r::P] for r in range(P)]  # rank r spills batches r, r + P, ...
    ref = oracle.count(b"".join(texts), k)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    res = _spill_ranks(G, P, per_rank, k, 7, 1, bytes([40 + P + k % 50]) * 128, n_bins=64)
    got = sorted(r for buf, _ in res for r in _records(buf, k))
    assert got == want  # every k-mer exactly once, on its owner, with the global count
    sts = [s for _, s in res]
    assert sum(s["count_sum"] for s in sts) == ref.windows == sum(s["valid_windows"] for s in sts)
    assert sum(s["distinct"] for s in sts) == ref.distinct
    assert all(s["count_sum"] == s["owned_windows"] for s in sts)
    assert all(s["bytes_recv"] > 0 for s in sts)


def test_spill_ranks_min_count_and_empty_rank(G):
    # rank 1 spills nothing at all; min_count 2
    P, k = 2, 40
    texts = _batches(31, n=3, reads=1000)
    ref = oracle.count(b"".join(texts), k, 2)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    res = _spill_ranks(G, P, [texts, []], k, 7, 2, b"\x5a" * 128, n_bins=32)
    assert sorted(r for buf, _ in res for r in _records(buf, k)) == want
    assert res[1][1]["valid_windows"] == 0 and res[1][1]["count_sum"] > 0
