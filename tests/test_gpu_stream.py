"""Streaming e2e entry point (gerbil_count_host_stream): the compaction kernel
writes the paper's binary records (App. C) straight into
page-locked host memory. Records are compared byte-exact, as a multiset (the
record order is unspecified), with the oracle's own App. C encoder."""
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


def split_records(buf: bytes, k: int) -> list[bytes]:
    """The test's own App. C parser: counter (1 byte, or 0xFF + 4), then ceil(k/4) bytes."""
    kb = (k + 3) // 4
    out, i = [], 0
    while i < len(buf):
        n = (5 if buf[i] == 0xFF else 1) + kb
        out.append(bytes(buf[i:i + n]))
        i += n
    assert i == len(buf), "record stream does not end on a record boundary"
    return out


def _text(seed: int, rep_reads: int = 300) -> bytes:
    w = synth.Workload(seed=seed, genome_len=20_000, read_len=120, n_reads=3000, err=0.003, nrate=0.002)
    rep = b"ACGTTGCAAGT" * 11  # counts >= 255 → 5-byte counters
    return synth.fastx(w, synth.FASTQ) + b"".join(b"@r\n" + rep + b"\n+\n" + b"I" * len(rep) + b"\n"
                                                  for _ in range(rep_reads))


@pytest.mark.parametrize("k,min_count", [(28, 1), (32, 1), (40, 1), (40, 3), (46, 2), (64, 1), (101, 1)])
def test_stream_records_match_oracle(G, k, min_count):
    text = _text(31 + k)
    ref = oracle.count(text, k, min_count)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    assert max(ref.counts) >= 255
    pb = G.pack_reads(text)
    out = _pinned(sum(len(r) for r in want) + 4096)
    with G.Gerbil() as g:
        n = g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 7, min_count, out=out)
        keys, counts = g.fetch(sorted=True)  # the device results stay valid
        st = g.stats()
    assert n == sum(len(r) for r in want)
    got = sorted(split_records(out[:n].tobytes(), k))
    assert got == want
    assert len(counts) == len(ref.counts) == st["kept"]


def test_stream_emergency_path(G):
    # θ = 1 and an over-full table: records of the emergency pass are streamed too
    k = 40
    w = synth.Workload(seed=41, genome_len=50_000, read_len=250, n_reads=800, err=0.01)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, k)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    pb = G.pack_reads(text)
    out = _pinned(sum(len(r) for r in want))
    with G.Gerbil(max_probes=1, target_load=1.6, distinct_ratio=0.3, n_bins=4) as g:
        n = g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 9, 1, out=out)
        st = g.stats()
    assert st["overflow_kmers"] > 0
    assert sorted(split_records(out[:n].tobytes(), k)) == want


def test_stream_recount_path(G):
    # ρ̂ far too small: the waves are recounted; the byte stream restarts cleanly
    w = synth.Workload(seed=42, genome_len=200_000, read_len=100, n_reads=4000, err=0.01)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 40)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    pb = G.pack_reads(text)
    out = _pinned(sum(len(r) for r in want))
    with G.Gerbil(distinct_ratio=0.001, max_probes=2) as g:
        n = g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, 40, 7, 1, out=out)
    assert sorted(split_records(out[:n].tobytes(), 40)) == want


def test_stream_capacity_and_buffer_errors(G):
    text = _text(5, rep_reads=10)
    k = 40
    ref = oracle.count(text, k)
    need = sum(len(oracle.encode_entry(x, c)) for x, c in zip(ref.kmers, ref.counts))
    pb = G.pack_reads(text)
    with G.Gerbil() as g:
        # sizing call: no buffer
        with pytest.raises(G.GerbilError) as e:
            g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 7, 1, out=None)
        assert e.value.needed_bytes == need
        # too small: error + size; the device results are still complete
        small = _pinned(need // 2)
        with pytest.raises(G.GerbilError) as e:
            g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 7, 1, out=small)
        assert e.value.needed_bytes == need
        keys, counts = g.fetch(sorted=True)
        assert len(counts) == len(ref.counts)
        # pageable memory is refused
        with pytest.raises(G.GerbilError):
            g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 7, 1,
                                out=np.zeros(need, np.uint8))
        # exact capacity works
        out = _pinned(need)
        assert g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, k, 7, 1, out=out) == need


def test_stream_empty_input(G):
    pb = G.pack_reads(b">a\nACGT\n")
    out = _pinned(16)
    with G.Gerbil() as g:
        assert g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, 28, 7, 1, out=out) == 0


@pytest.mark.parametrize("chunks", [2, 7, 64])
def test_chunked_upload_parity(G, chunks, monkeypatch):
    # the host batch is uploaded in chunks and step (b) runs per chunk: results are identical
    monkeypatch.setenv("GERBIL_UPLOAD_CHUNKS", str(chunks))
    w = synth.Workload(seed=50 + chunks, genome_len=60_000, read_len=150, n_reads=6000, err=0.005, nrate=0.003)
    text = synth.fastx(w, synth.FASTQ) + b"@e\n\n+\n\n" + b"@s\nACGTNACG\n+\nIIIIIIII\n"
    ref = oracle.count(text, 31)
    want = sorted(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    pb = G.pack_reads(text)
    out = _pinned(sum(len(r) for r in want))
    with G.Gerbil() as g:
        n = g.count_host_stream(pb.codes, pb.nmask, pb.read_start, pb.n_reads, 31, 7, 1, out=out)
        assert sorted(split_records(out[:n].tobytes(), 31)) == want
        g.count_host_packed(pb.codes, pb.nmask, pb.read_start, pb.n_reads, 31, 7, 1)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    from tests.helpers import compare

    compare(keys, counts, 31, ref)
    assert st["valid_windows"] == ref.windows
