"""Step (a) on the device (gerbil_parse_text / gerbil_count_text, SURVEY.md §8(f)
NEXT(4)): the GPU parser's packed batch must equal the host reader's
(gerbil_pack_reads) bit for bit on every text shape the host reader takes
(except FASTQ with empty lines between records, which it must refuse), and
counting from text on the device must equal the oracle's histogram."""
from __future__ import annotations

import random

import numpy as np
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


def _same(a, b):
    assert a.n_bases == b.n_bases and a.n_reads == b.n_reads
    nw, nm = (a.n_bases + 31) // 32, (a.n_bases + 63) // 64
    assert np.array_equal(a.read_start[: a.n_reads + 1], b.read_start[: b.n_reads + 1])
    assert np.array_equal(a.codes[:nw], b.codes[:nw])
    assert np.array_equal(a.nmask[:nm], b.nmask[:nm])


def _wrap(seq: bytes, width: int) -> bytes:
    return b"\n".join(seq[i:i + width] for i in range(0, len(seq), width)) if seq else b""


def _shapes():
    rnd = random.Random(5)
    alpha = b"ACGTacgtNnRYKM.- "
    seqs = [bytes(rnd.choice(alpha if rnd.random() < 0.1 else b"ACGT") for _ in range(rnd.randint(0, 300)))
            for _ in range(400)]
    fasta1 = b"".join(b">r%d\n" % i + s + b"\n" for i, s in enumerate(seqs))
    fasta_wrapped = b"".join(b">r%d desc\n" % i + _wrap(s, 61) + b"\n" for i, s in enumerate(seqs))
    fasta_blank = b"\n\n" + b"".join(b">r\n\n" + _wrap(s, 40) + b"\n\n" for s in seqs) + b">empty\n>e2\n"
    fasta_crlf = fasta_wrapped.replace(b"\n", b"\r\n")
    fasta_midcr = b">a\nAC\rGT\rNA\n>b\n\r\rACGT\r\n"
    fastq = b"".join(b"@q%d\n" % i + s + b"\n+\n" + b"I" * len(s) + b"\n" for i, s in enumerate(seqs))
    fastq_crlf = fastq.replace(b"\n", b"\r\n")
    fastq_noeol = fastq[:-1]
    fastq_trailing = fastq + b"\n\n\n"
    fastq_leading = b"\n\n" + fastq
    raw = b"\n".join(seqs) + b"\n"
    raw_blank = b"\n\n".join(seqs)
    return {"fasta1": fasta1, "fasta_wrapped": fasta_wrapped, "fasta_blank": fasta_blank, "fasta_crlf": fasta_crlf,
            "fasta_midcr": fasta_midcr, "fastq": fastq, "fastq_crlf": fastq_crlf, "fastq_noeol": fastq_noeol,
            "fastq_trailing": fastq_trailing, "fastq_leading": fastq_leading, "raw": raw, "raw_blank": raw_blank,
            "single": b"ACGTN", "empty": b"", "only_newlines": b"\n\n\n", "header_only": b">x\n"}


@pytest.mark.parametrize("name", list(_shapes()))
def test_device_parse_equals_host_reader(G, name):
    text = _shapes()[name]
    host = G.pack_reads(text)
    with G.Gerbil() as g:
        dev = g.parse_text(text)
    _same(dev, host)


def test_device_parse_synthetic_and_device_input(G):
    import torch

    w = synth.Workload(seed=3, genome_len=500_000, read_len=150, n_reads=200_000, err=0.004, nrate=0.003)
    for fmt in (synth.FASTQ, synth.FASTA, synth.RAW):
        text = synth.fastx(w, fmt)
        host = G.pack_reads(text)
        with G.Gerbil() as g:
            _same(g.parse_text(text), host)
            dt = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
            _same(g.parse_text(dt), host)  # text already in device memory


@pytest.mark.parametrize("bad,why", [
    (b"@a\nACGT\n+\nIIII\nxx\nACGT\n+\nIIII\n", "'@'"),
    (b"@a\nACGT\n-\nIIII\n", "'+'"),
    (b"@a\nACGT\n+\nIII\n", "quality"),
    (b"@a\nACGT\n+\n", "truncated"),
    (b"@a\nACGT\n+\nIIII\n\n@b\nAC\n+\nII\n", "empty line"),
])
def test_device_parse_errors(G, bad, why):
    with G.Gerbil() as g:
        with pytest.raises(G.GerbilError) as e:
            g.parse_text(bad)
        assert e.value.status == G.E_IO and why in str(e.value)


@pytest.mark.parametrize("k", [28, 40, 65])
def test_count_text_on_device(G, k):
    w = synth.Workload(seed=11, genome_len=100_000, read_len=100, n_reads=10_000, err=0.0025, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ).replace(b"\n", b"\r\n")
    ref = oracle.count(text, k)
    with G.Gerbil(n_bins=16) as g:
        g.count_text(text, k, 7, 1)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    compare(keys, counts, k, ref)
    assert st["valid_windows"] == ref.windows
