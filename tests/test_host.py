"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol include/gerbil.h declares; the host reader (step a) packs exactly what
the text says; the seeded generator is deterministic and its packed twin
matches its ASCII output. No compute call needs a GPU here."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

import synth
from tests.helpers import decode_packed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "gerbil.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gerbil_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1607_06618_b200 import gerbil

    lib = ctypes.CDLL(gerbil.library_path())
    declared = _declared_symbols()
    assert "gerbil_count" in declared and "gerbil_fetch" in declared and "gerbil_init" in declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/gerbil.h but not exported"
    assert sorted(gerbil.EXPORTED) == declared


def test_product_does_not_import_oracle():
    # the product path must never route through the oracle
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_1607_06618_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def _texts(reads):
    fa = b"".join(b">r%d\n" % i + r + b"\n" for i, r in enumerate(reads))
    fa_ml = b"".join(b">r%d\n" % i + b"\n".join(r[j:j + 13] for j in range(0, len(r), 13)) + b"\n"
                     for i, r in enumerate(reads))
    fq = b"".join(b"@r%d\n" % i + r + b"\n+\n" + b"I" * len(r) + b"\n" for i, r in enumerate(reads))
    return [fa, fa_ml, fq, fa.replace(b"\n", b"\r\n"), b"".join(r + b"\n" for r in reads if r)]


def test_reader_packs_exactly():
    from paper_1607_06618_b200 import gerbil

    rnd = random.Random(1)
    reads = [bytes(rnd.choice(b"ACGTacgtNnRY.") for _ in range(rnd.randint(1, 150))) for _ in range(97)]
    for t in _texts(reads):
        for threads in (1, 3, 8):
            p = gerbil.pack_reads(text=t, threads=threads)
            assert p.n_reads == len(reads)
            assert p.n_bases == sum(len(r) for r in reads)
            for i, r in enumerate(reads):
                s, e = int(p.read_start[i]), int(p.read_start[i + 1])
                expect = bytes(c if c in b"ACGT" else ord("N") for c in r.upper())
                assert decode_packed(p.codes, p.nmask, s, e - s) == expect


def test_reader_empty_and_errors(tmp_path):
    from paper_1607_06618_b200 import gerbil

    p = gerbil.pack_reads(text=b"")
    assert p.n_reads == 0 and p.n_bases == 0
    with pytest.raises(gerbil.GerbilError):
        gerbil.pack_reads(text=b"@r\nACGT\n-\nIIII\n")
    with pytest.raises(gerbil.GerbilError):
        gerbil.pack_reads(text=b"@r\nACGT\n+\nIII\n")
    with pytest.raises(gerbil.GerbilError):
        gerbil.pack_reads(paths=[str(tmp_path / "missing.fa")])
    f1, f2 = tmp_path / "a.fa", tmp_path / "b.fq"
    f1.write_bytes(b">x\nACGTACGTAC\n")
    f2.write_bytes(b"@y\nGGGNNTTT\n+\nIIIIIIII\n")
    p = gerbil.pack_reads(paths=[str(f1), str(f2)])
    assert p.n_reads == 2 and list(p.read_start) == [0, 10, 18]
    assert decode_packed(p.codes, p.nmask, 0, 18) == b"ACGTACGTACGGGNNTTT"


def test_synth_deterministic_and_shardable():
    w = synth.Workload(seed=5, genome_len=50_000, read_len=100, n_reads=300, err=0.01, nrate=0.002)
    a, b = synth.fastx(w, synth.RAW), synth.fastx(w, synth.RAW)
    assert a == b
    lines = a.split(b"\n")[:-1]
    assert len(lines) == 300 and all(len(l) == 100 for l in lines)
    s0, s1 = w.shard(0, 2), w.shard(1, 2)
    assert synth.fastx(s0, synth.RAW) + synth.fastx(s1, synth.RAW) == a
    # N rate and substitution rate roughly as requested
    n_frac = a.count(b"N") / 30000
    assert 0 < n_frac < 0.01
    w2 = synth.Workload(seed=6, genome_len=50_000, read_len=100, n_reads=300)
    assert synth.fastx(w2, synth.RAW) != synth.fastx(w, synth.RAW)


def test_synth_packed_twin_matches_ascii():
    w = synth.Workload(seed=3, genome_len=20_000, read_len=77, n_reads=211, err=0.02, nrate=0.01)
    codes, nmask, rs = synth.packed_host(w, threads=4)
    text = synth.fastx(w, synth.RAW).split(b"\n")[:-1]
    assert list(rs) == [i * 77 for i in range(212)]
    for i, r in enumerate(text):
        assert decode_packed(codes, nmask, i * 77, 77) == r


def test_reader_matches_synth_packing():
    from paper_1607_06618_b200 import gerbil

    w = synth.Workload(seed=9, genome_len=30_000, read_len=100, n_reads=500, err=0.01, nrate=0.003)
    codes, nmask, rs = synth.packed_host(w)
    p = gerbil.pack_reads(text=synth.fastx(w, synth.FASTQ))
    assert np.array_equal(p.read_start, rs)
    assert np.array_equal(p.codes[: len(codes)], codes)
    assert np.array_equal(p.nmask[: len(nmask)], nmask)


def test_reader_compressed_inputs(tmp_path):
    # PAPER.md:94 (§2.3.1 step 1) / App. B: FASTA/FASTQ "and compressed files of
    # these formats" — gzip (also several concatenated members, as BGZF writes) and bzip2
    # (also concatenated streams) decode to exactly the plain file's packed batch
    import bz2
    import gzip

    from paper_1607_06618_b200 import gerbil

    w = synth.Workload(seed=11, genome_len=40_000, read_len=150, n_reads=900, err=0.01, nrate=0.004)
    fq = synth.fastx(w, synth.FASTQ)
    fa = synth.fastx(w, synth.FASTA, line_width=60)
    plain = tmp_path / "r.fq"
    plain.write_bytes(fq)
    ref = gerbil.pack_reads(paths=[str(plain)])
    half = fq.index(b"\n@", len(fq) // 2) + 1
    variants = {
        "r.fq.gz": gzip.compress(fq),
        "r2.fq.gz": gzip.compress(fq[:half], 1) + gzip.compress(fq[half:], 9),  # two members
        "r.fq.bz2": bz2.compress(fq),
        "r2.fq.bz2": bz2.compress(fq[:half]) + bz2.compress(fq[half:]),          # two streams
    }
    for name, data in variants.items():
        f = tmp_path / name
        f.write_bytes(data)
        for threads in (1, 4):
            p = gerbil.pack_reads(paths=[str(f)], threads=threads)
            assert p.n_reads == ref.n_reads and p.n_bases == ref.n_bases, name
            assert np.array_equal(p.read_start, ref.read_start), name
            assert np.array_equal(p.codes, ref.codes) and np.array_equal(p.nmask, ref.nmask), name
    # several files, mixed codecs, loaded in parallel but packed in order
    (tmp_path / "a.fa.gz").write_bytes(gzip.compress(fa))
    both = gerbil.pack_reads(paths=[str(tmp_path / "a.fa.gz"), str(tmp_path / "r.fq.bz2"), str(plain)], threads=3)
    assert both.n_reads == 3 * ref.n_reads and both.n_bases == 3 * ref.n_bases
    nb = int(ref.n_bases)
    assert decode_packed(both.codes, both.nmask, nb, nb) == decode_packed(ref.codes, ref.nmask, 0, nb)
    assert decode_packed(both.codes, both.nmask, 2 * nb, nb) == decode_packed(ref.codes, ref.nmask, 0, nb)
    # damaged inputs fail with an I/O error naming the file
    for name, data in {"t.fq.gz": gzip.compress(fq)[:-40], "c.fq.gz": gzip.compress(fq)[:30] + b"\xff" * 64,
                       "t.fq.bz2": bz2.compress(fq)[:-30]}.items():
        f = tmp_path / name
        f.write_bytes(data)
        with pytest.raises(gerbil.GerbilError) as e:
            gerbil.pack_reads(paths=[str(f)])
        assert name in str(e.value)


@pytest.mark.parametrize("W,threads", [(1, 1), (2, 4), (7, 3)])
def test_merge_sorted_lists(W, threads):
    # host k-way merge of per-rank sorted results: disjoint key sets interleave
    # into one sorted list; a key in several lists sums its counts; empty lists are fine
    from paper_1607_06618_b200 import gerbil

    rng = np.random.default_rng(W)
    n_total = 200_000
    keys = np.unique(rng.integers(0, 2**63, size=(n_total, W), dtype=np.uint64), axis=0)
    counts = rng.integers(1, 1000, size=keys.shape[0]).astype(np.uint32)
    owner = rng.integers(0, 4, size=keys.shape[0])
    lists = [(keys[owner == r], counts[owner == r]) for r in range(4)] + [(np.zeros((0, W), np.uint64),
                                                                          np.zeros(0, np.uint32))]
    mk, mc = gerbil.merge_sorted(lists, threads=threads)
    assert np.array_equal(mk, keys) and np.array_equal(mc, counts)
    # overlapping lists (two independent jobs): union with summed counts
    a = (keys[::2], counts[::2])
    b = (keys[::3], counts[::3])
    mk, mc = gerbil.merge_sorted([a, b], threads=threads)
    idx2, idx3 = set(range(0, keys.shape[0], 2)), set(range(0, keys.shape[0], 3))
    both = sorted(idx2 | idx3)
    assert np.array_equal(mk, keys[both])
    exp = np.array([(counts[i] if i in idx2 else 0) + (counts[i] if i in idx3 else 0) for i in both], np.uint32)
    assert np.array_equal(mc, exp)
