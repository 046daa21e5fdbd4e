"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs — bit-exact sorted (k-mer, count) lists.

Covers every key-word boundary up to k=479, several m / bin counts / thresholds,
both read entry points (host reader, device-resident batch), the emergency
(overflow) path, step (b) properties, invariances and degenerate inputs.
"""
import random
import threading

import numpy as np
import pytest

import oracle
import synth
from tests.helpers import compare, decode_keys, decode_packed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1607_06618_b200 import gerbil

    return gerbil


# configs[0] of BASELINE.json: 10k synthetic 100-bp reads (1 Mbp), k=28, m=7, single bin, min_count=1
C0 = synth.Workload(seed=1, genome_len=100_000, read_len=100, n_reads=10_000, err=0.0025, nrate=0.001)


def _gpu_count_text(G, text, k, m=0, min_count=1, **kw):
    with G.Gerbil(**kw) as g:
        g.count(k, m, min_count, text=text)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    return keys, counts, st


def test_c0_parity_host_reader(G):
    text = synth.fastx(C0, synth.FASTQ)
    ref = oracle.count(text, 28, 1)
    keys, counts, st = _gpu_count_text(G, text, 28, 7, 1, n_bins=1)
    compare(keys, counts, 28, ref)
    assert st["valid_windows"] == ref.windows == st["count_sum"]
    assert st["distinct"] == ref.distinct


def test_c0_parity_device_batch(G):
    import torch

    text = synth.fastx(C0, synth.FASTQ)
    ref = oracle.count(text, 28, 1)
    codes, nmask, rs = synth.packed_device(C0)
    torch.cuda.synchronize()
    with G.Gerbil(n_bins=1) as g:
        g.count_device(codes, nmask, rs, C0.n_reads, 28, 7, 1)
        keys, counts = g.fetch(sorted=True)
    compare(keys, counts, 28, ref)


def test_device_twin_equals_host_twin(G):
    import torch

    w = synth.Workload(seed=4, genome_len=40_000, read_len=150, n_reads=3001, err=0.01, nrate=0.01)
    hc, hn, hr = synth.packed_host(w)
    dc, dn, dr = synth.packed_device(w)
    torch.cuda.synchronize()
    assert np.array_equal(dc.cpu().numpy().view(np.uint64)[: len(hc)], hc)
    assert np.array_equal(dn.cpu().numpy().view(np.uint64)[: len(hn)], hn)
    assert np.array_equal(dr.cpu().numpy().view(np.uint64), hr)


KS = [28, 31, 32, 33, 40, 56, 63, 64, 65, 96, 97, 100, 128, 129, 160, 161, 192, 193, 200]


@pytest.mark.parametrize("k", KS)
def test_parity_every_word_boundary(G, k):
    w = synth.Workload(seed=100 + k, genome_len=60_000, read_len=260, n_reads=700, err=0.004, nrate=0.0005)
    text = synth.fastx(w, synth.FASTA, line_width=61)
    ref = oracle.count(text, k, 1)
    keys, counts, st = _gpu_count_text(G, text, k, 11 if k > 100 else 7, 1, n_bins=64)
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows


# k beyond 200, up to the paper's maximum 479 (App. A "-k: Supported k range from
# 8 to 479"): every key-word boundary of W = 7..15 on 700-bp reads
KS_WIDE = [201, 223, 224, 225, 256, 257, 300, 383, 384, 385, 448, 449, 479]


@pytest.mark.parametrize("k", KS_WIDE)
def test_parity_wide_keys(G, k):
    w = synth.Workload(seed=300 + k, genome_len=80_000, read_len=700, n_reads=400, err=0.004, nrate=0.0005)
    text = synth.fastx(w, synth.FASTA, line_width=80)
    ref = oracle.count(text, k, 1)
    with G.Gerbil(n_bins=64) as g:
        g.count(k, 11, 1, text=text)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
        binary = g.encode_results(G.FMT_BINARY, sorted=True) if k in (300, 479) else None
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows and st["W"] == (k + 31) // 32
    if binary is not None:  # App. C records: ceil(k/4) = 75 / 120 key bytes
        assert binary == b"".join(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))


@pytest.mark.parametrize("m,B", [(5, 1), (7, 8), (9, 512), (11, 4096), (15, 100), (3, 7)])
def test_parity_invariant_in_m_and_bins(G, m, B):
    w = synth.Workload(seed=77, genome_len=30_000, read_len=100, n_reads=3000, err=0.003, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 40, 1)
    keys, counts, _ = _gpu_count_text(G, text, 40, m, 1, n_bins=B)
    compare(keys, counts, 40, ref)


@pytest.mark.parametrize("min_count", [1, 2, 3, 7])
def test_parity_threshold(G, min_count):
    w = synth.Workload(seed=5, genome_len=20_000, read_len=100, n_reads=3000, err=0.003, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 56, min_count)
    keys, counts, st = _gpu_count_text(G, text, 56, 7, min_count)
    compare(keys, counts, 56, ref)
    assert st["count_sum"] == ref.windows and st["distinct"] == ref.distinct


def test_parity_lex_ordering(G):
    w = synth.Workload(seed=8, genome_len=20_000, read_len=120, n_reads=1000, err=0.01)
    text = synth.fastx(w, synth.FASTA)
    ref = oracle.count(text, 33, 1)
    keys, counts, _ = _gpu_count_text(G, text, 33, 6, 1, ordering=G.ORDER_LEX, n_bins=32)
    compare(keys, counts, 33, ref)


# ---- degenerate inputs ----------------------------------------------------------
def test_empty_and_short_inputs(G):
    for text in (b"", b">a\nACGT\n", b">a\nACGTNACGTACG\n>b\n\n", b"@q\n\n+\n\n"):
        keys, counts, st = _gpu_count_text(G, text, 8)
        ref = oracle.count(text, 8)
        compare(keys, counts, 8, ref)
        assert st["count_sum"] == ref.windows


def test_all_a_heavy_contention(G):
    # every window is the same canonical key: maximal claim/count contention on one slot
    text = b"".join(b">a\n" + b"A" * 1000 + b"\n" for _ in range(2000)) + b">t\n" + b"T" * 5000 + b"\n"
    for k in (8, 32, 33, 64, 65, 200):
        keys, counts, _ = _gpu_count_text(G, text, k)
        assert decode_keys(keys, k) == [b"A" * k]
        assert int(counts[0]) == 2000 * (1000 - k + 1) + (5000 - k + 1)


def test_low_complexity_and_n_runs(G):
    rnd = random.Random(3)
    reads = []
    for _ in range(400):
        unit = bytes(rnd.choice(b"ACGT") for _ in range(rnd.randint(1, 4)))
        r = (unit * 200)[: rnd.randint(20, 300)]
        r = bytearray(r)
        for _ in range(rnd.randint(0, 5)):
            p = rnd.randrange(len(r))
            r[p:p + rnd.randint(1, 10)] = b"N" * len(r[p:p + rnd.randint(1, 10)])
        reads.append(bytes(r))
    text = b"".join(b">r\n" + r + b"\n" for r in reads)
    for k in (12, 31, 47):
        ref = oracle.count(text, k)
        keys, counts, _ = _gpu_count_text(G, text, k)
        compare(keys, counts, k, ref)


def test_de_bruijn_on_gpu(G):
    from tests.test_oracle import _de_bruijn

    s = _de_bruijn(9)
    keys, counts, _ = _gpu_count_text(G, b">db\n" + s + b"\n", 9, 4, n_bins=16)
    assert len(counts) == 4**9 // 2 and set(counts.tolist()) == {2}


def test_rc_input_doubles_counts_gpu(G):
    w = synth.Workload(seed=13, genome_len=20_000, read_len=90, n_reads=2000, err=0.01)
    reads = synth.fastx(w, synth.RAW).split(b"\n")[:-1]
    t1 = b"".join(b">r\n" + r + b"\n" for r in reads)
    t2 = t1 + b"".join(b">q\n" + oracle.reverse_complement(r) + b"\n" for r in reads)
    k1, c1, _ = _gpu_count_text(G, t1, 45)
    k2, c2, _ = _gpu_count_text(G, t2, 45)
    assert np.array_equal(k1, k2) and np.array_equal(2 * c1.astype(np.int64), c2.astype(np.int64))


# ---- emergency mechanism ------------------------------------------
@pytest.mark.parametrize("k", [28, 65, 200, 479])
def test_overflow_path_exact(G, k):
    w = synth.Workload(seed=21, genome_len=50_000, read_len=max(250, k + 200), n_reads=800, err=0.01)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, k)
    # θ = 1 bucket and an over-full table: many k-mers take the emergency path
    keys, counts, st = _gpu_count_text(G, text, k, 9, 1, max_probes=1, target_load=1.6,
                                       distinct_ratio=0.3, n_bins=4, count_mode=G.COUNT_L2)
    compare(keys, counts, k, ref)
    assert st["overflow_kmers"] > 0 and st["overflow_passes"] == 1


def test_recount_when_emergency_area_exhausted(G):
    w = synth.Workload(seed=22, genome_len=200_000, read_len=100, n_reads=4000, err=0.01)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 40)
    # ρ̂ far too small: overflow exceeds the emergency area → waves are recounted
    keys, counts, st = _gpu_count_text(G, text, 40, 7, 1, distinct_ratio=0.001, max_probes=2,
                                       count_mode=G.COUNT_L2)
    compare(keys, counts, 40, ref)
    assert st["ratio_used"] > 0.001


def test_repeated_calls_and_ratio_adaptation(G):
    w = synth.Workload(seed=23, genome_len=30_000, read_len=100, n_reads=3000, err=0.003)
    text = synth.fastx(w, synth.FASTQ)
    ref = oracle.count(text, 40)
    with G.Gerbil() as g:
        for _ in range(3):
            g.count(40, 7, 1, text=text)
            keys, counts = g.fetch(sorted=True)
            compare(keys, counts, 40, ref)
        assert g.stats()["ratio_used"] < 0.5  # adapted to the observed distinct/total ratio


# ---- step (b) properties ----------------------------------------------------------------
@pytest.mark.parametrize("kernel", ["tile", "reads"])
def test_fig1_supermers_on_gpu(G, kernel, monkeypatch):
    # PAPER.md:58 Fig. 1 with the lexicographic ordering (strand-symmetric gives the same cuts)
    monkeypatch.setenv("GERBIL_SUPERMER_KERNEL", kernel)
    p = G.pack_reads(text=b">fig1\nCAAGAACAGTG\n")
    with G.Gerbil(ordering=G.ORDER_LEX, n_bins=4) as g:
        pos, nwin, b, mu = g.debug_supermers(p, 4, 3)
    order = np.argsort(pos)
    sms = [decode_packed(p.codes, p.nmask, int(pos[i]), int(nwin[i]) + 3) for i in order]
    assert sms == [b"CAAGA", b"AGAA", b"GAACA", b"ACAG", b"CAGTG"]


@pytest.mark.parametrize("kernel", ["tile", "reads"])
@pytest.mark.parametrize("k", [12, 28, 40, 56, 65])
def test_both_supermer_kernels_parity(G, kernel, k, monkeypatch):
    # step (b) has a tile kernel and a read-per-lane kernel (w <= 64); both must give the
    # oracle's histogram on reads with N runs, varied lengths, reads shorter than k
    monkeypatch.setenv("GERBIL_SUPERMER_KERNEL", kernel)
    rnd = random.Random(k)
    reads = []
    for _ in range(3000):
        r = bytearray(rnd.choice(b"ACGT") for _ in range(rnd.randint(1, 400)))
        for _ in range(rnd.randint(0, 3)):
            p = rnd.randrange(len(r))
            r[p:p + 3] = b"NNN"[: len(r[p:p + 3])]
        reads.append(bytes(r))
    text = b"".join(b">r\n" + r + b"\n" for r in reads)
    ref = oracle.count(text, k)
    keys, counts, st = _gpu_count_text(G, text, k, 7, 1, n_bins=64)
    compare(keys, counts, k, ref)
    assert st["valid_windows"] == ref.windows


@pytest.mark.parametrize("kernel", ["tile", "reads"])
@pytest.mark.parametrize("k,m,ordering", [(28, 7, 0), (40, 9, 0), (65, 11, 1), (200, 15, 0), (9, 3, 0)])
def test_supermer_properties(G, k, m, ordering, kernel, monkeypatch):
    monkeypatch.setenv("GERBIL_SUPERMER_KERNEL", kernel)
    w = synth.Workload(seed=31, genome_len=10_000, read_len=300, n_reads=200, err=0.01, nrate=0.003)
    text = synth.fastx(w, synth.RAW)
    p = G.pack_reads(text=text)
    with G.Gerbil(ordering=ordering, n_bins=97) as g:
        pos, nwin, b, mu = g.debug_supermers(p, k, m)
    reads = text.split(b"\n")[:-1]
    # window multiset: super-mer windows == valid (N-free, in-read) windows
    valid = []
    for i, r in enumerate(reads):
        for j in range(len(r) - k + 1):
            if b"N" not in r[j:j + k]:
                valid.append(i * 300 + j)
    got = np.sort(np.concatenate([np.arange(int(a), int(a) + int(n)) for a, n in zip(pos, nwin)]))
    assert np.array_equal(got, np.array(sorted(valid), dtype=got.dtype))
    # every window has the super-mer's minimizer (oracle definition), bin is a function of it
    rnd = random.Random(1)
    mask = (1 << (2 * m)) - 1
    bin_of = {}
    for i in rnd.sample(range(len(pos)), min(300, len(pos))):
        mmer = bytes(b"ACGT"[(int(mu[i]) & mask) >> (2 * (m - 1 - t)) & 3] for t in range(m))
        for j in range(int(nwin[i])):
            q = int(pos[i]) + j
            kmer = reads[q // 300][q % 300: q % 300 + k]
            assert oracle.minimizer(kmer, m, ordering) == mmer
        assert bin_of.setdefault(int(mu[i]), int(b[i])) == int(b[i])


# ---- usage errors (include/gerbil.h validation) ---------------------------------------
def test_usage_errors(G):
    with G.Gerbil() as g:
        with pytest.raises(G.GerbilError) as e:
            g.fetch()
        assert e.value.status == G.E_STATE
        for k, m, l in ((7, 3, 1), (480, 7, 1), (28, 28, 1), (28, 16, 1), (28, 7, 0)):
            with pytest.raises(G.GerbilError) as e:
                g.count(k, m, l, text=b">a\nACGT\n")
            assert e.value.status == G.E_USAGE
        with pytest.raises(G.GerbilError) as e:
            g.count(28, 7, 1, text=b"@r\nACGT\n+\nII\n")
        assert e.value.status == G.E_IO


# ---- the exchange path on one GPU: NCCL (1-rank communicator) and loopback -------------
@pytest.mark.parametrize("backend", [0, 1])
def test_forced_exchange_single_rank(G, backend):
    # world = 1 but the full multi-rank shuffle runs: histogram all-gather, LPT owners,
    # pack into the send buffer, grouped send/recv to self, regroup of received super-mers
    w = synth.Workload(seed=43, genome_len=30_000, read_len=120, n_reads=4000, err=0.004, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    for k in (33, 65):
        ref = oracle.count(text, k)
        keys, counts, st = _gpu_count_text(G, text, k, 7, 1, force_exchange=True, comm_backend=backend,
                                           n_bins=128)
        compare(keys, counts, k, ref)
        assert st["count_sum"] == ref.windows


@pytest.mark.parametrize("backend", [0, 1])
def test_forced_group_exchange_single_rank(G, backend):
    # world = 1, exchange forced, 2^16 bins: the group exchange path (NCCL to self / loopback)
    w = synth.Workload(seed=44, genome_len=30_000, read_len=150, n_reads=4000, err=0.004, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ)
    for k in (40, 65, 130):
        ref = oracle.count(text, k)
        keys, counts, st = _gpu_count_text(G, text, k, 15, 1, force_exchange=True, comm_backend=backend,
                                           n_bins=1 << 16)
        compare(keys, counts, k, ref)
        assert st["count_sum"] == ref.windows and st["smem_windows"] > 0


# ---- multi-rank shard logic: loopback group (P virtual ranks on one GPU) ---------------
@pytest.mark.parametrize("P", [2, 3, 4])
def test_loopback_ranks_parity(G, P):
    w = synth.Workload(seed=41, genome_len=40_000, read_len=100, n_reads=6000, err=0.004, nrate=0.001)
    ref = oracle.count(synth.fastx(w, synth.FASTQ), 56)
    uid = bytes([P]) * 128
    results = [None] * P
    errors = []

    def rank(r):
        try:
            with G.Gerbil(rank=r, world=P, unique_id=uid, comm_backend=1, n_bins=256) as g:
                g.count(56, 7, 1, text=synth.fastx(w.shard(r, P), synth.FASTQ))
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
    strs = decode_keys(keys, 56)
    order = sorted(range(len(strs)), key=lambda i: strs[i])
    compare(keys[order], counts[order], 56, ref)
    assert sum(r[2]["count_sum"] for r in results) == ref.windows
    assert all(r[2]["bytes_recv"] > 0 for r in results)


# ---- NEXT(2): -d non-canonical mode and the paper's output encodings ----------------------
@pytest.mark.parametrize("k", [12, 31, 32, 33, 40, 64, 65, 100])
def test_parity_non_canonical(G, k):
    # PAPER.md:483 `-d`: a k-mer and its reverse complement are different k-mers
    w = synth.Workload(seed=300 + k, genome_len=20_000, read_len=150, n_reads=1500, err=0.004, nrate=0.001)
    text = synth.fastx(w, synth.FASTQ) + b"@t\n" + b"T" * 80 + b"\n+\n" + b"I" * 80 + b"\n"
    ref = oracle.count(text, k, 1, canonical=False)
    keys, counts, st = _gpu_count_text(G, text, k, 7, 1, canonical=False, n_bins=32)
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows


@pytest.mark.parametrize("k,min_count", [(28, 1), (40, 2), (65, 1)])
def test_binary_and_csv_output(G, k, min_count, tmp_path):
    # App. C records byte-exact against the oracle's encoder, counts >= 255
    # exercised by a repeated read; CSV (`-x h`) line-exact
    w = synth.Workload(seed=7, genome_len=5_000, read_len=100, n_reads=2000, err=0.002)
    rep = b"ACGTTGCA" * 12
    text = synth.fastx(w, synth.FASTQ) + b"".join(b"@r\n" + rep + b"\n+\n" + b"I" * len(rep) + b"\n"
                                                  for _ in range(300))
    ref = oracle.count(text, k, min_count)
    with G.Gerbil() as g:
        g.count(k, 7, min_count, text=text)
        binary = g.encode_results(G.FMT_BINARY, sorted=True)
        csv = g.encode_results(G.FMT_CSV, sorted=True)
        g.write_results(str(tmp_path / "out.bin"), G.FMT_BINARY, sorted=True)
    assert binary == b"".join(oracle.encode_entry(x, c) for x, c in zip(ref.kmers, ref.counts))
    assert max(ref.counts) >= 255
    assert csv == b"".join(x + b"," + str(c).encode() + b"\n" for x, c in zip(ref.kmers, ref.counts))
    assert (tmp_path / "out.bin").read_bytes() == binary


# ---- compressed input: gzip / bzip2 files through gerbil_count(paths) --------
@pytest.mark.parametrize("codec", ["gzip", "bz2"])
def test_parity_compressed_files(G, codec, tmp_path):
    import bz2
    import gzip

    w = synth.Workload(seed=61, genome_len=60_000, read_len=150, n_reads=4000, err=0.004, nrate=0.002)
    fq = synth.fastx(w, synth.FASTQ)
    fq2 = synth.fastx(w.shard(0, 2), synth.FASTQ)
    comp = gzip.compress if codec == "gzip" else bz2.compress
    paths = [tmp_path / f"a.fq.{codec}", tmp_path / f"b.fq.{codec}"]
    paths[0].write_bytes(comp(fq))
    paths[1].write_bytes(comp(fq2))
    # the harness decompresses with Python's own codec; the oracle counts the plain texts
    plain = b"".join((gzip.decompress if codec == "gzip" else bz2.decompress)(p.read_bytes()) for p in paths)
    ref = oracle.count(plain, 40, 1)
    with G.Gerbil() as g:
        g.count(40, 11, 1, paths=[str(p) for p in paths])
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    compare(keys, counts, 40, ref)
    assert st["count_sum"] == ref.windows


# ---- world > 1 with the device bin plan: whole groups of 1024 bins exchanged ----------------
@pytest.mark.parametrize("P,k", [(2, 40), (4, 40), (3, 65), (2, 150), (4, 201)])
def test_loopback_group_exchange(G, P, k):
    # 2^16 bins (the device plan): every rank groups its super-mers, the per-group histograms are
    # all-gathered, whole groups go to their LPT owner in one grouped all-to-all (descriptors,
    # bins, payload), and each owner counts its groups with the shared-memory / reference tables
    w = synth.Workload(seed=90 + k, genome_len=60_000, read_len=250, n_reads=3000, err=0.006, nrate=0.001)
    ref = oracle.count(synth.fastx(w, synth.FASTQ), k)
    uid = bytes([P + 16 * (k % 7)]) * 128
    results = [None] * P
    errors = []

    def rank(r):
        try:
            with G.Gerbil(rank=r, world=P, unique_id=uid, comm_backend=1, n_bins=1 << 16) as g:
                g.count(k, 15, 1, text=synth.fastx(w.shard(r, P), synth.FASTQ))
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
    strs = decode_keys(keys, k)
    order = sorted(range(len(strs)), key=lambda i: strs[i])
    compare(keys[order], counts[order], k, ref)
    assert sum(r[2]["count_sum"] for r in results) == ref.windows
    assert all(r[2]["smem_windows"] > 0 and r[2]["bytes_recv"] > 0 for r in results)


def test_loopback_auto_bins_agree(G):
    # n_bins = 0 (auto) with world > 1: the ranks derive B from the all-gathered totals
    P, k = 2, 40
    w = synth.Workload(seed=5, genome_len=40_000, read_len=120, n_reads=4000, err=0.004)
    ref = oracle.count(synth.fastx(w, synth.FASTQ), k)
    uid = b"\x7f" * 128
    results, errors = [None] * P, []

    def rank(r):
        try:
            with G.Gerbil(rank=r, world=P, unique_id=uid, comm_backend=1) as g:
                g.count(k, 15, 1, text=synth.fastx(w.shard(r, P), synth.FASTQ))
                results[r] = g.fetch(sorted=True) + (g.stats(),)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    assert results[0][2]["n_bins"] == results[1][2]["n_bins"]
    keys = np.concatenate([r[0] for r in results])
    counts = np.concatenate([r[1] for r in results])
    strs = decode_keys(keys, k)
    order = sorted(range(len(strs)), key=lambda i: strs[i])
    compare(keys[order], counts[order], k, ref)


# ---- sorted fetch: device LSD radix sort (sort.cu) ------------------------------------------
@pytest.mark.parametrize("k,read_len", [(28, 150), (40, 150), (100, 300), (479, 700)])
def test_device_sorted_fetch_matches_lexsort(G, k, read_len):
    # the sorted fetch (device radix sort over the 2k meaningful bits) equals numpy's lexicographic
    # sort of the unsorted fetch, for ~10^6 results (hundreds of tiles, ragged tail)
    w = synth.Workload(seed=k, genome_len=2_000_000, read_len=read_len, n_reads=max(2000, 3_000_000 // read_len),
                       err=0.01)
    codes, nmask, rs = synth.packed_device(w)
    import torch

    torch.cuda.synchronize()
    with G.Gerbil() as g:
        g.count_device(codes, nmask, rs, w.n_reads, k, 15, 1)
        uk, uc = g.fetch(sorted=False)
        sk, sc = g.fetch(sorted=True)
        sk2, sc2 = g.fetch(sorted=False)  # stays sorted on the device
    assert uk.shape[0] > 100_000
    order = np.lexsort(tuple(uk[:, j] for j in reversed(range(uk.shape[1]))))
    assert np.array_equal(sk, uk[order]) and np.array_equal(sc, uc[order])
    assert np.array_equal(sk2, sk) and np.array_equal(sc2, sc)


@pytest.mark.parametrize("k,bins", [(40, 1 << 16), (28, 1 << 22)])
def test_group_shuffle_wide_counters(G, monkeypatch, k, bins):
    # the bin shuffle's 64-bit-counter regroup instance (needed only when a fine bin could hold
    # 2^32 windows) forced on a small input: same histogram
    import torch

    monkeypatch.setenv("GERBIL_REGROUP_WIDE", "1")
    text = synth.fastx(C0, synth.FASTQ)
    ref = oracle.count(text, k, 1)
    codes, nmask, rs = synth.packed_device(C0)
    torch.cuda.synchronize()
    with G.Gerbil(n_bins=bins) as g:
        g.count_device(codes, nmask, rs, C0.n_reads, k, 15, 1)
        keys, counts = g.fetch(sorted=True)
        st = g.stats()
    compare(keys, counts, k, ref)
    assert st["count_sum"] == ref.windows
