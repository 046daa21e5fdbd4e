"""ctypes wrapper of liboracle.so — the CPU ORACLE (see oracle/oracle.cpp).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package. The product
(paper_1607_06618_b200/) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise ImportError(f"{_PATH} missing; run build_native.py")
        L = C.CDLL(_PATH)
        P = C.c_void_p
        L.oracle_count.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_char_p, C.c_uint64]
        L.oracle_count.restype = P
        L.oracle_count_sampled.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
                                           C.c_char_p, C.c_uint64]
        L.oracle_count_sampled.restype = P
        for f in ("oracle_result_n", "oracle_result_windows", "oracle_result_distinct"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = C.c_uint64
        L.oracle_result_get.argtypes = [P, C.c_char_p, C.POINTER(C.c_uint64)]
        L.oracle_result_free.argtypes = [P]
        L.oracle_sample_keep.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64]
        L.oracle_reverse_complement.argtypes = [C.c_char_p, C.c_uint32, C.c_char_p]
        L.oracle_canonical.argtypes = [C.c_char_p, C.c_uint32, C.c_char_p]
        L.oracle_minimizer.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_char_p]
        L.oracle_supermers.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                       C.c_char_p, C.c_uint64]
        L.oracle_supermers.restype = C.c_uint64
        U32P = C.POINTER(C.c_uint32)
        L.oracle_minimizer_t.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, U32P, C.c_char_p]
        L.oracle_order_key.argtypes = [C.c_char_p, C.c_uint32, C.c_int, U32P]
        L.oracle_order_key.restype = C.c_uint32
        L.oracle_supermers_t.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int, U32P,
                                         C.c_char_p, C.c_uint64]
        L.oracle_supermers_t.restype = C.c_uint64
        L.oracle_dfp_table.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, U32P]
        L.oracle_dfp_table.restype = C.c_int
        L.oracle_minimizer_stats.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, U32P,
                                             C.POINTER(C.c_uint64)]
        L.oracle_minimizer_stats.restype = C.c_int64
        _lib = L
    return _lib


KMC2, LEX, CGAT, ROBERTS, RANDOM, DFP = 0, 1, 2, 3, 4, 5


def _table(table):
    """DFP key table (a dfp_table() result, or any sequence of 4^m ints) → ctypes array, or None."""
    if table is None or isinstance(table, C.Array):
        return table
    return (C.c_uint32 * len(table))(*[int(x) for x in table])


class Result:
    """Sorted (k-mer string, count) list plus totals."""

    def __init__(self, kmers: list[bytes], counts: list[int], windows: int, distinct: int):
        self.kmers, self.counts, self.windows, self.distinct = kmers, counts, windows, distinct

    def as_dict(self) -> dict[bytes, int]:
        return dict(zip(self.kmers, self.counts))


def _collect(h, k: int) -> Result:
    L = lib()
    n = L.oracle_result_n(h)
    buf = C.create_string_buffer(max(n * k, 1))
    cnt = (C.c_uint64 * max(n, 1))()
    L.oracle_result_get(h, buf, cnt)
    raw = buf.raw
    kmers = [raw[i * k:(i + 1) * k] for i in range(n)]
    res = Result(kmers, list(cnt[:n]), L.oracle_result_windows(h), L.oracle_result_distinct(h))
    L.oracle_result_free(h)
    return res


def count(text: bytes, k: int, min_count: int = 1, canonical: bool = True) -> Result:
    err = C.create_string_buffer(512)
    h = lib().oracle_count(text, len(text), k, min_count, 1 if canonical else 0, err, 512)
    if not h:
        raise ValueError(err.value.decode())
    return _collect(h, k)


def count_sampled(text: bytes, k: int, min_count: int = 1, mod: int = 4096, threads: int = 0) -> Result:
    err = C.create_string_buffer(512)
    h = lib().oracle_count_sampled(text, len(text), k, min_count, mod, threads, err, 512)
    if not h:
        raise ValueError(err.value.decode())
    return _collect(h, k)


def sample_keep(kmer: bytes, mod: int) -> bool:
    return bool(lib().oracle_sample_keep(kmer, len(kmer), mod))


def reverse_complement(x: bytes) -> bytes:
    out = C.create_string_buffer(len(x))
    lib().oracle_reverse_complement(x, len(x), out)
    return out.raw


def canonical(x: bytes) -> bytes:
    out = C.create_string_buffer(len(x))
    lib().oracle_canonical(x, len(x), out)
    return out.raw


def minimizer(kmer: bytes, m: int, ordering: int = KMC2, symmetric: bool = True, table=None) -> bytes:
    out = C.create_string_buffer(m)
    lib().oracle_minimizer_t(kmer, len(kmer), m, ordering, 1 if symmetric else 0, _table(table), out)
    return out.raw


def order_key(mmer: bytes, ordering: int, table=None) -> int:
    """The oracle's ordering key of one m-mer (x before y iff key(x) < key(y))."""
    return lib().oracle_order_key(mmer, len(mmer), ordering, _table(table))


def supermers(seq: bytes, k: int, m: int, ordering: int = LEX, symmetric: bool = False, table=None) -> list[bytes]:
    L = lib()
    t = _table(table)
    need = L.oracle_supermers_t(seq, len(seq), k, m, ordering, 1 if symmetric else 0, t, None, 0)
    buf = C.create_string_buffer(max(need, 1))
    L.oracle_supermers_t(seq, len(seq), k, m, ordering, 1 if symmetric else 0, t, buf, need)
    return [s for s in buf.raw[:need].split(b"\n") if s]


def dfp_table(text: bytes, m: int, pivot: float, stride: int):
    """dfp(p) keys of all 4^m m-mers from the sampled frequencies (oracle_dfp_table)."""
    out = (C.c_uint32 * (1 << (2 * m)))()
    if lib().oracle_dfp_table(text, len(text), m, pivot, stride, out) != 0:
        raise ValueError("parse error")
    return out  # a ctypes uint32 array (indexable, list(out) for a copy)


def minimizer_stats(text: bytes, k: int, m: int, ordering: int, table=None) -> tuple[int, int]:
    """(max distinct canonical k-mers per minimizer, minimizers owning >= 1 k-mer)."""
    n = C.c_uint64(0)
    mx = lib().oracle_minimizer_stats(text, len(text), k, m, ordering, _table(table), C.byref(n))
    if mx < 0:
        raise ValueError("parse error")
    return int(mx), n.value


def encode_entry(kmer: bytes, count: int) -> bytes:
    """App. C output record of one (k-mer, count) pair."""
    L = lib()
    L.oracle_encode_entry.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_char_p]
    L.oracle_encode_entry.restype = C.c_uint64
    n = L.oracle_encode_entry(kmer, len(kmer), count, None)
    buf = C.create_string_buffer(n)
    L.oracle_encode_entry(kmer, len(kmer), count, buf)
    return buf.raw[:n]
