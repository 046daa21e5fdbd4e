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
        _lib = L
    return _lib


KMC2, LEX = 0, 1


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


def minimizer(kmer: bytes, m: int, ordering: int = KMC2, symmetric: bool = True) -> bytes:
    out = C.create_string_buffer(m)
    lib().oracle_minimizer(kmer, len(kmer), m, ordering, 1 if symmetric else 0, out)
    return out.raw


def supermers(seq: bytes, k: int, m: int, ordering: int = LEX, symmetric: bool = False) -> list[bytes]:
    L = lib()
    need = L.oracle_supermers(seq, len(seq), k, m, ordering, 1 if symmetric else 0, None, 0)
    buf = C.create_string_buffer(max(need, 1))
    L.oracle_supermers(seq, len(seq), k, m, ordering, 1 if symmetric else 0, buf, need)
    return [s for s in buf.raw[:need].split(b"\n") if s]


def encode_entry(kmer: bytes, count: int) -> bytes:
    """App. C output record of one (k-mer, count) pair."""
    L = lib()
    L.oracle_encode_entry.argtypes = [C.c_char_p, C.c_uint32, C.c_uint64, C.c_char_p]
    L.oracle_encode_entry.restype = C.c_uint64
    n = L.oracle_encode_entry(kmer, len(kmer), count, None)
    buf = C.create_string_buffer(n)
    L.oracle_encode_entry(kmer, len(kmer), count, buf)
    return buf.raw[:n]
