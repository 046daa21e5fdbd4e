"""Test-harness helpers: its OWN decoder of the library's key layout
(include/gerbil.h: W u64 words, base 0 in bits 63:62), comparison against the
oracle, and small synthetic texts. Shares no code with the CUDA path."""
from __future__ import annotations

import numpy as np

LETTERS = np.frombuffer(b"ACGT", dtype=np.uint8)


def decode_keys(keys: np.ndarray, k: int) -> list[bytes]:
    """keys[n, W] uint64 → list of k-letter byte strings."""
    n = keys.shape[0]
    if n == 0:
        return []
    out = np.empty((n, k), np.uint8)
    for i in range(k):
        w = keys[:, i // 32]
        out[:, i] = LETTERS[((w >> np.uint64(62 - 2 * (i % 32))) & np.uint64(3)).astype(np.int64)]
    return [bytes(r) for r in out]


def decode_packed(codes: np.ndarray, nmask: np.ndarray, start: int, length: int) -> bytes:
    """Bases [start, start+length) of a packed batch; N-mask bits decode as 'N'."""
    idx = np.arange(start, start + length, dtype=np.uint64)
    c = (codes[(idx >> np.uint64(5)).astype(np.int64)] >> (np.uint64(62) - np.uint64(2) * (idx & np.uint64(31)))) & np.uint64(3)
    nm = (nmask[(idx >> np.uint64(6)).astype(np.int64)] >> (np.uint64(63) - (idx & np.uint64(63)))) & np.uint64(1)
    s = LETTERS[c.astype(np.int64)].copy()
    s[nm.astype(bool)] = ord("N")
    return bytes(s)


def as_dict(strings: list[bytes], counts) -> dict[bytes, int]:
    return dict(zip(strings, (int(c) for c in counts)))


def compare(gpu_keys: np.ndarray, gpu_counts: np.ndarray, k: int, ref) -> None:
    """Element-by-element comparison of sorted GPU output with the oracle's sorted list."""
    got = decode_keys(gpu_keys, k)
    n = min(len(got), len(ref.kmers))
    for i in range(n):
        if got[i] != ref.kmers[i] or int(gpu_counts[i]) != ref.counts[i]:
            raise AssertionError(
                f"first mismatch at {i}: gpu ({got[i]!r}, {int(gpu_counts[i])}) vs oracle "
                f"({ref.kmers[i]!r}, {ref.counts[i]}); gpu n={len(got)} oracle n={len(ref.kmers)}")
    assert len(got) == len(ref.kmers), f"gpu n={len(got)} oracle n={len(ref.kmers)}"
