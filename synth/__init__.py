"""ctypes wrapper of libsynth.so — the seeded synthetic read generator.

Shared by the oracle side (ASCII FASTA/FASTQ) and the CUDA side (packed batch
written straight into device memory). Holds no arithmetic of the counting
method; see synth/synth_core.h for the recipe.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None

RAW, FASTA, FASTQ = 0, 1, 2


class Params(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("genome_len", C.c_uint64),
        ("read_len", C.c_uint64),
        ("n_reads", C.c_uint64),
        ("first_read", C.c_uint64),
        ("n_thr", C.c_uint32),
        ("s_thr", C.c_uint32),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise ImportError(f"{_PATH} missing; run build_native.py")
        L = C.CDLL(_PATH)
        L.synth_fastx.argtypes = [C.POINTER(Params), C.c_int, C.c_uint32, C.c_void_p, C.c_uint64, C.c_int]
        L.synth_fastx.restype = C.c_uint64
        L.synth_packed_host.argtypes = [C.POINTER(Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        L.synth_packed_device.argtypes = [C.POINTER(Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.synth_packed_device.restype = C.c_int
        _lib = L
    return _lib


def _thr(p: float) -> int:
    return min(int(round(p * 2**32)), 2**32 - 1)


@dataclass
class Workload:
    """Synthetic reads shaped like a paper dataset."""
    seed: int
    genome_len: int
    read_len: int
    n_reads: int
    err: float = 0.0       # substitution probability per base
    nrate: float = 0.0     # probability a base is 'N'
    first_read: int = 0

    def params(self) -> Params:
        return Params(self.seed, self.genome_len, self.read_len, self.n_reads, self.first_read,
                      _thr(self.nrate), _thr(self.err))

    @property
    def n_bases(self) -> int:
        return self.n_reads * self.read_len

    def shard(self, rank: int, world: int) -> "Workload":
        per = (self.n_reads + world - 1) // world
        a = min(self.n_reads, rank * per)
        b = min(self.n_reads, a + per)
        return Workload(self.seed, self.genome_len, self.read_len, b - a, self.err, self.nrate,
                        self.first_read + a)


def fastx(w: Workload, fmt: int = FASTQ, line_width: int = 0, threads: int = 0) -> bytes:
    p = w.params()
    need = lib().synth_fastx(C.byref(p), fmt, line_width, None, 0, threads)
    buf = C.create_string_buffer(need)
    lib().synth_fastx(C.byref(p), fmt, line_width, buf, need, threads)
    return buf.raw[:need]


def packed_host(w: Workload, threads: int = 0):
    """(codes, nmask, read_start) numpy arrays in the include/gerbil.h layout."""
    nb = w.n_bases
    codes = np.zeros(max((nb + 31) // 32, 1), np.uint64)
    nmask = np.zeros(max((nb + 63) // 64, 1), np.uint64)
    rs = np.zeros(w.n_reads + 1, np.uint64)
    p = w.params()
    lib().synth_packed_host(C.byref(p), codes.ctypes.data, nmask.ctypes.data, rs.ctypes.data, threads)
    return codes, nmask, rs


def packed_device(w: Workload, device="cuda", stream: int | None = None):
    """Same batch generated in device memory (torch tensors)."""
    import torch

    nb = w.n_bases
    codes = torch.empty(max((nb + 31) // 32, 1) + 1, dtype=torch.int64, device=device)
    nmask = torch.empty(max((nb + 63) // 64, 1) + 1, dtype=torch.int64, device=device)
    rs = torch.empty(w.n_reads + 1, dtype=torch.int64, device=device)
    p = w.params()
    if stream is None:
        stream = torch.cuda.current_stream(device).cuda_stream
    st = lib().synth_packed_device(C.byref(p), codes.data_ptr(), nmask.data_ptr(), rs.data_ptr(), stream)
    if st != 0:
        raise RuntimeError(f"synth_packed_device failed: cuda error {st}")
    return codes, nmask, rs
