"""Thin ctypes binding of the C ABI in include/gerbil.h (argument marshalling only).

Every step of the counting path runs in libgerbil.so; this module only moves
pointers and sizes across the boundary. Importing it without the built library
fails loudly: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libgerbil.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"{_LIB_PATH} is missing: build it with `python build_native.py`"
    )
_lib = C.CDLL(_LIB_PATH)

OK, E_USAGE, E_IO, E_INTERNAL, E_NOMEM, E_CUDA, E_NCCL, E_STATE = range(8)
FMT_BINARY, FMT_CSV = 0, 1
ORDER_KMC2, ORDER_LEX, ORDER_CGAT, ORDER_ROBERTS, ORDER_RANDOM, ORDER_DFP = 0, 1, 2, 3, 4, 5
COUNT_AUTO, COUNT_L2, COUNT_SMEM = 0, 1, 2  # gerbil_config.count_mode


class GerbilError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"gerbil status {status}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [
        ("struct_size", C.c_uint32),
        ("device", C.c_int32),
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("nccl_unique_id", C.c_void_p),
        ("comm_backend", C.c_int32),
        ("n_bins", C.c_uint32),
        ("ordering", C.c_int32),
        ("device_mem_cap", C.c_uint64),
        ("host_threads", C.c_int32),
        ("max_probes", C.c_uint32),
        ("distinct_ratio", C.c_double),
        ("target_load", C.c_double),
        ("wave_table_bytes", C.c_uint64),
        ("stream", C.c_void_p),
        ("timing", C.c_int32),
        ("force_exchange", C.c_int32),
        ("disable_normalization", C.c_int32),
        ("dfp_pivot", C.c_double),
        ("order_sample_stride", C.c_uint32),
        ("count_mode", C.c_int32),
    ]


class Reads(C.Structure):
    _fields_ = [
        ("paths", C.POINTER(C.c_char_p)),
        ("n_paths", C.c_uint32),
        ("text", C.c_char_p),
        ("text_len", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("input_bases", C.c_uint64),
        ("input_reads", C.c_uint64),
        ("valid_windows", C.c_uint64),
        ("supermers", C.c_uint64),
        ("owned_windows", C.c_uint64),
        ("distinct", C.c_uint64),
        ("kept", C.c_uint64),
        ("count_sum", C.c_uint64),
        ("overflow_kmers", C.c_uint64),
        ("probe_first", C.c_uint64),
        ("probe_more", C.c_uint64),
        ("probe_max", C.c_uint64),
        ("overflow_passes", C.c_uint32),
        ("waves", C.c_uint32),
        ("n_bins", C.c_uint32),
        ("W", C.c_uint32),
        ("max_bin_windows", C.c_uint64),
        ("bytes_sent", C.c_uint64),
        ("bytes_recv", C.c_uint64),
        ("ratio_used", C.c_double),
        ("ratio_observed", C.c_double),
        ("ms_h2d", C.c_double),
        ("ms_supermer", C.c_double),
        ("ms_shuffle", C.c_double),
        ("ms_count", C.c_double),
        ("ms_compact", C.c_double),
        ("ms_overflow", C.c_double),
        ("ms_total", C.c_double),
        ("ms_reader", C.c_double),
        ("launches_count", C.c_uint32),
        ("launches_compact", C.c_uint32),
        ("launches_total", C.c_uint32),
        ("smem_bins", C.c_uint64),
        ("smem_failed", C.c_uint64),
        ("smem_windows", C.c_uint64),
        ("smem_slots", C.c_uint32),
        ("launches_smem", C.c_uint32),
        ("ms_smem", C.c_double),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)
_lib.gerbil_config_default.argtypes = [C.POINTER(Config)]
_lib.gerbil_exchange_plan.argtypes = [C.c_void_p, C.c_uint32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
_lib.gerbil_init.argtypes = [C.POINTER(Config), C.POINTER(_P)]
_lib.gerbil_nccl_unique_id.argtypes = [_P, C.c_size_t]
_lib.gerbil_count.argtypes = [_P, C.POINTER(Reads), C.c_uint32, C.c_uint32, C.c_uint32]
_lib.gerbil_count_device.argtypes = [_P, _P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
_lib.gerbil_count_host_packed.argtypes = [_P, _P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
_lib.gerbil_minimizer_stats.argtypes = [_P, _U64P, _U64P]
_lib.gerbil_spill_begin.argtypes = [_P, C.c_uint32, C.c_uint32]
_lib.gerbil_parse_text.argtypes = [_P, _P, C.c_uint64, C.c_int32, _P, _P, _P, _U64P, _U64P]
_lib.gerbil_count_text.argtypes = [_P, _P, C.c_uint64, C.c_int32, C.c_uint32, C.c_uint32, C.c_uint32]
_lib.gerbil_spill_add.argtypes = [_P, _P, _P, _P, C.c_uint64]
_lib.gerbil_spill_finish.argtypes = [_P, C.c_uint32, _P, C.c_uint64, _U64P]
_lib.gerbil_count_host_stream.argtypes = [_P, _P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _P,
                                          C.c_uint64, _U64P]
_lib.gerbil_pack_reads.argtypes = [C.POINTER(Reads), C.c_int32, _P, _P, _P, _U64P, _U64P, C.c_char_p, C.c_size_t]
_lib.gerbil_fetch.argtypes = [_P, _P, _P, C.c_uint64, _U64P, C.c_int]
_lib.gerbil_merge_sorted.argtypes = [C.c_uint32, _P, _P, _P, C.c_uint32, C.c_int32, _P, _P, C.c_uint64, _U64P]
_lib.gerbil_results_device.argtypes = [_P, C.POINTER(_P), C.POINTER(_P), _U64P, C.POINTER(C.c_uint32)]
_lib.gerbil_get_stats.argtypes = [_P, C.POINTER(Stats)]
_lib.gerbil_last_error.argtypes = [_P]
_lib.gerbil_last_error.restype = C.c_char_p
_lib.gerbil_finalize.argtypes = [_P]
_lib.gerbil_encode_results.argtypes = [_P, C.c_int32, C.c_int, _P, C.c_uint64, _U64P]
_lib.gerbil_write_results.argtypes = [_P, C.c_char_p, C.c_int32, C.c_int]
_lib.gerbil_debug_supermers.argtypes = [_P, _P, _P, _P, C.c_uint64, C.c_uint32, C.c_uint32,
                                        _P, _P, _P, _P, C.c_uint64, _U64P]
for _f in ("gerbil_init", "gerbil_nccl_unique_id", "gerbil_count", "gerbil_count_device",
           "gerbil_count_host_packed", "gerbil_count_host_stream", "gerbil_minimizer_stats", "gerbil_pack_reads",
           "gerbil_spill_begin", "gerbil_spill_add", "gerbil_spill_finish", "gerbil_parse_text",
           "gerbil_count_text", "gerbil_fetch", "gerbil_results_device",
           "gerbil_get_stats", "gerbil_debug_supermers", "gerbil_encode_results", "gerbil_write_results",
           "gerbil_exchange_plan"):
    getattr(_lib, _f).restype = C.c_int

EXPORTED = [
    "gerbil_config_default", "gerbil_init", "gerbil_nccl_unique_id", "gerbil_count",
    "gerbil_count_device", "gerbil_count_host_packed", "gerbil_count_host_stream", "gerbil_pack_reads",
    "gerbil_fetch", "gerbil_minimizer_stats", "gerbil_spill_begin", "gerbil_spill_add", "gerbil_spill_finish",
    "gerbil_parse_text", "gerbil_count_text",
    "gerbil_results_device", "gerbil_get_stats", "gerbil_last_error", "gerbil_finalize",
    "gerbil_debug_supermers", "gerbil_encode_results", "gerbil_write_results", "gerbil_exchange_plan",
    "gerbil_merge_sorted",
]


def library_path() -> str:
    return _LIB_PATH


def _ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (host or device), or None."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _lib.gerbil_nccl_unique_id(buf, 128)
    if st != OK:
        raise GerbilError(st, "ncclGetUniqueId failed")
    return buf.raw


@dataclass
class ExchangePlan:
    owner: np.ndarray          # [n_bins] int32 owner rank of each bin
    send_desc_off: np.ndarray  # [world + 1] this rank's send layout (descriptors) by destination
    send_word_off: np.ndarray  # [world + 1] ... (payload words)
    recv_desc_off: np.ndarray  # [world + 1] receive layout by source
    recv_word_off: np.ndarray


def exchange_plan(hist: np.ndarray, rank: int) -> ExchangePlan:
    """Step (c) plan (host only): hist[world, 3, n_bins] u64 = per-rank windows, super-mers and
    payload words of every bin (the all-gathered step-(b) histograms)."""
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    world, three, n_bins = h.shape
    assert three == 3
    owner = np.zeros(n_bins, np.int32)
    offs = [np.zeros(world + 1, np.uint64) for _ in range(4)]
    st = _lib.gerbil_exchange_plan(_ptr(h), n_bins, world, rank, _ptr(owner), *(_ptr(o) for o in offs))
    if st != OK:
        raise GerbilError(st, "gerbil_exchange_plan failed")
    return ExchangePlan(owner, *offs)


def merge_sorted(lists: list[tuple[np.ndarray, np.ndarray]], threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """k-way merge (host, gerbil_merge_sorted) of sorted (keys[n, W] u64, counts[n] u32) lists —
    e.g. the sorted fetches of every rank — into one sorted list; equal keys sum their counts."""
    W = next((int(k.shape[1]) for k, _ in lists if k.ndim == 2), 1)
    ks = [np.ascontiguousarray(k, dtype=np.uint64).reshape(-1, W) for k, _ in lists]
    cs = [np.ascontiguousarray(c, dtype=np.uint32) for _, c in lists]
    kp = (C.c_void_p * max(len(ks), 1))(*[k.ctypes.data for k in ks])
    cp = (C.c_void_p * max(len(cs), 1))(*[c.ctypes.data for c in cs])
    n = np.array([k.shape[0] for k in ks], np.uint64)
    m = C.c_uint64()
    st = _lib.gerbil_merge_sorted(len(ks), C.cast(kp, C.c_void_p), C.cast(cp, C.c_void_p), _ptr(n), W, threads,
                                  None, None, 0, C.byref(m))
    if st != OK:
        raise GerbilError(st, "gerbil_merge_sorted failed")
    ok = np.zeros((m.value, W), np.uint64)
    oc = np.zeros(m.value, np.uint32)
    st = _lib.gerbil_merge_sorted(len(ks), C.cast(kp, C.c_void_p), C.cast(cp, C.c_void_p), _ptr(n), W, threads,
                                  _ptr(ok), _ptr(oc), m.value, C.byref(m))
    if st != OK:
        raise GerbilError(st, "gerbil_merge_sorted failed")
    return ok, oc


@dataclass
class PackedReads:
    codes: np.ndarray
    nmask: np.ndarray
    read_start: np.ndarray
    n_bases: int
    n_reads: int


def pack_reads(text: bytes | None = None, paths: list[str] | None = None, threads: int = 0) -> PackedReads:
    """Step (a) alone: FASTA/FASTQ → packed batch (include/gerbil.h layout)."""
    r, keep = _reads(text, paths)
    nb, nr = C.c_uint64(), C.c_uint64()
    err = C.create_string_buffer(512)
    st = _lib.gerbil_pack_reads(C.byref(r), threads, None, None, None, C.byref(nb), C.byref(nr), err, 512)
    if st != OK:
        raise GerbilError(st, err.value.decode())
    codes = np.zeros(max((nb.value + 31) // 32, 1), np.uint64)
    nmask = np.zeros(max((nb.value + 63) // 64, 1), np.uint64)
    rs = np.zeros(nr.value + 1, np.uint64)
    st = _lib.gerbil_pack_reads(C.byref(r), threads, _ptr(codes), _ptr(nmask), _ptr(rs), C.byref(nb),
                                C.byref(nr), err, 512)
    if st != OK:
        raise GerbilError(st, err.value.decode())
    del keep
    return PackedReads(codes, nmask, rs, nb.value, nr.value)


def _reads(text, paths):
    r = Reads()
    keep = []
    if text is not None:
        r.text = text
        r.text_len = len(text)
        keep.append(text)
    if paths:
        arr = (C.c_char_p * len(paths))(*[p.encode() for p in paths])
        r.paths = C.cast(arr, C.POINTER(C.c_char_p))
        r.n_paths = len(paths)
        keep.append(arr)
    return r, keep


class Gerbil:
    """One counting context (= one rank = one GPU)."""

    def __init__(self, device: int = -1, n_bins: int = 0, ordering: int = ORDER_KMC2, rank: int = 0,
                 world: int = 1, unique_id: bytes | None = None, comm_backend: int = 0,
                 max_probes: int = 0, distinct_ratio: float = 0.0, target_load: float = 0.0,
                 wave_table_bytes: int = 0, host_threads: int = 0, stream: int | None = None,
                 timing: bool = False, force_exchange: bool = False, canonical: bool = True,
                 dfp_pivot: float = 0.5, order_sample_stride: int = 0, count_mode: int = 0):
        cfg = Config()
        _lib.gerbil_config_default(C.byref(cfg))
        cfg.device = device
        cfg.n_bins = n_bins
        cfg.ordering = ordering
        cfg.rank = rank
        cfg.world = world
        self._uid = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
        cfg.nccl_unique_id = C.cast(self._uid, C.c_void_p) if self._uid is not None else None
        cfg.comm_backend = comm_backend
        cfg.max_probes = max_probes
        cfg.distinct_ratio = distinct_ratio
        cfg.target_load = target_load
        cfg.wave_table_bytes = wave_table_bytes
        cfg.host_threads = host_threads
        cfg.stream = stream
        cfg.timing = 1 if timing else 0
        cfg.force_exchange = 1 if force_exchange else 0
        cfg.disable_normalization = 0 if canonical else 1
        cfg.dfp_pivot = dfp_pivot
        cfg.order_sample_stride = order_sample_stride
        cfg.count_mode = count_mode
        h = C.c_void_p()
        st = _lib.gerbil_init(C.byref(cfg), C.byref(h))
        if st != OK:
            raise GerbilError(st, "gerbil_init failed")
        self._h = h
        self.k = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.gerbil_finalize(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st: int) -> None:
        if st != OK:
            raise GerbilError(st, _lib.gerbil_last_error(self._h).decode(errors="replace"))

    # ---- counting entry points ---------------------------------------------
    def count(self, k: int, m: int = 0, min_count: int = 1, text: bytes | None = None,
              paths: list[str] | None = None) -> None:
        r, keep = _reads(text, paths)
        self._check(_lib.gerbil_count(self._h, C.byref(r), k, m, min_count))
        del keep
        self.k = k

    def count_device(self, codes, nmask, read_start, n_reads: int, k: int, m: int = 0,
                     min_count: int = 1) -> None:
        """Packed batch already in device memory (torch tensors or raw addresses)."""
        self._check(_lib.gerbil_count_device(self._h, _ptr(codes), _ptr(nmask), _ptr(read_start), n_reads,
                                             k, m, min_count))
        self.k = k

    def count_host_packed(self, codes, nmask, read_start, n_reads: int, k: int, m: int = 0,
                          min_count: int = 1) -> None:
        self._check(_lib.gerbil_count_host_packed(self._h, _ptr(codes), _ptr(nmask), _ptr(read_start),
                                                  n_reads, k, m, min_count))
        self.k = k

    # ---- results ---------------------------------------------------------------
    def n_results(self) -> int:
        n = C.c_uint64()
        self._check(_lib.gerbil_fetch(self._h, None, None, 0, C.byref(n), 0))
        return n.value

    def count_host_stream(self, codes, nmask, read_start, n_reads: int, k: int, m: int = 0, min_count: int = 1,
                          out: np.ndarray | None = None) -> int:
        """Host batch in, App. C binary records streamed into `out` (a uint8 array in page-locked
        memory, e.g. a pinned torch tensor's .numpy()); returns the record bytes. Raises GerbilError
        (status GERBIL_E_USAGE) when `out` is too small — `needed_bytes` on the error holds the size."""
        n = C.c_uint64(0)
        cap = 0 if out is None else out.nbytes
        rc = _lib.gerbil_count_host_stream(self._h, _ptr(codes), _ptr(nmask), _ptr(read_start), n_reads, k, m,
                                           min_count, _ptr(out) if out is not None else None, cap, C.byref(n))
        self.k = k
        if rc != 0:
            err = GerbilError(rc, _lib.gerbil_last_error(self._h).decode(errors="replace"))
            err.needed_bytes = n.value
            raise err
        return n.value

    # ---- step (a) on the device (include/gerbil.h gerbil_parse_text / gerbil_count_text) ----
    @staticmethod
    def _text_arg(text):
        """bytes / numpy uint8 (host) or a CUDA uint8 tensor → (pointer, length, on_device, keepalive)."""
        if isinstance(text, (bytes, bytearray)):
            buf = C.create_string_buffer(bytes(text), len(text))
            return C.cast(buf, C.c_void_p).value, len(text), 0, buf
        if isinstance(text, np.ndarray):
            return text.ctypes.data, text.nbytes, 0, text
        # torch tensor
        on_dev = 1 if getattr(text, "is_cuda", False) else 0
        return text.data_ptr(), text.numel() * text.element_size(), on_dev, text

    def parse_text(self, text) -> PackedReads:
        """Parse FASTA / FASTQ / raw text on the GPU → the packed batch (host arrays)."""
        ptr, n, dev, keep = self._text_arg(text)
        nb, nr = C.c_uint64(), C.c_uint64()
        self._check(_lib.gerbil_parse_text(self._h, ptr, n, dev, None, None, None, C.byref(nb), C.byref(nr)))
        codes = np.zeros(max((nb.value + 31) // 32, 1), np.uint64)
        nmask = np.zeros(max((nb.value + 63) // 64, 1), np.uint64)
        rs = np.zeros(nr.value + 1, np.uint64)
        self._check(_lib.gerbil_parse_text(self._h, ptr, n, dev, _ptr(codes), _ptr(nmask), _ptr(rs), C.byref(nb),
                                           C.byref(nr)))
        del keep
        return PackedReads(codes, nmask, rs, nb.value, nr.value)

    def count_text(self, text, k: int, m: int = 0, min_count: int = 1) -> None:
        """Steps (a)..(e) on the GPU from FASTA / FASTQ / raw text (host bytes or a CUDA uint8 tensor)."""
        ptr, n, dev, keep = self._text_arg(text)
        self._check(_lib.gerbil_count_text(self._h, ptr, n, dev, k, m, min_count))
        self.k = k
        del keep

    # ---- out-of-core counting (include/gerbil.h gerbil_spill_*) ---------------
    def spill_begin(self, k: int, m: int = 0) -> None:
        self._check(_lib.gerbil_spill_begin(self._h, k, m))
        self.k = k

    def spill_add(self, codes, nmask, read_start, n_reads: int) -> None:
        self._check(_lib.gerbil_spill_add(self._h, _ptr(codes), _ptr(nmask), _ptr(read_start), n_reads))

    def spill_finish(self, min_count: int = 1, out: np.ndarray | None = None) -> int:
        """Phase two; App. C records into `out` (page-locked uint8 array). Returns the record bytes;
        GerbilError with needed_bytes when `out` is missing or too small."""
        n = C.c_uint64(0)
        cap = 0 if out is None else out.nbytes
        rc = _lib.gerbil_spill_finish(self._h, min_count, _ptr(out) if out is not None else None, cap, C.byref(n))
        if rc != 0:
            err = GerbilError(rc, _lib.gerbil_last_error(self._h).decode(errors="replace"))
            err.needed_bytes = n.value
            raise err
        return n.value

    def minimizer_stats(self) -> tuple[int, int]:
        """(max distinct k-mers per minimizer, minimizers owning >= 1 k-mer) of the last count."""
        mx, n = C.c_uint64(0), C.c_uint64(0)
        self._check(_lib.gerbil_minimizer_stats(self._h, C.byref(mx), C.byref(n)))
        return mx.value, n.value

    def fetch(self, sorted: bool = True, out_keys: np.ndarray | None = None,
              out_counts: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
        """(keys[n, W] uint64, counts[n] uint32) of this rank."""
        n = self.n_results()
        W = (self.k + 31) // 32
        keys = out_keys if out_keys is not None else np.empty((n, W), np.uint64)
        counts = out_counts if out_counts is not None else np.empty(n, np.uint32)
        got = C.c_uint64()
        self._check(_lib.gerbil_fetch(self._h, _ptr(keys), _ptr(counts), keys.shape[0], C.byref(got),
                                      1 if sorted else 0))
        return keys[: got.value], counts[: got.value]

    def encode_results(self, fmt: int = FMT_BINARY, sorted: bool = True) -> bytes:
        """Results in the paper's binary format (App. C) or as CSV (`-x h`)."""
        n = C.c_uint64()
        self._check(_lib.gerbil_encode_results(self._h, fmt, 1 if sorted else 0, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        self._check(_lib.gerbil_encode_results(self._h, fmt, 1 if sorted else 0, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def write_results(self, path: str, fmt: int = FMT_BINARY, sorted: bool = True) -> None:
        self._check(_lib.gerbil_write_results(self._h, path.encode(), fmt, 1 if sorted else 0))

    def results_device(self) -> tuple[int, int, int, int]:
        """(kmers_ptr, counts_ptr, n, W) of the device-resident results."""
        kp, cp = C.c_void_p(), C.c_void_p()
        n, W = C.c_uint64(), C.c_uint32()
        self._check(_lib.gerbil_results_device(self._h, C.byref(kp), C.byref(cp), C.byref(n), C.byref(W)))
        return kp.value or 0, cp.value or 0, n.value, W.value

    def stats(self) -> dict:
        s = Stats()
        self._check(_lib.gerbil_get_stats(self._h, C.byref(s)))
        return s.as_dict()

    def debug_supermers(self, packed: PackedReads, k: int, m: int):
        """Step (b) alone on a host batch: (pos, nwin, bin, mu) arrays."""
        n = C.c_uint64()
        args = (self._h, _ptr(packed.codes), _ptr(packed.nmask), _ptr(packed.read_start), packed.n_reads, k, m)
        self._check(_lib.gerbil_debug_supermers(*args, None, None, None, None, 0, C.byref(n)))
        pos = np.empty(n.value, np.uint64)
        nwin = np.empty(n.value, np.uint32)
        b = np.empty(n.value, np.uint32)
        mu = np.empty(n.value, np.uint32)
        self._check(_lib.gerbil_debug_supermers(*args, _ptr(pos), _ptr(nwin), _ptr(b), _ptr(mu), n.value,
                                                C.byref(n)))
        return pos, nwin, b, mu
