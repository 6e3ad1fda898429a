"""ctypes binding of include/reseq_cuda.h.

The library is built in-tree (paper_1404_3456_b200/libreseq_cuda.so) by
`paper_1404_3456_b200.build`.  There is no CPU fallback: if the shared object is missing
the import fails loudly, and on a machine without a CUDA device every compute call
raises `NoDeviceError`.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libreseq_cuda.so"

OK, INVALID_ARGUMENT, TEXT_TOO_LARGE, SCAN_OVERFLOW, CUDA_ERROR, OUT_OF_MEMORY, NO_DEVICE, BUFFER_TOO_SMALL = range(8)
MAX_TEXT = 0xFFFFFFFE


class ReseqError(RuntimeError):
    """reseq::error (errors.hpp:9-11)."""


class TextTooLargeError(ReseqError):
    """reseq::text_too_large_error (errors.hpp:58-61)."""


class ScanOverflowError(ReseqError):
    """reseq::scan_overflow_error (errors.hpp:54-56)."""


class NoDeviceError(ReseqError):
    pass


class SaStats(C.Structure):
    _fields_ = [
        ("alphabet", C.c_uint32),
        ("init_symbols", C.c_uint32),
        ("rounds", C.c_uint32),
        ("sort_passes", C.c_uint32),
        ("kernel_launches", C.c_uint64),
        ("refined_tile", C.c_uint64),
        ("refined_global", C.c_uint64),
    ]


class KernelProfile(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_uint64), ("total_ms", C.c_double)]


class PrefixRelations(C.Structure):
    _fields_ = [("q", C.c_size_t),
                ("prefixes_off", C.POINTER(C.c_uint64)), ("extensions_off", C.POINTER(C.c_uint64)),
                ("exact_off", C.POINTER(C.c_uint64)),
                ("prefixes", C.POINTER(C.c_uint32)), ("extensions", C.POINTER(C.c_uint32)),
                ("exact", C.POINTER(C.c_uint32))]


class Overlaps(C.Structure):
    _fields_ = [
        ("count", C.c_uint64),
        ("i", C.POINTER(C.c_uint32)),
        ("j", C.POINTER(C.c_uint32)),
        ("w", C.POINTER(C.c_uint32)),
        ("contained", C.POINTER(C.c_uint8)),
        ("queries", C.c_uint64),
        ("device_ms", C.c_double),
    ]


_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p

# name -> (restype, argtypes).  Kept in one table so tests can check the export list against
# include/reseq_cuda.h.
SIGNATURES = {
    "reseq_cuda_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "reseq_cuda_ctx_destroy": (None, [_vp]),
    "reseq_cuda_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "reseq_cuda_ctx_synchronize": (C.c_int, [_vp]),
    "reseq_cuda_ctx_launch_count": (C.c_uint64, [_vp]),
    "reseq_cuda_ctx_workspace_bytes": (C.c_size_t, [_vp]),
    "reseq_cuda_ctx_set_option": (C.c_int, [_vp, C.c_char_p, C.c_longlong]),
    "reseq_cuda_ctx_profile": (C.c_int, [_vp, C.c_int]),
    "reseq_cuda_ctx_profile_read": (C.c_size_t, [_vp, C.POINTER(KernelProfile), C.c_size_t]),
    "reseq_cuda_last_error": (C.c_char_p, []),
    "reseq_cuda_version": (C.c_char_p, []),
    "reseq_cuda_exclusive_scan": (C.c_int, [_vp, _vp, C.c_size_t, _vp]),
    "reseq_cuda_exclusive_scan_device": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _u64p]),
    "reseq_cuda_split_by_bit": (C.c_int, [_vp, _vp, _vp, C.c_size_t, C.c_uint, _vp, _vp]),
    "reseq_cuda_split_destinations": (C.c_int, [_vp, _vp, C.c_size_t, C.c_uint, _vp, _u32p]),
    "reseq_cuda_is_sorted": (C.c_int, [_vp, _vp, C.c_size_t, C.POINTER(C.c_int)]),
    "reseq_cuda_radix_sort": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "reseq_cuda_radix_sort_device": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "reseq_cuda_chunked_radix_sort": (C.c_int, [_vp, _vp, _vp, C.c_size_t, C.c_uint, _vp, _vp]),
    "reseq_cuda_build_sa": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _vp, C.POINTER(SaStats)]),
    "reseq_cuda_build_sa_device": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _vp, C.POINTER(SaStats)]),
    "reseq_cuda_sa_shard_create": (C.c_int, [_vp, _vp, C.c_size_t, C.POINTER(_vp), C.POINTER(C.c_int)]),
    "reseq_cuda_sa_shard_destroy": (None, [_vp]),
    "reseq_cuda_sa_shard_records": (C.c_int, [_vp, C.c_uint64, C.c_size_t, _vp]),
    "reseq_cuda_sa_shard_finish": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _u64p]),
    "reseq_cuda_sa_shard_uniform_info": (C.c_int, [_vp, _u32p, _u64p]),
    "reseq_cuda_sa_shard_uniform_records": (C.c_int, [_vp, C.c_uint64, C.c_size_t, _vp]),
    "reseq_cuda_sa_shard_uniform_sort_link": (C.c_int, [_vp, _vp, C.c_size_t, _vp]),
    "reseq_cuda_sa_shard_uniform_finish": (C.c_int, [_vp, _vp, _vp, _u64p]),
    "reseq_cuda_inverse_device": (C.c_int, [_vp, _vp, C.c_size_t, _vp]),
    "reseq_cuda_sa_shard_prefix_hist": (C.c_int, [_vp, C.c_uint64, C.c_size_t, _vp]),
    "reseq_cuda_sa_shard_bucket_size": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _u64p]),
    "reseq_cuda_sa_shard_bucket_records": (C.c_int, [_vp, _vp]),
    "reseq_cuda_rank_shard_partition": (C.c_int, [_vp, _vp, C.c_size_t, C.c_uint64, C.c_uint64, C.c_int, _vp, _u64p]),
    "reseq_cuda_rank_shard_finish": (C.c_int, [_vp, _vp, C.c_size_t, _vp]),
    "reseq_cuda_checksum_u32_device": (C.c_int, [_vp, _vp, C.c_size_t, _u64p]),
    "reseq_cuda_index_create": (C.c_int, [_vp, _vp, C.c_size_t, _vp, C.c_size_t, C.POINTER(_vp)]),
    "reseq_cuda_index_destroy": (None, [_vp]),
    "reseq_cuda_index_text_len": (C.c_size_t, [_vp]),
    "reseq_cuda_index_fragments": (C.c_size_t, [_vp]),
    "reseq_cuda_index_get": (C.c_int, [_vp, _vp, _vp, _vp]),
    "reseq_cuda_index_start_fragments": (C.c_int, [_vp, _vp]),
    "reseq_cuda_index_device_ptrs": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "reseq_cuda_index_locate_batch": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "reseq_cuda_index_locate_residuals": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "reseq_cuda_index_prefix_related_batch": (C.c_int, [_vp, _vp, _vp, C.c_size_t, C.POINTER(PrefixRelations)]),
    "reseq_cuda_prefix_relations_free": (None, [C.POINTER(PrefixRelations)]),
    "reseq_cuda_index_overlaps": (C.c_int, [_vp, C.c_uint32, C.POINTER(Overlaps)]),
    "reseq_cuda_index_overlaps_range": (C.c_int, [_vp, C.c_uint32, C.c_size_t, C.c_size_t, C.POINTER(Overlaps)]),
    "reseq_cuda_overlaps_free": (None, [C.POINTER(Overlaps)]),
    "reseq_cuda_index_overlaps_into": (C.c_int, [_vp, C.c_uint32, C.c_size_t, C.c_size_t, _vp, _vp, _vp, C.c_size_t, _vp,
                                                 C.POINTER(Overlaps)]),
    "reseq_greedy_superstring": (C.c_int, [_vp, C.c_size_t, _vp, C.c_size_t, C.POINTER(Overlaps), C.c_uint32,
                                           _vp, C.POINTER(C.c_size_t), _vp, C.POINTER(C.c_size_t)]),
    "reseq_synth_random_dna": (None, [C.c_size_t, C.c_uint64, _vp]),
    "reseq_synth_random_keys": (None, [C.c_size_t, C.c_uint64, _vp, _vp]),
    "reseq_synth_read_text": (C.c_int, [C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, C.c_uint64, _vp, _vp]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libreseq_cuda.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` "
            "(there is no CPU fallback for the reseq B200 backend)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError here == the ABI and the header diverged
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == OK:
        return
    msg = load().reseq_cuda_last_error().decode("utf-8", "replace")
    if status == INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == TEXT_TOO_LARGE:
        raise TextTooLargeError(msg)
    if status == SCAN_OVERFLOW:
        raise ScanOverflowError(msg)
    if status == OUT_OF_MEMORY:
        raise MemoryError(msg)
    if status == NO_DEVICE:
        raise NoDeviceError(msg)
    raise ReseqError(msg)
