"""Host-side mirror of the reference's `reseq` interface for the hot path, over the C ABI.

Names, argument meaning and error behaviour follow proj/include/reseq/*.hpp so that the
parity tests read like the reference's own:

    reference (C++)                                  here (Python, numpy arrays)
    executor(executor_config{w, chunk})              Executor(device=0)
    exclusive_scan(values, exec)                     exclusive_scan(values, exec)
    split_by_bit(key_array, bit, exec)               split_by_bit(keys, payload, bit, exec)
    radix_sort(key_array, exec)                      radix_sort(keys, payload, exec)
    chunked_radix_sort(key_array, exec, bits)        chunked_radix_sort(keys, payload, exec, bits)
    build_parallel(text, exec) -> {sa, rank}         build_parallel(text, exec) -> SuffixArray
    make_fragment_set(frags, alphabet)               make_fragment_set(frags, alphabet)
    fragment_index(set, builder, exec)               FragmentIndex(set, exec)
      .locate_prefix_range(p)                          .locate_prefix_range(p) / .locate_batch(ps)
      .start_rank_list()                               .start_rank_list()
    build_overlap_graph(set)                         FragmentIndex.overlaps(min_overlap) (sparse)
    greedy_superstring_with_order(set)               greedy_superstring_with_order(set, ...)

All computation happens in libreseq_cuda.so (CUDA kernels; the greedy merge is host C++).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (NoDeviceError, ReseqError, SaStats, ScanOverflowError,  # noqa: F401
                   TextTooLargeError)


def _host_array(count: int, dtype) -> np.ndarray:
    """A numpy array over page-locked memory when a CUDA device is there (PCIe-speed D2H), plain otherwise."""
    try:
        import torch
        if torch.cuda.is_available():
            t = torch.empty(int(count) * np.dtype(dtype).itemsize, dtype=torch.uint8).pin_memory()
            return t.numpy().view(dtype)
    except Exception:
        pass
    return np.empty(int(count), dtype)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u32(a, name="array") -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.uint32)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional")
    return arr


def _bytes_array(b) -> np.ndarray:
    if isinstance(b, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(b), dtype=np.uint8)
    if isinstance(b, str):
        return np.frombuffer(b.encode("latin-1"), dtype=np.uint8)
    return np.ascontiguousarray(b, dtype=np.uint8)


class Executor:
    """The device backend that stands where the reference passes `const executor&`
    (executor.hpp:28-145).  `workers` / `chunk_size` are accepted for source compatibility;
    results are independent of them on the device just as the reference guarantees on the
    host (executor.hpp:23-27)."""

    def __init__(self, device: int = 0, workers: int = 1, chunk_size: int = 1 << 15):
        self.workers = max(1, int(workers))
        self.chunk_size = max(1, int(chunk_size))
        self._lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self._lib.reseq_cuda_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def set_stream(self, cuda_stream: Optional[int]) -> None:
        """Launch on the given cudaStream_t.  `None` restores the context's own stream.  The integer
        0 -- what `torch.cuda.current_stream().cuda_stream` returns for torch's default stream -- means
        the legacy default stream (RESEQ_CUDA_STREAM_LEGACY), so that library kernels are ordered
        with torch's and NCCL's work on that stream."""
        if cuda_stream is None:
            handle = 0
        elif int(cuda_stream) == 0:
            handle = 1   # RESEQ_CUDA_STREAM_LEGACY == cudaStreamLegacy
        else:
            handle = int(cuda_stream)
        _lib.check(self._lib.reseq_cuda_ctx_set_stream(self._h, C.c_void_p(handle)))

    def synchronize(self) -> None:
        _lib.check(self._lib.reseq_cuda_ctx_synchronize(self._h))

    @property
    def launch_count(self) -> int:
        return int(self._lib.reseq_cuda_ctx_launch_count(self._h))

    @property
    def workspace_bytes(self) -> int:
        return int(self._lib.reseq_cuda_ctx_workspace_bytes(self._h))

    def set_option(self, name: str, value: int) -> None:
        _lib.check(self._lib.reseq_cuda_ctx_set_option(self._h, name.encode(), int(value)))

    def profile(self, enable: bool) -> None:
        """Start (and clear) or stop per-kernel event timing."""
        _lib.check(self._lib.reseq_cuda_ctx_profile(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        """{kernel name: (launches, total device ms)} since profile(True)."""
        buf = (_lib.KernelProfile * 64)()
        m = int(self._lib.reseq_cuda_ctx_profile_read(self._h, buf, 64))
        return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(min(m, 64))}

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.reseq_cuda_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_exec: Optional[Executor] = None


def default_executor() -> Executor:
    global _default_exec
    if _default_exec is None:
        _default_exec = Executor()
    return _default_exec


# ---- L0 primitives -----------------------------------------------------------------

def exclusive_scan(values, exec: Optional[Executor] = None) -> np.ndarray:
    """scan.hpp:32-56.  Raises ScanOverflowError when the total exceeds 2^32-1."""
    ex = exec or default_executor()
    v = _u32(values, "values")
    out = np.empty_like(v)
    _lib.check(ex._lib.reseq_cuda_exclusive_scan(ex.handle, _ptr(v), v.size, _ptr(out)))
    return out


def _pair(keys, payload):
    k = _u32(keys, "keys")
    p = None
    if payload is not None and len(payload) != 0:
        p = _u32(payload, "payload")
        if p.size != k.size:
            raise ValueError("payload must be empty or as long as keys")
    return k, p


def split_by_bit(keys, payload=None, bit: int = 0, exec: Optional[Executor] = None):
    """radix_sort.hpp:126-139: stable partition, keys whose bit is 0 first."""
    ex = exec or default_executor()
    k, p = _pair(keys, payload)
    ko = np.empty_like(k)
    po = None if p is None else np.empty_like(p)
    _lib.check(ex._lib.reseq_cuda_split_by_bit(ex.handle, _ptr(k), _ptr(p), k.size, int(bit), _ptr(ko), _ptr(po)))
    return ko, (po if po is not None else np.empty(0, np.uint32))


def split_destinations(keys, bit: int = 0, exec: Optional[Executor] = None):
    """detail::split_destinations, radix_sort.hpp:35-52 (Alg. 1): (destinations, total_false)."""
    ex = exec or default_executor()
    k = _u32(keys, "keys")
    d = np.empty_like(k)
    tof = C.c_uint32(0)
    _lib.check(ex._lib.reseq_cuda_split_destinations(ex.handle, _ptr(k), k.size, int(bit), _ptr(d), C.byref(tof)))
    return d, int(tof.value)


def is_sorted(keys, exec: Optional[Executor] = None) -> bool:
    """detail::phase_is_sorted, radix_sort.hpp:54-66."""
    ex = exec or default_executor()
    k = _u32(keys, "keys")
    flag = C.c_int(1)
    _lib.check(ex._lib.reseq_cuda_is_sorted(ex.handle, _ptr(k), k.size, C.byref(flag)))
    return bool(flag.value)


def radix_sort(keys, payload=None, exec: Optional[Executor] = None):
    """radix_sort.hpp:143-161: stable ascending sort on keys, payload carried."""
    ex = exec or default_executor()
    k, p = _pair(keys, payload)
    ko = np.empty_like(k)
    po = None if p is None else np.empty_like(p)
    _lib.check(ex._lib.reseq_cuda_radix_sort(ex.handle, _ptr(k), _ptr(p), k.size, _ptr(ko), _ptr(po)))
    return ko, (po if po is not None else np.empty(0, np.uint32))


def chunked_radix_sort(keys, payload=None, exec: Optional[Executor] = None, digit_bits: int = 4):
    """radix_sort.hpp:169-303: same result as radix_sort; digit_bits outside 1..8 raises
    ValueError (std::invalid_argument, :171-172) before any device work."""
    if digit_bits < 1 or digit_bits > 8:
        raise ValueError("digit_bits must be in 1..8")
    ex = exec or default_executor()
    k, p = _pair(keys, payload)
    ko = np.empty_like(k)
    po = None if p is None else np.empty_like(p)
    _lib.check(ex._lib.reseq_cuda_chunked_radix_sort(ex.handle, _ptr(k), _ptr(p), k.size, int(digit_bits),
                                                     _ptr(ko), _ptr(po)))
    return ko, (po if po is not None else np.empty(0, np.uint32))


# ---- L1 suffix array ------------------------------------------------------------------

@dataclass
class SuffixArray:
    """suffix_array.hpp:21-26."""
    sa: np.ndarray
    rank: np.ndarray
    stats: Optional[SaStats] = None

    def text_len(self) -> int:
        return int(self.sa.size)


def build_parallel(text, exec: Optional[Executor] = None) -> SuffixArray:
    """suffix_array.hpp:61-124.  The device path accepts up to 2^32-2 bytes (the reference
    stops at 2^31-1, :64); longer texts raise TextTooLargeError."""
    ex = exec or default_executor()
    t = _bytes_array(text)
    sa = np.empty(t.size, np.uint32)
    rank = np.empty(t.size, np.uint32)
    st = SaStats()
    _lib.check(ex._lib.reseq_cuda_build_sa(ex.handle, _ptr(t), t.size, _ptr(sa), _ptr(rank), C.byref(st)))
    return SuffixArray(sa, rank, st)


# ---- fragment sets (host; sequence.hpp) -------------------------------------------------

class EmptyFragmentError(ReseqError):
    """errors.hpp:13-18."""


class InvalidByteError(ReseqError):
    """errors.hpp:20-28."""


class OffsetOutOfRangeError(ReseqError):
    """errors.hpp:30-34."""


@dataclass
class FragmentSet:
    """sequence.hpp:60-92: concat = f0 \\0 f1 \\0 ... ; starts[i] = offset of fragment i."""
    concat: np.ndarray
    starts: np.ndarray
    alphabet: str

    def size(self) -> int:
        return int(self.starts.size)

    def length(self, i: int) -> int:
        end = int(self.starts[i + 1]) - 1 if i + 1 < self.starts.size else int(self.concat.size) - 1
        return end - int(self.starts[i])

    def lengths(self) -> np.ndarray:
        ends = np.append(self.starts[1:], np.uint32(self.concat.size)).astype(np.int64) - 1
        return (ends - self.starts.astype(np.int64)).astype(np.uint32)

    def bytes(self, i: int) -> bytes:
        s = int(self.starts[i])
        return self.concat[s:s + self.length(i)].tobytes()


def make_fragment_set(fragments: Sequence, alphabet: str = "dna") -> FragmentSet:
    """sequence.hpp:103-124, including its validation: empty fragments and bytes outside
    the alphabet are errors; the total is capped (here at 2^32-2, see build_parallel)."""
    if alphabet not in ("dna", "generic_byte"):
        raise ValueError("alphabet must be 'dna' or 'generic_byte'")
    frs = [bytes(f) if not isinstance(f, str) else f.encode("latin-1") for f in fragments]
    allowed = np.zeros(256, bool)
    if alphabet == "dna":
        allowed[[65, 67, 71, 84]] = True
    else:
        allowed[33:127] = True
    total = 0
    for i, f in enumerate(frs):
        if len(f) == 0:
            raise EmptyFragmentError(f"empty fragment at index {i}")
        a = np.frombuffer(f, np.uint8)
        bad = np.flatnonzero(~allowed[a])
        if bad.size:
            raise InvalidByteError(f"invalid byte {int(a[bad[0]])} at position {int(bad[0])} of fragment {i}")
        total += len(f)
    if total + len(frs) > _lib.MAX_TEXT:
        raise TextTooLargeError(f"text of length {total + len(frs)} exceeds 2^32-2")
    concat = np.zeros(total + len(frs), np.uint8)
    starts = np.zeros(len(frs), np.uint32)
    o = 0
    for i, f in enumerate(frs):
        starts[i] = o
        concat[o:o + len(f)] = np.frombuffer(f, np.uint8)
        o += len(f) + 1
    return FragmentSet(concat, starts, alphabet)


def fragment_set_from_text(concat, starts, alphabet: str = "dna") -> FragmentSet:
    """Wraps an already concatenated text (e.g. from synth_read_text)."""
    return FragmentSet(_bytes_array(concat), _u32(starts, "starts"), alphabet)


# ---- L2 index ---------------------------------------------------------------------------

@dataclass
class OverlapList:
    """Non-zero entries of overlap_graph.weight (overlap.hpp:26-45) with w >= min_overlap,
    sorted by (i, j); `contained[i]` = absorb_contained would drop fragment i (:51-67)."""
    i: np.ndarray
    j: np.ndarray
    w: np.ndarray
    contained: np.ndarray
    queries: int
    device_ms: float
    min_overlap: int

    def dense(self, k: int) -> np.ndarray:
        m = np.zeros((k, k), np.uint32)
        m[self.i, self.j] = self.w
        return m


class FragmentIndex:
    """fragment_index (fragment_index.hpp:30-167) resident in HBM."""

    def __init__(self, fset: FragmentSet, exec: Optional[Executor] = None):
        self.set = fset
        self.exec = exec or default_executor()
        self._lib = self.exec._lib
        h = C.c_void_p()
        _lib.check(self._lib.reseq_cuda_index_create(self.exec.handle, _ptr(fset.concat), fset.concat.size,
                                                     _ptr(fset.starts), fset.starts.size, C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.reseq_cuda_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _get(self, which: int) -> np.ndarray:
        n, k = self.set.concat.size, self.set.starts.size
        out = np.empty(k if which == 2 else n, np.uint32)
        args = [None, None, None]
        args[which] = _ptr(out)
        _lib.check(self._lib.reseq_cuda_index_get(self._h, *args))
        return out

    def sa(self) -> np.ndarray:
        return self._get(0)

    def rank(self) -> np.ndarray:
        return self._get(1)

    def start_rank_list(self) -> np.ndarray:
        return self._get(2)

    def locate_batch(self, patterns: Iterable) -> tuple[np.ndarray, np.ndarray]:
        pats = [bytes(p) if not isinstance(p, str) else p.encode("latin-1") for p in patterns]
        off = np.zeros(len(pats) + 1, np.uint64)
        for i, p in enumerate(pats):
            off[i + 1] = off[i] + len(p)
        blob = np.frombuffer(b"".join(pats), np.uint8) if pats else np.zeros(0, np.uint8)
        lo = np.empty(len(pats), np.uint32)
        hi = np.empty(len(pats), np.uint32)
        _lib.check(self._lib.reseq_cuda_index_locate_batch(self._h, _ptr(blob), _ptr(off), len(pats),
                                                           _ptr(lo), _ptr(hi)))
        return lo, hi

    def locate_prefix_range(self, pattern) -> tuple[int, int]:
        """fragment_index.hpp:65-70."""
        lo, hi = self.locate_batch([pattern])
        return int(lo[0]), int(hi[0])

    def locate_residuals(self, frag, off) -> tuple[np.ndarray, np.ndarray]:
        f, o = _u32(frag, "frag"), _u32(off, "off")
        if f.size != o.size:
            raise ValueError("frag and off must have the same length")
        lo = np.empty(f.size, np.uint32)
        hi = np.empty(f.size, np.uint32)
        try:
            _lib.check(self._lib.reseq_cuda_index_locate_residuals(self._h, _ptr(f), _ptr(o), f.size,
                                                                   _ptr(lo), _ptr(hi)))
        except ValueError as e:
            raise OffsetOutOfRangeError(str(e)) from None
        return lo, hi

    def prefix_related_batch(self, frag, off):
        """fragment_index::prefix_related (fragment_index.hpp:72-109) for a batch of residuals.
        Returns a list of (prefixes_of, extensions_of, exact_matches) id arrays, each
        ascending by id."""
        f, o = _u32(frag, "frag"), _u32(off, "off")
        if f.size != o.size:
            raise ValueError("frag and off must have the same length")
        rel = _lib.PrefixRelations()
        try:
            try:
                _lib.check(self._lib.reseq_cuda_index_prefix_related_batch(self._h, _ptr(f), _ptr(o), f.size,
                                                                           C.byref(rel)))
            except ValueError as e:
                raise OffsetOutOfRangeError(str(e)) from None
            out = []
            for i in range(f.size):
                row = []
                for offp, idp in ((rel.prefixes_off, rel.prefixes), (rel.extensions_off, rel.extensions),
                                  (rel.exact_off, rel.exact)):
                    a, b = int(offp[i]), int(offp[i + 1])
                    row.append(np.array([idp[t] for t in range(a, b)], np.uint32))
                out.append(tuple(row))
            return out
        finally:
            self._lib.reseq_cuda_prefix_relations_free(C.byref(rel))

    def prefix_related(self, frag: int, off: int = 0):
        """prefix_related(residual{frag, off}) (fragment_index.hpp:78-80)."""
        return self.prefix_related_batch([frag], [off])[0]

    def prefix_related_patterns(self, patterns: Iterable):
        """fragment_index::prefix_related(std::string_view) (fragment_index.hpp:82-109) for arbitrary
        byte patterns (non-empty, no separator byte).  The interval searches -- one per distinct
        fragment length below |pattern| plus one for the whole pattern -- run on the device as one
        batch (at each length the reference's narrowed interval equals locate_prefix_range of that
        prefix, :75-80); the classification over start_rank_list is the reference's, on the host.
        Like the reference (:91), a pattern whose interval empties at an intermediate length returns
        at once: its prefixes_of then stay in (length, rank) order instead of ascending ids."""
        pats = [bytes(p) if not isinstance(p, str) else p.encode("latin-1") for p in patterns]
        if any(len(p) == 0 for p in pats):
            raise ValueError("patterns must be non-empty (fragment_index.hpp:63-64)")
        lens = self.set.lengths()
        lengths = np.unique(lens)
        queries, spans = [], []
        for p in pats:
            cuts = [int(c) for c in lengths if c < len(p)]
            spans.append((len(queries), cuts))
            queries.extend(p[:c] for c in cuts)
            queries.append(p)
        lo, hi = self.locate_batch(queries) if queries else (np.zeros(0, np.uint32), np.zeros(0, np.uint32))
        if not hasattr(self, "_start_rank"):
            self._start_rank = self._get(2)
            sf = np.empty(self.set.starts.size, np.uint32)
            _lib.check(self._lib.reseq_cuda_index_start_fragments(self._h, _ptr(sf)))
            self._start_frag = sf
        out = []
        for p, (q0, cuts) in zip(pats, spans):
            prefixes, early = [], False
            for t, c in enumerate(cuts):
                l, h = int(lo[q0 + t]), int(hi[q0 + t])
                if l == h:
                    early = True
                    break
                a, b = np.searchsorted(self._start_rank, [l, h], side="left")
                ids = self._start_frag[a:b]
                prefixes.extend(ids[lens[ids] == c].tolist())      # ranks ascending (collect_starts_of_length, :150-158)
            if early:
                out.append((np.array(prefixes, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32)))
                continue
            l, h = int(lo[q0 + len(cuts)]), int(hi[q0 + len(cuts)])
            a, b = np.searchsorted(self._start_rank, [l, h], side="left")
            ids = self._start_frag[a:b]
            out.append((np.sort(np.array(prefixes, np.uint32)), np.sort(ids[lens[ids] > len(p)]).astype(np.uint32),
                        np.sort(ids[lens[ids] == len(p)]).astype(np.uint32)))
        return out

    def overlaps(self, min_overlap: int = 1, frag_begin: int = 0, frag_end: Optional[int] = None,
                 reuse_buffers: bool = False) -> OverlapList:
        """Sparse overlap graph; [frag_begin, frag_end) restricts the querying fragments (the
        unit of sharding across GPUs).  The device writes the triples straight into the arrays of
        the returned OverlapList (reseq_cuda_index_overlaps_into).  With `reuse_buffers` those
        arrays are page-locked buffers kept by this index (PCIe-speed transfer, no allocation per
        call) and stay valid only until the next such call."""
        k = self.set.starts.size
        if frag_end is None:
            frag_end = k
        cap = getattr(self, "_ov_cap", 0) or max(1024, 32 * (int(frag_end) - int(frag_begin)))
        while True:
            if reuse_buffers:
                bufs = getattr(self, "_ov_bufs", None)
                if bufs is None or bufs[0].size < cap or bufs[3].size < k:
                    bufs = tuple(_host_array(cap, np.uint32) for _ in range(3)) + (_host_array(max(1, k), np.uint8),)
                    self._ov_bufs = bufs
                i, j, w, contained = bufs
            else:
                i, j, w = (np.empty(cap, np.uint32) for _ in range(3))
                contained = np.empty(max(1, k), np.uint8)
            ov = _lib.Overlaps()
            st = self._lib.reseq_cuda_index_overlaps_into(self._h, int(min_overlap), int(frag_begin), int(frag_end),
                                                          _ptr(i), _ptr(j), _ptr(w), i.size, _ptr(contained), C.byref(ov))
            if st == _lib.BUFFER_TOO_SMALL:
                cap = int(ov.count) + int(ov.count) // 8 + 1024
                continue
            _lib.check(st)
            break
        m = int(ov.count)
        self._ov_cap = m + m // 8 + 1024          # the next call on this index starts with room to spare
        return OverlapList(i[:m], j[:m], w[:m], contained[:k], int(ov.queries), float(ov.device_ms),
                           max(1, int(min_overlap)))


# ---- L3 host merge ---------------------------------------------------------------------------

def greedy_superstring_from_overlaps(fset: FragmentSet, ov: OverlapList) -> tuple[bytes, np.ndarray]:
    """The scalable host merge (host/greedy.cpp) over an OverlapList."""
    lib = _lib.load()
    i, j, w = _u32(ov.i), _u32(ov.j), _u32(ov.w)
    contained = np.ascontiguousarray(ov.contained, np.uint8)
    c_ov = _lib.Overlaps()
    c_ov.count = i.size
    c_ov.i = i.ctypes.data_as(C.POINTER(C.c_uint32))
    c_ov.j = j.ctypes.data_as(C.POINTER(C.c_uint32))
    c_ov.w = w.ctypes.data_as(C.POINTER(C.c_uint32))
    c_ov.contained = contained.ctypes.data_as(C.POINTER(C.c_uint8))
    k = fset.starts.size
    sup = np.empty(max(1, int(fset.concat.size) - k), np.uint8)
    order = np.empty(max(1, k), np.uint32)
    sl, ol = C.c_size_t(0), C.c_size_t(0)
    _lib.check(lib.reseq_greedy_superstring(_ptr(fset.concat), fset.concat.size, _ptr(fset.starts), k,
                                            C.byref(c_ov), int(ov.min_overlap), _ptr(sup), C.byref(sl),
                                            _ptr(order), C.byref(ol)))
    return sup[:sl.value].tobytes(), order[:ol.value].copy()


def greedy_superstring_with_order(fset: FragmentSet, index: Optional[FragmentIndex] = None,
                                  min_overlap: int = 1, exec: Optional[Executor] = None):
    """overlap.hpp:80-113: (superstring, original ids in concatenation order).  Overlaps come
    from the device index; the merge itself runs on the host."""
    ix = index or FragmentIndex(fset, exec)
    return greedy_superstring_from_overlaps(fset, ix.overlaps(min_overlap))


# ---- synthetic workloads -----------------------------------------------------------------------

def synth_random_dna(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.uint8)
    _lib.load().reseq_synth_random_dna(n, seed, _ptr(out))
    return out


def synth_random_keys(n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    k, p = np.empty(n, np.uint32), np.empty(n, np.uint32)
    _lib.load().reseq_synth_random_keys(n, seed, _ptr(k), _ptr(p))
    return k, p


def synth_read_text(genome_len: int, read_len: int, k: int, genome_seed: int = 1, read_seed: int = 2,
                    pinned: bool = False):
    """SURVEY.md 8(d) read text: returns (concat uint8[k*(L+1)], starts uint32[k])."""
    n = k * (read_len + 1)
    if pinned:
        import torch
        t = torch.empty(n, dtype=torch.uint8).pin_memory()
        out = t.numpy()
    else:
        out = np.empty(n, np.uint8)
    starts = np.empty(k, np.uint32)
    _lib.check(_lib.load().reseq_synth_read_text(genome_len, read_len, k, genome_seed, read_seed,
                                                  _ptr(out), _ptr(starts)))
    return out, starts
