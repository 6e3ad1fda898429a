"""ctypes wrappers of the test oracle (oracle/liboracle.so) and of the real reference
(oracle/_ref/libreseq_ref.so).  TEST INFRASTRUCTURE: imported only from tests/."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def vp(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def u8(b) -> np.ndarray:
    if isinstance(b, str):
        b = b.encode("latin-1")
    if isinstance(b, (bytes, bytearray)):
        return np.frombuffer(bytes(b), np.uint8).copy()
    return np.ascontiguousarray(b, np.uint8)


def u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.uint32)


def blob(frags):
    frs = [f.encode("latin-1") if isinstance(f, str) else bytes(f) for f in frags]
    off = np.zeros(len(frs) + 1, np.uint64)
    for i, f in enumerate(frs):
        off[i + 1] = off[i] + len(f)
    return u8(b"".join(frs)), off


def concat_of(frags):
    """fragment_set layout (sequence.hpp:60-62): returns (concat, starts, lens)."""
    frs = [f.encode("latin-1") if isinstance(f, str) else bytes(f) for f in frags]
    starts, lens, out = [], [], bytearray()
    for f in frs:
        starts.append(len(out))
        lens.append(len(f))
        out += f + b"\0"
    return u8(bytes(out)), u32(starts), u32(lens)


class Oracle:
    def __init__(self):
        self.lib = C.CDLL(str(ROOT / "oracle" / "liboracle.so"))
        L = self.lib
        L.orc_verify_sa.restype = C.c_uint64
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_checksum_u32.restype = C.c_uint64
        L.orc_checksum_u32_from.restype = C.c_uint64
        L.orc_overlap_list.restype = C.c_uint64
        L.orc_overlap_list_fast.restype = C.c_uint64
        L.orc_absorb_contained.restype = C.c_size_t
        L.orc_overlap_weight.restype = C.c_uint32

    def build_sa(self, text):
        t = u8(text)
        sa, rank = np.empty(t.size, np.uint32), np.empty(t.size, np.uint32)
        assert self.lib.orc_build_sa(vp(t), C.c_size_t(t.size), vp(sa), vp(rank)) == 0
        return sa, rank

    def verify_sa(self, text, sa, threads=8) -> int:
        t = u8(text)
        return int(self.lib.orc_verify_sa(vp(t), C.c_size_t(t.size), vp(u32(sa)), C.c_uint(threads)))

    def suffix_less(self, text, i, j) -> bool:
        t = u8(text)
        return bool(self.lib.orc_suffix_less(vp(t), C.c_size_t(t.size), C.c_uint32(i), C.c_uint32(j)))

    def exclusive_scan(self, v):
        v = u32(v)
        out = np.empty_like(v)
        return self.lib.orc_exclusive_scan(vp(v), C.c_size_t(v.size), vp(out)), out

    def split_by_bit(self, k, p, bit):
        k = u32(k)
        p = None if p is None else u32(p)
        ko = np.empty_like(k)
        po = None if p is None else np.empty_like(p)
        self.lib.orc_split_by_bit(vp(k), vp(p), C.c_size_t(k.size), C.c_uint(bit), vp(ko), vp(po))
        return ko, po

    def split_destinations(self, k, bit):
        k = u32(k)
        d = np.empty_like(k)
        tof = C.c_uint32(0)
        self.lib.orc_split_destinations(vp(k), C.c_size_t(k.size), C.c_uint(bit), vp(d), C.byref(tof))
        return d, int(tof.value)

    def is_sorted(self, k) -> bool:
        k = u32(k)
        return bool(self.lib.orc_is_sorted(vp(k), C.c_size_t(k.size)))

    def stable_sort(self, k, p):
        k = u32(k)
        p = None if p is None else u32(p)
        ko = np.empty_like(k)
        po = None if p is None else np.empty_like(p)
        self.lib.orc_stable_sort(vp(k), vp(p), C.c_size_t(k.size), vp(ko), vp(po))
        return ko, po

    def fnv1a64(self, b) -> int:
        b = u8(b)
        return int(self.lib.orc_fnv1a64(vp(b), C.c_size_t(b.size)))

    def checksum_u32(self, v) -> int:
        v = u32(v)
        return int(self.lib.orc_checksum_u32(vp(v), C.c_size_t(v.size)))

    def checksum_keys(self, keys, payload) -> int:
        k, p = u32(keys), u32(payload)
        h = self.checksum_u32(k)
        return int(self.lib.orc_checksum_u32_from(vp(p), C.c_size_t(p.size), C.c_uint64(h)))

    def locate(self, text, sa, pat):
        t, p = u8(text), u8(pat)
        lo, hi = C.c_uint32(), C.c_uint32()
        self.lib.orc_locate(vp(t), C.c_size_t(t.size), vp(u32(sa)), vp(p), C.c_size_t(p.size),
                            C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def start_rank_list(self, rank, starts):
        s = u32(starts)
        out = np.empty(s.size, np.uint32)
        self.lib.orc_start_rank_list(vp(u32(rank)), vp(s), C.c_size_t(s.size), vp(out))
        return out

    def prefix_related(self, text, starts, lens, pat):
        t, s, l, p = u8(text), u32(starts), u32(lens), u8(pat)
        k = s.size
        a, b, c = (np.empty(k, np.uint32) for _ in range(3))
        na, nb, nc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self.lib.orc_prefix_related(vp(t), vp(s), vp(l), C.c_size_t(k), vp(p), C.c_size_t(p.size), vp(a),
                                    C.byref(na), vp(b), C.byref(nb), vp(c), C.byref(nc))
        return a[:na.value].copy(), b[:nb.value].copy(), c[:nc.value].copy()

    def overlap_weight(self, a, b) -> int:
        a, b = u8(a), u8(b)
        return int(self.lib.orc_overlap_weight(vp(a), C.c_size_t(a.size), vp(b), C.c_size_t(b.size)))

    def overlap_graph(self, text, starts, lens):
        t, s, l = u8(text), u32(starts), u32(lens)
        w = np.empty((s.size, s.size), np.uint32)
        self.lib.orc_overlap_graph(vp(t), vp(s), vp(l), C.c_size_t(s.size), vp(w))
        return w

    def overlap_list(self, text, starts, lens, min_ov=1):
        t, s, l = u8(text), u32(starts), u32(lens)
        cap = 1 << 16
        while True:
            oi, oj, ow = (np.empty(cap, np.uint32) for _ in range(3))
            m = int(self.lib.orc_overlap_list(vp(t), vp(s), vp(l), C.c_size_t(s.size), C.c_uint32(min_ov),
                                              vp(oi), vp(oj), vp(ow), C.c_uint64(cap)))
            if m <= cap:
                return oi[:m].copy(), oj[:m].copy(), ow[:m].copy()
            cap = m

    def overlap_list_fast(self, text, starts, lens, min_ov=1, threads=8, cap=None):
        """orc_overlap_list_fast: the same list by per-length hash tables over `threads` host threads
        (BASELINE configs 1 and 2 at full size)."""
        t, s, l = u8(text), u32(starts), u32(lens)
        cap = int(cap or max(1 << 16, 40 * s.size))
        while True:
            oi, oj, ow = (np.empty(cap, np.uint32) for _ in range(3))
            m = int(self.lib.orc_overlap_list_fast(vp(t), vp(s), vp(l), C.c_size_t(s.size), C.c_uint32(min_ov),
                                                   C.c_uint(threads), vp(oi), vp(oj), vp(ow), C.c_uint64(cap)))
            if m <= cap:
                return oi[:m].copy(), oj[:m].copy(), ow[:m].copy()
            cap = m

    def make_read_text(self, G, L, k, genome_seed=1, read_seed=2):
        out = np.empty(k * (L + 1), np.uint8)
        assert self.lib.orc_make_read_text(C.c_size_t(G), C.c_size_t(L), C.c_size_t(k), C.c_uint64(genome_seed),
                                           C.c_uint64(read_seed), vp(out)) == 0
        return out

    def absorb_contained(self, text, starts, lens):
        t, s, l = u8(text), u32(starts), u32(lens)
        keep = np.empty(s.size, np.uint32)
        m = self.lib.orc_absorb_contained(vp(t), vp(s), vp(l), C.c_size_t(s.size), vp(keep))
        return keep[:m].copy()

    def greedy(self, text, starts, lens):
        t, s, l = u8(text), u32(starts), u32(lens)
        sup = np.empty(max(1, int(l.sum())), np.uint8)
        order = np.empty(max(1, s.size), np.uint32)
        sl, ol = C.c_size_t(), C.c_size_t()
        self.lib.orc_greedy(vp(t), vp(s), vp(l), C.c_size_t(s.size), vp(sup), C.byref(sl), vp(order),
                            C.byref(ol))
        return sup[:sl.value].tobytes(), order[:ol.value].copy()


class Reference:
    """The unmodified reference, through oracle/ref_shim.cpp."""

    PATH = ROOT / "oracle" / "_ref" / "libreseq_ref.so"

    @classmethod
    def try_load(cls):
        if not cls.PATH.exists():
            return None
        try:
            return cls()
        except OSError:
            return None

    def __init__(self):
        self.lib = C.CDLL(str(self.PATH))
        L = self.lib
        L.ref_fnv1a64.restype = C.c_uint64
        L.ref_checksum_u32.restype = C.c_uint64
        L.ref_index_create.restype = C.c_void_p
        L.ref_index_text_len.restype = C.c_size_t
        L.ref_overlap_weight.restype = C.c_uint32
        L.ref_hardware_concurrency.restype = C.c_uint

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def build_naive(self, text):
        t = u8(text)
        sa, rank = np.empty(t.size, np.uint32), np.empty(t.size, np.uint32)
        assert self.lib.ref_build_naive(vp(t), C.c_size_t(t.size), vp(sa), vp(rank)) == 0
        return sa, rank

    def build_parallel(self, text, workers=1, chunk=1 << 15):
        t = u8(text)
        sa, rank = np.empty(t.size, np.uint32), np.empty(t.size, np.uint32)
        st = self.lib.ref_build_parallel(vp(t), C.c_size_t(t.size), C.c_uint(workers), C.c_size_t(chunk),
                                         vp(sa), vp(rank))
        return st, sa, rank

    def exclusive_scan(self, v, workers=1, chunk=1 << 15):
        v = u32(v)
        out = np.empty_like(v)
        st = self.lib.ref_exclusive_scan(vp(v), C.c_size_t(v.size), C.c_uint(workers), C.c_size_t(chunk), vp(out))
        return st, out

    def _sort(self, fn, k, p, *extra, workers=1, chunk=1 << 15):
        k = u32(k)
        p = None if p is None else u32(p)
        ko = np.empty_like(k)
        po = None if p is None else np.empty_like(p)
        st = fn(vp(k), vp(p), C.c_size_t(k.size), *extra, vp(ko), vp(po))
        return st, ko, po

    def split_by_bit(self, k, p, bit, workers=1, chunk=1 << 15):
        return self._sort(self.lib.ref_split_by_bit, k, p, C.c_uint(bit), C.c_uint(workers), C.c_size_t(chunk))

    def split_destinations(self, k, bit, workers=1, chunk=1 << 15):
        k = u32(k)
        d = np.empty_like(k)
        tof = C.c_uint32(0)
        st = self.lib.ref_split_destinations(vp(k), C.c_size_t(k.size), C.c_uint(bit), C.c_uint(workers),
                                             C.c_size_t(chunk), vp(d), C.byref(tof))
        assert st == 0
        return d, int(tof.value)

    def is_sorted(self, k, workers=1, chunk=1 << 15) -> bool:
        k = u32(k)
        flag = C.c_int(0)
        assert self.lib.ref_is_sorted(vp(k), C.c_size_t(k.size), C.c_uint(workers), C.c_size_t(chunk), C.byref(flag)) == 0
        return bool(flag.value)

    def radix_sort(self, k, p, workers=1, chunk=1 << 15):
        return self._sort(self.lib.ref_radix_sort, k, p, C.c_uint(workers), C.c_size_t(chunk))

    def chunked_radix_sort(self, k, p, digit_bits=4, workers=1, chunk=1 << 15):
        return self._sort(self.lib.ref_chunked_radix_sort, k, p, C.c_uint(workers), C.c_size_t(chunk),
                          C.c_uint(digit_bits))

    def fnv1a64(self, b) -> int:
        b = u8(b)
        return int(self.lib.ref_fnv1a64(vp(b), C.c_size_t(b.size)))

    def checksum_u32(self, v) -> int:
        v = u32(v)
        return int(self.lib.ref_checksum_u32(vp(v), C.c_size_t(v.size)))

    def make_random_dna(self, n, seed):
        out = np.empty(n, np.uint8)
        self.lib.ref_make_random_dna(C.c_size_t(n), C.c_uint64(seed), vp(out))
        return out

    def make_random_keys(self, n, seed):
        k, p = np.empty(n, np.uint32), np.empty(n, np.uint32)
        self.lib.ref_make_random_keys(C.c_size_t(n), C.c_uint64(seed), vp(k), vp(p))
        return k, p

    def make_read_text(self, G, L, k, genome_seed=1, read_seed=2):
        out = np.empty(k * (L + 1), np.uint8)
        assert self.lib.ref_make_read_text(C.c_size_t(G), C.c_size_t(L), C.c_size_t(k), C.c_uint64(genome_seed),
                                           C.c_uint64(read_seed), vp(out)) == 0
        return out

    def index(self, frags, alphabet="dna", builder=0, workers=1, chunk=1 << 15):
        return RefIndex(self, frags, alphabet, builder, workers, chunk)

    def overlap_weight(self, a, b) -> int:
        a, b = u8(a), u8(b)
        return int(self.lib.ref_overlap_weight(vp(a), C.c_size_t(a.size), vp(b), C.c_size_t(b.size)))

    def overlap_graph(self, frags, alphabet="dna"):
        b, off = blob(frags)
        k = len(frags)
        w = np.empty((k, k), np.uint32)
        assert self.lib.ref_overlap_graph(vp(b), vp(off), C.c_size_t(k), 0 if alphabet == "dna" else 1, vp(w)) == 0
        return w

    def greedy(self, frags, alphabet="dna"):
        b, off = blob(frags)
        k = len(frags)
        sup = np.empty(max(1, b.size), np.uint8)
        order = np.empty(max(1, k), np.uint32)
        sl, ol = C.c_size_t(), C.c_size_t()
        assert self.lib.ref_greedy(vp(b), vp(off), C.c_size_t(k), 0 if alphabet == "dna" else 1, vp(sup),
                                   C.byref(sl), vp(order), C.byref(ol)) == 0
        return sup[:sl.value].tobytes(), order[:ol.value].copy()

    def absorb_contained(self, frags, alphabet="dna"):
        b, off = blob(frags)
        k = len(frags)
        keep = np.empty(max(1, k), np.uint32)
        m = C.c_size_t()
        assert self.lib.ref_absorb_contained(vp(b), vp(off), C.c_size_t(k), 0 if alphabet == "dna" else 1,
                                             vp(keep), C.byref(m)) == 0
        return keep[:m.value].copy()

    def double_cut(self, seq, m, n, cut_seed, shuffle_seed):
        s = u8(seq)
        k = C.c_size_t()
        st = self.lib.ref_double_cut(vp(s), C.c_size_t(s.size), C.c_size_t(m), C.c_size_t(n),
                                     C.c_uint64(cut_seed), C.c_uint64(shuffle_seed), None, None, C.byref(k))
        assert st == 0
        b = np.empty(s.size * 2, np.uint8)
        off = np.empty(k.value + 1, np.uint64)
        self.lib.ref_double_cut(vp(s), C.c_size_t(s.size), C.c_size_t(m), C.c_size_t(n), C.c_uint64(cut_seed),
                                C.c_uint64(shuffle_seed), vp(b), vp(off), C.byref(k))
        return [b[int(off[i]):int(off[i + 1])].tobytes() for i in range(k.value)]


class RefIndex:
    def __init__(self, ref, frags, alphabet, builder, workers, chunk):
        self.ref = ref
        self.k = len(frags)
        b, off = blob(frags)
        self.h = ref.lib.ref_index_create(vp(b), vp(off), C.c_size_t(self.k), 0 if alphabet == "dna" else 1,
                                          int(builder), C.c_uint(workers), C.c_size_t(chunk))
        assert self.h, "reference index construction failed"
        self.n = int(ref.lib.ref_index_text_len(C.c_void_p(self.h)))

    def arrays(self):
        concat = np.empty(self.n, np.uint8)
        starts = np.empty(self.k, np.uint32)
        sa, rank = np.empty(self.n, np.uint32), np.empty(self.n, np.uint32)
        srl = np.empty(self.k, np.uint32)
        self.ref.lib.ref_index_get(C.c_void_p(self.h), vp(concat), vp(starts), vp(sa), vp(rank), vp(srl))
        return concat, starts, sa, rank, srl

    def locate(self, pat):
        p = u8(pat)
        lo, hi = C.c_uint32(), C.c_uint32()
        self.ref.lib.ref_index_locate(C.c_void_p(self.h), vp(p), C.c_size_t(p.size), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def prefix_related(self, pat):
        p = u8(pat)
        a, b, c = (np.empty(max(1, self.k), np.uint32) for _ in range(3))
        na, nb, nc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        self.ref.lib.ref_index_prefix_related(C.c_void_p(self.h), vp(p), C.c_size_t(p.size), vp(a), C.byref(na),
                                              vp(b), C.byref(nb), vp(c), C.byref(nc))
        return a[:na.value].copy(), b[:nb.value].copy(), c[:nc.value].copy()

    def close(self):
        if self.h:
            self.ref.lib.ref_index_destroy(C.c_void_p(self.h))
            self.h = None

    def __del__(self):
        self.close()
