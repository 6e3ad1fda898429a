"""The C-ABI library loads, exports exactly the symbols include/reseq_cuda.h declares, and
refuses to compute without a device (no CPU fallback).  CPU only: no compute calls."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = (ROOT / "include" / "reseq_cuda.h").read_text()


def declared_functions():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    return sorted(set(re.findall(r"\b(reseq_[a-z0-9_]+)\s*\(", body)))


def test_header_declares_what_the_binding_binds(rq):
    names = declared_functions()
    assert len(names) >= 30
    assert sorted(rq._lib.SIGNATURES) == names


def test_library_exports_every_declared_symbol(rq):
    lib = rq._lib.load()
    out = subprocess.run(["nm", "-D", "--defined-only", str(rq._lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (reseq_[a-z0-9_]+)", out))
    for name in declared_functions():
        assert name in exported, f"{name} declared in reseq_cuda.h but not exported"
        assert getattr(lib, name) is not None
    assert b"sm_100a" in lib.reseq_cuda_version()


def test_header_compiles_as_c(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "reseq_cuda.h"\nint main(void){ reseq_sa_stats s; (void)s; return RESEQ_OK; }\n')
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-c", str(src), "-o",
                    str(tmp_path / "t.o")], check=True)


def test_sm100a_code_is_embedded(rq):
    out = subprocess.run(["cuobjdump", "-lelf", str(rq._lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback(rq):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rq.NoDeviceError):
        rq.Executor(0)
    with pytest.raises(rq.NoDeviceError):
        rq.build_parallel(b"banana")


def test_argument_validation_needs_no_device(rq):
    # digit_bits is validated before any device work (radix_sort.hpp:171-172)
    with pytest.raises(ValueError):
        rq.chunked_radix_sort([1, 2], None, None, 0)
    with pytest.raises(ValueError):
        rq.chunked_radix_sort([1, 2], None, None, 9)
    lib = rq._lib.load()
    assert lib.reseq_cuda_split_by_bit(None, None, None, 0, 40, None, None) == rq._lib.INVALID_ARGUMENT
    assert lib.reseq_cuda_chunked_radix_sort(None, None, None, 0, 12, None, None) == rq._lib.INVALID_ARGUMENT


def test_fragment_set_layout_and_validation(rq):
    # test_sequence.cpp:9-25
    fs = rq.make_fragment_set([b"GA", b"TT"], "dna")
    assert fs.concat.tobytes() == b"GA\0TT\0" and fs.starts.tolist() == [0, 3]
    fs = rq.make_fragment_set([b"abthatb", b"hatbpaab", b"tbabhhatbpaa", b"paabtabh", b"bhaabtpb"], "generic_byte")
    assert fs.concat.size == 43 + 5 and fs.lengths().tolist() == [7, 8, 12, 8, 8]
    assert fs.bytes(2) == b"tbabhhatbpaa" and fs.length(4) == 8
    with pytest.raises(rq.EmptyFragmentError):
        rq.make_fragment_set([b"GA", b""], "dna")
    with pytest.raises(rq.InvalidByteError):
        rq.make_fragment_set([b"GAX"], "dna")
    with pytest.raises(rq.InvalidByteError):
        rq.make_fragment_set([b"a b"], "generic_byte")
