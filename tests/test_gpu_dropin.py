"""The drop-in proven on the reference's own classes: oracle/_ref/dropin_test is the reference's
fragment_index (with the `builder::cuda` patch of INTEGRATION.md section 2), its assembler and its parallel
operators (with the executor_config::device patch of section 3) compiled against libreseq_cuda.so by
oracle/make_dropin.py -- here it runs on the GPU: the KATs of proj/tests/test_fragment_index.cpp:33-53,
82-104,129-138, its 3000 random prefix_related queries (:106-127) and the naive == indexed assembler check
of proj/tests/test_assembler.cpp:241-269, all over a suffix array built on the device."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "oracle" / "_ref" / "dropin_test"


@pytest.mark.gpu
def test_reference_classes_run_over_the_device_library(_built):
    if not EXE.exists():
        pytest.skip("oracle/_ref/dropin_test was not built (needs /root/reference at build time)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "drop-in ok" in r.stdout


def test_the_patch_applies_to_the_reference_headers(_built):
    """CPU: where the reference is present the patch anchors must all be found and the program must
    compile (build() does both); the binary is what travels to the GPU box."""
    if not Path("/root/reference/proj/include").is_dir():
        pytest.skip("no reference tree here")
    assert EXE.exists()
