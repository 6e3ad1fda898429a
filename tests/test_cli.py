"""The command-line tool (tools/reseq_b200.cpp): the reference tool's `build-sa` and `bench`
subcommands (proj/tools/reseq.cpp:267-314) with its file formats -- SURVEY.md section 8(f) row 3."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
TOOL = ROOT / "paper_1404_3456_b200" / "reseq_b200"


def run(*args):
    return subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True)


def test_tool_is_built_and_prints_usage(_built):
    assert TOOL.exists()
    r = run()
    assert r.returncode == 2 and "build-sa" in r.stderr and "bench" in r.stderr
    assert run("build-sa", "only-input").returncode == 2          # -o is required (tools/reseq.cpp:131-132)
    assert run("frobnicate").returncode == 2


def test_missing_input_is_an_io_error(_built, tmp_path):
    r = run("build-sa", tmp_path / "absent.fa", "-o", tmp_path / "sa.bin")
    assert r.returncode == 1 and "cannot open" in r.stderr         # io_error, io.hpp:61-62


@pytest.mark.gpu
def test_build_sa_formats_match_the_reference_tool(rq, oracle, tmp_path):
    """The reference's own command lines (tools/reseq.cpp:71-83,130-134): app-level --format /
    --alphabet, default format txt (decimal lines), default alphabet auto."""
    # FASTA with a header, lower case, blank lines and a trailing space: io.hpp:44-58
    rng = np.random.default_rng(3)
    seq = bytes(rng.choice([65, 67, 71, 84], 5000).astype(np.uint8)).decode()
    fasta = tmp_path / "t.fa"
    fasta.write_text(">chr1 test\n" + seq[:2000].lower() + "\n\n" + seq[2000:4000] + " \n>chr2\n" + seq[4000:] + "\n")
    want, _ = oracle.build_sa(np.frombuffer(seq.encode(), np.uint8))
    # the reference's default: `build-sa in -o out` writes decimal lines (format = "txt", :76, :279-281)
    r = run("build-sa", fasta, "-o", tmp_path / "sa.txt")
    assert r.returncode == 0, r.stderr
    assert r.stderr.strip() == f"wrote 5000 entries to {tmp_path / 'sa.txt'}"   # tools/reseq.cpp:282
    assert (tmp_path / "sa.txt").read_text() == "".join(f"{v}\n" for v in want)
    # app-level option before the subcommand, as CLI11 parses it; raw little-endian u32 (:273-278)
    r = run("--format", "bin", "build-sa", fasta, "-o", tmp_path / "sa.bin")
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "sa.bin").read_bytes() == want.astype("<u4").tobytes()
    # ... and after it; `txt` is accepted, any value other than bin writes decimals (:279)
    for fmt in ("txt", "text"):
        r = run("build-sa", fasta, "--out", tmp_path / f"sa2.{fmt}", "--format", fmt)
        assert r.returncode == 0, r.stderr
        assert (tmp_path / f"sa2.{fmt}").read_text() == "".join(f"{v}\n" for v in want)
    # --alphabet auto (the default): a text with other letters is a byte text and keeps its case
    raw = tmp_path / "g.txt"
    raw.write_text("abthatb hatbpaab\n")
    want_g, _ = oracle.build_sa(np.frombuffer(b"abthatbhatbpaab", np.uint8))
    for extra in ([], ["--alphabet", "byte"], ["--alphabet", "auto"]):
        r = run(*extra, "--format", "bin", "build-sa", raw, "-o", tmp_path / "g.bin")
        assert r.returncode == 0, r.stderr
        assert (tmp_path / "g.bin").read_bytes() == want_g.astype("<u4").tobytes()
    # --alphabet dna on it: upper-cased, then invalid_byte_error from the sequence constructor
    r = run("--alphabet", "dna", "build-sa", raw, "-o", tmp_path / "g2.bin")
    assert r.returncode == 1 and "invalid byte 66 at position 1 of fragment 0" in r.stderr   # 'B'
    # values outside auto|dna|byte are rejected by the option check (:81-82); the old spelling was `generic`
    assert run("--alphabet", "generic", "build-sa", raw, "-o", tmp_path / "g3.bin").returncode == 2
    # a control byte inside a byte text is stripped by the reader, a byte > 126 is invalid
    (tmp_path / "hi.txt").write_bytes(b"ab\xffcd\n")
    r = run("--alphabet", "byte", "build-sa", tmp_path / "hi.txt", "-o", tmp_path / "hi.bin")
    assert r.returncode == 1 and "invalid byte 255 at position 2" in r.stderr


@pytest.mark.gpu
def test_bench_csv_reproduces_the_reference_checksums(rq, tmp_path):
    """bench.hpp:166-171 columns; the checksums are the ones the reference tool prints for the same
    (op, n, seed = 1): BASELINE.md section 2.  One block per worker count (tools/reseq.cpp:295-296)."""
    out = tmp_path / "b.csv"
    r = run("--chunk-size", 4096, "bench", "--ops", "build_parallel,radix_sort,chunked_radix_sort", "--sizes", 1 << 20,
            "--workers", "1,3", "--reps", 2, "-o", out)
    assert r.returncode == 0, r.stderr
    assert r.stderr.strip() == f"wrote 12 rows to {out}"            # tools/reseq.cpp:311
    lines = out.read_text().splitlines()
    assert lines[0] == "op,n,workers,chunk_size,rep,wall_time_ns,checksum"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 12
    by_op = {}
    for op, n, workers, chunk, rep, ns, checksum in rows:
        assert n == str(1 << 20) and int(ns) > 0 and workers in ("1", "3") and chunk == "4096"
        by_op.setdefault(op, set()).add(int(checksum))
    assert by_op["build_parallel"] == {7546189330682201289}
    assert by_op["radix_sort"] == {91396105105168530}
    assert by_op["chunked_radix_sort"] == {91396105105168530}
    # default sizes: every power of two 2^10 .. 2^20 (tools/reseq.cpp:61-65)
    r = run("bench", "--ops", "radix_sort", "--workers", 1, "--reps", 1)
    assert r.returncode == 0, r.stderr
    sizes = [int(ln.split(",")[1]) for ln in r.stdout.splitlines()[1:]]
    assert sizes == [1 << e for e in range(10, 21)]
    assert run("bench", "--sizes", 1000, "--strict-sizes").returncode != 0
