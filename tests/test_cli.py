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
    # FASTA with a header, lower case, blank lines and a trailing space: io.hpp:44-58
    rng = np.random.default_rng(3)
    seq = bytes(rng.choice([65, 67, 71, 84], 5000).astype(np.uint8)).decode()
    fasta = tmp_path / "t.fa"
    fasta.write_text(">chr1 test\n" + seq[:2000].lower() + "\n\n" + seq[2000:4000] + " \n>chr2\n" + seq[4000:] + "\n")
    want, _ = oracle.build_sa(np.frombuffer(seq.encode(), np.uint8))
    r = run("build-sa", fasta, "-o", tmp_path / "sa.bin")
    assert r.returncode == 0, r.stderr
    assert r.stderr.strip() == f"wrote 5000 entries to {tmp_path / 'sa.bin'}"   # tools/reseq.cpp:282
    assert (tmp_path / "sa.bin").read_bytes() == want.astype("<u4").tobytes()   # raw little-endian u32, :273-278
    r = run("build-sa", fasta, "--out", tmp_path / "sa.txt", "--format", "text")
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "sa.txt").read_text() == "".join(f"{v}\n" for v in want)  # :280
    # generic alphabet keeps the case (io.hpp:53-55): a different text, a different array
    raw = tmp_path / "g.txt"
    raw.write_text("abthatb hatbpaab\n")
    r = run("build-sa", raw, "-o", tmp_path / "g.bin", "--alphabet", "generic")
    assert r.returncode == 0, r.stderr
    want, _ = oracle.build_sa(np.frombuffer(b"abthatbhatbpaab", np.uint8))
    assert (tmp_path / "g.bin").read_bytes() == want.astype("<u4").tobytes()


@pytest.mark.gpu
def test_bench_csv_reproduces_the_reference_checksums(rq, tmp_path):
    """bench.hpp:166-171 columns; the checksums are the ones the reference tool prints for the same
    (op, n, seed = 1): BASELINE.md section 2."""
    out = tmp_path / "b.csv"
    r = run("bench", "--ops", "build_parallel,radix_sort,chunked_radix_sort", "--sizes", 1 << 20, "--reps", 2, "-o", out)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "op,n,workers,chunk_size,rep,wall_time_ns,checksum"
    rows = [ln.split(",") for ln in lines[1:]]
    assert len(rows) == 6
    by_op = {}
    for op, n, workers, chunk, rep, ns, checksum in rows:
        assert n == str(1 << 20) and int(ns) > 0
        by_op.setdefault(op, set()).add(int(checksum))
    assert by_op["build_parallel"] == {7546189330682201289}
    assert by_op["radix_sort"] == {91396105105168530}
    assert by_op["chunked_radix_sort"] == {91396105105168530}
