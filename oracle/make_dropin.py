"""TEST INFRASTRUCTURE -- builds oracle/_ref/dropin_test: the REFERENCE'S OWN fragment_index, assembler and
parallel operators compiled against libreseq_cuda.so through the two plug points of SURVEY.md 8(b).

Nothing of the reference is copied into the repository: a scratch copy of /root/reference/proj/include is
made in a temporary directory, patched there exactly as INTEGRATION.md sections 2 and 3 describe --

  * fragment_index.hpp:32-38   `builder::cuda`: the constructor takes sa_ from reseq_cuda_build_sa;
  * executor.hpp:13-15         `int device = -1;` in executor_config;
  * suffix_array.hpp:61, scan.hpp:32, radix_sort.hpp:126,143,169   one forwarding line at the top of
    build_parallel / exclusive_scan / split_by_bit / radix_sort / chunked_radix_sort;

-- and tests/cpp/test_dropin.cpp is compiled against the patched headers.  Only the binary is kept
(oracle/_ref/ is git-ignored; it travels to the GPU box with the snapshot, where /root/reference does
not exist).  Fails loudly if a patch anchor is not found: the patch is then out of date.
"""
from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/proj/include")
OUT = ROOT / "oracle" / "_ref" / "dropin_test"
LIB = ROOT / "paper_1404_3456_b200" / "libreseq_cuda.so"


def sub(text: str, old: str, new: str, what: str) -> str:
    if text.count(old) != 1:
        raise RuntimeError(f"patch anchor for {what} found {text.count(old)} times (expected once)")
    return text.replace(old, new)


def patch(inc: Path) -> None:
    f = inc / "reseq" / "fragment_index.hpp"
    s = f.read_text()
    s = sub(s, '#include "reseq/suffix_array.hpp"\n', '#include "reseq/suffix_array.hpp"\n#include "reseq_cuda.h"\n', "fragment_index include")
    s = sub(s, "enum class builder { direct, scan_radix };", "enum class builder { direct, scan_radix, cuda };", "builder enum")
    s = sub(s, """        sa_ = b == builder::scan_radix ? build_parallel(set.concat(), exec)
                                       : build_naive(set.concat());
""", """        if (b == builder::cuda) {
            reseq_cuda_ctx* ctx = nullptr;
            if (reseq_cuda_ctx_create(0, &ctx) != RESEQ_OK) throw error(reseq_cuda_last_error());
            const auto& text = set.concat();
            sa_.sa.resize(text.size());
            sa_.rank.resize(text.size());
            const int st = reseq_cuda_build_sa(ctx, reinterpret_cast<const uint8_t*>(text.data()), text.size(),
                                               sa_.sa.data(), sa_.rank.data(), nullptr);
            reseq_cuda_ctx_destroy(ctx);
            if (st == RESEQ_TEXT_TOO_LARGE) throw text_too_large_error(text.size());
            if (st != RESEQ_OK) throw error(reseq_cuda_last_error());
        } else {
            sa_ = b == builder::scan_radix ? build_parallel(set.concat(), exec)
                                           : build_naive(set.concat());
        }
""", "fragment_index constructor")
    f.write_text(s)

    f = inc / "reseq" / "executor.hpp"
    s = f.read_text()
    s = sub(s, "    std::size_t chunk_size = std::size_t{1} << 15;\n", "    std::size_t chunk_size = std::size_t{1} << 15;\n    int device = -1;   // >= 0: the operators run on that CUDA device\n", "executor_config")
    f.write_text(s)

    f = inc / "reseq" / "suffix_array.hpp"
    s = f.read_text()
    s = sub(s, """inline suffix_array build_parallel(std::string_view text,
                                   const executor& exec = executor()) {
""", """}  // namespace reseq
#include "reseq_b200/executor_dispatch.hpp"
namespace reseq {
inline suffix_array build_parallel(std::string_view text,
                                   const executor& exec = executor()) {
    if (exec.config().device >= 0) return cuda::dispatch::build_parallel<suffix_array>(text, exec.config().device);
""", "build_parallel")
    f.write_text(s)

    f = inc / "reseq" / "scan.hpp"
    s = f.read_text()
    head = s[s.index("inline std::vector<std::uint32_t> exclusive_scan(std::span<const std::uint32_t> values,"):]
    sig = head[:head.index("{\n") + 2]
    s = sub(s, sig, "}  // namespace reseq\n#include \"reseq_b200/executor_dispatch.hpp\"\nnamespace reseq {\n" + sig +
            "    if (exec.config().device >= 0) return cuda::dispatch::exclusive_scan(values, exec.config().device);\n", "exclusive_scan")
    f.write_text(s)

    f = inc / "reseq" / "radix_sort.hpp"
    s = f.read_text()
    for name, call in (("split_by_bit(const key_array& arr, unsigned bit,", "split_by_bit(arr, bit, exec.config().device)"),
                       ("radix_sort(const key_array& arr, const executor& exec = executor()) {", "radix_sort(arr, exec.config().device)"),
                       ("chunked_radix_sort(const key_array& arr, const executor& exec,", "chunked_radix_sort(arr, digit_bits, exec.config().device)")):
        start = s.index("inline key_array " + name)
        brace = s.index("{\n", start) + 2
        s = s[:brace] + f"    if (exec.config().device >= 0) return cuda::dispatch::{call};\n" + s[brace:]
    s = sub(s, "inline key_array split_by_bit(const key_array& arr, unsigned bit,",
            "}  // namespace reseq\n#include \"reseq_b200/executor_dispatch.hpp\"\nnamespace reseq {\ninline key_array split_by_bit(const key_array& arr, unsigned bit,", "radix_sort include")
    f.write_text(s)


def main() -> int:
    if not REF.is_dir():
        print("make_dropin: /root/reference absent; keeping the prebuilt binary if any")
        return 0
    if not LIB.exists():
        raise SystemExit("make_dropin: build libreseq_cuda.so first")
    src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    deps = [src, Path(__file__), LIB, ROOT / "include" / "reseq_b200" / "executor_dispatch.hpp", ROOT / "include" / "reseq_cuda.h"]
    if OUT.exists() and all(OUT.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return 0
    OUT.parent.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory(prefix="reseq_dropin_") as tmp:
        inc = Path(tmp) / "include"
        shutil.copytree(REF, inc)
        patch(inc)
        cmd = ["g++", "-std=c++20", "-O1", "-pthread", "-I", str(inc), "-I", str(ROOT / "include"), str(src), str(LIB),
               "-Wl,-rpath,$ORIGIN/../../paper_1404_3456_b200", "-o", str(OUT)]
        r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        if r.returncode != 0:
            raise SystemExit("make_dropin: compile failed\n" + r.stdout)
    print(OUT)
    return 0


if __name__ == "__main__":
    sys.exit(main())
