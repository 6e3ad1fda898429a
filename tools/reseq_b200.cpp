// reseq-b200 command line: the two subcommands of the reference tool that sit on the hot path,
// with the reference's flags, defaults and file formats, so that the same command line writes the
// same bytes (proj/tools/reseq.cpp).
//
//   reseq_b200 [global options] build-sa <input> -o <out>
//       proj/tools/reseq.cpp:130-134,267-284 -- input: FASTA or raw text ('>' lines dropped, bytes
//       <= 32 and 127 stripped, DNA folded to upper case: io.hpp:42-58); output: the suffix array,
//       one decimal per line, or raw little-endian u32 with --format bin (any other value writes
//       decimals, as the reference does, :273-281); "wrote N entries to <out>" on stderr.
//   reseq_b200 [global options] bench [--ops a,b] [--sizes n,m] [--workers w,...] [--reps R]
//                                     [--digit-bits B] [--strict-sizes] [-o csv]
//       proj/tools/reseq.cpp:136-159,286-314, bench.hpp:106-171 -- CSV
//       "op,n,workers,chunk_size,rep,wall_time_ns,checksum" over radix_sort / chunked_radix_sort /
//       build_parallel on the reference's synthetic inputs (make_random_keys / make_random_dna,
//       bench.hpp:54-72) with the reference's FNV-1a checksums (bench.hpp:31-52): the checksum column
//       equals the reference tool's for the same (op, n, seed).  One block of rows per requested worker
//       count, like the reference (default 1 and the core count, :295-296); on the device the count
//       changes nothing but the column.  Default sizes: every power of two 2^10..2^20 (:61-65).
//   global options (the reference's, :71-83; accepted before or after the subcommand):
//       --format bin|txt (default txt)   --alphabet auto|dna|byte (default auto: detect_alphabet,
//       io.hpp:109-122; a byte outside the alphabet is invalid_byte_error, sequence.hpp:20-33)
//       --seed S   --workers N   --chunk-size N   --config file (workers / chunk_size: no device meaning)
//       --device N (this tool only)
//
// The reference CLI itself needs CLI11 and nlohmann-json (absent here, proj/.gitignore:2), hence
// this small hand-rolled parser; `reconstruct`, `overlap`, `shotgun`, `verify` are not on the
// accelerated path and are not offered.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "reseq_b200/reseq_cuda.hpp"

namespace {

namespace rc = reseq::cuda;

std::string read_sequence_text(std::istream& in, bool fold_upper) {   // io.hpp:44-58
    std::string text, line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.front() == '>') continue;
        for (char c : line) {
            const auto u = static_cast<unsigned char>(c);
            if (u <= 32 || u == 127) continue;
            text.push_back(fold_upper ? static_cast<char>(std::toupper(u)) : c);
        }
    }
    return text;
}

bool is_dna_text(const std::string& text) {   // detect_alphabet, io.hpp:109-122
    for (char c : text) {
        const int u = std::toupper(static_cast<unsigned char>(c));
        if (u != 'A' && u != 'C' && u != 'G' && u != 'T') return false;
    }
    return true;
}

// sequence's constructor (sequence.hpp:39-41, validate_bytes :26-33) with the message of
// invalid_byte_error (errors.hpp:20-28).
void validate_bytes(const std::string& text, bool dna) {
    for (std::size_t i = 0; i < text.size(); ++i) {
        const auto c = static_cast<unsigned char>(text[i]);
        const bool ok = dna ? (c == 'A' || c == 'C' || c == 'G' || c == 'T') : (c >= 33 && c <= 126);
        if (!ok)
            throw std::runtime_error("invalid byte " + std::to_string(int(c)) + " at position " + std::to_string(i) +
                                     " of fragment 0");
    }
}

std::string load_sequence(const std::string& path, const std::string& alphabet) {   // tools/reseq.cpp:47-59
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::string text = read_sequence_text(in, alphabet == "dna");
    if (text.empty()) throw std::runtime_error(path + " holds no sequence data");
    bool dna = alphabet == "dna";
    if (alphabet == "auto") {
        dna = is_dna_text(text);
        if (dna)
            for (auto& c : text) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
    }
    validate_bytes(text, dna);
    return text;
}

std::uint64_t fnv1a64(const unsigned char* b, std::size_t n, std::uint64_t h) {   // bench.hpp:31-38
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}
std::uint64_t checksum_u32(const std::vector<std::uint32_t>& v, std::uint64_t h = 14695981039346656037ull) {
    for (std::uint32_t x : v) {   // bench.hpp:40-48: over the little-endian bytes
        const unsigned char le[4] = {static_cast<unsigned char>(x), static_cast<unsigned char>(x >> 8),
                                     static_cast<unsigned char>(x >> 16), static_cast<unsigned char>(x >> 24)};
        h = fnv1a64(le, 4, h);
    }
    return h;
}

std::vector<std::string> split_csv(const std::string& s) {
    std::vector<std::string> out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) if (!item.empty()) out.push_back(item);
    return out;
}

int usage() {
    std::cerr << "usage: reseq_b200 [--format bin|txt] [--alphabet auto|dna|byte] [--seed S] [--workers N] [--chunk-size N]\n"
                 "                  [--config file] [--device N] <subcommand> ...\n"
                 "       reseq_b200 build-sa <input> -o <out>\n"
                 "       reseq_b200 bench [--ops radix_sort,chunked_radix_sort,build_parallel] [--sizes n,...] [--workers w,...]\n"
                 "                        [--reps R] [--digit-bits B] [--strict-sizes] [-o out.csv]\n";
    return 2;
}

// The reference's app-level options (tools/reseq.cpp:71-83), taken wherever they stand.
struct Globals {
    unsigned workers = 0;             // 0: default = core count
    std::size_t chunk_size = std::size_t{1} << 15;
    std::uint64_t seed = 1;
    std::string format = "txt";
    std::string alphabet = "auto";
    std::string config;
    int device = 0;
    bool bad = false;
};

// Consumes a global option at argv[i] (advancing i past its value); false if argv[i] is not one.
bool take_global(Globals& g, int argc, char** argv, int& i, bool in_bench) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
        if (i + 1 < argc) return argv[++i];
        g.bad = true;
        return std::string();
    };
    if (a == "--format") g.format = next();
    else if (a == "--alphabet") {
        g.alphabet = next();
        if (g.alphabet != "auto" && g.alphabet != "dna" && g.alphabet != "byte") g.bad = true;   // CLI::IsMember, :81-82
    }
    else if (a == "--seed") g.seed = std::stoull(next());
    else if (a == "--workers" && !in_bench) g.workers = static_cast<unsigned>(std::stoul(next()));
    else if (a == "--chunk-size") g.chunk_size = std::stoull(next());
    else if (a == "--config") g.config = next();
    else if (a == "--device") g.device = std::atoi(next().c_str());
    else return false;
    return true;
}

int cmd_build_sa(Globals& g, int argc, char** argv) {
    std::string input, out_path;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        if (take_global(g, argc, argv, i, false)) continue;
        if (a == "-o" || a == "--out") { if (i + 1 < argc) out_path = argv[++i]; else return usage(); }
        else if (!a.empty() && a[0] != '-' && input.empty()) input = a;
        else return usage();
    }
    if (g.bad || input.empty() || out_path.empty()) return usage();
    const std::string text = load_sequence(input, g.alphabet);
    rc::device_executor dev(g.device);
    const rc::suffix_array sa = rc::build_parallel(text, dev);
    std::ofstream out(out_path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open " + out_path);
    if (g.format == "bin") {   // tools/reseq.cpp:273-278
        std::vector<char> le(4 * sa.sa.size());
        for (std::size_t i = 0; i < sa.sa.size(); ++i) {
            const std::uint32_t v = sa.sa[i];
            le[4 * i] = static_cast<char>(v);
            le[4 * i + 1] = static_cast<char>(v >> 8);
            le[4 * i + 2] = static_cast<char>(v >> 16);
            le[4 * i + 3] = static_cast<char>(v >> 24);
        }
        out.write(le.data(), static_cast<std::streamsize>(le.size()));
    } else {                   // every other value: decimal lines (:279-281)
        for (std::uint32_t v : sa.sa) out << v << "\n";
    }
    std::cerr << "wrote " << sa.sa.size() << " entries to " << out_path << "\n";
    return 0;
}

int cmd_bench(Globals& g, int argc, char** argv) {
    std::vector<std::string> ops{"radix_sort", "chunked_radix_sort", "build_parallel"};
    std::vector<std::size_t> sizes;
    std::vector<unsigned> workers;
    unsigned reps = 3, digit_bits = 4;
    bool strict = false;
    std::string out_path;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        if (take_global(g, argc, argv, i, true)) continue;
        auto next = [&]() -> std::string { if (i + 1 < argc) return argv[++i]; g.bad = true; return std::string(); };
        if (a == "--ops") ops = split_csv(next());
        else if (a == "--sizes") { sizes.clear(); for (auto& s : split_csv(next())) sizes.push_back(std::stoull(s)); }
        else if (a == "--workers") { workers.clear(); for (auto& s : split_csv(next())) workers.push_back(static_cast<unsigned>(std::stoul(s))); }
        else if (a == "--reps") reps = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--digit-bits") digit_bits = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--strict-sizes") strict = true;
        else if (a == "--unit" || a == "--reconstruct-mode") next();   // reconstruct only: accepted, unused
        else if (a == "-o" || a == "--out") out_path = next();
        else return usage();
    }
    if (g.bad) return usage();
    if (sizes.empty()) for (std::size_t n = 1 << 10; n <= (1 << 20); n <<= 1) sizes.push_back(n);   // tools/reseq.cpp:61-65
    if (strict)
        for (auto s : sizes)
            if (s < (1 << 10) || s > (1 << 20) || (s & (s - 1))) {   // :289-294
                std::cerr << "--sizes: " << s << " is not a power of two in 2^10..2^20\n";
                return 105;   // CLI::ValidationError's exit code
            }
    if (workers.empty()) {   // :295-296
        unsigned hw = g.workers ? g.workers : std::thread::hardware_concurrency();
        if (hw == 0) hw = 1;
        workers = {1u, hw};
    }
    rc::device_executor dev(g.device);
    std::ofstream file;
    if (!out_path.empty()) {
        file.open(out_path, std::ios::binary);
        if (!file) throw std::runtime_error("cannot open " + out_path);
    }
    std::ostream& out = out_path.empty() ? std::cout : file;
    out << "op,n,workers,chunk_size,rep,wall_time_ns,checksum\n";   // bench.hpp:167
    std::size_t rows = 0;
    for (const auto& op : ops) {
        for (std::size_t size : sizes) {
            rc::key_array keys;
            std::string text;
            if (op == "radix_sort" || op == "chunked_radix_sort") {   // make_random_keys, bench.hpp:54-64
                std::mt19937_64 rng(g.seed);
                keys.keys.resize(size);
                keys.payload.resize(size);
                for (std::size_t i = 0; i < size; ++i) {
                    keys.keys[i] = static_cast<std::uint32_t>(rng());
                    keys.payload[i] = static_cast<std::uint32_t>(i);
                }
            } else if (op == "build_parallel") {                      // make_random_dna, bench.hpp:66-72
                std::mt19937_64 rng(g.seed);
                static const char bases[] = "ACGT";
                text.resize(size);
                for (auto& c : text) c = bases[rng() & 3];
            } else {
                continue;   // `reconstruct` is not on the accelerated path
            }
            for (unsigned w : workers) {
                for (unsigned rep = 0; rep < reps; ++rep) {
                    std::uint64_t checksum = 0;
                    rc::key_array sorted;
                    rc::suffix_array sa;
                    const auto t0 = std::chrono::steady_clock::now();   // the operation only, as bench.hpp:85-91
                    if (op == "radix_sort") sorted = rc::radix_sort(keys, dev);
                    else if (op == "chunked_radix_sort") sorted = rc::chunked_radix_sort(keys, dev, digit_bits);
                    else sa = rc::build_parallel(text, dev);
                    const auto t1 = std::chrono::steady_clock::now();
                    if (op == "build_parallel") checksum = checksum_u32(sa.sa);
                    else checksum = checksum_u32(sorted.payload, checksum_u32(sorted.keys));
                    const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
                    out << op << ',' << size << ',' << w << ',' << g.chunk_size << ',' << rep << ',' << ns << ',' << checksum << '\n';
                    ++rows;
                }
            }
        }
    }
    if (!out_path.empty()) std::cerr << "wrote " << rows << " rows to " << out_path << "\n";   // tools/reseq.cpp:311
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        Globals g;
        int i = 1;
        while (i < argc && take_global(g, argc, argv, i, false)) ++i;   // app-level options before the subcommand
        if (i >= argc || g.bad) return usage();
        const std::string cmd = argv[i];
        if (cmd == "build-sa") return cmd_build_sa(g, argc - i - 1, argv + i + 1);
        if (cmd == "bench") return cmd_bench(g, argc - i - 1, argv + i + 1);
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";   // tools/reseq.cpp:336-338
        return 1;
    }
}
