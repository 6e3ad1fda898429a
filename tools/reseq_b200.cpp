// reseq-b200 command line: the two subcommands of the reference tool that sit on the hot path,
// with the reference's file formats, so that outputs can be diffed byte for byte.
//
//   reseq_b200 build-sa <input> -o <out> [--format bin|text] [--alphabet dna|generic] [--device N]
//       proj/tools/reseq.cpp:267-284 -- input: FASTA or raw text ('>' lines dropped, bytes <= 32 and
//       127 stripped, DNA folded to upper case: io.hpp:42-58); output: the suffix array as raw
//       little-endian u32 (bin) or one decimal per line (text); "wrote N entries to <out>" on stderr.
//   reseq_b200 bench [--ops a,b] [--sizes n,m] [--reps R] [--digit-bits B] [--seed S] [-o csv]
//       bench.hpp:106-171 -- CSV "op,n,workers,chunk_size,rep,wall_time_ns,checksum" over
//       radix_sort / chunked_radix_sort / build_parallel on the reference's synthetic inputs
//       (make_random_keys / make_random_dna, bench.hpp:54-72) with the reference's FNV-1a checksums
//       (bench.hpp:31-52): the checksum column must equal the reference tool's for the same
//       (op, n, seed).  workers is reported as 0 (device), chunk_size as 0.
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
#include <string>
#include <vector>

#include "reseq_b200/reseq_cuda.hpp"

namespace {

namespace rc = reseq::cuda;

std::string read_sequence_text(std::istream& in, bool dna) {   // io.hpp:44-58
    std::string text, line;
    while (std::getline(in, line)) {
        if (!line.empty() && line.front() == '>') continue;
        for (char c : line) {
            const auto u = static_cast<unsigned char>(c);
            if (u <= 32 || u == 127) continue;
            text.push_back(dna ? static_cast<char>(std::toupper(u)) : c);
        }
    }
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
    std::cerr << "usage: reseq_b200 build-sa <input> -o <out> [--format bin|text] [--alphabet dna|generic] [--device N]\n"
                 "       reseq_b200 bench [--ops radix_sort,chunked_radix_sort,build_parallel] [--sizes n,...]\n"
                 "                        [--reps R] [--digit-bits B] [--seed S] [--device N] [-o out.csv]\n";
    return 2;
}

int cmd_build_sa(int argc, char** argv) {
    std::string input, out_path, format = "bin", alphabet = "dna";
    int device = 0;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : std::string(); };
        if (a == "-o" || a == "--out") out_path = next();
        else if (a == "--format") format = next();
        else if (a == "--alphabet") alphabet = next();
        else if (a == "--device") device = std::atoi(next().c_str());
        else if (!a.empty() && a[0] != '-' && input.empty()) input = a;
        else return usage();
    }
    if (input.empty() || out_path.empty() || (format != "bin" && format != "text") ||
        (alphabet != "dna" && alphabet != "generic"))
        return usage();
    std::ifstream in(input, std::ios::binary);
    if (!in) { std::cerr << "error: cannot open " << input << "\n"; return 1; }
    const std::string text = read_sequence_text(in, alphabet == "dna");
    if (text.empty()) { std::cerr << "error: " << input << " holds no sequence data\n"; return 1; }
    rc::device_executor dev(device);
    const rc::suffix_array sa = rc::build_parallel(text, dev);
    std::ofstream out(out_path, std::ios::binary);
    if (!out) { std::cerr << "error: cannot open " << out_path << "\n"; return 1; }
    if (format == "bin") {
        std::vector<char> le(4 * sa.sa.size());
        for (std::size_t i = 0; i < sa.sa.size(); ++i) {
            const std::uint32_t v = sa.sa[i];
            le[4 * i] = static_cast<char>(v);
            le[4 * i + 1] = static_cast<char>(v >> 8);
            le[4 * i + 2] = static_cast<char>(v >> 16);
            le[4 * i + 3] = static_cast<char>(v >> 24);
        }
        out.write(le.data(), static_cast<std::streamsize>(le.size()));
    } else {
        for (std::uint32_t v : sa.sa) out << v << "\n";
    }
    std::cerr << "wrote " << sa.sa.size() << " entries to " << out_path << "\n";
    return 0;
}

int cmd_bench(int argc, char** argv) {
    std::vector<std::string> ops{"radix_sort", "chunked_radix_sort", "build_parallel"};
    std::vector<std::size_t> sizes;
    unsigned reps = 3, digit_bits = 4;
    std::uint64_t seed = 1;
    int device = 0;
    std::string out_path;
    for (int i = 0; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> std::string { return i + 1 < argc ? argv[++i] : std::string(); };
        if (a == "--ops") ops = split_csv(next());
        else if (a == "--sizes") { sizes.clear(); for (auto& s : split_csv(next())) sizes.push_back(std::stoull(s)); }
        else if (a == "--reps") reps = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--digit-bits") digit_bits = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--seed") seed = std::stoull(next());
        else if (a == "--device") device = std::atoi(next().c_str());
        else if (a == "-o" || a == "--out") out_path = next();
        else return usage();
    }
    if (sizes.empty()) for (int e = 10; e <= 20; e += 2) sizes.push_back(std::size_t{1} << e);   // tools/reseq.cpp:61-65
    rc::device_executor dev(device);
    std::ofstream file;
    if (!out_path.empty()) {
        file.open(out_path);
        if (!file) { std::cerr << "error: cannot open " << out_path << "\n"; return 1; }
    }
    std::ostream& out = out_path.empty() ? std::cout : file;
    out << "op,n,workers,chunk_size,rep,wall_time_ns,checksum\n";   // bench.hpp:167
    for (const auto& op : ops) {
        for (std::size_t size : sizes) {
            rc::key_array keys;
            std::string text;
            if (op == "radix_sort" || op == "chunked_radix_sort") {   // make_random_keys, bench.hpp:54-64
                std::mt19937_64 rng(seed);
                keys.keys.resize(size);
                keys.payload.resize(size);
                for (std::size_t i = 0; i < size; ++i) {
                    keys.keys[i] = static_cast<std::uint32_t>(rng());
                    keys.payload[i] = static_cast<std::uint32_t>(i);
                }
            } else if (op == "build_parallel") {                      // make_random_dna, bench.hpp:66-72
                std::mt19937_64 rng(seed);
                static const char bases[] = "ACGT";
                text.resize(size);
                for (auto& c : text) c = bases[rng() & 3];
            } else {
                continue;   // `reconstruct` is not on the accelerated path
            }
            for (unsigned rep = 0; rep < reps; ++rep) {
                std::uint64_t checksum = 0;
                const auto t0 = std::chrono::steady_clock::now();
                if (op == "radix_sort") {
                    const auto r = rc::radix_sort(keys, dev);
                    checksum = checksum_u32(r.payload, checksum_u32(r.keys));
                } else if (op == "chunked_radix_sort") {
                    const auto r = rc::chunked_radix_sort(keys, dev, digit_bits);
                    checksum = checksum_u32(r.payload, checksum_u32(r.keys));
                } else {
                    const auto r = rc::build_parallel(text, dev);
                    checksum = checksum_u32(r.sa);
                }
                const auto t1 = std::chrono::steady_clock::now();
                const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
                out << op << ',' << size << ",0,0," << rep << ',' << ns << ',' << checksum << '\n';
            }
        }
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    try {
        const std::string cmd = argv[1];
        if (cmd == "build-sa") return cmd_build_sa(argc - 2, argv + 2);
        if (cmd == "bench") return cmd_bench(argc - 2, argv + 2);
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
