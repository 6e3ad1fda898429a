// Synthetic workloads of SURVEY.md section 8(d), host side.
//
// The definitions (not the code) come from the reference's bench generators:
//   random DNA   -- bench.hpp:66-72   one mt19937_64 draw per base, "ACGT"[x & 3]
//   random keys  -- bench.hpp:54-64   (uint32_t) draw, payload = index
//   bounded draw -- shotgun.hpp:20-27 rejection sampling so results do not depend on a
//                                     library distribution
//   read text    -- sequence.hpp:103-124  reads joined and terminated by byte 0
// std::mt19937_64 is specified bit-exactly by the C++ standard, so these reproduce the
// reference's inputs (pinned by the SA fingerprints in tests/test_synth.py).
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "reseq_cuda.h"

namespace {

uint64_t draw_below(std::mt19937_64& rng, uint64_t bound) {
    // largest multiple of `bound` that fits: values at or above it are redrawn
    const uint64_t all = ~uint64_t{0};
    const uint64_t limit = all - all % bound;
    uint64_t x = rng();
    while (x >= limit) x = rng();
    return x % bound;
}

}  // namespace

extern "C" {

void reseq_synth_random_dna(size_t n, uint64_t seed, uint8_t* out) {
    static const char kBases[4] = {'A', 'C', 'G', 'T'};
    std::mt19937_64 rng(seed);
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<uint8_t>(kBases[rng() & 3]);
}

void reseq_synth_random_keys(size_t n, uint64_t seed, uint32_t* keys, uint32_t* payload) {
    std::mt19937_64 rng(seed);
    for (size_t i = 0; i < n; ++i) {
        keys[i] = static_cast<uint32_t>(rng());
        if (payload) payload[i] = static_cast<uint32_t>(i);
    }
}

int reseq_synth_read_text(size_t genome_len, size_t read_len, size_t k, uint64_t genome_seed,
                          uint64_t read_seed, uint8_t* out, uint32_t* starts) {
    if (read_len == 0 || read_len > genome_len) return RESEQ_INVALID_ARGUMENT;
    if (k * (read_len + 1) > RESEQ_CUDA_MAX_TEXT) return RESEQ_TEXT_TOO_LARGE;
    std::vector<uint8_t> genome(genome_len);
    reseq_synth_random_dna(genome_len, genome_seed, genome.data());
    std::mt19937_64 rng(read_seed);
    const uint64_t span = genome_len - read_len + 1;
    uint8_t* dst = out;
    for (size_t i = 0; i < k; ++i) {
        const uint64_t s = draw_below(rng, span);
        if (starts) starts[i] = static_cast<uint32_t>(dst - out);
        std::memcpy(dst, genome.data() + s, read_len);
        dst += read_len;
        *dst++ = 0;
    }
    return RESEQ_OK;
}

}  // extern "C"
