/*
 * reseq_cuda.h -- C ABI of the B200 (sm_100a) backend for the `reseq` hot path:
 * suffix-array construction over sentinel-joined read sets, the data-parallel
 * primitives it is made of, SA-driven prefix-range / overlap queries, and the host
 * greedy superstring merge.
 *
 * Every entry point replaces one reference interface (cited as
 * proj/include/reseq/<file>:<line>, relative to the reference root).  The reference
 * is a header-only C++ library with no FFI of its own; its extension points are the
 * `const executor&` argument and `fragment_index::builder`.  INTEGRATION.md shows the
 * binding a reference maintainer would add (a `builder::cuda` enumerator and an
 * executor backend that forward to these symbols).
 *
 * Conventions
 *   - plain pointers + sizes; no C++/torch types; no exception crosses this boundary.
 *   - every function returns an int status (RESEQ_OK == 0); reseq_cuda_last_error()
 *     gives the message of the calling thread's most recent failure.
 *   - "host" entry points take HOST buffers and perform H2D / D2H internally
 *     (pinned buffers are copied at full PCIe rate; pageable ones work too).
 *   - "_device" entry points take DEVICE pointers (HBM-resident data) and enqueue on
 *     the context's stream; call reseq_cuda_ctx_synchronize() before reading results.
 *   - outputs are pre-sized by the caller (value semantics of the reference's
 *     std::vector returns are provided by the C++ shim in include/reseq_b200/).
 *   - empty inputs are valid and produce empty outputs (suffix_array.hpp:66,
 *     scan.hpp:35, radix_sort.hpp:146).
 *   - one host thread per context at a time (executor.hpp:39-40 has the same rule);
 *     a finished index is immutable and may be queried concurrently from several
 *     contexts.
 *   - there is NO CPU fallback: without a CUDA device every compute entry point
 *     fails with RESEQ_NO_DEVICE.
 */
#ifndef RESEQ_CUDA_H
#define RESEQ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ shim maps them back to the reference's exception types
 * (errors.hpp:9-11,54-61; radix_sort.hpp:171-172). */
enum reseq_status {
    RESEQ_OK = 0,
    RESEQ_INVALID_ARGUMENT = 1, /* std::invalid_argument (e.g. digit_bits not in 1..8) */
    RESEQ_TEXT_TOO_LARGE = 2,   /* reseq::text_too_large_error */
    RESEQ_SCAN_OVERFLOW = 3,    /* reseq::scan_overflow_error */
    RESEQ_CUDA_ERROR = 4,       /* reseq::error carrying the CUDA message */
    RESEQ_OUT_OF_MEMORY = 5,
    RESEQ_NO_DEVICE = 6,
    RESEQ_BUFFER_TOO_SMALL = 7  /* caller-provided output arrays too short; the needed size is reported */
};

/* Largest text the device path accepts.  The reference caps at 2^31-1
 * (suffix_array.hpp:64, sequence.hpp:113-114); positions and rank+1 are u32, so the
 * device path relaxes the cap to 2^32-2 (needed for the 3 Gbp configuration). */
#define RESEQ_CUDA_MAX_TEXT 0xFFFFFFFEull

typedef struct reseq_cuda_ctx reseq_cuda_ctx;     /* device + stream + workspace arena */
typedef struct reseq_cuda_index reseq_cuda_index; /* device-resident fragment index */

/* ---- context ------------------------------------------------------------------ */

/* Replaces: executor construction, executor.hpp:28-37 (the BSP thread pool becomes a
 * device + stream; `workers`/`chunk_size` have no device meaning). */
int reseq_cuda_ctx_create(int device, reseq_cuda_ctx** out);
void reseq_cuda_ctx_destroy(reseq_cuda_ctx* ctx);
/* Launch on an externally owned cudaStream_t (e.g. torch's current stream) so callers
 * can bracket work with their own events and order it against their own kernels and NCCL.
 * NULL restores the context's own (non-blocking) stream.  The legacy default stream -- whose
 * cudaStream_t value is also 0, which is what torch.cuda.current_stream().cuda_stream returns
 * unless a side stream is current -- is selected with RESEQ_CUDA_STREAM_LEGACY (the value of
 * cudaStreamLegacy); RESEQ_CUDA_STREAM_PER_THREAD likewise (cudaStreamPerThread). */
#define RESEQ_CUDA_STREAM_LEGACY ((void*)0x1)
#define RESEQ_CUDA_STREAM_PER_THREAD ((void*)0x2)
int reseq_cuda_ctx_set_stream(reseq_cuda_ctx* ctx, void* cuda_stream);
int reseq_cuda_ctx_synchronize(reseq_cuda_ctx* ctx);
/* Number of kernels this context has launched since creation (bench `gpu_launches`). */
uint64_t reseq_cuda_ctx_launch_count(const reseq_cuda_ctx* ctx);
/* Bytes currently held by the context's workspace arena. */
size_t reseq_cuda_ctx_workspace_bytes(const reseq_cuda_ctx* ctx);
/* Tuning / test knobs; results never depend on them.  Unknown names are RESEQ_INVALID_ARGUMENT.
 *   "sa_uniform"      0 switches off the path for uniform read sets (k reads of one length:
 *                     transposed 16-base records, one verified overlap per read); default 1
 *   "sa_ragged"       0 switches off the path for ragged read sets (reads of mixed lengths <= 254 bases: the
 *                     uniform path's flow with looked-up terminator distances); default 1.  "sa_uniform" = 0
 *                     switches off both and leaves the general DNA records
 *   "sa_text_rounds"  maximum number of shared-memory group-refinement rounds (keys fetched from
 *                     the packed text) the DNA paths run before handing over to prefix doubling;
 *                     0 forces pure prefix doubling; default 16
 *   "sa_shortcut"     0 switches off the sentinel-distance shortcut of the general DNA path
 *   "sort_cfg"        onesweep tile shape, 0 (default tuning) .. 9
 *   "sa_doubling_local" 0: prefix-doubling rounds always sort (group, rank2) pairs of all suffixes with the
 *                     global digit passes (default 1: each CTA orders the groups of its tile in shared
 *                     memory; the global form runs only for groups that outgrow a CTA's window)
 *   "sa_speculate"    0: never start a build on the previous build's route (default 1: a context that
 *                     has just built a uniform read set of n bytes queues the next n-byte build on the
 *                     same route without a host round trip; the route's premises are re-checked on the
 *                     device and a text of another kind is rebuilt the ordinary way)
 *   "sa_graph"        0: never replay the speculative route as a CUDA graph (default 1: a device-resident
 *                     build whose text, outputs, workspace, stream and options are those of the previous
 *                     build is ONE cudaGraphLaunch; needs a stream of the caller's or the context's own --
 *                     capture is not allowed on the legacy default stream -- and no per-kernel profiling)
 *   "inverse_mode"    how rank = sa^-1 is computed above 2^22 suffixes: 0 two partition passes + a
 *                     shared-memory window scatter, 1 one partition pass + an L2-window scatter */
int reseq_cuda_ctx_set_option(reseq_cuda_ctx* ctx, const char* name, long long value);
/* Per-kernel device timing, measured with CUDA events recorded on the launching stream
 * around every launch while enabled.  reseq_cuda_ctx_profile(ctx, 1) clears and starts,
 * (ctx, 0) stops; reseq_cuda_ctx_profile_read synchronises the stream and writes up to
 * `cap` per-kernel-name aggregates, returning how many names exist. */
typedef struct reseq_kernel_profile {
    char name[48];
    uint64_t launches;
    double total_ms;
} reseq_kernel_profile;
int reseq_cuda_ctx_profile(reseq_cuda_ctx* ctx, int enable);
size_t reseq_cuda_ctx_profile_read(reseq_cuda_ctx* ctx, reseq_kernel_profile* out, size_t cap);
const char* reseq_cuda_last_error(void);
const char* reseq_cuda_version(void);

/* ---- L0 primitives ------------------------------------------------------------ */

/* Replaces exclusive_scan, scan.hpp:32-56: out[i] = sum(values[0..i)).  A grand total
 * above 0xFFFFFFFF returns RESEQ_SCAN_OVERFLOW (scan.hpp:38) and leaves `out`
 * unspecified. */
int reseq_cuda_exclusive_scan(reseq_cuda_ctx* ctx, const uint32_t* values, size_t n,
                              uint32_t* out);
int reseq_cuda_exclusive_scan_device(reseq_cuda_ctx* ctx, const uint32_t* d_values, size_t n,
                                     uint32_t* d_out, uint64_t* total_out /* host, nullable */);

/* Replaces split_by_bit, radix_sort.hpp:126-139: stable partition, bit==0 first.
 * `payload`/`payload_out` may both be NULL (key_array without payload,
 * radix_sort.hpp:16-23).  bit > 31 is RESEQ_INVALID_ARGUMENT. */
int reseq_cuda_split_by_bit(reseq_cuda_ctx* ctx, const uint32_t* keys, const uint32_t* payload,
                            size_t n, unsigned bit, uint32_t* keys_out, uint32_t* payload_out);

/* Replaces detail::split_destinations, radix_sort.hpp:35-52 (the paper's Alg. 1 dataflow,
 * PAPER.md:310-348): b = bit value, e = 1 - b, f = exclusive scan of e, tof = e[n-1] + f[n-1],
 * destinations[i] = b[i] ? i - f[i] + tof : f[i]; *total_false = tof (0 for n = 0).
 * bit > 31 is RESEQ_INVALID_ARGUMENT. */
int reseq_cuda_split_destinations(reseq_cuda_ctx* ctx, const uint32_t* keys, size_t n, unsigned bit,
                                  uint32_t* destinations, uint32_t* total_false);
/* Replaces detail::phase_is_sorted, radix_sort.hpp:54-66 (radix_sort's early exit, :151):
 * *sorted = 1 iff keys[i-1] <= keys[i] for all i. */
int reseq_cuda_is_sorted(reseq_cuda_ctx* ctx, const uint32_t* keys, size_t n, int* sorted);

/* Replaces radix_sort, radix_sort.hpp:143-161: stable ascending sort on keys, payload
 * carried.  Implemented as an 8-bit-digit LSD "onesweep" radix sort; passes whose
 * digit is constant over the whole array are skipped (the analogue of the
 * reference's sortedness early-exit, radix_sort.hpp:151). */
int reseq_cuda_radix_sort(reseq_cuda_ctx* ctx, const uint32_t* keys, const uint32_t* payload,
                          size_t n, uint32_t* keys_out, uint32_t* payload_out);
int reseq_cuda_radix_sort_device(reseq_cuda_ctx* ctx, const uint32_t* d_keys,
                                 const uint32_t* d_payload, size_t n, uint32_t* d_keys_out,
                                 uint32_t* d_payload_out);

/* Replaces chunked_radix_sort, radix_sort.hpp:169-303: same result as radix_sort;
 * `digit_bits` selects the radix width of the device passes and must be in 1..8,
 * otherwise RESEQ_INVALID_ARGUMENT (radix_sort.hpp:171-172). */
int reseq_cuda_chunked_radix_sort(reseq_cuda_ctx* ctx, const uint32_t* keys,
                                  const uint32_t* payload, size_t n, unsigned digit_bits,
                                  uint32_t* keys_out, uint32_t* payload_out);

/* ---- L1 suffix array ---------------------------------------------------------- */

/* Per-build statistics (all optional output). */
typedef struct reseq_sa_stats {
    uint32_t alphabet;      /* 0 = 2-bit DNA path (bytes in {0,A,C,G,T}), 1 = generic bytes */
    uint32_t init_symbols;  /* symbols ranked by the initial k-mer sort */
    uint32_t rounds;        /* prefix-doubling rounds executed */
    uint32_t sort_passes;   /* radix digit passes executed in total */
    uint64_t kernel_launches;
    uint64_t refined_tile;  /* elements re-sorted by the shared-memory group-refine kernel */
    uint64_t refined_global;/* elements re-sorted by the global radix fallback */
} reseq_sa_stats;

/* Replaces build_parallel, suffix_array.hpp:61-124 (and therefore build_naive,
 * :45-54, whose result it equals): sa = suffix positions in the total order of
 * suffix_less (:28-41), rank = inverse permutation.  n == 0 is valid.
 * n > RESEQ_CUDA_MAX_TEXT returns RESEQ_TEXT_TOO_LARGE.  `rank` may be NULL. */
int reseq_cuda_build_sa(reseq_cuda_ctx* ctx, const uint8_t* text, size_t n, uint32_t* sa,
                        uint32_t* rank, reseq_sa_stats* stats /* nullable */);
int reseq_cuda_build_sa_device(reseq_cuda_ctx* ctx, const uint8_t* d_text, size_t n,
                               uint32_t* d_sa, uint32_t* d_rank,
                               reseq_sa_stats* stats /* nullable, filled after sync */);

/* ---- multi-GPU building blocks (one process per GPU; see paper_1404_3456_b200/sharded.py) ----
 * A sample-sort partitioned build of the same suffix array: the text is replicated on every
 * rank, each rank makes the 64-bit records of a slice of positions (shard_records:
 * key24 << 40 | terminator byte << 32 | position, key24 = the first 12 bases), the records are
 * exchanged by splitter range on the key's top 16 bits (NCCL all-to-all, done by the caller), and
 * each rank finishes its bucket (shard_finish).  The concatenation of the buckets in splitter order is the array
 * reseq_cuda_build_sa returns.  Only the 2-bit DNA path shards (a text with other bytes is
 * built replicated).  shard_finish reports `unfinished` > 0 when a group exceeded the refine
 * kernel's window; the caller then falls back to the replicated single-device build. */
typedef struct reseq_cuda_sa_shard reseq_cuda_sa_shard;
int reseq_cuda_sa_shard_create(reseq_cuda_ctx* ctx, const uint8_t* d_text, size_t n,
                               reseq_cuda_sa_shard** out, int* is_dna /* nullable */);
void reseq_cuda_sa_shard_destroy(reseq_cuda_sa_shard* shard);
/* d_records[i] = record of suffix pos_begin + i, i < count. */
int reseq_cuda_sa_shard_records(reseq_cuda_sa_shard* shard, uint64_t pos_begin, size_t count,
                                uint64_t* d_records);
/* Sorts (stable, by key24; the input array is clobbered) and refines a bucket of m records
 * that arrive in ascending position order within equal keys; d_sa_out receives the m suffix
 * positions in suffix order. */
int reseq_cuda_sa_shard_finish(reseq_cuda_sa_shard* shard, uint64_t* d_records, size_t m,
                               uint32_t* d_sa_out, uint64_t* unfinished);
/* The same for a uniform read set (k reads of one length, see reseq_cuda_build_sa): shard_create
 * detects it; *period = read length + 1 (0: not uniform -- use shard_records / shard_finish).
 *   uniform_records    records key32 << 32 | position of the suffixes of reads [read_begin,
 *                      read_begin + read_count), transposed: d_records[t * read_count + r] is the
 *                      suffix of read read_begin + r with t symbols before its sentinel.
 *   (the caller partitions by splitter range, exchanges, and brings the bucket into (t, position)
 *    order: a stable sort of the received slices on t = period - 1 - position mod period)
 *   uniform_sort_link  sorts the bucket (4 digit passes; the array is clobbered) and proves, per whole
 *                      read found in it, its predecessor's suffixes to be prefixes: d_cov[read] = t
 *                      (one byte per read of the WHOLE set, zeroed by the caller; combine the ranks'
 *                      tables with an all-reduce MAX before finishing).
 *   uniform_finish     accepts / refines the bucket under the combined table: d_sa_out = its m suffix
 *                      positions in suffix order.  Must follow uniform_sort_link on the same shard. */
int reseq_cuda_sa_shard_uniform_info(const reseq_cuda_sa_shard* shard, uint32_t* period, uint64_t* reads);
int reseq_cuda_sa_shard_uniform_records(reseq_cuda_sa_shard* shard, uint64_t read_begin, size_t read_count,
                                        uint64_t* d_records);
int reseq_cuda_sa_shard_uniform_sort_link(reseq_cuda_sa_shard* shard, uint64_t* d_records, size_t m,
                                          uint8_t* d_cov);
int reseq_cuda_sa_shard_uniform_finish(reseq_cuda_sa_shard* shard, const uint8_t* d_cov, uint32_t* d_sa_out,
                                       uint64_t* unfinished);
/* Bucket-local record generation (no record travels: the text is replicated).
 *   prefix_hist     d_hist[4096] (device, u32) = histogram of the 12-bit key prefix (6 bases, zero padded
 *                   from the terminator on) over the suffixes of `unit_count` units from `unit_begin`:
 *                   reads for a uniform read set, positions otherwise.  The ranks' histograms are summed
 *                   (all-reduce) and the G - 1 splitters read off the cumulative counts.
 *   bucket_size     *m = number of suffixes of the WHOLE text whose prefix lies in [prefix_lo, prefix_hi)
 *                   (a count sweep over all suffix keys + one scan, kept on the shard)
 *   bucket_records  writes those m records (same layouts as uniform_records / shard_records) in the
 *                   order the stable digit passes start from: (terminator distance, position) for a
 *                   uniform read set, position otherwise.  Must follow bucket_size on the same shard. */
int reseq_cuda_sa_shard_prefix_hist(reseq_cuda_sa_shard* shard, uint64_t unit_begin, size_t unit_count,
                                    uint32_t* d_hist);
int reseq_cuda_sa_shard_bucket_size(reseq_cuda_sa_shard* shard, uint32_t prefix_lo, uint32_t prefix_hi, uint64_t* m);
int reseq_cuda_sa_shard_bucket_records(reseq_cuda_sa_shard* shard, uint64_t* d_records);
/* rank sharded by POSITION (suffix_array.hpp:118-122 without replicating the inverse): rank g owns the
 * positions [floor(n g / G), floor(n (g+1) / G)).
 *   rank_shard_partition  for a bucket of the suffix array (positions d_sa_bucket[0..m), global indices
 *                         global_offset + i): d_records_out (m entries) = records
 *                         (position - owner's base) << 32 | global index, grouped by owner;
 *                         counts_out[g] (host, `world` entries) = records for owner g.  These go through
 *                         ONE all-to-all.
 *   rank_shard_finish     on the owner: `len` received records (a permutation of its slice; clobbered)
 *                         -> d_rank_slice[p - base] = global index. */
int reseq_cuda_rank_shard_partition(reseq_cuda_ctx* ctx, const uint32_t* d_sa_bucket, size_t m, uint64_t global_offset,
                                    uint64_t n, int world, uint64_t* d_records_out, uint64_t* counts_out);
int reseq_cuda_rank_shard_finish(reseq_cuda_ctx* ctx, uint64_t* d_records, size_t len, uint32_t* d_rank_slice);
/* d_rank[d_sa[i]] = i (suffix_array.hpp:118-122). */
int reseq_cuda_inverse_device(reseq_cuda_ctx* ctx, const uint32_t* d_sa, size_t n, uint32_t* d_rank);

/* FNV-1a-64 over the little-endian bytes of a device u32 array == bench::checksum_u32,
 * bench.hpp:31-48 (host-side fold of per-block partials is exact: FNV is sequential, so
 * this copies the array back in chunks and folds on the host; a parity fingerprint, not
 * a timed operator). */
int reseq_cuda_checksum_u32_device(reseq_cuda_ctx* ctx, const uint32_t* d_v, size_t n,
                                   uint64_t* out);

/* ---- L2 fragment index -------------------------------------------------------- */

/* Replaces fragment_index::fragment_index(set, builder::scan_radix, exec),
 * fragment_index.hpp:34-56.  `concat` is fragment_set::concat() (f0 \0 f1 \0 ...,
 * sequence.hpp:60-92), `starts` fragment_set::starts().  The index owns device copies
 * of the text (raw + 2-bit packed when DNA), SA, rank, start_rank_list and a k-mer
 * directory over the SA.  Host inputs need not outlive the call. */
int reseq_cuda_index_create(reseq_cuda_ctx* ctx, const uint8_t* concat, size_t n,
                            const uint32_t* starts, size_t k, reseq_cuda_index** out);
void reseq_cuda_index_destroy(reseq_cuda_index* ix);
size_t reseq_cuda_index_text_len(const reseq_cuda_index* ix);
size_t reseq_cuda_index_fragments(const reseq_cuda_index* ix);
/* Copies of fragment_index::sa().sa / .rank / start_rank_list() (fragment_index.hpp:59-61);
 * any pointer may be NULL. */
int reseq_cuda_index_get(const reseq_cuda_index* ix, uint32_t* sa, uint32_t* rank,
                         uint32_t* start_rank_list);
/* start_fragments[t] = frag_at_start_[sa[start_rank_list[t]]] (fragment_index.hpp:44,98): the id of
 * the fragment whose start suffix has the t-th smallest rank; k entries. */
int reseq_cuda_index_start_fragments(const reseq_cuda_index* ix, uint32_t* start_fragments);
/* Device pointers to the same arrays (valid until destroy). */
int reseq_cuda_index_device_ptrs(const reseq_cuda_index* ix, const uint32_t** d_sa,
                                 const uint32_t** d_rank, const uint32_t** d_start_rank_list);

/* Replaces q calls of fragment_index::locate_prefix_range, fragment_index.hpp:65-70 (the
 * binary searches of narrow(), :114-148).  Pattern i is pats[pat_off[i] .. pat_off[i+1]);
 * patterns must be non-empty and free of byte 0.  lo[i], hi[i] receive the half-open SA
 * interval; an absent pattern yields lo == hi at the lower-bound insertion point. */
int reseq_cuda_index_locate_batch(reseq_cuda_index* ix, const uint8_t* pats,
                                  const uint64_t* pat_off, size_t q, uint32_t* lo, uint32_t* hi);

/* Same query where every pattern is a suffix of a fragment already in the text:
 * pattern i = fragment frag[i] from offset off[i] to its end (a `residual`,
 * sequence.hpp:96-101).  Nothing but (frag, off) crosses PCIe. */
int reseq_cuda_index_locate_residuals(reseq_cuda_index* ix, const uint32_t* frag,
                                      const uint32_t* off, size_t q, uint32_t* lo, uint32_t* hi);

/* Replaces q calls of fragment_index::prefix_related, fragment_index.hpp:72-109, for
 * patterns given as residuals (the assembler's use, assembler.hpp:74-78,117).  Results are
 * CSR: list i of each kind occupies [*_off[i], *_off[i+1]) of the malloc'ed id arrays
 * (each list ascending by id, fragment_index.hpp:105-107).  Free with
 * reseq_cuda_prefix_relations_free(). */
typedef struct reseq_prefix_relations {
    size_t q;
    uint64_t *prefixes_off, *extensions_off, *exact_off; /* q+1 each */
    uint32_t *prefixes, *extensions, *exact;
} reseq_prefix_relations;
int reseq_cuda_index_prefix_related_batch(reseq_cuda_index* ix, const uint32_t* frag,
                                          const uint32_t* off, size_t q,
                                          reseq_prefix_relations* out);
void reseq_cuda_prefix_relations_free(reseq_prefix_relations* r);

/* The sparse overlap graph: every (i, j, w) with i != j and
 * w = overlap_weight(f_i, f_j) >= min_overlap (overlap.hpp:16-23, :35-45 restricted to
 * non-zero entries), sorted by (i, j).  One query per (fragment, offset) pair with
 * remaining length >= min_overlap.  Also reports, per fragment, whether
 * detail::absorb_contained (overlap.hpp:51-67) would drop it.  Arrays are malloc'ed;
 * free with reseq_cuda_overlaps_free(). */
typedef struct reseq_overlaps {
    uint64_t count;       /* number of (i, j, w) triples */
    uint32_t *i, *j, *w;  /* count entries each, sorted by (i, j) */
    uint8_t* contained;   /* k flags */
    uint64_t queries;     /* number of locate-equivalent queries executed */
    double device_ms;     /* device time of the query + enumeration kernels */
} reseq_overlaps;
int reseq_cuda_index_overlaps(reseq_cuda_index* ix, uint32_t min_overlap, reseq_overlaps* out);
/* The same restricted to queries of fragments [frag_begin, frag_end) (still against all
 * fragments): the unit of sharding across GPUs -- concatenating the per-range results in
 * fragment order gives reseq_cuda_index_overlaps; `contained` is filled for the range only. */
int reseq_cuda_index_overlaps_range(reseq_cuda_index* ix, uint32_t min_overlap, size_t frag_begin,
                                    size_t frag_end, reseq_overlaps* out);
void reseq_cuda_overlaps_free(reseq_overlaps* o);
/* The same into arrays the caller owns (i, j, w: `capacity` entries each; contained: k bytes) --
 * page-locked arrays receive the result at PCIe speed with no intermediate copy.  `out` is filled as
 * above with its pointers set to the caller's arrays (do not pass it to reseq_cuda_overlaps_free).
 * If more than `capacity` triples exist nothing is copied, out->count holds the number needed and
 * the call returns RESEQ_BUFFER_TOO_SMALL. */
int reseq_cuda_index_overlaps_into(reseq_cuda_index* ix, uint32_t min_overlap, size_t frag_begin, size_t frag_end,
                                   uint32_t* i, uint32_t* j, uint32_t* w, size_t capacity, uint8_t* contained,
                                   reseq_overlaps* out);

/* ---- L3 host merge (stays on the host by design) -------------------------------- */

/* Replaces greedy_superstring_with_order, overlap.hpp:80-113, at scale: consumes the
 * sparse overlap list (>= min_overlap) and the containment flags from
 * reseq_cuda_index_overlaps, finishes sub-threshold overlaps among the surviving contigs
 * exactly, and returns the same superstring and id order the reference's O(k^3) loop
 * produces.  `superstring` must hold sum(lens) bytes, `order` k entries.  Pure host code;
 * needs no device. */
int reseq_greedy_superstring(const uint8_t* concat, size_t n, const uint32_t* starts, size_t k,
                             const reseq_overlaps* ov, uint32_t min_overlap,
                             uint8_t* superstring, size_t* superstring_len, uint32_t* order,
                             size_t* order_len);

/* ---- synthetic workloads (bench.hpp:54-72, shotgun.hpp:20-27) - */

/* genome = "ACGT"[mt19937_64(genome_seed)() & 3] per base. */
void reseq_synth_random_dna(size_t n, uint64_t seed, uint8_t* out);
/* keys[i] = (uint32_t) mt19937_64(seed)(), payload[i] = i. */
void reseq_synth_random_keys(size_t n, uint64_t seed, uint32_t* keys, uint32_t* payload);
/* k reads of length L drawn forward-strand, error-free, start = bounded rejection draw
 * from mt19937_64(read_seed); out receives k*(L+1) bytes: read, 0, read, 0, ...;
 * starts (nullable) receives the k fragment offsets. */
int reseq_synth_read_text(size_t genome_len, size_t read_len, size_t k, uint64_t genome_seed,
                          uint64_t read_seed, uint8_t* out, uint32_t* starts);

#ifdef __cplusplus
}
#endif
#endif /* RESEQ_CUDA_H */
