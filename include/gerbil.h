/*
 * gerbil.h — C ABI of the B200-native Gerbil counting phase.
 *
 * What the library computes (Abstract): the histogram of all
 * length-k substrings of a set of reads, counting each k-mer under its
 * canonical representation min(x, rc(x)) (§2.4.2), ignoring
 * every k-mer that contains an undetermined base (§2.4.1),
 * and reporting the (k-mer, count) pairs whose count reaches a threshold
 * (App. A `-l`).
 *
 * How (§2): reads are cut into minimizer super-mers
 * (§2.1) and every super-mer is assigned to a bin, so that all
 * occurrences of a k-mer fall in one bin; bins are shuffled to
 * their owner GPU (NCCL all-to-all, world > 1) and counted independently in a
 * bucketised open-addressing hash table (PAPER.md:63-84, Alg. 1; :171-178,
 * §3.3.1) with an exact emergency path for k-mers that exhaust θ probes
 * (§3.4.3). Steps (a)-(e) of SURVEY.md §8(a).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - 2-bit base code: A=0, C=1, G=2, T=3 (App. C).
 *  - Packed base stream: base i of a batch lives in 64-bit word i/32, bits
 *    [63-2(i%32) : 62-2(i%32)] (first base in the most significant bits,
 *    PAPER.md:517-518).
 *  - N-mask: bit (63 - i%64) of word i/64 is 1 iff base i is undetermined
 *    (any byte outside {A,C,G,T,a,c,g,t} in the text).
 *  - read_start[0..n_reads]: base offset of read r is read_start[r]; its
 *    length is read_start[r+1]-read_start[r]; read_start[0] == 0. k-mers never
 *    span two reads.
 *  - Result key layout: W = ceil(k/32) u64 words per k-mer; word 0 holds bases
 *    0..31 with base 0 in bits 63:62; the last word is left-aligned and
 *    zero-padded. A big-endian dump of the words truncated to ceil(k/4) bytes
 *    is exactly the appendix k-mer byte encoding, and the
 *    numeric order of the word arrays equals A<C<G<T string order.
 *
 * Ownership: the caller owns every input buffer; inputs are read-only during
 * the call and never retained. The library owns its device memory, streams
 * and results until the next gerbil_count* call or gerbil_finalize.
 * gerbil_fetch copies into caller-allocated buffers. Calls on one context
 * must be serialised by the caller. No C++ exception crosses this ABI.
 *
 * Errors: every call returns a gerbil_status. GERBIL_E_USAGE for invalid
 * arguments (nothing is changed); GERBIL_E_IO for unreadable/malformed input
 * (message with file and line via gerbil_last_error); GERBIL_E_INTERNAL when
 * the Σcount == #valid-windows invariant fails; GERBIL_E_CUDA /
 * GERBIL_E_NCCL poison the context (only gerbil_finalize is then valid);
 * GERBIL_E_STATE for gerbil_fetch before a successful count.
 */
#ifndef GERBIL_H
#define GERBIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GERBIL_ABI_VERSION 1

typedef struct gerbil_ctx gerbil_ctx;

typedef enum {
  GERBIL_OK = 0,
  GERBIL_E_USAGE = 1,
  GERBIL_E_IO = 2,
  GERBIL_E_INTERNAL = 3,
  GERBIL_E_NOMEM = 4,
  GERBIL_E_CUDA = 5,
  GERBIL_E_NCCL = 6,
  GERBIL_E_STATE = 7
} gerbil_status;

/* Minimizer orderings (§3.1).
 * KMC2 is Gerbil's choice; LEX (A<C<G<T) is the ordering of
 * Fig. 1; CGAT (C<G<A<T), ROBERTS (even positions
 * complemented, then C<A<T<G), RANDOM (a fixed bijection of the m-mers) and
 * DFP (distance from pivot dfp_pivot in the sampled frequency order; m <= 12)
 * are the alternatives the paper evaluates. Results never depend on the
 * ordering; super-mers, bins and the Fig. Minimizer metrics do. */
typedef enum {
  GERBIL_ORDER_KMC2 = 0, GERBIL_ORDER_LEX = 1, GERBIL_ORDER_CGAT = 2,
  GERBIL_ORDER_ROBERTS = 3, GERBIL_ORDER_RANDOM = 4, GERBIL_ORDER_DFP = 5
} gerbil_ordering;

typedef struct {
  uint32_t struct_size;    /* sizeof(gerbil_config); ABI versioning */
  int32_t device;          /* CUDA device ordinal of this rank; -1 = current */
  int32_t rank, world;     /* multi-process mode, one GPU per rank; 0/1 = single */
  const void* nccl_unique_id; /* 128-byte ncclUniqueId when world > 1, else NULL */
  int32_t comm_backend;    /* 0 = NCCL (one process per GPU); 1 = loopback: `world`
                              contexts in ONE process on one GPU, driven from `world`
                              host threads, exchanging by device copies (test seam;
                              nccl_unique_id = any 128-byte group key) */
  uint32_t n_bins;         /* B (temporary-file analogue, PAPER.md:459 `-f`); 0 = auto (>= 512) */
  int32_t ordering;        /* gerbil_ordering; 0 = KMC2 */
  uint64_t device_mem_cap; /* out-of-core budget (`-e`): gerbil_spill_finish counts bin
                             groups of at most device_mem_cap / 2 bytes of super-mers; 0 = 16 GiB groups.
                             The in-core calls size their buffers from the input and do not read it. */
  int32_t host_threads;    /* host reader threads; 0 = all cores (`-t`) */
  uint32_t max_probes;     /* θ in buckets; 0 = 32; capped at 2^20 */
  double distinct_ratio;   /* initial ρ̂ = distinct/total estimate; 0 = 0.5 */
  double target_load;      /* α: table load factor target; 0 = 0.7 */
  uint64_t wave_table_bytes; /* per-wave table budget (kept L2-resident); 0 = 128 MiB */
  void* stream;            /* cudaStream_t to launch on; NULL = library-owned stream */
  int32_t timing;          /* 1 = record per-kernel CUDA-event times into gerbil_stats */
  int32_t force_exchange;  /* 1 = run the multi-rank shuffle even when world == 1 (test
                              seam: exercises the NCCL all-gather / send / recv path on one
                              GPU; a 1-rank communicator is created internally) */
  int32_t disable_normalization; /* 1 = `-d`: count each k-mer as it occurs;
                                    x and rc(x) are different k-mers. 0 = canonical (default) */
  double dfp_pivot;        /* DFP ordering: pivot p in [0, 1] */
  uint32_t order_sample_stride; /* DFP ordering: sample every stride-th 1024-base tile; 0 = 16 */
  int32_t count_mode;      /* step (d) table placement ("Kernel (d)"):
                              0 = auto: a bin predicted (ρ̂ · windows) to fit an on-chip table
                                  is counted there — one warp's shared-memory table of whole
                                  keys (k <= 96), or a CTA's table of occurrence references
                                  (k > 96; and the second tier of mostly distinct data); bins
                                  too large go to hash-class passes (k > 96) or L2-resident
                                  wave tables; n_bins = 0 then picks enough bins (up to 2^22)
                                  when m >= 11 makes bins that small;
                              1 = L2 wave tables only;
                              2 = try the on-chip tables for every bin (test seam: bins that
                                  overflow them are recounted in the wave tables).
                              Results never depend on it; the streaming call uses the same
                              placement. */
} gerbil_config;

/* Result encodings (App. C). */
typedef enum {
  GERBIL_FMT_BINARY = 0, /* per k-mer: count < 255 → 1 byte; else 0xFF + 4-byte big-endian
                            count; then ceil(k/4) bytes, 4 bases per byte A=00 C=01 G=10 T=11,
                            first base in the most significant bits, pad bits 0 */
  GERBIL_FMT_CSV = 1     /* `-x h` human readable: one "KMER,COUNT\n" line per k-mer */
} gerbil_format;

/* Exactly one source must be set. */
typedef struct {
  const char* const* paths; uint32_t n_paths; /* FASTA/FASTQ files (App. B) */
  const char* text; uint64_t text_len;        /* one in-memory FASTA or FASTQ document */
} gerbil_reads;

typedef struct {
  /* sizes (whole job = all ranks, except where noted "local") */
  uint64_t input_bases;      /* local: all input bases incl. undetermined ones */
  uint64_t input_reads;      /* local */
  uint64_t valid_windows;    /* local: n_k, k-mer windows with no undetermined base */
  uint64_t supermers;        /* local: super-mers produced by step (b) */
  uint64_t owned_windows;    /* windows counted on this rank after the shuffle */
  uint64_t distinct;         /* distinct canonical k-mers counted on this rank */
  uint64_t kept;             /* of which count >= min_count (returned by fetch) */
  uint64_t count_sum;        /* Σ counts over all table slots + overflow (== owned_windows) */
  uint64_t overflow_kmers;   /* k-mer occurrences that exhausted θ probes (emergency path) */
  uint64_t probe_first;      /* inserts resolved in the first bucket */
  uint64_t probe_more;       /* inserts that needed more than one bucket */
  uint64_t probe_max;        /* most buckets probed by one insert */
  uint32_t overflow_passes;  /* extra counting passes spent on the emergency path */
  uint32_t waves;            /* table waves run by step (d) */
  uint32_t n_bins;
  uint32_t W;                /* key words per k-mer */
  uint64_t max_bin_windows;  /* largest bin (global), for skew reporting */
  uint64_t bytes_sent, bytes_recv; /* step (c) NVLink traffic of this rank */
  double ratio_used;         /* ρ̂ used to size this call's tables */
  double ratio_observed;     /* max over waves of distinct / windows */
  /* per-stage device milliseconds (timing=1). Steps (d)+(e) run in two
     overlapping wave lanes by default: ms_count is then the span of both
     steps and ms_compact is 0 (GERBIL_WAVE_LANES=1: separate, serial). */
  double ms_h2d, ms_supermer, ms_shuffle, ms_count, ms_compact, ms_overflow, ms_total;
  /* host reader (step a) wall milliseconds */
  double ms_reader;
  uint32_t launches_count, launches_compact, launches_total;
  /* step (d) in shared memory (count_mode != 1) */
  uint64_t smem_bins;        /* bins counted in on-chip (shared-memory) tables, all tiers */
  uint64_t smem_failed;      /* of which abandoned (too many distinct k-mers) by a tier and passed on */
  uint64_t smem_windows;     /* windows of the bins that completed in shared memory */
  uint32_t smem_slots;       /* first-tier table slots (per warp, or per CTA for reference tables) */
  uint32_t launches_smem;    /* shared-memory count launches (included in launches_count) */
  double ms_smem;            /* their device time (included in ms_count) */
} gerbil_stats;

/* Fills cfg with defaults (struct_size set, everything else "auto"). */
void gerbil_config_default(gerbil_config* cfg);

/* Creates a context on cfg->device. world > 1 requires nccl_unique_id (from
 * gerbil_nccl_unique_id on rank 0, broadcast by the caller). */
gerbil_status gerbil_init(const gerbil_config* cfg, gerbil_ctx** out);

/* Writes a fresh ncclUniqueId (128 bytes) into id_out. */
gerbil_status gerbil_nccl_unique_id(void* id_out, size_t id_len);

/* Full path (a)→(e): host reader parses FASTA/FASTQ (PAPER.md:94-95,
 * §2.3.1 steps 1-2), packs 2 bits/base, copies to the device, then counts.
 * Validation: 8 <= k <= 200 (PAPER.md:447 allows 8..479; this build stops at
 * 200), 1 <= m <= min(k-1, 15) or m == 0 (auto = 7),
 * min_count >= 1, exactly one read source. */
gerbil_status gerbil_count(gerbil_ctx* ctx, const gerbil_reads* reads,
                           uint32_t k, uint32_t m, uint32_t min_count);

/* Steps (b)→(e) on a packed batch already resident on this rank's device
 * (layout above; nmask may be NULL when no base is undetermined). The
 * headline timed region. n_reads may be 0. */
gerbil_status gerbil_count_device(gerbil_ctx* ctx, const uint64_t* d_codes,
                                  const uint64_t* d_nmask,
                                  const uint64_t* d_read_start, uint64_t n_reads,
                                  uint32_t k, uint32_t m, uint32_t min_count);

/* Same as gerbil_count_device but from HOST buffers (the H2D copy is part of
 * the call). Host buffers should be pinned for full PCIe bandwidth. */
gerbil_status gerbil_count_host_packed(gerbil_ctx* ctx, const uint64_t* codes,
                                       const uint64_t* nmask,
                                       const uint64_t* read_start, uint64_t n_reads,
                                       uint32_t k, uint32_t m, uint32_t min_count);

/* Streaming end-to-end call (steps b→e from HOST buffers to HOST records):
 * gerbil_count_host_packed, and in the same pass the compaction kernel encodes
 * every k-mer with count >= min_count as the paper's binary record (App. C,
 * PAPER.md:512-521; GERBIL_FORMAT_BINARY: 1-byte counter, or 0xFF + 32-bit
 * big-endian counter when >= 255, then ceil(k/4) bytes, 4 bases per byte MSB
 * first, zero-padded) and writes it straight into out[0, capacity) over PCIe
 * while later waves are still being counted — the download overlaps step (d).
 * Record order is unspecified. out must be page-locked host memory
 * (cudaHostAlloc / cudaHostRegister) — GERBIL_E_USAGE otherwise — and is
 * owned by the caller. *n_bytes = size of the complete encoding. If capacity
 * is too small (capacity = 0 and out = NULL is a sizing call), out's contents
 * are unspecified, *n_bytes holds the size needed and GERBIL_E_USAGE is
 * returned; the (k-mer, count) results stay on the device either way
 * (gerbil_fetch / gerbil_encode_results work as after gerbil_count_device). */
gerbil_status gerbil_count_host_stream(gerbil_ctx* ctx, const uint64_t* codes,
                                       const uint64_t* nmask,
                                       const uint64_t* read_start, uint64_t n_reads,
                                       uint32_t k, uint32_t m, uint32_t min_count,
                                       uint8_t* out, uint64_t capacity, uint64_t* n_bytes);

/* Host reader alone (step a): parse FASTA/FASTQ and pack. Two-call pattern:
 * with codes == NULL, returns the sizes (n_bases, n_reads) only. Buffers:
 * codes[ceil(n_bases/32)], nmask[ceil(n_bases/64)], read_start[n_reads+1]. */
gerbil_status gerbil_pack_reads(const gerbil_reads* reads, int32_t threads,
                                uint64_t* codes, uint64_t* nmask,
                                uint64_t* read_start, uint64_t* n_bases,
                                uint64_t* n_reads, char* err, size_t err_len);

/* Copies this rank's results (count >= min_count) into kmers[n*W] and
 * counts[n]. kmers == NULL → only *n_out is written (two-call pattern).
 * capacity is in entries. sorted != 0 → ascending key order (A<C<G<T).
 * Fails with GERBIL_E_USAGE if capacity < n. */
gerbil_status gerbil_fetch(gerbil_ctx* ctx, uint64_t* kmers, uint32_t* counts,
                           uint64_t capacity, uint64_t* n_out, int sorted);

/* Encodes this rank's results (count >= min_count) in `format` (gerbil_format)
 * into out[capacity] bytes; out == NULL → only *n_bytes is written (two-call
 * pattern). sorted != 0 → ascending k-mer order (the CSV of PAPER.md:521 is
 * for small data sets; SPEC.md:475 sorts it). GERBIL_E_USAGE if capacity is
 * too small, GERBIL_E_STATE before a successful count. */
gerbil_status gerbil_encode_results(gerbil_ctx* ctx, int32_t format, int sorted, uint8_t* out,
                                    uint64_t capacity, uint64_t* n_bytes);

/* Same, written to a file (GERBIL_E_IO if it cannot be written). */
gerbil_status gerbil_write_results(gerbil_ctx* ctx, const char* path, int32_t format, int sorted);

/* Host-only k-way merge of n_lists SORTED result lists — e.g. the sorted fetches of the
 * ranks of one job, whose key sets are disjoint (every bin has one owner) —
 * into one list in ascending key order (SURVEY.md §3.4 "cross-GPU merge").
 * keys[l] holds n[l] * W words, counts[l] n[l] counts (caller-owned, unchanged). Keys present
 * in several lists are merged into one entry with the summed count (merging histograms of
 * independent jobs). out_keys == NULL → only *n_out (the merged entry count) is written;
 * otherwise out_keys[*n_out * W] / out_counts[*n_out] receive the list (capacity = entries).
 * threads <= 0 = all host cores. GERBIL_E_USAGE on bad arguments or a too small capacity. */
gerbil_status gerbil_merge_sorted(uint32_t n_lists, const uint64_t* const* keys, const uint32_t* const* counts,
                                  const uint64_t* n, uint32_t W, int32_t threads, uint64_t* out_keys,
                                  uint32_t* out_counts, uint64_t capacity, uint64_t* n_out);

/* ---- step (a) on the device --------------------
 * "Phase one on the GPU" (the paper's future work): a FASTA /
 * FASTQ / raw document (App. B) is parsed by kernels into the
 * packed batch layout above — identical, bit for bit, to gerbil_pack_reads
 * on the same text (readings Q3/Q4). text is host memory (on_device = 0,
 * copied to the device; page-locked for full PCIe speed) or device memory
 * (on_device = 1, not modified). gerbil_parse_text returns the batch in host
 * arrays sized as for gerbil_pack_reads (NULL arrays: only *n_bases and
 * *n_reads — the sizing call). gerbil_count_text runs steps (a)…(e) on the
 * device (results as after gerbil_count_device). GERBIL_E_IO (message with
 * the line number) for malformed FASTQ, and for FASTQ with empty lines
 * between records, which the device parser does not take (the host reader
 * does). */
gerbil_status gerbil_parse_text(gerbil_ctx* ctx, const char* text, uint64_t len, int32_t on_device,
                                uint64_t* codes, uint64_t* nmask, uint64_t* read_start,
                                uint64_t* n_bases, uint64_t* n_reads);
gerbil_status gerbil_count_text(gerbil_ctx* ctx, const char* text, uint64_t len, int32_t on_device,
                                uint32_t k, uint32_t m, uint32_t min_count);

/* ---- out-of-core counting ---------------------
 * The paper's two-phase design with the temporary
 * files in page-locked host memory, for inputs given in several batches or
 * larger than the device: (1) gerbil_spill_begin fixes k, m and the bins
 * (cfg.n_bins, 0 → 4096); (2) gerbil_spill_add (any number of times) runs
 * step (b) on one HOST packed batch (layout as gerbil_count_device) and moves
 * its super-mers, grouped by bin, to host memory owned by the context;
 * (3) gerbil_spill_finish counts the bins in groups that fit the device
 * budget (cfg.device_mem_cap / 2, 0 → 16 GiB per group) — every group's
 * super-mers from every batch are uploaded, regrouped by bin and counted
 * (steps d, e) — and streams the App. C records of every k-mer with count
 * >= min_count into out (page-locked, as gerbil_count_host_stream; capacity 0
 * = sizing: *n_bytes is the size needed, GERBIL_E_USAGE). A sizing call, or a
 * buffer that is too small, keeps the spilled job: call gerbil_spill_finish
 * again with a buffer of *n_bytes (phase one is not repeated); a successful
 * call or any other error ends the job. The histogram is
 * the same as one gerbil_count over the concatenated batches. No device
 * result set remains (gerbil_fetch → GERBIL_E_STATE); stats describe the whole
 * job. world > 1: each rank spills its own batches and gerbil_spill_finish is
 * collective (every rank calls it): the bins are split into contiguous ranges
 * of about equal global windows, rank d counts range d (its records: the k-mers
 * of those bins, with counts over every rank's batches), the groups move in
 * rounds of one grouped all-to-all each; the job parameters (bins, k, m,
 * ordering, disable_normalization) must agree (else GERBIL_E_USAGE), and the
 * job is kept on every rank unless every rank's records fit (then every rank
 * returns GERBIL_E_USAGE with its own *n_bytes, and all call again).
 * The DFP ordering is refused (its table is per batch); force_exchange is
 * refused. GERBIL_E_STATE when called out of order. */
gerbil_status gerbil_spill_begin(gerbil_ctx* ctx, uint32_t k, uint32_t m);
gerbil_status gerbil_spill_add(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                               const uint64_t* read_start, uint64_t n_reads);
gerbil_status gerbil_spill_finish(gerbil_ctx* ctx, uint32_t min_count, uint8_t* out,
                                  uint64_t capacity, uint64_t* n_bytes);

/* Fig. Minimizer metrics of the last count: the number of
 * distinct k-mers (count >= min_count) per minimizer under the context's
 * ordering — *max_per_minimizer = its maximum, *n_minimizers = minimizers
 * owning at least one k-mer (this rank). The total number of super-mers is
 * gerbil_stats.supermers (step (b) also cuts super-mers at 1024-window tile
 * boundaries). Needs m <= 12; GERBIL_E_STATE before a successful count. */
gerbil_status gerbil_minimizer_stats(gerbil_ctx* ctx, uint64_t* max_per_minimizer,
                                     uint64_t* n_minimizers);

/* Device-side view of this rank's results (valid until the next count). */
gerbil_status gerbil_results_device(gerbil_ctx* ctx, const uint64_t** d_kmers,
                                    const uint32_t** d_counts, uint64_t* n,
                                    uint32_t* W);

/* Step (c) exchange plan (host only, no device needed): what every rank computes,
 * identically, from the all-gathered per-bin histograms before the NCCL
 * all-to-all (PAPER.md:49 — all occurrences of a k-mer go to one temporary
 * file, here one owner rank; the LPT ownership replaces the paper's load
 * balancer).
 *   hist:  [world][3][n_bins] u64, rank-major: windows, super-mers and payload
 *          words of every bin produced by step (b) on that rank (input, not retained).
 *   owner: [n_bins] out — owner rank of each bin: bins sorted by total windows
 *          (heaviest first, ties by bin index) go to the least-loaded rank (ties
 *          by rank index), so every rank derives the same map.
 *   send_desc_off, send_word_off: [world + 1] out — this rank's send buffer
 *          layout: descriptors / payload words for destination d occupy
 *          [off[d], off[d+1]), bins in increasing order inside a destination.
 *   recv_desc_off, recv_word_off: [world + 1] out — receive layout by source.
 * GERBIL_E_USAGE on a NULL pointer, world < 1, rank outside [0, world) or
 * n_bins == 0. */
gerbil_status gerbil_exchange_plan(const uint64_t* hist, uint32_t n_bins, int32_t world, int32_t rank,
                                   int32_t* owner, uint64_t* send_desc_off, uint64_t* send_word_off,
                                   uint64_t* recv_desc_off, uint64_t* recv_word_off);

gerbil_status gerbil_get_stats(const gerbil_ctx* ctx, gerbil_stats* out);
const char* gerbil_last_error(const gerbil_ctx* ctx);
void gerbil_finalize(gerbil_ctx* ctx);

/* ---- debug / test entry points (step b in isolation) ------------------- */
/* Runs step (b) only and copies the super-mers to host: pos[i] = base offset
 * of the first window, nwin[i] = number of windows, bin[i], minimizer key
 * mu[i] (ordering key of the canonical minimizer). Two-call
 * pattern with pos == NULL. Order of super-mers is unspecified. */
gerbil_status gerbil_debug_supermers(gerbil_ctx* ctx, const uint64_t* codes,
                                     const uint64_t* nmask,
                                     const uint64_t* read_start, uint64_t n_reads,
                                     uint32_t k, uint32_t m, uint64_t* pos,
                                     uint32_t* nwin, uint32_t* bin, uint32_t* mu,
                                     uint64_t capacity, uint64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* GERBIL_H */
