// api_internal.h — host orchestration internals shared by the library's translation units
// (api.cu: context life cycle + entry points; pipeline.cu: steps (b)-(e) of one call;
// waves.cu: bin plans, shared-memory / reference / L2 wave passes, the group exchange;
// io.cu: host batches, device parsing; spill.cu: out-of-core jobs; results.cu: fetch,
// sort, encodings). Not part of the public boundary (include/gerbil.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gerbil.h"
#include "comm.h"
#include "common.cuh"
#include "kernels.h"
#include "output.h"
#include "reader.h"
#include "table.cuh"
#include "table_inline.cuh"

using namespace gerbil;


namespace gerbil_api {
using namespace gerbil;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    release();
    size_t want = std::max<size_t>(n + n / 8, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      want = std::max<size_t>(n, 256);
      e = cudaMalloc(&p, want);
    }
    if (e == cudaSuccess) bytes = want;
    else p = nullptr;
    return e;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Device-side counters, zeroed per pass, read back once.
struct Counters {
  unsigned long long n_supermers, n_windows, ovf_n, out_n, sum_counts, distinct;
  unsigned long long probe[4];
  unsigned long long read_work;  // dynamic read counter of supermer_reads_kernel
};

// Step-(b) kernel choice: the tile kernel (supermer.cu) by default — on B200 it
// beat the read-per-lane kernel (supermer_reads.cu: 49 vs 40 ms on C1, smem
// rings cap it at 10 warps/SM); GERBIL_SUPERMER_KERNEL=reads selects the latter
// where it applies (tests run both).
inline bool use_reads_kernel(uint32_t k, uint32_t m, uint64_t n_bases, uint64_t n_reads) {
  const char* e = getenv("GERBIL_SUPERMER_KERNEL");
  if (e && strcmp(e, "reads") == 0) return n_reads > 0 && k - m + 1 <= 64;
  (void)n_bases;
  return false;
}

enum Kind { K_SUPERMER, K_SHUFFLE, K_COUNT, K_COMPACT, K_OVERFLOW, K_H2D, K_SMEM, K_NKIND };

struct TimedEvent {
  int kind;
  cudaEvent_t a, b;
};

// A host batch uploaded in chunks (gerbil_count_host_packed): after ev[c],
// bases [0, base_end[c]) and read_start[0, read_end[c]] are resident.
struct UploadPlan {
  uint64_t n_bases = 0;
  std::vector<uint64_t> base_end, read_end;
  std::vector<cudaEvent_t> ev;
};

// Out-of-core state (gerbil_spill_*): phase one leaves every batch's
// super-mers grouped by bin in page-locked host memory (the paper's temporary
// files, PAPER.md:47-49 / :97), phase two counts them bin group by bin group.
struct SpillBatch {
  uint64_t* desc = nullptr;     // [n_sm] pos (relative to payload) << 11 | nwin-1, bin order
  uint32_t* bin = nullptr;      // [n_sm]
  uint64_t* payload = nullptr;  // [n_words] word-aligned packed super-mers
  uint64_t n_sm = 0, n_words = 0;
  std::vector<uint64_t> d_off, w_off;  // [B+1] per-bin offsets into desc / payload
};
// Page-locked blocks reused across spill jobs: pinning host memory costs far
// more than the PCIe copies themselves (~2 GB/s), so blocks go back to the
// pool instead of being freed.
struct PinnedPool {
  std::vector<std::pair<void*, size_t>> free_blocks;
  void* get(size_t n) {
    size_t best = SIZE_MAX, bi = 0;
    for (size_t i = 0; i < free_blocks.size(); ++i)
      if (free_blocks[i].second >= n && free_blocks[i].second < best) best = free_blocks[i].second, bi = i;
    if (best != SIZE_MAX) {
      void* p = free_blocks[bi].first;
      free_blocks.erase(free_blocks.begin() + bi);
      sizes.push_back({p, best});
      return p;
    }
    void* p = nullptr;
    const size_t want = n + n / 8 + 4096;  // room for a slightly larger batch next time
    if (cudaHostAlloc(&p, want, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    sizes.push_back({p, want});
    return p;
  }
  void put(void* p) {
    if (!p) return;
    for (size_t i = 0; i < sizes.size(); ++i)
      if (sizes[i].first == p) {
        free_blocks.push_back(sizes[i]);
        sizes.erase(sizes.begin() + i);
        return;
      }
  }
  void clear() {
    for (auto& b : free_blocks) cudaFreeHost(b.first);
    for (auto& b : sizes) cudaFreeHost(b.first);
    free_blocks.clear();
    sizes.clear();
  }
  std::vector<std::pair<void*, size_t>> sizes;  // blocks in use
};

struct SpillState {
  bool active = false;
  uint32_t k = 0, m = 0, B = 0;
  std::vector<SpillBatch> batches;
  std::vector<uint64_t> win, cnt, words;  // [B] totals over batches
  uint64_t bases = 0, reads = 0, windows = 0, supermers = 0;
  PinnedPool pool;
  void release() {  // blocks return to the pool
    for (auto& b : batches) {
      pool.put(b.desc);
      pool.put(b.bin);
      pool.put(b.payload);
    }
    batches.clear();
    active = false;
  }
};

// Page-locked host staging buffer (grown on demand): per-bin tables of 10^6 bins move
// at PCIe speed instead of through pageable bounce buffers.
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    const size_t want = std::max<size_t>(n + n / 8, 4096);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct Wave {
  uint64_t d0, d1;   // descriptor range (bin-ordered)
  uint64_t windows;
  uint64_t nb;       // buckets
};

}  // namespace gerbil_api

using namespace gerbil_api;

struct gerbil_ctx {
  gerbil_config cfg;
  int device = 0, sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t lane_stream = nullptr;             // second wave lane (steps d+e)
  cudaStream_t pcie_stream = nullptr;             // record copies to the host (streaming call)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  std::vector<cudaEvent_t> wave_ev;               // "wave w compacted" (streaming call)
  bool poisoned = false;
  std::string err;
  double rho = 0.5;
  bool rho_seen = false;  // rho was measured (an earlier call) or given (cfg.distinct_ratio)
  Comm* comm = nullptr;
  int rank = 0, world = 1;
  // device buffers
  DevBuf in_codes, in_nmask, in_rstart;  // uploads of host batches
  DevBuf desc_pre, bin_pre, mu_dbg, desc_sorted, rs_bits;
  DevBuf counters;
  DevBuf hist;  // [3][B] windows, super-mers, payload words (ull)
  DevBuf hist_all, cursor, cursor2, seg_base;
  DevBuf table, ovf, out_keys, out_counts, wave_distinct;
  DevBuf rec_stage, rec_meta;
  DevBuf rec_stage2, rec_snap_d;  // streaming call, shared-memory pass: record staging, result snapshots
  DevBuf order_rank, order_freq;  // DFP ordering: key table [4^m] and its sample histogram
  DevBuf text_buf, p_cnt, p_off, p_ls, p_cr, p_eff, p_first, p_seq, p_rflag, p_pos, p_ridx, p_tmp, p_misc;  // parser
  uint32_t m = 0;  // streaming call: per-lane record staging; counters/snapshots/offsets
  DevBuf send_desc, send_bin, send_payload, recv_desc, recv_bin, recv_payload;
  DevBuf smem_range, smem_failed, rest_desc, rest_range, rest_off;  // step (d) in shared memory
  int smem_optin = 0;  // max dynamic shared memory per block (bytes)
  size_t mem_total = 0;  // device memory (bytes), read once
  PinnedBuf h_hist, h_rng, h_fail;  // per-bin histogram download, bin list upload, abandoned bins
  DevBuf bin_off_d, plan_sums;  // device-side bin plan (many bins, one rank)
  bool results_sorted = false;   // out_keys already in A<C<G<T order (a sorted fetch ran)
  Counters* h_counters = nullptr;  // pinned
  // results
  bool have_result = false;
  uint64_t n_out = 0;
  uint32_t W = 0, k = 0;
  gerbil_stats stats;
  // timing
  std::vector<TimedEvent> evs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  uint32_t n_launch[K_NKIND] = {0};
  // streaming record sink of the current call (gerbil_count_host_stream)
  uint8_t* rec_out = nullptr;
  uint64_t rec_cap = 0, rec_bytes = 0;
  unsigned long long* h_snap = nullptr;  // pinned: per-wave record byte counters (streaming call)
  size_t h_snap_n = 0;
  const UploadPlan* upload = nullptr;     // chunked upload of the current call, or null
  std::vector<cudaEvent_t> chunk_ev;
  bool want_words = false;   // step (b) also histograms payload words per bin (exchange / spill)
  uint64_t rec_base = 0;     // streamed records already in rec_out (spill groups append)
  SpillState spill;
};

namespace gerbil_api {

inline gerbil_status fail(gerbil_ctx* c, gerbil_status st, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (st == GERBIL_E_CUDA || st == GERBIL_E_NCCL) c->poisoned = true;
  }
  return st;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, GERBIL_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKS(expr)                              \
  do {                                         \
    gerbil_status s_ = (expr);                 \
    if (s_ != GERBIL_OK) return s_;            \
  } while (0)

inline cudaEvent_t get_event(gerbil_ctx* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}

// Counts one launch of `kind`; with timing on and `timed`, a CUDA-event pair
// brackets it on stream `st`. A span timer (launches = 0) brackets a phase.
struct Timer {
  gerbil_ctx* ctx;
  cudaStream_t st;
  cudaEvent_t b = nullptr;
  Timer(gerbil_ctx* c, int kind, cudaStream_t s = nullptr, bool timed = true, uint32_t launches = 1)
      : ctx(c), st(s ? s : c->stream) {
    ctx->n_launch[kind] += launches;
    if (ctx->cfg.timing && timed) {
      cudaEvent_t a = get_event(ctx);
      b = get_event(ctx);
      cudaEventRecord(a, st);
      ctx->evs.push_back({kind, a, b});
    }
  }
  ~Timer() {
    if (b) cudaEventRecord(b, st);
  }
};

// Wave lanes: with 2, consecutive waves alternate between two half-budget
// tables on two streams, so one wave's compaction and launch tail overlap the
// next wave's counting (GERBIL_WAVE_LANES=1 restores the serial schedule).
inline int wave_lanes() {
  const char* e = getenv("GERBIL_WAVE_LANES");
  if (e && *e) return atoi(e) <= 1 ? 1 : 2;
  return 2;
}

inline gerbil_status validate(gerbil_ctx* ctx, uint32_t k, uint32_t& m, uint32_t min_count) {
  if (!ctx) return GERBIL_E_USAGE;
  if (ctx->poisoned) return fail(ctx, GERBIL_E_STATE, "context poisoned by an earlier CUDA/NCCL error");
  if (k < 8 || k > 479) return fail(ctx, GERBIL_E_USAGE, "k must be in [8, 479]");
  if (m == 0) m = std::min<uint32_t>(7, k - 1);
  if (m > 15 || m >= k) return fail(ctx, GERBIL_E_USAGE, "m must be in [1, min(k-1, 15)]");
  if (min_count < 1) return fail(ctx, GERBIL_E_USAGE, "min_count must be >= 1");
  if (ctx->cfg.ordering == GERBIL_ORDER_DFP && m > 12)
    return fail(ctx, GERBIL_E_USAGE, "the DFP ordering needs m <= 12");
  return GERBIL_OK;
}

uint32_t smem_slots_for(gerbil_ctx* ctx, uint32_t k);
// The first counting tier uses the CTA-wide reference tables (count_ref.cu) for long keys
// (W >= 4), per-warp tables of whole keys otherwise (measured: for W <= 3 the reference tables
// as first tier cost 1.5-2x on the C2/C3 shards; they serve as the second tier there).
inline bool ref_tier1(const gerbil_ctx* ctx, uint32_t k) {
  (void)ctx;
  return key_words(k) >= 4;
}
// CTAs per SM of the first reference-table tier: 2 = two bins in flight per SM on half tables
// (a bin's warps wait at its barriers while the other bin's keep the SM busy; bins that do not fit
// go to the full-table second tier), 1 = one bin per SM (GERBIL_REF_CTAS overrides)
int ref_tier1_ctas();
// from this many bins up, a single rank plans steps (c)-(e) on the device
constexpr uint32_t kDevicePlanBins = 1u << 16;
gerbil_status count_local_device_plan(gerbil_ctx* ctx, const uint64_t* codes, uint64_t n_sm, uint32_t B,
                                      uint32_t cap, uint32_t k, uint32_t min_count, uint64_t windows,
                                      uint64_t n_bases);

inline uint32_t choose_bins(gerbil_ctx* ctx, uint64_t n_bases, uint64_t n_reads, uint32_t W, uint32_t k, uint32_t m) {
  if (ctx->cfg.n_bins) return ctx->cfg.n_bins;
  // Shared-memory counting (count_smem.cu for W <= 3, the CTA-wide reference tables of
  // count_ref.cu for W >= 4) wants bins whose distinct k-mers fit one table: ~0.35 of its
  // slots on average leaves room for skew. Bins are hashes of minimizers, so that needs many
  // more minimizers than bins (m >= 11: >= 2M canonical m-mers) — else the L2 policy below.
  // Windows are estimated from the mean read length (exact for equal-length reads): k = 100 on
  // 100-bp reads has one window per 100 bases.
  double windows = (double)n_bases;
  if (n_reads > 0) {
    const double len = (double)n_bases / (double)n_reads;
    windows = std::min(windows, (double)n_reads * std::max(0.0, len - (double)k + 1.0));
  }
  const uint32_t cap = m < 11 ? 0u : smem_slots_for(ctx, k);
  if (cap) {
    const double want = ctx->rho * windows / (0.35 * cap);
    uint32_t B = 512;
    while ((double)B < want && B < (1u << 22)) B <<= 1;
    while (B < 64u * (uint32_t)ctx->world) B <<= 1;
    return B;
  }
  // Enough bins that one L2-sized wave packs ~16 of them (waves are unions of
  // whole bins), at least 512 (the paper's default F) and at
  // least 64 per rank.
  const double slot = 8.0 + 8.0 * W;
  const double table = ctx->rho * windows * slot / ctx->cfg.target_load;
  const double per_bin = (double)ctx->cfg.wave_table_bytes / 16.0;
  uint32_t B = 512;
  while ((double)B * per_bin < table && B < 8192) B <<= 1;
  while (B < 64u * (uint32_t)ctx->world) B <<= 1;
  return B;
}

// Step (c) plan from the all-gathered histograms H[world][3][B] (windows, super-mers,
// payload words): LPT bin owners (heaviest bin first to the least-loaded rank; ties to
// the lower bin / rank, so every rank derives the same map), this rank's send layout
// by destination and receive layout by source (inside each, owned bins in bin order).
inline void exchange_plan(const uint64_t* H, uint32_t B, int P, int r, int32_t* owner, uint64_t* sd_off,
                   uint64_t* sw_off, uint64_t* rd_off, uint64_t* rw_off) {
  auto Hw = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + b]; };
  auto Hc = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + B + b]; };
  auto Hp = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + 2 * B + b]; };
  std::vector<uint64_t> gw(B, 0);
  for (int s = 0; s < P; ++s)
    for (uint32_t b = 0; b < B; ++b) gw[b] += Hw(s, b);
  std::vector<uint32_t> order(B);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return gw[a] > gw[b]; });
  std::vector<uint64_t> load(P, 0);
  for (uint32_t b : order) {
    int best = 0;
    for (int p = 1; p < P; ++p)
      if (load[p] < load[best]) best = p;
    owner[b] = best;
    load[best] += gw[b];
  }
  for (int i = 0; i <= P; ++i) sd_off[i] = sw_off[i] = rd_off[i] = rw_off[i] = 0;
  for (uint32_t b = 0; b < B; ++b) {
    sd_off[owner[b] + 1] += Hc(r, b);
    sw_off[owner[b] + 1] += Hp(r, b);
  }
  for (int d = 0; d < P; ++d) {
    sd_off[d + 1] += sd_off[d];
    sw_off[d + 1] += sw_off[d];
  }
  for (int s = 0; s < P; ++s) {
    uint64_t cd = 0, cw = 0;
    for (uint32_t b = 0; b < B; ++b)
      if (owner[b] == r) {
        cd += Hc(s, b);
        cw += Hp(s, b);
      }
    rd_off[s + 1] = rd_off[s] + cd;
    rw_off[s + 1] = rw_off[s] + cw;
  }
}

// Small device → page-locked host read on ctx->stream. During a streaming call the copy engine
// is busy with the record copies (GB), behind which a cudaMemcpy would queue: a kernel writes the
// words through the mapping instead.
inline cudaError_t d2h_small(gerbil_ctx* ctx, void* host_pinned, const void* dev, size_t bytes) {
  if (!ctx->rec_out) return cudaMemcpyAsync(host_pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream);
  unsigned long long* mapped = nullptr;
  cudaError_t e = cudaHostGetDevicePointer((void**)&mapped, host_pinned, 0);
  if (e != cudaSuccess) return e;
  return launch_copy_words_mapped(mapped, reinterpret_cast<const unsigned long long*>(dev), (bytes + 7) / 8,
                                  ctx->stream);
}

// results (W key words + u32 count) a fixed 1/div share of the device memory holds (>= 1)
inline uint64_t result_budget_entries(gerbil_ctx* ctx, uint32_t W, uint32_t div) {
  if (!ctx->mem_total) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      tot = 64ull << 30;
    }
    ctx->mem_total = tot;
  }
  const uint64_t n = (uint64_t)(ctx->mem_total / div) / (W * 8ull + 4ull);
  return n ? n : 1;
}

inline double wall_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// GERBIL_TRACE=1: host wall-clock milestones of a call on stderr (diagnostics)
inline void trace(const char* what) {
  static const bool on = getenv("GERBIL_TRACE") && *getenv("GERBIL_TRACE") == '1';
  static double t0 = 0;
  if (!on) return;
  const double t = wall_ms();
  if (strcmp(what, "call") == 0) t0 = t;
  fprintf(stderr, "[gerbil] %9.3f ms  %s\n", t - t0, what);
}

// ---------------------------------------------------------------------------
// Grow b to n bytes keeping its first `keep` bytes (results of an earlier pass).
inline cudaError_t ensure_keep(DevBuf& b, size_t n, size_t keep, cudaStream_t s) {
  if (n <= b.bytes && b.p) return cudaSuccess;
  if (keep == 0 || !b.p) return b.ensure(n);
  DevBuf nb;
  cudaError_t e = nb.ensure(n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(nb.p, b.p, keep, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  std::swap(b.p, nb.p);
  std::swap(b.bytes, nb.bytes);
  return cudaSuccess;
}


// ---- cross-unit steps -----------------------------------------------------------------------
struct Preset;
struct RestBin;
uint32_t smem_slots_for(gerbil_ctx* ctx, uint32_t k);
uint32_t smem_max_fill(const gerbil_ctx* ctx, uint32_t cap, uint32_t k);
uint64_t smem_window_threshold(const gerbil_ctx* ctx, uint32_t max_fill);
gerbil_status count_waves(gerbil_ctx* ctx, const uint64_t* stream_codes, const uint64_t* desc,
                          const std::vector<uint64_t>& bin_off, const std::vector<uint64_t>& bin_win,
                          const std::vector<uint32_t>& bins, uint32_t k, uint32_t min_count,
                          uint64_t total_windows);
gerbil_status group_shuffle(gerbil_ctx* ctx, const uint64_t* desc_in, const uint32_t* bin_in, uint64_t n, uint32_t B,
                            uint64_t* tmp_desc, uint32_t* tmp_bin, uint64_t* desc_alt, uint64_t max_windows);
gerbil_status exchange_groups(gerbil_ctx* ctx, const uint64_t* codes, uint64_t n_sm, uint32_t B, uint32_t cap,
                              uint32_t k, uint32_t min_count, uint64_t& owned_windows);
gerbil_status build_dfp_table(gerbil_ctx* ctx, const SupermerArgs& a, uint64_t n_bases, uint32_t m);
gerbil_status run_supermer(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                           const uint64_t* rstart, uint64_t n_reads, uint64_t n_bases, uint32_t k,
                           uint32_t m, uint32_t B, bool want_mu, uint64_t& n_sm, bool want_hist = true);
void begin_call(gerbil_ctx* ctx);
gerbil_status count_device_impl(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                uint32_t min_count, bool fresh = true);
}  // namespace gerbil_api

// entry-point helpers shared by io.cu and spill.cu (C linkage, not exported by gerbil.h)
extern "C" {
gerbil_status upload_batch(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask, const uint64_t* rstart,
                           uint64_t n_reads, UploadPlan& plan);
}
