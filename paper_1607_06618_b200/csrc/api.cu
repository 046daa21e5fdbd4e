// api.cu — C ABI (include/gerbil.h) and host orchestration of steps (a)-(e).
//
// One context = one rank = one GPU. gerbil_count_device runs, on the
// context's stream:
//   (b) supermer kernel → descriptors + per-bin histogram     (supermer.cu)
//   [host] read the histogram; world > 1: all-gather it, assign bins to
//          owner ranks (LPT), pack + NCCL all-to-all          (comm.cu)
//   (c) bin scatter: descriptors grouped by bin                (shuffle.cu)
//   [host] plan table waves (groups of bins whose table fits the budget)
//   (d)+(e) per wave: count kernel, compaction kernel          (count.cu, compact.cu)
//   emergency pass for overflowed k-mers; Σ-count invariant check.
// Table waves reuse one table buffer sized to stay L2-resident
// (cfg.wave_table_bytes, default 128 MiB ≈ the 126 MB L2), so the hash-table
// atomics are served by L2 and HBM sees the streaming traffic only.
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

namespace {

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
bool use_reads_kernel(uint32_t k, uint32_t m, uint64_t n_bases, uint64_t n_reads) {
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

}  // namespace

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
  DevBuf order_rank, order_freq;  // DFP ordering: key table [4^m] and its sample histogram
  DevBuf text_buf, p_cnt, p_off, p_ls, p_cr, p_eff, p_first, p_seq, p_rflag, p_pos, p_ridx, p_tmp, p_misc;  // parser
  uint32_t m = 0;  // streaming call: per-lane record staging; counters/snapshots/offsets
  DevBuf send_desc, send_bin, send_payload, recv_desc, recv_bin, recv_payload;
  DevBuf smem_range, smem_failed, rest_desc, rest_range, rest_off;  // step (d) in shared memory
  int smem_optin = 0;  // max dynamic shared memory per block (bytes)
  PinnedBuf h_hist, h_rng;  // per-bin histogram download, shared-memory bin list upload
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

namespace {

gerbil_status fail(gerbil_ctx* c, gerbil_status st, const std::string& msg) {
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

cudaEvent_t get_event(gerbil_ctx* ctx) {
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
int wave_lanes() {
  const char* e = getenv("GERBIL_WAVE_LANES");
  if (e && *e) return atoi(e) <= 1 ? 1 : 2;
  return 2;
}

gerbil_status validate(gerbil_ctx* ctx, uint32_t k, uint32_t& m, uint32_t min_count) {
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
// from this many bins up, a single rank plans steps (c)-(e) on the device
constexpr uint32_t kDevicePlanBins = 1u << 16;
gerbil_status count_local_device_plan(gerbil_ctx* ctx, const uint64_t* codes, uint64_t n_sm, uint32_t B,
                                      uint32_t cap, uint32_t k, uint32_t min_count, uint64_t windows,
                                      uint64_t n_bases);

uint32_t choose_bins(gerbil_ctx* ctx, uint64_t n_bases, uint64_t n_reads, uint32_t W, uint32_t k, uint32_t m) {
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
  const uint32_t cap = (ctx->rec_out || m < 11) ? 0u : smem_slots_for(ctx, k);
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
void exchange_plan(const uint64_t* H, uint32_t B, int P, int r, int32_t* owner, uint64_t* sd_off,
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

double wall_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// GERBIL_TRACE=1: host wall-clock milestones of a call on stderr (diagnostics)
void trace(const char* what) {
  static const bool on = getenv("GERBIL_TRACE") && *getenv("GERBIL_TRACE") == '1';
  static double t0 = 0;
  if (!on) return;
  const double t = wall_ms();
  if (strcmp(what, "call") == 0) t0 = t;
  fprintf(stderr, "[gerbil] %9.3f ms  %s\n", t - t0, what);
}

// ---------------------------------------------------------------------------
// Grow b to n bytes keeping its first `keep` bytes (results of an earlier pass).
cudaError_t ensure_keep(DevBuf& b, size_t n, size_t keep, cudaStream_t s) {
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

// Results already produced by the shared-memory pass of this call: the wave
// pass appends after them (out_n, Σcount and distinct start from these).
struct Preset {
  unsigned long long out_n = 0, sum_counts = 0, distinct = 0;
};

// Steps (d)+(e) in L2-resident wave tables over the bin-ordered descriptors
// of `bins` (consecutive in desc).
gerbil_status count_waves_l2(gerbil_ctx* ctx, const uint64_t* stream_codes, const uint64_t* desc,
                             const std::vector<uint64_t>& bin_off, const std::vector<uint64_t>& bin_win,
                             const std::vector<uint32_t>& bins, uint32_t k, uint32_t min_count,
                             uint64_t total_windows, const Preset& pre) {
  const uint32_t W = key_words(k);
  const uint64_t bb = table_inline(k) ? kInlineBucketBytes : table_bucket_bytes(k);
  const double slot_bytes = (double)bb / kSlotsPerBucket;
  double alpha = ctx->cfg.target_load;  // lowered on a retry once rho can grow no further
  const uint32_t theta = std::min<uint32_t>(ctx->cfg.max_probes, 1u << 20);  // probe counters are 24-bit
  const int lanes = wave_lanes();
  const double budget = (double)ctx->cfg.wave_table_bytes / lanes;  // per-lane table bytes
  Counters& hc = *ctx->h_counters;
  for (int attempt = 0;; ++attempt) {
    const double rho = ctx->rho;
    // plan waves: consecutive owned bins until the table budget is reached
    std::vector<Wave> waves;
    uint64_t max_nb = 1, out_bound = 0;
    {
      double acc = 0;
      Wave cur{0, 0, 0, 0};
      bool open = false;
      auto close = [&] {
        if (!open) return;
        const double slots = std::max(64.0, std::ceil(rho * (double)cur.windows / alpha));
        cur.nb = (uint64_t)std::ceil(slots / kSlotsPerBucket);
        max_nb = std::max(max_nb, cur.nb);
        out_bound += std::min<uint64_t>(cur.nb * kSlotsPerBucket, cur.windows);
        waves.push_back(cur);
        open = false;
        acc = 0;
      };
      for (uint32_t b : bins) {
        const double need = rho * (double)bin_win[b] / alpha * slot_bytes;
        if (open && acc + need > budget) close();
        if (!open) {
          cur = Wave{bin_off[b], bin_off[b], 0, 0};
          open = true;
        }
        cur.d1 = bin_off[b + 1] - bin_off[b] + cur.d1;
        cur.windows += bin_win[b];
        acc += need;
      }
      close();
    }
    const uint64_t ovf_cap = std::max<uint64_t>(1 << 16, total_windows / 32);
    const uint64_t lane_bytes = (max_nb * bb + 255) & ~255ull;
    CK(ctx->table.ensure(lanes * lane_bytes));
    CK(ctx->ovf.ensure(ovf_cap * W * 8));
    // Result buffer: the waves' distinct bound can exceed device memory when most k-mers are
    // singletons and min_count > 1 drops them (C4: ~1.5e10 bound, ~3.6e8 kept per GPU), so it is
    // sized for at most a quarter of the free memory and grown between waves when the bound of
    // the next wave might not fit (a sync reads how many results the earlier waves kept).
    uint64_t out_chunk = out_bound;
    {
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
        const uint64_t fit = (uint64_t)(fr / 4) / (W * 8 + 4);
        uint64_t big_wave = 0;
        for (const Wave& wv : waves) big_wave = std::max(big_wave, std::min<uint64_t>(wv.nb * kSlotsPerBucket, wv.windows));
        out_chunk = std::min(out_bound, std::max(fit, 2 * big_wave));
      }
    }
    uint64_t out_cap = pre.out_n + out_chunk + ovf_cap;
    CK(ensure_keep(ctx->out_keys, out_cap * W * 8, pre.out_n * W * 8, ctx->stream));
    CK(ensure_keep(ctx->out_counts, out_cap * 4, pre.out_n * 4, ctx->stream));
    uint64_t out_committed = pre.out_n, bound_left = out_bound;  // results possibly written / still to come
    // [0, n): distinct per wave; [n, 2n): dynamic work counters of the count launches
    const size_t nw = std::max<size_t>(waves.size(), 1);
    CK(ctx->wave_distinct.ensure(2 * nw * 8));
    CK(cudaMemsetAsync(ctx->table.p, 0, lanes * lane_bytes, ctx->stream));
    CK(cudaMemsetAsync(ctx->wave_distinct.p, 0, 2 * nw * 8, ctx->stream));
    Counters* dc = ctx->counters.as<Counters>();
    CK(cudaMemsetAsync(&dc->ovf_n, 0, sizeof(Counters) - offsetof(Counters, ovf_n), ctx->stream));
    if (pre.out_n || pre.sum_counts || pre.distinct) {
      static_assert(offsetof(Counters, sum_counts) == offsetof(Counters, out_n) + 8 &&
                        offsetof(Counters, distinct) == offsetof(Counters, out_n) + 16,
                    "preset copy assumes out_n, sum_counts, distinct are adjacent");
      hc.out_n = pre.out_n;  // pinned staging for the copy
      hc.sum_counts = pre.sum_counts;
      hc.distinct = pre.distinct;
      CK(cudaMemcpyAsync(&dc->out_n, &hc.out_n, 24, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }

    TableArgs t{};
    t.table = ctx->table.as<unsigned char>();
    t.max_probes = theta;
    t.ovf = ctx->ovf.as<uint64_t>();
    t.ovf_cap = ovf_cap;
    t.ovf_n = &dc->ovf_n;
    t.probe_hist = dc->probe;
    CompactArgs ca{};
    ca.table = t.table;
    ca.k = k;
    ca.min_count = min_count;
    ca.out_keys = ctx->out_keys.as<uint64_t>();
    ca.out_counts = ctx->out_counts.as<uint32_t>();
    ca.cap = out_cap;
    ca.out_n = &dc->out_n;
    ca.sum_counts = &dc->sum_counts;
    ca.distinct = &dc->distinct;
    // Streaming call: each lane's compactions append App. C records to the
    // lane's HBM staging area; after compact(w) the lane's byte counter is
    // copied to pinned host memory (h_snap[w]) and an event marks wave w.
    // Once every wave is launched, this thread waits for the waves in order
    // and has the copy engine move [end of the lane's previous wave,
    // h_snap[w]) of the staging area to the caller's buffer — DMA behind the
    // counting, no SMs taken from the count kernels. rec_meta: 2 lane counters.
    const bool streaming = ctx->rec_out != nullptr;
    const bool two = lanes > 1 && waves.size() > 1;
    unsigned long long* lane_ctr = nullptr;
    uint64_t lane_stage_off[2] = {0, 0}, lane_cap[2] = {0, 0};
    struct Pending {
      int lane;
      size_t wi;
    };
    std::vector<Pending> pending;
    uint64_t lane_done[2] = {0, 0}, host_off = ctx->rec_base;
    if (streaming) {
      const uint64_t rec_max = 5 + (k + 3) / 4;
      uint64_t lb[2] = {0, 0};
      for (size_t w = 0; w < waves.size(); ++w)
        lb[two ? (w & 1) : 0] += std::min<uint64_t>(waves[w].nb * kSlotsPerBucket, waves[w].windows) * rec_max;
      lb[0] += ovf_cap * rec_max;
      lane_stage_off[1] = (lb[0] + 64 + 255) & ~255ull;
      lane_cap[0] = lb[0];
      lane_cap[1] = lb[1];
      CK(ctx->rec_stage.ensure(lane_stage_off[1] + lb[1] + 64));
      CK(ctx->rec_meta.ensure(2 * 8));
      CK(cudaMemsetAsync(ctx->rec_meta.p, 0, 2 * 8, ctx->stream));
      lane_ctr = ctx->rec_meta.as<unsigned long long>();
      if (ctx->h_snap_n < nw + 1) {
        if (ctx->h_snap) cudaFreeHost(ctx->h_snap);
        ctx->h_snap = nullptr;
        ctx->h_snap_n = 0;
        CK(cudaMallocHost((void**)&ctx->h_snap, (nw + 1) * 8));
        ctx->h_snap_n = nw + 1;
      }
      while (ctx->wave_ev.size() < nw + 1) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        ctx->wave_ev.push_back(ev);
      }
    }
    // after compact(wi) on st: snapshot lane L's byte counter, mark the wave
    auto stream_wave = [&](int L, size_t wi, cudaStream_t st) -> gerbil_status {
      CK(cudaMemcpyAsync(ctx->h_snap + wi, lane_ctr + L, 8, cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(ctx->wave_ev[wi], st));
      pending.push_back({L, wi});
      return GERBIL_OK;
    };
    // wait for each marked wave in order and DMA its records to the caller
    auto drain_copies = [&]() -> gerbil_status {
      for (const Pending& pw : pending) {
        CK(cudaEventSynchronize(ctx->wave_ev[pw.wi]));
        const uint64_t end = ctx->h_snap[pw.wi], start = lane_done[pw.lane], len = end - start;
        if (len && host_off + len <= ctx->rec_cap)
          CK(cudaMemcpyAsync(ctx->rec_out + host_off, ctx->rec_stage.as<uint8_t>() + lane_stage_off[pw.lane] + start,
                             len, cudaMemcpyDeviceToHost, ctx->pcie_stream));
        lane_done[pw.lane] = end;
        host_off += len;
      }
      pending.clear();
      return GERBIL_OK;
    };
    trace("waves planned, buffers ready");
    {
      // with two lanes the per-launch events would overlap: one span timer
      // covers steps (d)+(e) and is reported as ms_count (ms_compact = 0)
      Timer span(ctx, K_COUNT, ctx->stream, two, 0);
      if (two) {
        CK(cudaEventRecord(ctx->fork_ev, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->lane_stream, ctx->fork_ev, 0));
      }
      for (size_t w = 0; w < waves.size(); ++w) {
        const int lane = two ? (int)(w & 1) : 0;
        cudaStream_t st = lane ? ctx->lane_stream : ctx->stream;
        const uint64_t wb = std::min<uint64_t>(waves[w].nb * kSlotsPerBucket, waves[w].windows);
        if (!streaming && out_committed + wb + ovf_cap > out_cap) {
          // the next wave might not fit: settle how many results the launched waves kept
          if (two) CK(cudaStreamSynchronize(ctx->lane_stream));
          CK(cudaMemcpyAsync(&hc.out_n, &dc->out_n, 8, cudaMemcpyDeviceToHost, ctx->stream));
          CK(cudaStreamSynchronize(ctx->stream));
          out_committed = hc.out_n;
          if (out_committed + wb + ovf_cap > out_cap) {
            out_cap = out_committed + std::max(std::min(bound_left, out_chunk), wb) + ovf_cap;
            CK(ensure_keep(ctx->out_keys, out_cap * W * 8, out_committed * W * 8, ctx->stream));
            CK(ensure_keep(ctx->out_counts, out_cap * 4, out_committed * 4, ctx->stream));
            ca.out_keys = ctx->out_keys.as<uint64_t>();
            ca.out_counts = ctx->out_counts.as<uint32_t>();
            ca.cap = out_cap;
          }
          if (two) {  // the lane stream continues after everything issued on the main stream
            CK(cudaEventRecord(ctx->fork_ev, ctx->stream));
            CK(cudaStreamWaitEvent(ctx->lane_stream, ctx->fork_ev, 0));
          }
        }
        out_committed += wb;
        bound_left -= std::min(bound_left, wb);
        t.table = ctx->table.as<unsigned char>() + lane * lane_bytes;
        t.nb = waves[w].nb;
        CountArgs a{stream_codes, desc, waves[w].d0, waves[w].d1, k, t,
                    ctx->wave_distinct.as<unsigned long long>() + nw + w,
                    ctx->cfg.disable_normalization ? 0u : 1u,
                    count_dpc((double)waves[w].windows / (double)std::max<uint64_t>(1, waves[w].d1 - waves[w].d0))};
        {
          Timer tm(ctx, K_COUNT, st, !two);
          CK(launch_count(a, W, ctx->sms, st));
        }
        ca.table = t.table;
        ca.nb = waves[w].nb;
        ca.wave_distinct = ctx->wave_distinct.as<unsigned long long>() + w;
        if (streaming) {
          ca.rec_out = ctx->rec_stage.as<uint8_t>() + lane_stage_off[lane];
          ca.rec_cap = lane_cap[lane];
          ca.rec_n = lane_ctr + lane;
        }
        {
          Timer tm(ctx, K_COMPACT, st, !two);
          CK(launch_compact(ca, ctx->sms, st));
        }
        if (streaming) CKS(stream_wave(lane, w, st));
      }
      if (two) {
        CK(cudaEventRecord(ctx->join_ev, ctx->lane_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
      }
    }
    trace("waves launched");
    if (streaming) CKS(drain_copies());
    CK(cudaMemcpyAsync(ctx->h_counters, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<unsigned long long> wd(waves.size());
    if (!waves.empty())
      CK(cudaMemcpyAsync(wd.data(), ctx->wave_distinct.p, waves.size() * 8, cudaMemcpyDeviceToHost,
                         ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    // observed distinct/total ratio: max over waves large enough to be a fair
    // sample (a tiny wave of a few singletons would read 1.0 and bloat every
    // table of the next call); small inputs fall back to the pooled ratio
    double observed = 0;
    uint64_t big = 0, pooled_w = 0, pooled_d = 0;
    for (size_t w = 0; w < waves.size(); ++w) {
      big = std::max(big, waves[w].windows);
      pooled_w += waves[w].windows;
      pooled_d += wd[w];
    }
    for (size_t w = 0; w < waves.size(); ++w)
      if (waves[w].windows >= std::max<uint64_t>(big / 4, 1))
        observed = std::max(observed, (double)wd[w] / (double)waves[w].windows);
    if (pooled_w) observed = std::max(observed, (double)pooled_d / (double)pooled_w);
    ctx->stats.waves = (uint32_t)waves.size();
    ctx->stats.ratio_used = rho;
    ctx->stats.ratio_observed = observed;
    ctx->stats.overflow_kmers = hc.ovf_n;
    ctx->stats.overflow_passes = 0;
    ctx->stats.probe_first = hc.probe[0];
    ctx->stats.probe_more = hc.probe[1];
    ctx->stats.probe_max = hc.probe[2];
    const uint64_t ovf_n = hc.ovf_n;
    trace("waves done (synced)");
    if (ovf_n > ovf_cap) {
      // emergency area exhausted: redo the waves with larger tables (after
      // this attempt's record copies, which write the same host buffer)
      if (streaming) {
        CK(cudaStreamSynchronize(ctx->pcie_stream));
        lane_done[0] = lane_done[1] = 0;
        host_off = ctx->rec_base;
      }
      ctx->rho = std::min(1.0, std::max(2.0 * rho, 1.25 * observed + 0.02));
      // rho is capped at 1 (distinct <= windows): with alpha > 1 the tables would keep their
      // size on every retry, so shrink the load target instead
      if (ctx->rho <= rho && alpha > 0.5) alpha = std::max(0.5, alpha * 0.5);
      if (attempt > 8) return fail(ctx, GERBIL_E_INTERNAL, "table sizing did not converge");
      continue;
    }
    if (ovf_n > 0) {
      // emergency mechanism: count the overflowed k-mers
      // exactly in a table with room for all of them and θ = every bucket.
      const uint64_t nb2 = std::max<uint64_t>(8, (uint64_t)std::ceil((double)ovf_n / (0.5 * kSlotsPerBucket)));
      CK(ctx->table.ensure(nb2 * bb));
      t.table = ctx->table.as<unsigned char>();
      CK(cudaMemsetAsync(ctx->table.p, 0, nb2 * bb, ctx->stream));
      // overflow keys must not be overwritten while re-inserted: θ = nb2 never overflows
      TableArgs t2 = t;
      t2.table = ctx->table.as<unsigned char>();
      t2.nb = nb2;
      t2.max_probes = (uint32_t)std::min<uint64_t>(nb2, 0xffffffffu);
      t2.ovf_cap = 0;
      CountKeysArgs ka{ctx->ovf.as<uint64_t>(), ovf_n, k, t2};
      {
        Timer tm(ctx, K_OVERFLOW);
        CK(launch_count_keys(ka, W, ctx->sms, ctx->stream));
      }
      CompactArgs c2 = ca;
      c2.table = t2.table;
      c2.nb = nb2;
      c2.wave_distinct = nullptr;
      if (streaming) {  // lane 0's staging area has room for the emergency pass
        c2.rec_out = ctx->rec_stage.as<uint8_t>();
        c2.rec_cap = lane_cap[0];
        c2.rec_n = lane_ctr;
      }
      {
        Timer tm(ctx, K_OVERFLOW);
        CK(launch_compact(c2, ctx->sms, ctx->stream));
      }
      if (streaming) {
        CKS(stream_wave(0, nw, ctx->stream));
        CKS(drain_copies());
      }
      CK(cudaMemcpyAsync(ctx->h_counters, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->stats.overflow_passes = 1;
      if (hc.ovf_n != ovf_n) return fail(ctx, GERBIL_E_INTERNAL, "emergency pass overflowed");
    }
    if (hc.out_n > out_cap) return fail(ctx, GERBIL_E_INTERNAL, "result buffer bound violated");
    // ratio adaptation for the next call ("we dynamically adjust the ratio")
    if (observed > 0) ctx->rho = std::min(1.0, std::max(observed * 1.15 + 0.01, 0.02));
    ctx->n_out = hc.out_n;
    if (streaming) {  // wait for the last record copies
      CK(cudaStreamSynchronize(ctx->pcie_stream));
      ctx->rec_bytes = host_off;
      trace("record copies done (synced)");
    }
    ctx->stats.kept = hc.out_n;
    ctx->stats.distinct = hc.distinct;
    ctx->stats.count_sum = hc.sum_counts;
    ctx->stats.owned_windows = total_windows;
    return GERBIL_OK;
  }
}

// Shared-memory table slots per warp for this k (0 = shared-memory path off).
uint32_t smem_slots_for(gerbil_ctx* ctx, uint32_t k) {
  if (ctx->cfg.count_mode == 1) return 0;
  if (!ctx->smem_optin &&
      cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  // W >= 4: one CTA-wide table of occurrence references per bin (count_ref.cu)
  const uint32_t cap = key_words(k) >= 4 ? ref_table_slots((size_t)ctx->smem_optin - 1024)
                                         : smem_table_slots(k, (size_t)ctx->smem_optin - 1024);
  return cap >= 128 ? cap : 0;
}

// Abandonment threshold of the shared-memory tables: a round inserts <= 32 k-mers, so
// a table never fills.
uint32_t smem_max_fill(uint32_t cap, uint32_t k) {
  return key_words(k) >= 4 ? ref_max_fill(cap) : cap - std::max<uint32_t>(64u, cap / 4);
}

// Windows up to which a bin goes to the shared-memory pass: predicted distinct
// (ρ̂ · windows) within the abandonment threshold; a miss costs only the bin's
// partial work (it is recounted in the wave tables). count_mode 2: every bin.
uint64_t smem_window_threshold(const gerbil_ctx* ctx, uint32_t max_fill) {
  if (ctx->cfg.count_mode == 2) return ~0ull;
  return std::max<uint64_t>(max_fill, (uint64_t)(0.95 * max_fill / std::max(ctx->rho, 1e-6)));
}

struct RestBin {
  uint64_t d0, d1, win;  // descriptor range and windows of a bin for the L2 wave tables
};

// Steps (d)+(e): the shared-memory pass over the n bins listed (device) in
// ctx->smem_range, then the bins of `rest` plus every bin the shared-memory pass
// abandoned, gathered into one contiguous descriptor range and counted in the
// L2-resident wave tables, whose results are appended.
gerbil_status count_waves_ranges(gerbil_ctx* ctx, const uint64_t* stream_codes, const uint64_t* desc, uint32_t n,
                                 uint64_t elig_windows, uint64_t out_bound, uint32_t cap, uint32_t max_fill,
                                 std::vector<RestBin>& rest, uint32_t k, uint32_t min_count,
                                 uint64_t total_windows) {
  const uint32_t W = key_words(k);
  CK(ctx->smem_failed.ensure((size_t)n * 16 + 16));
  // the shared-memory pass writes at most out_bound results, but with min_count > 1 on singleton-rich
  // input (C4) that bound can exceed device memory: the buffer is capped at a quarter of the free
  // memory and, if the kept results do not fit, the pass is rerun once with the exact size
  uint64_t out_cap = std::max<uint64_t>(out_bound, 1);
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
      out_cap = std::min<uint64_t>(out_cap, std::max<uint64_t>(1, (uint64_t)(fr / 4) / (W * 8 + 4)));
  }
  CK(ctx->out_keys.ensure(out_cap * W * 8));
  CK(ctx->out_counts.ensure(out_cap * 4));
  CK(ctx->counters.ensure(sizeof(Counters)));
  Counters* dc = ctx->counters.as<Counters>();
  CK(cudaMemsetAsync(&dc->ovf_n, 0, sizeof(Counters) - offsetof(Counters, ovf_n), ctx->stream));
  SmemCountArgs a{};
  a.codes = stream_codes;
  a.desc = desc;
  a.range = ctx->smem_range.as<unsigned long long>();
  a.n_list = n;
  a.k = k;
  a.min_count = min_count;
  a.canonical = ctx->cfg.disable_normalization ? 0u : 1u;
  a.cap = cap;
  a.max_fill = max_fill;
  a.out_n = &dc->out_n;
  a.sum_counts = &dc->sum_counts;
  a.distinct = &dc->distinct;
  a.failed = ctx->smem_failed.as<unsigned long long>();
  a.n_failed = &dc->read_work;
  Counters& hc = *ctx->h_counters;
  for (int attempt = 0;; ++attempt) {
    a.out_keys = ctx->out_keys.as<uint64_t>();
    a.out_counts = ctx->out_counts.as<uint32_t>();
    a.out_cap = out_cap;
    {
      Timer tm(ctx, K_SMEM);
      CK(launch_count_smem(a, ctx->sms, ctx->stream));
    }
    trace("smem count issued");
    CK(cudaMemcpyAsync(ctx->h_counters, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    trace("smem count done (synced)");
    if (hc.out_n > out_bound) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory result bound violated");
    if (hc.out_n <= out_cap) break;
    if (attempt > 0) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory pass: result size changed on rerun");
    out_cap = hc.out_n;  // exact: the rerun keeps the same k-mers
    CK(ctx->out_keys.ensure(out_cap * W * 8));
    CK(ctx->out_counts.ensure(out_cap * 4));
    CK(cudaMemsetAsync(&dc->ovf_n, 0, sizeof(Counters) - offsetof(Counters, ovf_n), ctx->stream));
  }
  const uint64_t n_failed = hc.read_work;
  Preset pre;
  pre.out_n = hc.out_n;
  pre.sum_counts = hc.sum_counts;
  pre.distinct = hc.distinct;
  uint64_t failed_windows = 0;
  if (n_failed) {
    std::vector<unsigned long long> fr(2 * n_failed);
    CK(cudaMemcpyAsync(fr.data(), ctx->smem_failed.p, fr.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint64_t i = 0; i < n_failed; ++i) {
      const uint64_t w = fr[2 * i + 1] >> kRangeWinShift;
      rest.push_back({fr[2 * i], fr[2 * i + 1] & kRangeEndMask, w});
      failed_windows += w;
    }
  }
  ctx->stats.smem_bins += n;
  ctx->stats.smem_failed += n_failed;
  uint64_t smem_windows = elig_windows - std::min(elig_windows, failed_windows);
  // Tier 2: bins too large for the many-warp tables get 4-warp tables (~4x the slots per
  // warp) in a second launch; what still does not fit goes to the wave tables.
  const int w1 = a.warps ? a.warps : smem_count_warps(k);
  const int w2n = std::max(1, w1 / 2);
  const uint32_t cap2 = w1 > 4 ? smem_table_slots(k, (size_t)ctx->smem_optin - 1024, w2n) : 0u;
  if (!rest.empty() && cap2 > cap) {
    const uint32_t mf2 = smem_max_fill(cap2, k);
    const uint64_t thr2 = smem_window_threshold(ctx, mf2);
    std::vector<RestBin> keep;
    uint64_t n2 = 0, w2 = 0, ob2 = 0;
    CK(ctx->h_rng.ensure(rest.size() * 16));
    unsigned long long* r2 = ctx->h_rng.as<unsigned long long>();
    for (const RestBin& rb : rest) {
      if (rb.win <= thr2) {
        r2[2 * n2] = rb.d0;
        r2[2 * n2 + 1] = rb.d1 | (std::min<uint64_t>(rb.win, (1u << 24) - 1) << kRangeWinShift);
        ++n2;
        w2 += rb.win;
        ob2 += smem_bin_out_bound(rb.win, cap2, mf2);
      } else {
        keep.push_back(rb);
      }
    }
    if (n2) {
      const uint64_t out2 = pre.out_n + ob2;
      CK(ensure_keep(ctx->out_keys, out2 * W * 8, pre.out_n * W * 8, ctx->stream));
      CK(ensure_keep(ctx->out_counts, out2 * 4, pre.out_n * 4, ctx->stream));
      CK(ctx->smem_range.ensure(n2 * 16));
      CK(ctx->smem_failed.ensure(n2 * 16 + 16));
      CK(cudaMemcpyAsync(ctx->smem_range.p, r2, n2 * 16, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemsetAsync(&dc->read_work, 0, 8, ctx->stream));
      SmemCountArgs a2 = a;
      a2.range = ctx->smem_range.as<unsigned long long>();
      a2.n_list = (uint32_t)n2;
      a2.cap = cap2;
      a2.max_fill = mf2;
      a2.warps = w2n;
      a2.out_keys = ctx->out_keys.as<uint64_t>();
      a2.out_counts = ctx->out_counts.as<uint32_t>();
      a2.out_cap = out2;
      a2.failed = ctx->smem_failed.as<unsigned long long>();
      {
        Timer tm(ctx, K_SMEM);
        CK(launch_count_smem(a2, ctx->sms, ctx->stream));
      }
      CK(cudaMemcpyAsync(ctx->h_counters, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (hc.out_n > out2) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory result bound violated");
      pre.out_n = hc.out_n;
      pre.sum_counts = hc.sum_counts;
      pre.distinct = hc.distinct;
      const uint64_t nf2 = hc.read_work;
      uint64_t fw2 = 0;
      if (nf2) {
        std::vector<unsigned long long> fr(2 * nf2);
        CK(cudaMemcpyAsync(fr.data(), ctx->smem_failed.p, fr.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (uint64_t i = 0; i < nf2; ++i) {
          const uint64_t w = fr[2 * i + 1] >> kRangeWinShift;
          keep.push_back({fr[2 * i], fr[2 * i + 1] & kRangeEndMask, w});
          fw2 += w;
        }
      }
      ctx->stats.smem_bins += n2;
      ctx->stats.smem_failed += nf2;
      smem_windows += w2 - std::min(w2, fw2);
      rest.swap(keep);
      trace("smem tier 2 done (synced)");
    }
  }
  ctx->stats.smem_windows += smem_windows;
  const double smem_obs = smem_windows ? (double)pre.distinct / (double)smem_windows : 0.0;
  gerbil_status st = GERBIL_OK;
  if (rest.empty()) {
    ctx->stats.waves = 0;
    ctx->stats.ratio_used = ctx->rho;
    ctx->stats.ratio_observed = smem_obs;
    ctx->stats.overflow_kmers = 0;
    ctx->stats.overflow_passes = 0;
    ctx->n_out = pre.out_n;
    ctx->stats.kept = pre.out_n;
    ctx->stats.distinct = pre.distinct;
    ctx->stats.count_sum = pre.sum_counts;
    ctx->stats.owned_windows = total_windows;
  } else {
    // gather the remaining bins' descriptors into one contiguous range (any bin order)
    const uint32_t R = (uint32_t)rest.size();
    CK(ctx->h_rng.ensure((size_t)R * 16 + (size_t)R * 8));
    unsigned long long* rr = ctx->h_rng.as<unsigned long long>();
    unsigned long long* ro = rr + 2 * (size_t)R;
    std::vector<uint64_t> off2(R + 1, 0), win2(R);
    std::vector<uint32_t> list2(R);
    for (uint32_t i = 0; i < R; ++i) {
      rr[2 * i] = rest[i].d0;
      rr[2 * i + 1] = rest[i].d1;
      ro[i] = off2[i];
      off2[i + 1] = off2[i] + (rest[i].d1 - rest[i].d0);
      win2[i] = rest[i].win;
      list2[i] = i;
    }
    CK(ctx->rest_range.ensure((size_t)R * 16));
    CK(ctx->rest_off.ensure((size_t)R * 8));
    CK(ctx->rest_desc.ensure(std::max<uint64_t>(off2[R], 1) * 8));
    CK(cudaMemcpyAsync(ctx->rest_range.p, rr, (size_t)R * 16, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->rest_off.p, ro, (size_t)R * 8, cudaMemcpyHostToDevice, ctx->stream));
    {
      Timer tm(ctx, K_SHUFFLE);
      CK(launch_gather_ranges(desc, ctx->rest_range.as<unsigned long long>(), ctx->rest_off.as<unsigned long long>(),
                              R, ctx->rest_desc.as<uint64_t>(), ctx->sms, ctx->stream));
    }
    st = count_waves_l2(ctx, stream_codes, ctx->rest_desc.as<uint64_t>(), off2, win2, list2, k, min_count,
                        total_windows, pre);
    if (st != GERBIL_OK) return st;
  }
  // ratio adaptation: the larger of the wave and shared-memory observations
  if (smem_obs > 0) ctx->rho = std::min(1.0, std::max(rest.empty() ? 0.0 : ctx->rho, std::max(smem_obs * 1.15 + 0.01, 0.02)));
  return st;
}

// Steps (d)+(e) over the bin-ordered descriptors of this rank, bins given on the
// host: the predicted-small bins go to the shared-memory pass, the rest (and any
// abandoned bin) to the L2 wave tables (count_waves_ranges); with no small bin the
// wave tables take the bins in place.
gerbil_status count_waves(gerbil_ctx* ctx, const uint64_t* stream_codes, const uint64_t* desc,
                          const std::vector<uint64_t>& bin_off, const std::vector<uint64_t>& bin_win,
                          const std::vector<uint32_t>& bins, uint32_t k, uint32_t min_count,
                          uint64_t total_windows) {
  const uint32_t cap = ctx->rec_out ? 0u : smem_slots_for(ctx, k);
  ctx->stats.smem_slots = cap;
  if (cap == 0) return count_waves_l2(ctx, stream_codes, desc, bin_off, bin_win, bins, k, min_count,
                                      total_windows, Preset{});
  const uint32_t max_fill = smem_max_fill(cap, k);
  const uint64_t thr = smem_window_threshold(ctx, max_fill);
  std::vector<uint32_t> elig;
  std::vector<RestBin> rest;
  for (uint32_t b : bins) {
    if (bin_off[b + 1] == bin_off[b]) continue;  // no super-mers, nothing to count
    if (bin_win[b] <= thr) elig.push_back(b);
    else rest.push_back({bin_off[b], bin_off[b + 1], bin_win[b]});
  }
  uint64_t elig_w = 0;
  for (uint32_t b : elig) elig_w += bin_win[b];
  // a shared-memory pass over a sliver of the windows would only add a launch and a
  // gather of every other bin (m < 11 gives few bins small enough): waves take all
  if (elig.empty() || (ctx->cfg.count_mode != 2 && elig_w * 20 < total_windows))
    return count_waves_l2(ctx, stream_codes, desc, bin_off, bin_win, bins, k, min_count, total_windows,
                          Preset{});
  trace("smem bins selected");
  const uint32_t n = (uint32_t)elig.size();
  CK(ctx->h_rng.ensure(2 * (size_t)n * 8));
  unsigned long long* rng = ctx->h_rng.as<unsigned long long>();
  uint64_t out_bound = 0, elig_windows = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t b = elig[i];
    rng[2 * i] = bin_off[b];
    rng[2 * i + 1] = bin_off[b + 1] | (std::min<uint64_t>(bin_win[b], (1u << 24) - 1) << kRangeWinShift);
    out_bound += smem_bin_out_bound(bin_win[b], cap, max_fill);
    elig_windows += bin_win[b];
  }
  CK(ctx->smem_range.ensure(2 * (size_t)n * 8));
  CK(cudaMemcpyAsync(ctx->smem_range.p, rng, 2 * (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // h_rng is reused by the wave pass
  return count_waves_ranges(ctx, stream_codes, desc, n, elig_windows, out_bound, cap, max_fill, rest, k,
                            min_count, total_windows);
}

// Single rank with many bins: the per-bin bookkeeping of steps (c)-(e) stays on the
// device — exclusive scan of the per-bin super-mer counts (bin offsets), scatter, and
// the split into the shared-memory list and the rest (plan_bins_kernel); only the
// rest bins (few) come to the host for the wave tables.
// (c) on one rank: group-major shuffle (shuffle.cu) of desc_in/bin_in into ctx->desc_sorted; the
// bins' offsets (ctx->bin_off_d) and windows (ctx->hist) come out of it. tmp_* are scratch of n.
gerbil_status group_shuffle(gerbil_ctx* ctx, const uint64_t* desc_in, const uint32_t* bin_in, uint64_t n, uint32_t B,
                            uint64_t* tmp_desc, uint32_t* tmp_bin, uint64_t* desc_alt) {
  if (n >= (1ull << 32)) return fail(ctx, GERBIL_E_USAGE, "more than 2^32 super-mers in one call: split the batch");
  CK(ctx->hist.ensure(3ull * B * 8));
  CK(ctx->bin_off_d.ensure(((size_t)B + 1) * 8));
  CK(ctx->desc_sorted.ensure(std::max<uint64_t>(n, 1) * 8));
  CK(ctx->p_tmp.ensure(group_shuffle_scratch_bytes(B)));
  GroupShuffleArgs gs{};
  gs.desc_in = desc_in;
  gs.bin_in = bin_in;
  gs.n = n;
  gs.n_bins = B;
  gs.tmp_desc = tmp_desc;
  gs.tmp_bin = tmp_bin;
  gs.desc_alt = desc_alt;
  gs.desc_out = ctx->desc_sorted.as<uint64_t>();
  gs.off = ctx->bin_off_d.as<unsigned long long>();
  gs.win = ctx->hist.as<unsigned long long>();
  gs.scratch = ctx->p_tmp.as<unsigned long long>();
  const uint32_t G = group_shuffle_groups(B);
  Timer tm(ctx, K_SHUFFLE, nullptr, true, G > 64 ? 5 : 4);
  CK(launch_group_shuffle(gs, ctx->sms, ctx->stream));
  return GERBIL_OK;
}

gerbil_status count_planned(gerbil_ctx* ctx, const uint64_t* codes, uint32_t B, uint32_t cap, uint32_t k,
                            uint32_t min_count, uint64_t windows);

gerbil_status count_local_device_plan(gerbil_ctx* ctx, const uint64_t* codes, uint64_t n_sm, uint32_t B,
                                      uint32_t cap, uint32_t k, uint32_t min_count, uint64_t windows,
                                      uint64_t n_bases) {
  (void)n_bases;
  CK(ctx->send_desc.ensure(std::max<uint64_t>(n_sm, 1) * 8));  // scratch (reuses the exchange buffers)
  CK(ctx->send_bin.ensure(std::max<uint64_t>(n_sm, 1) * 4));
  CKS(group_shuffle(ctx, ctx->desc_pre.as<uint64_t>(), ctx->bin_pre.as<uint32_t>(), n_sm, B,
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->desc_pre.as<uint64_t>()));
  return count_planned(ctx, codes, B, cap, k, min_count, windows);
}

// Step (c) across ranks with the device bin plan kept (many bins, shared-memory / reference
// tables): every rank groups its super-mers by bin (group_shuffle), bins are owned in GROUPS of
// 1024 consecutive bins (4096 groups at 2^22 bins) so the plan is small: the per-group windows /
// super-mers / payload words of all ranks are all-gathered (3 x 32 KB per rank) and every rank
// derives the same greedy LPT owner map (exchange_plan over groups; PAPER.md:210's load balance,
// all occurrences of a k-mer end up on one GPU). Each rank packs its groups into
// per-destination segments (descriptor with the position already rebased into the owner's receive
// buffer, bin, re-aligned payload) and ONE grouped ncclSend/ncclRecv moves all three; the owner
// regroups what it received by bin and counts it with the device plan (count_planned).
gerbil_status exchange_groups(gerbil_ctx* ctx, const uint64_t* codes, uint64_t n_sm, uint32_t B, uint32_t cap,
                              uint32_t k, uint32_t min_count, uint64_t& owned_windows) {
  const int P = ctx->world, r = ctx->rank;
  const uint32_t G = group_shuffle_groups(B);
  CK(ctx->send_desc.ensure(std::max<uint64_t>(n_sm, 1) * 8));
  CK(ctx->send_bin.ensure(std::max<uint64_t>(n_sm, 1) * 4));
  CKS(group_shuffle(ctx, ctx->desc_pre.as<uint64_t>(), ctx->bin_pre.as<uint32_t>(), n_sm, B,
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->desc_pre.as<uint64_t>()));
  // per-group statistics of every rank
  CK(ctx->hist_all.ensure(3ull * G * 8 * (P + 1)));
  unsigned long long* gst = ctx->hist_all.as<unsigned long long>();
  unsigned long long* gall = gst + 3ull * G;
  {
    Timer tm(ctx, K_SHUFFLE);
    CK(launch_group_stats(ctx->desc_sorted.as<uint64_t>(), ctx->bin_off_d.as<unsigned long long>(), B, k, gst,
                          ctx->stream));
  }
  if (!ctx->comm->allgather(gst, gall, 3ull * G * 8, ctx->stream)) return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
  std::vector<uint64_t> H(3ull * G * P);
  CK(cudaMemcpyAsync(H.data(), gall, H.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  trace("group histograms all-gathered");
  auto Hw = [&](int s, uint32_t g) { return H[(size_t)s * 3 * G + g]; };
  auto Hc = [&](int s, uint32_t g) { return H[(size_t)s * 3 * G + G + g]; };
  auto Hp = [&](int s, uint32_t g) { return H[(size_t)s * 3 * G + 2 * G + g]; };
  std::vector<int32_t> owner(G);
  std::vector<uint64_t> sd_off(P + 1), sw_off(P + 1), rd_off(P + 1), rw_off(P + 1);
  exchange_plan(H.data(), G, P, r, owner.data(), sd_off.data(), sw_off.data(), rd_off.data(), rw_off.data());
  // this rank's data starts, in destination d's receive buffer, after the lower ranks' data
  std::vector<uint64_t> rb(P, 0);
  for (int s = 0; s < r; ++s)
    for (uint32_t g = 0; g < G; ++g) rb[owner[g]] += Hp(s, g);
  std::vector<unsigned long long> base3(3ull * G);
  {
    std::vector<uint64_t> cd(sd_off.begin(), sd_off.end() - 1), cw(sw_off.begin(), sw_off.end() - 1);
    for (uint32_t g = 0; g < G; ++g) {
      const int d = owner[g];
      base3[g] = cd[d];
      base3[G + g] = cw[d];
      base3[2ull * G + g] = rb[d] + (cw[d] - sw_off[d]);
      cd[d] += Hc(r, g);
      cw[d] += Hp(r, g);
    }
  }
  owned_windows = 0;
  uint64_t max_group = 0;
  for (uint32_t g = 0; g < G; ++g)
    if (owner[g] == r) {
      uint64_t w = 0;
      for (int s = 0; s < P; ++s) w += Hw(s, g);
      owned_windows += w;
      max_group = std::max(max_group, w);
    }
  const uint64_t n_send = sd_off[P], w_send = sw_off[P], n_recv = rd_off[P], w_recv = rw_off[P];
  CK(ctx->seg_base.ensure(3ull * G * 8));
  CK(cudaMemcpyAsync(ctx->seg_base.p, base3.data(), base3.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(ctx->send_desc.ensure(std::max<uint64_t>(std::max(n_send, n_recv), 1) * 8));
  CK(ctx->send_bin.ensure(std::max<uint64_t>(std::max(n_send, n_recv), 1) * 4));
  CK(ctx->send_payload.ensure(std::max<uint64_t>(w_send, 1) * 8));
  CK(ctx->recv_desc.ensure(std::max<uint64_t>(n_recv, 1) * 8));
  CK(ctx->recv_bin.ensure(std::max<uint64_t>(n_recv, 1) * 4));
  CK(ctx->recv_payload.ensure(std::max<uint64_t>(w_recv, 1) * 8));
  {
    Timer tm(ctx, K_SHUFFLE);
    CK(launch_group_pack(ctx->desc_sorted.as<uint64_t>(), ctx->bin_off_d.as<unsigned long long>(), B, codes, k,
                         ctx->seg_base.as<unsigned long long>(), ctx->send_desc.as<uint64_t>(),
                         ctx->send_bin.as<uint32_t>(), ctx->send_payload.as<uint64_t>(), ctx->stream));
  }
  // one grouped all-to-all: descriptors, bins and payload to every owner
  std::vector<size_t> so[3], sb[3], ro[3], rbytes[3];
  const std::vector<uint64_t>* soff[3] = {&sd_off, &sd_off, &sw_off};
  const std::vector<uint64_t>* roff[3] = {&rd_off, &rd_off, &rw_off};
  const size_t elem[3] = {8, 4, 8};
  Comm::Xfer x[3];
  void* sbuf[3] = {ctx->send_desc.p, ctx->send_bin.p, ctx->send_payload.p};
  void* rbuf[3] = {ctx->recv_desc.p, ctx->recv_bin.p, ctx->recv_payload.p};
  for (int b = 0; b < 3; ++b) {
    so[b].resize(P);
    sb[b].resize(P);
    ro[b].resize(P);
    rbytes[b].resize(P);
    for (int p = 0; p < P; ++p) {
      so[b][p] = (*soff[b])[p] * elem[b];
      sb[b][p] = ((*soff[b])[p + 1] - (*soff[b])[p]) * elem[b];
      ro[b][p] = (*roff[b])[p] * elem[b];
      rbytes[b][p] = ((*roff[b])[p + 1] - (*roff[b])[p]) * elem[b];
    }
    x[b] = Comm::Xfer{sbuf[b], so[b].data(), sb[b].data(), rbuf[b], ro[b].data(), rbytes[b].data()};
  }
  {
    Timer tm(ctx, K_SHUFFLE);
    if (!ctx->comm->alltoallv_multi(x, 3, ctx->stream)) return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
  }
  trace("groups exchanged");
  ctx->stats.bytes_sent = (n_send - (sd_off[r + 1] - sd_off[r])) * 12 + (w_send - (sw_off[r + 1] - sw_off[r])) * 8;
  ctx->stats.bytes_recv = (n_recv - (rd_off[r + 1] - rd_off[r])) * 12 + (w_recv - (rw_off[r + 1] - rw_off[r])) * 8;
  // regroup what this rank owns by bin, then count it
  CKS(group_shuffle(ctx, ctx->recv_desc.as<uint64_t>(), ctx->recv_bin.as<uint32_t>(), n_recv, B,
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->recv_desc.as<uint64_t>()));
  return count_planned(ctx, ctx->recv_payload.as<uint64_t>(), B, cap, k, min_count, owned_windows);
}

// Steps (d)+(e) over ctx->desc_sorted with the bins' offsets / windows on the device (after
// group_shuffle): the device bin plan, shared-memory (or reference) tables, then the L2 waves.
gerbil_status count_planned(gerbil_ctx* ctx, const uint64_t* codes, uint32_t B, uint32_t cap, uint32_t k,
                            uint32_t min_count, uint64_t windows) {
  ctx->stats.smem_slots = cap;
  unsigned long long* d_win = ctx->hist.as<unsigned long long>();
  unsigned long long* d_off = ctx->bin_off_d.as<unsigned long long>();
  trace("scatter issued");
  const uint32_t max_fill = smem_max_fill(cap, k);
  CK(ctx->smem_range.ensure((size_t)B * 16));
  CK(ctx->rest_range.ensure((size_t)B * 24));
  CK(ctx->plan_sums.ensure(5 * 8));
  CK(cudaMemsetAsync(ctx->plan_sums.p, 0, 5 * 8, ctx->stream));
  PlanBinsArgs pa{};
  pa.win = d_win;
  pa.off = d_off;
  pa.n_bins = B;
  pa.thr = smem_window_threshold(ctx, max_fill);
  pa.max_fill = max_fill;
  pa.cap = cap;
  pa.elig = ctx->smem_range.as<unsigned long long>();
  pa.rest = ctx->rest_range.as<unsigned long long>();
  pa.sums = ctx->plan_sums.as<unsigned long long>();
  pa.max_win = pa.sums + 4;
  {
    Timer tm(ctx, K_SHUFFLE);
    CK(launch_plan_bins(pa, ctx->sms, ctx->stream));
  }
  unsigned long long sums[5];
  CK(cudaMemcpyAsync(sums, pa.sums, sizeof sums, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const uint64_t n_elig = sums[0], n_rest = sums[3];
  ctx->stats.max_bin_windows = sums[4];
  std::vector<RestBin> rest(n_rest);
  if (n_rest) {
    static_assert(sizeof(RestBin) == 24, "RestBin mirrors the device rest triples");
    CK(cudaMemcpyAsync(rest.data(), pa.rest, n_rest * 24, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  trace("bins planned on the device");
  if (n_elig == 0) {
    // nothing for shared memory: the wave tables take every bin
    std::vector<uint64_t> off2(n_rest + 1, 0), win2(n_rest);
    std::vector<uint32_t> list2(n_rest);
    std::sort(rest.begin(), rest.end(), [](const RestBin& x, const RestBin& y) { return x.d0 < y.d0; });
    // bins are consecutive in desc_sorted (all of them are rest bins): no gather needed
    for (uint64_t i = 0; i < n_rest; ++i) {
      off2[i] = rest[i].d0;
      off2[i + 1] = rest[i].d1;
      win2[i] = rest[i].win;
      list2[i] = (uint32_t)i;
    }
    return count_waves_l2(ctx, codes, ctx->desc_sorted.as<uint64_t>(), off2, win2, list2, k, min_count, windows,
                          Preset{});
  }
  return count_waves_ranges(ctx, codes, ctx->desc_sorted.as<uint64_t>(), (uint32_t)n_elig, sums[1], sums[2], cap,
                            max_fill, rest, k, min_count, windows);
}

// ---------------------------------------------------------------------------
// dfp(p) key table (reading Q23): sample m-mer
// frequencies on the device (all ranks' samples summed), sort by (frequency,
// A<C<G<T number), key = signed distance of the position from P = p·4^m.
gerbil_status build_dfp_table(gerbil_ctx* ctx, const SupermerArgs& a, uint64_t n_bases, uint32_t m) {
  const uint64_t M = 1ull << (2 * m);
  CK(ctx->rs_bits.ensure(supermer_scratch_words(n_bases) * 8));
  CK(ctx->order_freq.ensure(M * 4 * (ctx->comm ? ctx->world + 1 : 1)));
  CK(ctx->order_rank.ensure(M * 4));
  uint64_t* rs = ctx->rs_bits.as<uint64_t>();
  uint32_t* freq = ctx->order_freq.as<uint32_t>();
  CK(cudaMemsetAsync(freq, 0, M * 4, ctx->stream));
  if (n_bases > 0) {
    Timer tm(ctx, K_SUPERMER, nullptr, true, a.n_reads ? 2u : 1u);
    CK(supermer_prepare(a, rs, ctx->stream));
    CK(supermer_mark_reads(a, rs, 0, a.n_reads, ctx->sms, ctx->stream));
    CK(launch_dfp_sample(a.codes, a.nmask, rs, n_bases, m, ctx->cfg.order_sample_stride, freq, ctx->sms,
                         ctx->stream));
  }
  std::vector<uint64_t> f(M, 0);
  if (ctx->comm) {  // every rank must build the same table: sum all ranks' samples
    uint32_t* all = freq + M;
    if (!ctx->comm->allgather(freq, all, M * 4, ctx->stream)) return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
    std::vector<uint32_t> h(M * ctx->world);
    CK(cudaMemcpyAsync(h.data(), all, h.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < ctx->world; ++r)
      for (uint64_t v = 0; v < M; ++v) f[v] += h[(size_t)r * M + v];
  } else {
    std::vector<uint32_t> h(M);
    CK(cudaMemcpyAsync(h.data(), freq, M * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint64_t v = 0; v < M; ++v) f[v] = h[v];
  }
  std::vector<uint32_t> order(M);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return f[x] != f[y] ? f[x] < f[y] : x < y; });
  // re-sort by |position - 4^m p| (the real pivot; p * 4^m is exact in double), ties to the
  // smaller position (Q23); the key is the rank in that order
  const double x = ctx->cfg.dfp_pivot * (double)M;
  std::vector<uint32_t> bypiv(M);
  std::iota(bypiv.begin(), bypiv.end(), 0u);
  std::sort(bypiv.begin(), bypiv.end(), [&](uint32_t a, uint32_t b) {
    const double da = std::fabs((double)a - x), db = std::fabs((double)b - x);
    return da != db ? da < db : a < b;
  });
  std::vector<uint32_t> key(M);
  for (uint64_t r = 0; r < M; ++r) key[order[bypiv[r]]] = (uint32_t)r;
  CK(cudaMemcpyAsync(ctx->order_rank.p, key.data(), M * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // key is a host temporary
  return GERBIL_OK;
}

// ---------------------------------------------------------------------------
gerbil_status run_supermer(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                           const uint64_t* rstart, uint64_t n_reads, uint64_t n_bases, uint32_t k,
                           uint32_t m, uint32_t B, bool want_mu, uint64_t& n_sm, bool want_hist = true) {
  const uint32_t w = k - m + 1;
  uint64_t cap = (uint64_t)((double)n_bases * 2.0 / (w + 1) * 1.3) + (n_bases / kTile + 1) * 4 + 1024;
  Counters* dc = ctx->counters.as<Counters>();
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK(ctx->desc_pre.ensure(cap * 8));
    CK(ctx->bin_pre.ensure(cap * 4));
    if (want_mu) CK(ctx->mu_dbg.ensure(cap * 4));
    CK(cudaMemsetAsync(dc, 0, sizeof(Counters), ctx->stream));
    if (want_hist) CK(cudaMemsetAsync(ctx->hist.p, 0, 3ull * B * 8, ctx->stream));
    SupermerArgs a{};
    a.codes = codes;
    a.nmask = nmask;
    a.read_start = rstart;
    a.n_reads = n_reads;
    a.n_bases = n_bases;
    a.k = k;
    a.m = m;
    a.n_bins = B;
    a.ordering = (uint32_t)ctx->cfg.ordering;
    a.desc = ctx->desc_pre.as<uint64_t>();
    a.bin = ctx->bin_pre.as<uint32_t>();
    a.mu = want_mu ? ctx->mu_dbg.as<uint32_t>() : nullptr;
    a.cap = cap;
    a.n_supermers = &dc->n_supermers;
    a.n_windows = &dc->n_windows;
    unsigned long long* h = ctx->hist.as<unsigned long long>();
    a.bin_windows = want_hist ? h : nullptr;
    a.bin_supermers = want_hist ? h + B : nullptr;
    a.bin_words = (want_hist && (ctx->comm || ctx->want_words)) ? h + 2 * B : nullptr;
    const UploadPlan* up = ctx->upload;
    a.order_rank = nullptr;
    if (ctx->cfg.ordering == GERBIL_ORDER_DFP) {
      // dfp(p) needs the sampled frequencies before any minimizer: the whole
      // batch must be resident (no chunk overlap for this ordering)
      if (up)
        for (cudaEvent_t ev : up->ev) CK(cudaStreamWaitEvent(ctx->stream, ev, 0));
      up = nullptr;
      CKS(build_dfp_table(ctx, a, n_bases, m));
      a.order_rank = ctx->order_rank.as<uint32_t>();
    }
    if (use_reads_kernel(k, m, n_bases, n_reads)) {
      if (up)
        for (cudaEvent_t ev : up->ev) CK(cudaStreamWaitEvent(ctx->stream, ev, 0));
      Timer tm(ctx, K_SUPERMER);
      CK(launch_supermer_reads(a, &dc->read_work, ctx->sms, ctx->stream));
    } else if (up) {
      // chunked upload: mark each chunk's reads and run the tiles it completes
      // as soon as it lands, so step (b) runs behind the H2D copies
      CK(ctx->rs_bits.ensure(supermer_scratch_words(n_bases) * 8));
      uint64_t* rs = ctx->rs_bits.as<uint64_t>();
      const uint64_t n_tiles = supermer_tile_count(n_bases), reach = supermer_tile_reach();
      Timer tm(ctx, K_SUPERMER, nullptr, true, 0);
      CK(supermer_prepare(a, rs, ctx->stream));
      uint64_t r0 = 0, t0 = 0;
      for (size_t c = 0; c < up->ev.size(); ++c) {
        CK(cudaStreamWaitEvent(ctx->stream, up->ev[c], 0));
        const uint64_t r1 = up->read_end[c];
        if (r1 > r0) {
          CK(supermer_mark_reads(a, rs, r0, r1, ctx->sms, ctx->stream));
          ctx->n_launch[K_SUPERMER]++;
        }
        r0 = std::max(r0, r1);
        const bool last = c + 1 == up->ev.size();
        const uint64_t be = up->base_end[c];
        uint64_t t1 = last ? n_tiles : (be >= reach ? std::min(n_tiles, (be - reach) / 1024 + 1) : 0);
        t1 = std::max(t1, t0);
        if (t1 > t0) {
          CK(supermer_run_tiles(a, rs, t0, t1, ctx->sms, ctx->stream));
          ctx->n_launch[K_SUPERMER]++;
        }
        t0 = t1;
      }
    } else {
      CK(ctx->rs_bits.ensure(supermer_scratch_words(n_bases) * 8));
      Timer tm(ctx, K_SUPERMER, nullptr, true, n_reads ? 2u : 1u);  // rs_bits_kernel + supermer_kernel
      CK(launch_supermer(a, ctx->rs_bits.as<uint64_t>(), ctx->sms, ctx->stream));
    }
    CK(cudaMemcpyAsync(ctx->h_counters, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    n_sm = ctx->h_counters->n_supermers;
    if (n_sm <= cap) return GERBIL_OK;
    cap = n_sm + 1024;
  }
  return fail(ctx, GERBIL_E_INTERNAL, "super-mer buffer sizing did not converge");
}

// per-call timing/launch bookkeeping reset (before any timed work of the call)
void begin_call(gerbil_ctx* ctx) {
  ctx->evs.clear();
  ctx->ev_used = 0;
  for (auto& v : ctx->n_launch) v = 0;
}

gerbil_status count_device_impl(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                uint32_t min_count, bool fresh = true) {
  const double t0 = wall_ms();
  ctx->have_result = false;
  ctx->results_sorted = false;
  ctx->n_out = 0;
  if (fresh) begin_call(ctx);
  memset(&ctx->stats, 0, sizeof ctx->stats);
  const uint32_t W = key_words(k);
  ctx->W = W;
  ctx->k = k;
  ctx->m = m;
  uint64_t n_bases = 0;
  if (ctx->upload) {
    n_bases = ctx->upload->n_bases;  // host batch: known without waiting for the upload
  } else if (n_reads > 0) {
    CK(cudaMemcpyAsync(&ctx->h_counters->probe[3], rstart + n_reads, 8, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    n_bases = ctx->h_counters->probe[3];
  }
  // all ranks must agree on B: it is derived from the job's totals (all-gathered sizes)
  uint64_t tot_bases = n_bases, tot_reads = n_reads;
  if (ctx->comm && ctx->cfg.n_bins == 0) {
    CK(ctx->plan_sums.ensure(2ull * 8 * (ctx->world + 1)));
    uint64_t* sz = ctx->plan_sums.as<uint64_t>();
    ctx->h_counters->probe[0] = n_bases;
    ctx->h_counters->probe[1] = n_reads;
    CK(cudaMemcpyAsync(sz, ctx->h_counters->probe, 16, cudaMemcpyHostToDevice, ctx->stream));
    if (!ctx->comm->allgather(sz, sz + 2, 16, ctx->stream)) return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
    std::vector<uint64_t> all(2ull * ctx->world);
    CK(cudaMemcpyAsync(all.data(), sz + 2, all.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    tot_bases = tot_reads = 0;
    for (int p = 0; p < ctx->world; ++p) {
      tot_bases += all[2 * p];
      tot_reads += all[2 * p + 1];
    }
  }
  const uint32_t B = choose_bins(ctx, tot_bases, tot_reads, W, k, m);
  CK(ctx->counters.ensure(sizeof(Counters)));
  CK(ctx->hist.ensure(3ull * B * 8));
  ctx->stats.n_bins = B;
  ctx->stats.W = W;
  ctx->stats.input_bases = n_bases;
  ctx->stats.input_reads = n_reads;

  // the device-planned path (many bins) groups super-mers with the group-major shuffle, which
  // derives the bin histogram itself: step (b) then skips it. With world > 1 whole groups of
  // bins are exchanged (exchange_groups) and each owner plans its bins on the device.
  const uint64_t pos_lim = key_words(k) >= 4 ? (1ull << 39) : (1ull << 43);
  const uint32_t smem_cap = (!ctx->rec_out && B >= kDevicePlanBins && B <= (1u << 22) && n_bases < pos_lim &&
                             (!ctx->comm || tot_bases < pos_lim))
                                ? smem_slots_for(ctx, k)
                                : 0u;
  // (b)
  uint64_t n_sm = 0;
  trace("supermer issue");
  CKS(run_supermer(ctx, codes, nmask, rstart, n_reads, n_bases, k, m, B, false, n_sm, smem_cap == 0));
  trace("supermer done (synced)");
  const uint64_t local_windows = ctx->h_counters->n_windows;
  ctx->stats.supermers = n_sm;
  ctx->stats.valid_windows = local_windows;
  uint64_t owned_windows = 0;
  if (smem_cap && ctx->comm) {
    // many bins, several ranks: groups of bins exchanged, then planned on the device by the owner
    CKS(exchange_groups(ctx, codes, n_sm, B, smem_cap, k, min_count, owned_windows));
  } else if (smem_cap) {
    // many bins, one rank: steps (c)-(e) planned on the device (no per-bin host work)
    CKS(count_local_device_plan(ctx, codes, n_sm, B, smem_cap, k, min_count, local_windows, n_bases));
    owned_windows = local_windows;
  } else {
  CK(ctx->h_hist.ensure(3ull * B * 8));
  const unsigned long long* hist = ctx->h_hist.as<unsigned long long>();
  CK(cudaMemcpyAsync(ctx->h_hist.p, ctx->hist.p, 3ull * B * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  trace("histogram downloaded");

  std::vector<uint64_t> bin_win(B), bin_off(B + 1, 0);
  std::vector<uint32_t> owned;
  owned.reserve(B);
  const uint64_t* stream_codes = codes;
  if (!ctx->comm) {
    // (c) local: group descriptors by bin
    for (uint32_t b = 0; b < B; ++b) {
      bin_win[b] = hist[b];
      bin_off[b + 1] = bin_off[b] + hist[B + b];
      owned.push_back(b);
      owned_windows += hist[b];
    }
    ctx->stats.max_bin_windows = *std::max_element(bin_win.begin(), bin_win.end());
    CK(ctx->desc_sorted.ensure(std::max<uint64_t>(n_sm, 1) * 8));
    CK(ctx->cursor.ensure((size_t)B * 8));
    CK(cudaMemcpyAsync(ctx->cursor.p, bin_off.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    ScatterArgs s{};
    s.desc_in = ctx->desc_pre.as<uint64_t>();
    s.bin_in = ctx->bin_pre.as<uint32_t>();
    s.n = n_sm;
    s.n_bins = B;
    s.cursor = ctx->cursor.as<unsigned long long>();
    s.desc_out = ctx->desc_sorted.as<uint64_t>();
    {
      Timer tm(ctx, K_SHUFFLE);
      CK(launch_scatter(s, ctx->sms, ctx->stream));
    }
  } else {
    // (c) multi-GPU: all-gather histograms, LPT owners, pack, all-to-all, regroup
    const int P = ctx->world, r = ctx->rank;
    CK(ctx->hist_all.ensure(3ull * B * 8 * P));
    if (!ctx->comm->allgather(ctx->hist.p, ctx->hist_all.p, 3ull * B * 8, ctx->stream))
      return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
    std::vector<unsigned long long> H(3ull * B * P);
    CK(cudaMemcpyAsync(H.data(), ctx->hist_all.p, H.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    auto Hw = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + b]; };
    auto Hc = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + B + b]; };
    auto Hp = [&](int s, uint32_t b) { return H[(size_t)s * 3 * B + 2 * B + b]; };
    std::vector<uint64_t> gw(B, 0);
    for (int s = 0; s < P; ++s)
      for (uint32_t b = 0; b < B; ++b) gw[b] += Hw(s, b);
    ctx->stats.max_bin_windows = *std::max_element(gw.begin(), gw.end());
    // LPT owners and the send / receive layouts (exchange_plan, also gerbil_exchange_plan)
    std::vector<int32_t> owner(B);
    std::vector<uint64_t> sd_off(P + 1, 0), sw_off(P + 1, 0), rd_off(P + 1, 0), rw_off(P + 1, 0);
    exchange_plan(reinterpret_cast<const uint64_t*>(H.data()), B, P, r, owner.data(), sd_off.data(),
                  sw_off.data(), rd_off.data(), rw_off.data());
    // per-bin send cursors: inside a destination's range, bins in increasing order
    std::vector<unsigned long long> cur_d(B), cur_w(B), seg(B);
    {
      std::vector<uint64_t> cd(sd_off.begin(), sd_off.end() - 1), cw(sw_off.begin(), sw_off.end() - 1);
      for (uint32_t b = 0; b < B; ++b) {
        const int d = owner[b];
        cur_d[b] = cd[d];
        cur_w[b] = cw[d];
        seg[b] = sw_off[d];
        cd[d] += Hc(r, b);
        cw[d] += Hp(r, b);
      }
    }
    const uint64_t n_send = sd_off[P], w_send = sw_off[P], n_recv = rd_off[P], w_recv = rw_off[P];
    CK(ctx->send_desc.ensure(std::max<uint64_t>(n_send, 1) * 8));
    CK(ctx->send_bin.ensure(std::max<uint64_t>(n_send, 1) * 4));
    CK(ctx->send_payload.ensure(std::max<uint64_t>(w_send, 1) * 8));
    CK(ctx->recv_desc.ensure(std::max<uint64_t>(n_recv, 1) * 8));
    CK(ctx->recv_bin.ensure(std::max<uint64_t>(n_recv, 1) * 4));
    CK(ctx->recv_payload.ensure(std::max<uint64_t>(w_recv, 1) * 8));
    CK(ctx->cursor.ensure((size_t)B * 8));
    CK(ctx->cursor2.ensure((size_t)B * 8));
    CK(ctx->seg_base.ensure((size_t)B * 8));
    CK(cudaMemcpyAsync(ctx->cursor.p, cur_d.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->cursor2.p, cur_w.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->seg_base.p, seg.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    PackArgs pa{};
    pa.desc_in = ctx->desc_pre.as<uint64_t>();
    pa.bin_in = ctx->bin_pre.as<uint32_t>();
    pa.n = n_sm;
    pa.codes = codes;
    pa.k = k;
    pa.cur_desc = ctx->cursor.as<unsigned long long>();
    pa.cur_words = ctx->cursor2.as<unsigned long long>();
    pa.seg_word_base = ctx->seg_base.as<unsigned long long>();
    pa.send_desc = ctx->send_desc.as<uint64_t>();
    pa.send_bin = ctx->send_bin.as<uint32_t>();
    pa.send_payload = ctx->send_payload.as<uint64_t>();
    {
      Timer tm(ctx, K_SHUFFLE);
      CK(launch_pack(pa, ctx->sms, ctx->stream));
    }
    std::vector<size_t> so(P), sb(P), ro(P), rb(P);
    auto xchg = [&](const DevBuf& sbuf, const std::vector<uint64_t>& soff, DevBuf& rbuf,
                    const std::vector<uint64_t>& roff, size_t elem) {
      for (int p = 0; p < P; ++p) {
        so[p] = soff[p] * elem;
        sb[p] = (soff[p + 1] - soff[p]) * elem;
        ro[p] = roff[p] * elem;
        rb[p] = (roff[p + 1] - roff[p]) * elem;
      }
      return ctx->comm->alltoallv(sbuf.p, so.data(), sb.data(), rbuf.p, ro.data(), rb.data(), ctx->stream);
    };
    CK(cudaStreamSynchronize(ctx->stream));
    if (!xchg(ctx->send_desc, sd_off, ctx->recv_desc, rd_off, 8) ||
        !xchg(ctx->send_bin, sd_off, ctx->recv_bin, rd_off, 4) ||
        !xchg(ctx->send_payload, sw_off, ctx->recv_payload, rw_off, 8))
      return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
    ctx->stats.bytes_sent = (n_send - (sd_off[r + 1] - sd_off[r])) * 12 + (w_send - (sw_off[r + 1] - sw_off[r])) * 8;
    ctx->stats.bytes_recv = (n_recv - (rd_off[r + 1] - rd_off[r])) * 12 + (w_recv - (rw_off[r + 1] - rw_off[r])) * 8;
    // regroup received descriptors by bin, rebasing pos into recv_payload
    for (uint32_t b = 0; b < B; ++b) {
      uint64_t c = 0, wv = 0;
      if (owner[b] == r)
        for (int s = 0; s < P; ++s) {
          c += Hc(s, b);
          wv += Hw(s, b);
        }
      bin_off[b + 1] = bin_off[b] + c;
      bin_win[b] = wv;
      if (owner[b] == r) {
        owned.push_back(b);
        owned_windows += wv;
      }
    }
    CK(ctx->desc_sorted.ensure(std::max<uint64_t>(n_recv, 1) * 8));
    CK(cudaMemcpyAsync(ctx->cursor.p, bin_off.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (int s = 0; s < P; ++s) {
      ScatterArgs sa{};
      sa.desc_in = ctx->recv_desc.as<uint64_t>() + rd_off[s];
      sa.bin_in = ctx->recv_bin.as<uint32_t>() + rd_off[s];
      sa.n = rd_off[s + 1] - rd_off[s];
      sa.n_bins = B;
      sa.cursor = ctx->cursor.as<unsigned long long>();
      sa.desc_out = ctx->desc_sorted.as<uint64_t>();
      sa.pos_add = rw_off[s] * 32;
      Timer tm(ctx, K_SHUFFLE);
      CK(launch_scatter(sa, ctx->sms, ctx->stream));
    }
    stream_codes = ctx->recv_payload.as<uint64_t>();
  }

  // (d) + (e)
  trace("scatter issued");
  CKS(count_waves(ctx, stream_codes, ctx->desc_sorted.as<uint64_t>(), bin_off, bin_win, owned, k,
                  min_count, owned_windows));
  }
  // Σ-count invariant: every valid window counted exactly once
  if (ctx->stats.count_sum != owned_windows)
    return fail(ctx, GERBIL_E_INTERNAL,
                "invariant violated: sum of counts " + std::to_string(ctx->stats.count_sum) +
                    " != valid windows " + std::to_string(owned_windows));
  // timing
  if (ctx->cfg.timing) {
    double ms[K_NKIND] = {0};
    for (auto& e : ctx->evs) {
      float f = 0;
      cudaEventElapsedTime(&f, e.a, e.b);
      ms[e.kind] += f;
    }
    ctx->stats.ms_h2d = ms[K_H2D];
    ctx->stats.ms_supermer = ms[K_SUPERMER];
    ctx->stats.ms_shuffle = ms[K_SHUFFLE];
    ctx->stats.ms_count = ms[K_COUNT] + ms[K_SMEM];
    ctx->stats.ms_smem = ms[K_SMEM];
    ctx->stats.ms_compact = ms[K_COMPACT];
    ctx->stats.ms_overflow = ms[K_OVERFLOW];
  }
  // kernel launches of this call (copies are not launches)
  ctx->stats.launches_count = ctx->n_launch[K_COUNT] + ctx->n_launch[K_SMEM];
  ctx->stats.launches_smem = ctx->n_launch[K_SMEM];
  ctx->stats.launches_compact = ctx->n_launch[K_COMPACT];
  ctx->stats.launches_total = ctx->n_launch[K_SUPERMER] + ctx->n_launch[K_SHUFFLE] + ctx->n_launch[K_COUNT] +
                              ctx->n_launch[K_COMPACT] + ctx->n_launch[K_OVERFLOW] + ctx->n_launch[K_SMEM];
  ctx->stats.ms_total = wall_ms() - t0;
  ctx->have_result = true;
  return GERBIL_OK;
}

}  // namespace

// ============================================================== C ABI =====
extern "C" {

void gerbil_config_default(gerbil_config* cfg) {
  memset(cfg, 0, sizeof *cfg);
  cfg->struct_size = sizeof *cfg;
  cfg->device = -1;
  cfg->world = 1;
  cfg->dfp_pivot = 0.5;
}

gerbil_status gerbil_nccl_unique_id(void* id_out, size_t id_len) {
  if (!id_out || id_len < 128) return GERBIL_E_USAGE;
  std::string err;
  return nccl_get_unique_id(id_out, err) ? GERBIL_OK : GERBIL_E_NCCL;
}

gerbil_status gerbil_init(const gerbil_config* cfg_in, gerbil_ctx** out) {
  if (!cfg_in || !out) return GERBIL_E_USAGE;
  *out = nullptr;
  gerbil_config cfg;
  gerbil_config_default(&cfg);
  memcpy(&cfg, cfg_in, std::min<size_t>(cfg_in->struct_size ? cfg_in->struct_size : sizeof cfg, sizeof cfg));
  cfg.struct_size = sizeof cfg;
  if (cfg.world < 1) cfg.world = 1;
  if (cfg.rank < 0 || cfg.rank >= cfg.world) return GERBIL_E_USAGE;
  if (cfg.ordering < 0 || cfg.ordering > GERBIL_ORDER_DFP) return GERBIL_E_USAGE;
  if (!(cfg.dfp_pivot >= 0.0 && cfg.dfp_pivot <= 1.0)) return GERBIL_E_USAGE;
  if (cfg.order_sample_stride == 0) cfg.order_sample_stride = 16;
  if (cfg.world > 1 && !cfg.nccl_unique_id) return GERBIL_E_USAGE;
  if (cfg.n_bins > (1u << 22)) return GERBIL_E_USAGE;
  if (cfg.max_probes == 0) cfg.max_probes = 32;
  if (cfg.target_load <= 0) cfg.target_load = 0.7;
  if (cfg.target_load > 4.0) return GERBIL_E_USAGE;
  if (cfg.distinct_ratio < 0 || cfg.distinct_ratio > 1) return GERBIL_E_USAGE;
  if (cfg.wave_table_bytes == 0) cfg.wave_table_bytes = 128ull << 20;
  gerbil_ctx* ctx = new gerbil_ctx();
  ctx->cfg = cfg;
  ctx->rho = cfg.distinct_ratio > 0 ? cfg.distinct_ratio : 0.5;
  ctx->rank = cfg.rank;
  ctx->world = cfg.world;
  cudaError_t e = cudaSuccess;
  if (cfg.device >= 0) e = cudaSetDevice(cfg.device);
  if (e == cudaSuccess) e = cudaGetDevice(&ctx->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (e == cudaSuccess) {
    if (cfg.stream) {
      ctx->stream = (cudaStream_t)cfg.stream;
    } else {
      e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
      ctx->own_stream = true;
    }
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->lane_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->pcie_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocHost((void**)&ctx->h_counters, sizeof(Counters));
  if (e != cudaSuccess) {
    delete ctx;
    return GERBIL_E_CUDA;
  }
  if (cfg.world > 1 || cfg.force_exchange) {
    std::string err;
    unsigned char own_id[128] = {0};
    const void* id = cfg.nccl_unique_id;
    if (!id) {  // world == 1 with force_exchange: a private 1-rank group
      if (cfg.comm_backend == 0 && !nccl_get_unique_id(own_id, err)) {
        gerbil_finalize(ctx);
        return GERBIL_E_NCCL;
      }
      if (cfg.comm_backend != 0) snprintf((char*)own_id, sizeof own_id, "gerbil-self-%p", (void*)ctx);
      id = own_id;
    }
    ctx->comm = make_comm(cfg.comm_backend, id, cfg.rank, cfg.world, err);
    if (!ctx->comm) {
      gerbil_finalize(ctx);
      return GERBIL_E_NCCL;
    }
  }
  *out = ctx;
  return GERBIL_OK;
}

void gerbil_finalize(gerbil_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  delete ctx->comm;
  ctx->spill.release();
  ctx->spill.pool.clear();
  if (ctx->lane_stream) {
    cudaStreamSynchronize(ctx->lane_stream);
    cudaStreamDestroy(ctx->lane_stream);
  }
  if (ctx->pcie_stream) {
    cudaStreamSynchronize(ctx->pcie_stream);
    cudaStreamDestroy(ctx->pcie_stream);
  }
  for (auto ev : ctx->wave_ev) cudaEventDestroy(ev);
  for (auto ev : ctx->chunk_ev) cudaEventDestroy(ev);
  if (ctx->h_snap) cudaFreeHost(ctx->h_snap);
  if (ctx->fork_ev) cudaEventDestroy(ctx->fork_ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* gerbil_last_error(const gerbil_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

gerbil_status gerbil_exchange_plan(const uint64_t* hist, uint32_t n_bins, int32_t world, int32_t rank,
                                   int32_t* owner, uint64_t* send_desc_off, uint64_t* send_word_off,
                                   uint64_t* recv_desc_off, uint64_t* recv_word_off) {
  if (!hist || !owner || !send_desc_off || !send_word_off || !recv_desc_off || !recv_word_off || world < 1 ||
      rank < 0 || rank >= world || n_bins == 0)
    return GERBIL_E_USAGE;
  try {
    exchange_plan(hist, n_bins, world, rank, owner, send_desc_off, send_word_off, recv_desc_off, recv_word_off);
  } catch (...) {
    return GERBIL_E_NOMEM;
  }
  return GERBIL_OK;
}

gerbil_status gerbil_get_stats(const gerbil_ctx* ctx, gerbil_stats* out) {
  if (!ctx || !out) return GERBIL_E_USAGE;
  *out = ctx->stats;
  return GERBIL_OK;
}

gerbil_status gerbil_count_device(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                  const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                  uint32_t min_count) {
  CKS(validate(ctx, k, m, min_count));
  if (n_reads > 0 && (!codes || !rstart)) return fail(ctx, GERBIL_E_USAGE, "null device buffer");
  if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GERBIL_E_CUDA, "cudaSetDevice");
  return count_device_impl(ctx, codes, nmask, rstart, n_reads, k, m, min_count);
}

// Uploads a host packed batch into ctx->in_* in chunks on the copy stream
// (64-base-word boundaries); step (b) consumes each chunk as it lands
// (run_supermer with ctx->upload = &plan). GERBIL_UPLOAD_CHUNKS overrides the
// chunk count (tests force several chunks on small inputs).
gerbil_status upload_batch(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask, const uint64_t* rstart,
                           uint64_t n_reads, UploadPlan& plan) {
  const uint64_t nb = rstart[n_reads];
  const uint64_t ncw = std::max<uint64_t>((nb + 31) / 32, 1), nmw = std::max<uint64_t>((nb + 63) / 64, 1);
  CK(ctx->in_codes.ensure(ncw * 8));
  CK(ctx->in_nmask.ensure(nmw * 8));
  CK(ctx->in_rstart.ensure((n_reads + 1) * 8));
  // Upload in chunks on the copy stream (64-base-word boundaries); step (b)
  // consumes each chunk as it lands (run_supermer). GERBIL_UPLOAD_CHUNKS
  // overrides the count (tests force several chunks on small inputs).
  uint64_t nch = std::min<uint64_t>(16, std::max<uint64_t>(1, nb >> 26));
  if (const char* e = getenv("GERBIL_UPLOAD_CHUNKS"))
    if (*e) nch = std::max<uint64_t>(1, std::min<uint64_t>(strtoull(e, nullptr, 10), std::max<uint64_t>(nmw, 1)));
  plan.n_bases = nb;
  while (ctx->chunk_ev.size() < nch) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->chunk_ev.push_back(ev);
  }
  // the copies may start only after earlier work on the main stream (a
  // previous call still reading these buffers)
  CK(cudaEventRecord(ctx->fork_ev, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->pcie_stream, ctx->fork_ev, 0));
  {
    Timer tm(ctx, K_H2D, ctx->pcie_stream, true, 0);
    uint64_t w0 = 0, r0 = 0;
    for (uint64_t c = 0; c < nch; ++c) {
      const bool last = c + 1 == nch;
      const uint64_t w1 = last ? nmw : (c + 1) * nmw / nch;  // N-mask words [w0, w1)
      const uint64_t be = std::min<uint64_t>(w1 * 64, nb);
      const uint64_t cw0 = std::min<uint64_t>(2 * w0, (nb + 31) / 32), cw1 = std::min<uint64_t>(2 * w1, (nb + 31) / 32);
      const uint64_t r1 = last ? n_reads : (uint64_t)(std::lower_bound(rstart, rstart + n_reads, be) - rstart);
      if (cw1 > cw0)
        CK(cudaMemcpyAsync(ctx->in_codes.as<uint64_t>() + cw0, codes + cw0, (cw1 - cw0) * 8,
                           cudaMemcpyHostToDevice, ctx->pcie_stream));
      if (nmask && nb > 0 && w1 > w0)
        CK(cudaMemcpyAsync(ctx->in_nmask.as<uint64_t>() + w0, nmask + w0, (w1 - w0) * 8, cudaMemcpyHostToDevice,
                           ctx->pcie_stream));
      const uint64_t rs0 = c == 0 ? 0 : r0 + 1;  // read_start[r0] came with the previous chunk
      if (r1 + 1 > rs0)
        CK(cudaMemcpyAsync(ctx->in_rstart.as<uint64_t>() + rs0, rstart + rs0, (r1 + 1 - rs0) * 8,
                           cudaMemcpyHostToDevice, ctx->pcie_stream));
      CK(cudaEventRecord(ctx->chunk_ev[c], ctx->pcie_stream));
      plan.base_end.push_back(be);
      plan.read_end.push_back(r1);
      plan.ev.push_back(ctx->chunk_ev[c]);
      w0 = w1;
      r0 = r1;
    }
  }
  return GERBIL_OK;
}

gerbil_status gerbil_count_host_packed(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                       const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                       uint32_t min_count) {
  CKS(validate(ctx, k, m, min_count));
  if (!rstart) return fail(ctx, GERBIL_E_USAGE, "null host buffer");
  CK(cudaSetDevice(ctx->device));
  const uint64_t nb = rstart[n_reads];
  if (nb > 0 && !codes) return fail(ctx, GERBIL_E_USAGE, "null host buffer");
  trace("call");
  begin_call(ctx);
  UploadPlan plan;
  CKS(upload_batch(ctx, codes, nmask, rstart, n_reads, plan));
  ctx->upload = &plan;
  const gerbil_status st =
      count_device_impl(ctx, ctx->in_codes.as<uint64_t>(), nmask ? ctx->in_nmask.as<uint64_t>() : nullptr,
                        ctx->in_rstart.as<uint64_t>(), n_reads, k, m, min_count, false);
  ctx->upload = nullptr;
  // every chunk event has been waited on by the main stream unless the call
  // failed early; make sure no copy outlives the call
  if (st != GERBIL_OK) cudaStreamSynchronize(ctx->pcie_stream);
  return st;
}

gerbil_status gerbil_count_host_stream(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                       const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                       uint32_t min_count, uint8_t* out, uint64_t capacity, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return GERBIL_E_USAGE;
  *n_bytes = 0;
  if (capacity > 0) {
    if (!out) return fail(ctx, GERBIL_E_USAGE, "null output buffer");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, out) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return fail(ctx, GERBIL_E_USAGE, "output buffer must be page-locked host memory (cudaHostAlloc/Register)");
    }
  }
  // a dummy sink keeps the encoder on when capacity == 0 (sizing call: nothing is copied)
  ctx->rec_out = capacity > 0 ? out : reinterpret_cast<uint8_t*>(1);
  ctx->rec_cap = capacity;
  ctx->rec_base = 0;
  const gerbil_status st = gerbil_count_host_packed(ctx, codes, nmask, rstart, n_reads, k, m, min_count);
  ctx->rec_out = nullptr;
  ctx->rec_cap = 0;
  if (st != GERBIL_OK) return st;
  *n_bytes = ctx->rec_bytes;
  if (ctx->rec_bytes > capacity)
    return fail(ctx, GERBIL_E_USAGE, "output capacity " + std::to_string(capacity) + " < " +
                                         std::to_string(ctx->rec_bytes) + " record bytes");
  return GERBIL_OK;
}

// ---- step (a) on the device (parse.cu) ----------
// Parses d_text[0, len) into ctx->in_codes / in_nmask / in_rstart (the
// packed layout of include/gerbil.h), exactly as the host reader would.
gerbil_status parse_text_impl(gerbil_ctx* ctx, const uint8_t* d_text, uint64_t len, uint64_t& n_reads,
                              uint64_t& n_bases) {
  cudaStream_t st = ctx->stream;
  n_reads = n_bases = 0;
  const uint64_t nblk = parse_blocks(len);
  CK(ctx->p_cnt.ensure(std::max<uint64_t>(2 * nblk, 1) * 4));
  CK(ctx->p_off.ensure(std::max<uint64_t>(2 * nblk, 1) * 8));
  CK(ctx->p_misc.ensure(16 * 8));
  unsigned long long* misc = ctx->p_misc.as<unsigned long long>();  // [0,1] nl/cr totals, [2,3] first/last, [4] err, [5,6] totals
  uint32_t* cnt_nl = ctx->p_cnt.as<uint32_t>();
  uint32_t* cnt_cr = cnt_nl + nblk;
  uint64_t* off_nl = ctx->p_off.as<uint64_t>();
  uint64_t* off_cr = off_nl + nblk;
  CK(ctx->p_tmp.ensure(scan_tmp_words(std::max<uint64_t>(nblk, 1)) * 8 + 64));
  CK(cudaMemsetAsync(misc, 0, 16 * 8, st));
  CK(launch_parse_count(d_text, len, cnt_nl, cnt_cr, st));
  CK(launch_widen(cnt_nl, off_nl, 2 * nblk, ctx->sms, st));  // cnt_nl and cnt_cr are contiguous
  CK(launch_scan_u64(off_nl, off_nl, nblk, ctx->p_tmp.as<uint64_t>(), reinterpret_cast<uint64_t*>(misc), st));
  CK(launch_scan_u64(off_cr, off_cr, nblk, ctx->p_tmp.as<uint64_t>(), reinterpret_cast<uint64_t*>(misc + 1), st));
  uint64_t h[8] = {0};
  uint8_t last = '\n';
  CK(cudaMemcpyAsync(h, misc, 16, cudaMemcpyDeviceToHost, st));
  if (len) CK(cudaMemcpyAsync(&last, d_text + len - 1, 1, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const uint64_t n_nl = h[0], n_cr = h[1];
  const uint64_t n_lines = n_nl + (len > 0 && last != '\n' ? 1 : 0);
  if (n_lines == 0) return GERBIL_OK;
  CK(ctx->p_ls.ensure((n_lines + 2) * 8));
  CK(ctx->p_cr.ensure((n_cr + 1) * 8));
  uint64_t* ls = ctx->p_ls.as<uint64_t>();
  CK(cudaMemsetAsync(ls, 0, 8, st));
  CK(launch_parse_write(d_text, len, off_nl, off_cr, ls, ctx->p_cr.as<uint64_t>(), st));
  const uint64_t end_sentinel = len + 1;  // the last line has no '\n': it ends at len
  if (n_lines > n_nl) CK(cudaMemcpyAsync(ls + n_lines, &end_sentinel, 8, cudaMemcpyHostToDevice, st));
  CK(ctx->p_eff.ensure(n_lines * 4));
  CK(ctx->p_first.ensure(n_lines));
  const unsigned long long init[3] = {~0ull, 0ull, ~0ull};  // first, last non-empty line; error
  CK(cudaMemcpyAsync(misc + 2, init, 24, cudaMemcpyHostToDevice, st));
  CK(launch_parse_lines(d_text, ls, n_lines, ctx->p_cr.as<uint64_t>(), n_cr, ctx->p_eff.as<uint32_t>(),
                        ctx->p_first.as<uint8_t>(), misc + 2, ctx->sms, st));
  CK(cudaMemcpyAsync(h, misc + 2, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] == ~0ull) return GERBIL_OK;  // only empty lines
  const uint64_t f0 = h[0], n_eff = h[1] + 1;
  uint8_t c0 = 0;
  CK(cudaMemcpy(&c0, ctx->p_first.as<uint8_t>() + f0, 1, cudaMemcpyDeviceToHost));
  const int kind = c0 == '>' ? 0 : c0 == '@' ? 1 : 2;
  CK(ctx->p_seq.ensure(n_lines * 8));
  CK(ctx->p_rflag.ensure(n_lines * 8));
  CK(ctx->p_pos.ensure(n_lines * 8));
  CK(ctx->p_ridx.ensure(n_lines * 8));
  CK(ctx->p_tmp.ensure(scan_tmp_words(n_lines) * 8 + 64));
  CK(launch_parse_classify(ctx->p_eff.as<uint32_t>(), ctx->p_first.as<uint8_t>(), n_lines, f0, n_eff, kind,
                           ctx->p_seq.as<uint64_t>(), ctx->p_rflag.as<uint64_t>(), misc + 4, ctx->sms, st));
  CK(launch_scan_u64(ctx->p_seq.as<uint64_t>(), ctx->p_pos.as<uint64_t>(), n_lines, ctx->p_tmp.as<uint64_t>(),
                     reinterpret_cast<uint64_t*>(misc + 5), st));
  CK(launch_scan_u64(ctx->p_rflag.as<uint64_t>(), ctx->p_ridx.as<uint64_t>(), n_lines, ctx->p_tmp.as<uint64_t>(),
                     reinterpret_cast<uint64_t*>(misc + 6), st));
  CK(cudaMemcpyAsync(h, misc + 4, 24, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] != ~0ull) {
    static const char* what[] = {"", "FASTQ: expected '@'", "FASTQ: expected '+'",
                                 "FASTQ: quality length differs from sequence length", "FASTQ: truncated record",
                                 "FASTQ: empty line between records (not supported by the device parser; "
                                 "use the host reader)"};
    const uint64_t line = h[0] >> 8, code = h[0] & 0xff;
    return fail(ctx, GERBIL_E_IO,
                "<device>:" + std::to_string(line + 1) + ": " + (code < 6 ? what[code] : "parse error"));
  }
  n_bases = h[1];
  n_reads = h[2];
  const uint64_t ncw = std::max<uint64_t>((n_bases + 31) / 32, 1), nmw = std::max<uint64_t>((n_bases + 63) / 64, 1);
  CK(ctx->in_codes.ensure(ncw * 8));
  CK(ctx->in_nmask.ensure(nmw * 8));
  CK(ctx->in_rstart.ensure((n_reads + 1) * 8));
  CK(cudaMemsetAsync(ctx->in_codes.p, 0, ncw * 8, st));
  CK(cudaMemsetAsync(ctx->in_nmask.p, 0, nmw * 8, st));
  CK(launch_parse_read_starts(ctx->p_pos.as<uint64_t>(), ctx->p_rflag.as<uint64_t>(), ctx->p_ridx.as<uint64_t>(),
                              n_lines, ctx->in_rstart.as<uint64_t>(), ctx->sms, st));
  CK(cudaMemcpyAsync(ctx->in_rstart.as<uint64_t>() + n_reads, misc + 5, 8, cudaMemcpyDeviceToDevice, st));
  CK(launch_parse_pack(d_text, ls, ctx->p_seq.as<uint64_t>(), ctx->p_pos.as<uint64_t>(), n_lines,
                       ctx->in_codes.as<uint64_t>(), ctx->in_nmask.as<uint64_t>(), ctx->sms, st));
  return GERBIL_OK;
}

// text (host, or device when on_device) → aligned device copy
gerbil_status stage_text(gerbil_ctx* ctx, const char* text, uint64_t len, int on_device, const uint8_t*& d_text) {
  CK(ctx->text_buf.ensure(std::max<uint64_t>(len, 1) + 64));
  if (len)
    CK(cudaMemcpyAsync(ctx->text_buf.p, text, len, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream));
  d_text = ctx->text_buf.as<uint8_t>();
  return GERBIL_OK;
}

gerbil_status gerbil_parse_text(gerbil_ctx* ctx, const char* text, uint64_t len, int32_t on_device,
                                uint64_t* codes, uint64_t* nmask, uint64_t* rstart, uint64_t* n_bases,
                                uint64_t* n_reads) {
  if (!ctx || !n_bases || !n_reads || (len && !text)) return ctx ? fail(ctx, GERBIL_E_USAGE, "null argument")
                                                                  : GERBIL_E_USAGE;
  CK(cudaSetDevice(ctx->device));
  const uint8_t* d_text = nullptr;
  CKS(stage_text(ctx, text, len, on_device, d_text));
  uint64_t nr = 0, nb = 0;
  CKS(parse_text_impl(ctx, d_text, len, nr, nb));
  *n_bases = nb;
  *n_reads = nr;
  if (codes && nb) CK(cudaMemcpyAsync(codes, ctx->in_codes.p, ((nb + 31) / 32) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (nmask && nb) CK(cudaMemcpyAsync(nmask, ctx->in_nmask.p, ((nb + 63) / 64) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (rstart) {
    if (nr) CK(cudaMemcpyAsync(rstart, ctx->in_rstart.p, (nr + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    else rstart[0] = 0;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return GERBIL_OK;
}

gerbil_status gerbil_count_text(gerbil_ctx* ctx, const char* text, uint64_t len, int32_t on_device, uint32_t k,
                                uint32_t m, uint32_t min_count) {
  CKS(validate(ctx, k, m, min_count));
  if (len && !text) return fail(ctx, GERBIL_E_USAGE, "null text");
  CK(cudaSetDevice(ctx->device));
  begin_call(ctx);
  const uint8_t* d_text = nullptr;
  uint64_t nr = 0, nb = 0;
  {
    Timer tm(ctx, K_H2D, nullptr, true, 0);  // upload + parse (step a on the device) → ms_h2d
    CKS(stage_text(ctx, text, len, on_device, d_text));
    CKS(parse_text_impl(ctx, d_text, len, nr, nb));
  }
  if (nr == 0) {  // keep the stream layout valid for an empty batch
    CK(ctx->in_rstart.ensure(8));
    CK(cudaMemsetAsync(ctx->in_rstart.p, 0, 8, ctx->stream));
  }
  return count_device_impl(ctx, ctx->in_codes.as<uint64_t>(), ctx->in_nmask.as<uint64_t>(),
                           ctx->in_rstart.as<uint64_t>(), nr, k, m, min_count, false);
}

// ---- out-of-core counting ------------------------
// The paper's two phases with the temporary files in
// page-locked host memory: gerbil_spill_add runs step (b) on one host batch
// and moves its super-mers, grouped by bin (pack_kernel, one destination),
// to the host; gerbil_spill_finish then takes bins in groups that fit the
// device budget, uploads each group's super-mers from every batch, regroups
// them by bin (scatter with per-batch position rebasing) and runs steps
// (d)+(e) with the App. C records streamed to the caller's buffer.

gerbil_status gerbil_spill_begin(gerbil_ctx* ctx, uint32_t k, uint32_t m) {
  CKS(validate(ctx, k, m, 1));
  if (ctx->world > 1 || ctx->cfg.force_exchange)
    return fail(ctx, GERBIL_E_USAGE, "out-of-core counting runs on one rank (world = 1)");
  if (ctx->cfg.ordering == GERBIL_ORDER_DFP)  // its table is sampled per batch: bins would differ
    return fail(ctx, GERBIL_E_USAGE, "out-of-core counting needs a data-independent ordering (not DFP)");
  ctx->spill.release();
  SpillState& sp = ctx->spill;
  sp.win.clear();
  sp.cnt.clear();
  sp.words.clear();
  sp.bases = sp.reads = sp.windows = sp.supermers = 0;
  sp.active = true;
  sp.k = k;
  sp.m = m;
  sp.B = ctx->cfg.n_bins ? ctx->cfg.n_bins : 4096;  // fixed for every batch of the job
  sp.win.assign(sp.B, 0);
  sp.cnt.assign(sp.B, 0);
  sp.words.assign(sp.B, 0);
  ctx->have_result = false;
  return GERBIL_OK;
}

gerbil_status gerbil_spill_add(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                               const uint64_t* rstart, uint64_t n_reads) {
  if (!ctx) return GERBIL_E_USAGE;
  SpillState& sp = ctx->spill;
  if (!sp.active) return fail(ctx, GERBIL_E_STATE, "gerbil_spill_begin first");
  if (!rstart) return fail(ctx, GERBIL_E_USAGE, "null host buffer");
  CK(cudaSetDevice(ctx->device));
  const uint64_t nb = rstart[n_reads];
  if (nb > 0 && !codes) return fail(ctx, GERBIL_E_USAGE, "null host buffer");
  const uint32_t k = sp.k, m = sp.m, B = sp.B;
  begin_call(ctx);
  UploadPlan plan;
  CKS(upload_batch(ctx, codes, nmask, rstart, n_reads, plan));
  CK(ctx->counters.ensure(sizeof(Counters)));
  CK(ctx->hist.ensure(3ull * B * 8));
  uint64_t n_sm = 0;
  ctx->upload = &plan;
  ctx->want_words = true;
  const gerbil_status st = run_supermer(ctx, ctx->in_codes.as<uint64_t>(),
                                        nmask ? ctx->in_nmask.as<uint64_t>() : nullptr,
                                        ctx->in_rstart.as<uint64_t>(), n_reads, nb, k, m, B, false, n_sm);
  ctx->upload = nullptr;
  ctx->want_words = false;
  if (st != GERBIL_OK) {
    cudaStreamSynchronize(ctx->pcie_stream);
    return st;
  }
  const uint64_t windows = ctx->h_counters->n_windows;
  std::vector<unsigned long long> H(3ull * B);
  CK(cudaMemcpyAsync(H.data(), ctx->hist.p, 3ull * B * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  // bin-ordered layout of this batch (one destination: position = word offset * 32)
  SpillBatch sb;
  sb.d_off.assign(B + 1, 0);
  sb.w_off.assign(B + 1, 0);
  for (uint32_t b = 0; b < B; ++b) {
    sb.d_off[b + 1] = sb.d_off[b] + H[B + b];
    sb.w_off[b + 1] = sb.w_off[b] + H[2 * B + b];
  }
  sb.n_sm = sb.d_off[B];
  sb.n_words = sb.w_off[B];
  if (sb.n_sm != n_sm) return fail(ctx, GERBIL_E_INTERNAL, "spill: super-mer histogram mismatch");
  std::vector<unsigned long long> cur_d(sb.d_off.begin(), sb.d_off.end() - 1), cur_w(sb.w_off.begin(), sb.w_off.end() - 1),
      seg(B, 0);
  CK(ctx->send_desc.ensure(std::max<uint64_t>(n_sm, 1) * 8));
  CK(ctx->send_bin.ensure(std::max<uint64_t>(n_sm, 1) * 4));
  CK(ctx->send_payload.ensure(std::max<uint64_t>(sb.n_words, 1) * 8));
  CK(ctx->cursor.ensure((size_t)B * 8));
  CK(ctx->cursor2.ensure((size_t)B * 8));
  CK(ctx->seg_base.ensure((size_t)B * 8));
  CK(cudaMemcpyAsync(ctx->cursor.p, cur_d.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->cursor2.p, cur_w.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->seg_base.p, seg.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
  PackArgs pa{};
  pa.desc_in = ctx->desc_pre.as<uint64_t>();
  pa.bin_in = ctx->bin_pre.as<uint32_t>();
  pa.n = n_sm;
  pa.codes = ctx->in_codes.as<uint64_t>();
  pa.k = k;
  pa.cur_desc = ctx->cursor.as<unsigned long long>();
  pa.cur_words = ctx->cursor2.as<unsigned long long>();
  pa.seg_word_base = ctx->seg_base.as<unsigned long long>();
  pa.send_desc = ctx->send_desc.as<uint64_t>();
  pa.send_bin = ctx->send_bin.as<uint32_t>();
  pa.send_payload = ctx->send_payload.as<uint64_t>();
  {
    Timer tm(ctx, K_SHUFFLE);
    CK(launch_pack(pa, ctx->sms, ctx->stream));
  }
  // spill to page-locked host memory (the temporary files)
  if (n_sm) {
    sb.desc = static_cast<uint64_t*>(sp.pool.get(n_sm * 8));
    sb.bin = static_cast<uint32_t*>(sp.pool.get(n_sm * 4));
    sb.payload = static_cast<uint64_t*>(sp.pool.get(std::max<uint64_t>(sb.n_words, 1) * 8));
    if (!sb.desc || !sb.bin || !sb.payload) {
      sp.pool.put(sb.desc);
      sp.pool.put(sb.bin);
      sp.pool.put(sb.payload);
      return fail(ctx, GERBIL_E_NOMEM, "spill: cannot page-lock host memory");
    }
    CK(cudaMemcpyAsync(sb.desc, ctx->send_desc.p, n_sm * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(sb.bin, ctx->send_bin.p, n_sm * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(sb.payload, ctx->send_payload.p, sb.n_words * 8, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  for (uint32_t b = 0; b < B; ++b) {
    sp.win[b] += H[b];
    sp.cnt[b] += H[B + b];
    sp.words[b] += H[2 * B + b];
  }
  sp.bases += nb;
  sp.reads += n_reads;
  sp.windows += windows;
  sp.supermers += n_sm;
  sp.batches.push_back(std::move(sb));
  return GERBIL_OK;
}

gerbil_status gerbil_spill_finish(gerbil_ctx* ctx, uint32_t min_count, uint8_t* out, uint64_t capacity,
                                  uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return GERBIL_E_USAGE;
  *n_bytes = 0;
  SpillState& sp = ctx->spill;
  if (!sp.active) return fail(ctx, GERBIL_E_STATE, "gerbil_spill_begin first");
  if (min_count < 1) return fail(ctx, GERBIL_E_USAGE, "min_count must be >= 1");
  if (capacity > 0) {
    if (!out) return fail(ctx, GERBIL_E_USAGE, "null output buffer");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, out) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return fail(ctx, GERBIL_E_USAGE, "output buffer must be page-locked host memory (cudaHostAlloc/Register)");
    }
  }
  CK(cudaSetDevice(ctx->device));
  const uint32_t k = sp.k, B = sp.B;
  trace("call");
  begin_call(ctx);
  memset(&ctx->stats, 0, sizeof ctx->stats);
  ctx->W = key_words(k);
  ctx->k = k;
  ctx->m = sp.m;
  ctx->rec_out = capacity > 0 ? out : reinterpret_cast<uint8_t*>(1);
  ctx->rec_cap = capacity;
  ctx->rec_base = 0;
  ctx->rec_bytes = 0;
  // device budget per bin group: super-mer descriptors (8 + 4 + 8 sorted) and payload
  uint64_t budget = ctx->cfg.device_mem_cap ? ctx->cfg.device_mem_cap / 2 : (16ull << 30);
  if (const char* e = getenv("GERBIL_SPILL_GROUP_BYTES"))
    if (*e) budget = std::max<uint64_t>(1, strtoull(e, nullptr, 10));
  uint64_t distinct = 0, kept = 0, count_sum = 0, groups = 0, waves = 0, ovf = 0;
  gerbil_status st = GERBIL_OK;
  for (uint32_t b_lo = 0; b_lo < B && st == GERBIL_OK;) {
    uint32_t b_hi = b_lo;
    uint64_t bytes = 0;
    while (b_hi < B) {  // at least one bin per group
      const uint64_t add = sp.cnt[b_hi] * 20 + sp.words[b_hi] * 8;
      if (b_hi > b_lo && bytes + add > budget) break;
      bytes += add;
      ++b_hi;
    }
    uint64_t n_desc = 0, n_words = 0, g_windows = 0;
    for (uint32_t b = b_lo; b < b_hi; ++b) {
      n_desc += sp.cnt[b];
      n_words += sp.words[b];
      g_windows += sp.win[b];
    }
    if (n_desc == 0) {
      b_lo = b_hi;
      continue;
    }
    ++groups;
    CK(ctx->recv_desc.ensure(n_desc * 8));
    CK(ctx->recv_bin.ensure(n_desc * 4));
    CK(ctx->recv_payload.ensure(std::max<uint64_t>(n_words, 1) * 8));
    CK(ctx->desc_sorted.ensure(n_desc * 8));
    CK(ctx->cursor.ensure((size_t)B * 8));
    // upload every batch's segment of the group, then regroup by bin
    std::vector<uint64_t> bin_off(B + 1, 0), bin_win(B, 0);
    std::vector<uint32_t> owned;
    for (uint32_t b = 0; b < B; ++b) {
      const bool in = b >= b_lo && b < b_hi;
      bin_off[b + 1] = bin_off[b] + (in ? sp.cnt[b] : 0);
      bin_win[b] = in ? sp.win[b] : 0;
      if (in) owned.push_back(b);
    }
    CK(cudaMemcpyAsync(ctx->cursor.p, bin_off.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    uint64_t gd = 0, gw = 0;
    for (const SpillBatch& bt : sp.batches) {
      const uint64_t d0 = bt.d_off[b_lo], d1 = bt.d_off[b_hi], w0 = bt.w_off[b_lo], w1 = bt.w_off[b_hi];
      if (d1 == d0) continue;
      CK(cudaMemcpyAsync(ctx->recv_desc.as<uint64_t>() + gd, bt.desc + d0, (d1 - d0) * 8, cudaMemcpyHostToDevice,
                         ctx->stream));
      CK(cudaMemcpyAsync(ctx->recv_bin.as<uint32_t>() + gd, bt.bin + d0, (d1 - d0) * 4, cudaMemcpyHostToDevice,
                         ctx->stream));
      CK(cudaMemcpyAsync(ctx->recv_payload.as<uint64_t>() + gw, bt.payload + w0, (w1 - w0) * 8,
                         cudaMemcpyHostToDevice, ctx->stream));
      ScatterArgs sa{};
      sa.desc_in = ctx->recv_desc.as<uint64_t>() + gd;
      sa.bin_in = ctx->recv_bin.as<uint32_t>() + gd;
      sa.n = d1 - d0;
      sa.n_bins = B;
      sa.cursor = ctx->cursor.as<unsigned long long>();
      sa.desc_out = ctx->desc_sorted.as<uint64_t>();
      sa.pos_add = (gw - w0) * 32;  // batch payload positions → group payload positions (mod 2^64)
      {
        Timer tm(ctx, K_SHUFFLE);
        CK(launch_scatter(sa, ctx->sms, ctx->stream));
      }
      gd += d1 - d0;
      gw += w1 - w0;
    }
    trace("spill group uploaded + regrouped (issued)");
    st = count_waves(ctx, ctx->recv_payload.as<uint64_t>(), ctx->desc_sorted.as<uint64_t>(), bin_off, bin_win,
                     owned, k, min_count, g_windows);
    trace("spill group counted");
    if (st != GERBIL_OK) break;
    if (ctx->stats.count_sum != g_windows) {
      st = fail(ctx, GERBIL_E_INTERNAL, "invariant violated in a spill group: sum of counts != windows");
      break;
    }
    distinct += ctx->stats.distinct;
    kept += ctx->stats.kept;
    count_sum += ctx->stats.count_sum;
    waves += ctx->stats.waves;
    ovf += ctx->stats.overflow_kmers;
    ctx->rec_base = ctx->rec_bytes;
    b_lo = b_hi;
  }
  ctx->rec_out = nullptr;
  ctx->rec_cap = 0;
  const uint64_t total = ctx->rec_base;
  ctx->rec_base = 0;
  ctx->have_result = false;  // results were streamed group by group; no device-resident set remains
  if (st != GERBIL_OK) {
    sp.release();
    return st;
  }
  ctx->stats.input_bases = sp.bases;
  ctx->stats.input_reads = sp.reads;
  ctx->stats.valid_windows = sp.windows;
  ctx->stats.supermers = sp.supermers;
  ctx->stats.distinct = distinct;
  ctx->stats.kept = kept;
  ctx->stats.count_sum = count_sum;
  ctx->stats.owned_windows = sp.windows;
  ctx->stats.waves = (uint32_t)waves;
  ctx->stats.overflow_kmers = ovf;
  ctx->stats.n_bins = B;
  ctx->stats.W = ctx->W;
  *n_bytes = total;
  if (count_sum != sp.windows) {
    sp.release();
    return fail(ctx, GERBIL_E_INTERNAL, "invariant violated: sum of counts != valid windows");
  }
  // a sizing call (capacity 0) or a too-small buffer keeps the spilled job: call again with
  // a buffer of *n_bytes (phase one is not repeated)
  if (total > capacity)
    return fail(ctx, GERBIL_E_USAGE, "output capacity " + std::to_string(capacity) + " < " +
                                         std::to_string(total) + " record bytes");
  sp.release();
  return GERBIL_OK;
}

gerbil_status gerbil_pack_reads(const gerbil_reads* reads, int32_t threads, uint64_t* codes,
                                uint64_t* nmask, uint64_t* rstart, uint64_t* n_bases, uint64_t* n_reads,
                                char* err, size_t err_len) {
  if (!reads || !n_bases || !n_reads) return GERBIL_E_USAGE;
  const bool has_text = reads->text != nullptr, has_paths = reads->paths != nullptr && reads->n_paths > 0;
  if (has_text == has_paths) return GERBIL_E_USAGE;
  PackedBatch pb;
  std::string e;
  bool ok = true;
  if (has_text) ok = pack_text(reads->text, reads->text_len, threads, pb, e, "<memory>");
  else ok = pack_files(reads->paths, reads->n_paths, threads, pb, e);
  if (!ok) {
    if (err && err_len) {
      strncpy(err, e.c_str(), err_len - 1);
      err[err_len - 1] = 0;
    }
    return GERBIL_E_IO;
  }
  if (pb.read_start.empty()) pb.read_start.push_back(0);
  *n_bases = pb.n_bases;
  *n_reads = pb.n_reads;
  if (codes) {
    memcpy(codes, pb.codes.data(), pb.codes.size() * 8);
    if (nmask) memcpy(nmask, pb.nmask.data(), pb.nmask.size() * 8);
    if (rstart) memcpy(rstart, pb.read_start.data(), pb.read_start.size() * 8);
  }
  return GERBIL_OK;
}

gerbil_status gerbil_count(gerbil_ctx* ctx, const gerbil_reads* reads, uint32_t k, uint32_t m,
                           uint32_t min_count) {
  CKS(validate(ctx, k, m, min_count));
  if (!reads) return fail(ctx, GERBIL_E_USAGE, "null reads");
  const bool has_text = reads->text != nullptr, has_paths = reads->paths != nullptr && reads->n_paths > 0;
  if (has_text == has_paths) return fail(ctx, GERBIL_E_USAGE, "exactly one read source must be set");
  const double t0 = wall_ms();
  PackedBatch pb;
  std::string e;
  bool ok = true;
  if (has_text) ok = pack_text(reads->text, reads->text_len, ctx->cfg.host_threads, pb, e, "<memory>");
  else ok = pack_files(reads->paths, reads->n_paths, ctx->cfg.host_threads, pb, e);
  if (!ok) return fail(ctx, GERBIL_E_IO, e);
  if (pb.read_start.empty()) pb.read_start.push_back(0);
  const double t_reader = wall_ms() - t0;
  gerbil_status st = gerbil_count_host_packed(ctx, pb.codes.data(), pb.nmask.data(), pb.read_start.data(),
                                              pb.n_reads, k, m, min_count);
  ctx->stats.ms_reader = t_reader;
  return st;
}

gerbil_status gerbil_minimizer_stats(gerbil_ctx* ctx, uint64_t* max_per_minimizer, uint64_t* n_minimizers) {
  if (!ctx || !max_per_minimizer || !n_minimizers) return GERBIL_E_USAGE;
  if (!ctx->have_result) return fail(ctx, GERBIL_E_STATE, "no result: call gerbil_count first");
  if (ctx->m > 12) return fail(ctx, GERBIL_E_USAGE, "minimizer stats need m <= 12");
  CK(cudaSetDevice(ctx->device));
  const uint64_t hn = 2ull << (2 * ctx->m);  // every ordering key is < 2 * 4^m
  DevBuf hist, out;
  CK(hist.ensure(hn * 4));
  CK(out.ensure(16));
  CK(cudaMemsetAsync(hist.p, 0, hn * 4, ctx->stream));
  CK(cudaMemsetAsync(out.p, 0, 16, ctx->stream));
  CK(launch_minimizer_hist(ctx->out_keys.as<uint64_t>(), ctx->n_out, ctx->W, ctx->k, ctx->m,
                           (uint32_t)ctx->cfg.ordering, ctx->order_rank.as<uint32_t>(), hist.as<uint32_t>(), hn,
                           out.as<unsigned long long>(), ctx->sms, ctx->stream));
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, out.p, 16, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *max_per_minimizer = h[0];
  *n_minimizers = h[1];
  return GERBIL_OK;
}

gerbil_status gerbil_results_device(gerbil_ctx* ctx, const uint64_t** d_kmers, const uint32_t** d_counts,
                                    uint64_t* n, uint32_t* W) {
  if (!ctx) return GERBIL_E_USAGE;
  if (!ctx->have_result) return fail(ctx, GERBIL_E_STATE, "no successful count yet");
  if (d_kmers) *d_kmers = ctx->out_keys.as<uint64_t>();
  if (d_counts) *d_counts = ctx->out_counts.as<uint32_t>();
  if (n) *n = ctx->n_out;
  if (W) *W = ctx->W;
  return GERBIL_OK;
}

gerbil_status gerbil_fetch(gerbil_ctx* ctx, uint64_t* kmers, uint32_t* counts, uint64_t capacity,
                           uint64_t* n_out, int sorted) {
  if (!ctx || !n_out) return GERBIL_E_USAGE;
  if (!ctx->have_result) return fail(ctx, GERBIL_E_STATE, "no successful count yet");
  *n_out = ctx->n_out;
  if (!kmers) return GERBIL_OK;
  if (capacity < ctx->n_out) return fail(ctx, GERBIL_E_USAGE, "capacity too small");
  const uint64_t n = ctx->n_out, W = ctx->W;
  CK(cudaSetDevice(ctx->device));
  bool host_sort = false;
  if (sorted && n > 1 && !ctx->results_sorted) {
    // device LSD radix sort (sort.cu) of the results in place; only if its temporaries do not
    // fit does the host sort them after the copy
    DevBuf tk, tc, sc;
    if (tk.ensure(n * W * 8) == cudaSuccess && tc.ensure(n * 4) == cudaSuccess &&
        sc.ensure(sort_scratch_words(n) * 8) == cudaSuccess) {
      CK(launch_sort_results(ctx->out_keys.as<uint64_t>(), ctx->out_counts.as<uint32_t>(), n, (uint32_t)W, ctx->k,
                             tk.as<uint64_t>(), tc.as<uint32_t>(), sc.as<uint64_t>(), ctx->sms, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      ctx->results_sorted = true;
    } else {
      cudaGetLastError();
      host_sort = true;
    }
  }
  CK(cudaMemcpyAsync(kmers, ctx->out_keys.p, n * W * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (counts) CK(cudaMemcpyAsync(counts, ctx->out_counts.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (host_sort) {
    std::vector<uint64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0ull);
    std::sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
      return std::lexicographical_compare(kmers + a * W, kmers + a * W + W, kmers + b * W, kmers + b * W + W);
    });
    std::vector<uint64_t> kk(n * W);
    std::vector<uint32_t> cc(counts ? n : 0);
    for (uint64_t i = 0; i < n; ++i) {
      memcpy(&kk[i * W], kmers + idx[i] * W, W * 8);
      if (counts) cc[i] = counts[idx[i]];
    }
    memcpy(kmers, kk.data(), n * W * 8);
    if (counts) memcpy(counts, cc.data(), n * 4);
  }
  return GERBIL_OK;
}

gerbil_status gerbil_encode_results(gerbil_ctx* ctx, int32_t format, int sorted, uint8_t* out,
                                    uint64_t capacity, uint64_t* n_bytes) {
  if (!ctx || !n_bytes) return GERBIL_E_USAGE;
  if (format != GERBIL_FMT_BINARY && format != GERBIL_FMT_CSV) return fail(ctx, GERBIL_E_USAGE, "unknown format");
  if (!ctx->have_result) return fail(ctx, GERBIL_E_STATE, "no successful count yet");
  const uint64_t n = ctx->n_out, W = ctx->W;
  std::vector<uint64_t> keys(std::max<uint64_t>(n * W, 1));
  std::vector<uint32_t> counts(std::max<uint64_t>(n, 1));
  uint64_t got = 0;
  CKS(gerbil_fetch(ctx, keys.data(), counts.data(), n, &got, sorted));
  const uint64_t need = encode_results(format, keys.data(), counts.data(), got, ctx->k, (uint32_t)W, nullptr,
                                       ctx->cfg.host_threads);
  *n_bytes = need;
  if (!out) return GERBIL_OK;
  if (capacity < need) return fail(ctx, GERBIL_E_USAGE, "capacity too small");
  encode_results(format, keys.data(), counts.data(), got, ctx->k, (uint32_t)W, out, ctx->cfg.host_threads);
  return GERBIL_OK;
}

gerbil_status gerbil_merge_sorted(uint32_t n_lists, const uint64_t* const* keys, const uint32_t* const* counts,
                                  const uint64_t* n, uint32_t W, int32_t threads, uint64_t* out_keys,
                                  uint32_t* out_counts, uint64_t capacity, uint64_t* n_out) {
  if (!n_out || W == 0 || W > (uint32_t)kMaxW || (n_lists && (!keys || !counts || !n))) return GERBIL_E_USAGE;
  for (uint32_t l = 0; l < n_lists; ++l)
    if (n[l] && (!keys[l] || !counts[l])) return GERBIL_E_USAGE;
  const uint64_t m = merge_sorted(n_lists, keys, counts, n, W, nullptr, nullptr, threads);
  *n_out = m;
  if (!out_keys) return GERBIL_OK;
  if (!out_counts || capacity < m) return GERBIL_E_USAGE;
  merge_sorted(n_lists, keys, counts, n, W, out_keys, out_counts, threads);
  return GERBIL_OK;
}

gerbil_status gerbil_write_results(gerbil_ctx* ctx, const char* path, int32_t format, int sorted) {
  if (!ctx || !path) return GERBIL_E_USAGE;
  uint64_t nb = 0;
  CKS(gerbil_encode_results(ctx, format, sorted, nullptr, 0, &nb));
  std::vector<uint8_t> buf(std::max<uint64_t>(nb, 1));
  CKS(gerbil_encode_results(ctx, format, sorted, buf.data(), nb, &nb));
  FILE* f = fopen(path, "wb");
  if (!f) return fail(ctx, GERBIL_E_IO, std::string(path) + ": cannot open for writing");
  const bool ok = fwrite(buf.data(), 1, nb, f) == nb;
  if (fclose(f) != 0 || !ok) return fail(ctx, GERBIL_E_IO, std::string(path) + ": write failed");
  return GERBIL_OK;
}

gerbil_status gerbil_debug_supermers(gerbil_ctx* ctx, const uint64_t* codes, const uint64_t* nmask,
                                     const uint64_t* rstart, uint64_t n_reads, uint32_t k, uint32_t m,
                                     uint64_t* pos, uint32_t* nwin, uint32_t* bin, uint32_t* mu,
                                     uint64_t capacity, uint64_t* n_out) {
  // step (b) alone accepts the small k of the paper's Fig. 1 example (k=4, m=3)
  if (!ctx) return GERBIL_E_USAGE;
  if (k < 2 || k > 479 || m < 1 || m >= k || m > 15)
    return fail(ctx, GERBIL_E_USAGE, "debug_supermers: need 2 <= k <= 479, 1 <= m < k, m <= 15");
  if (!rstart || !n_out) return fail(ctx, GERBIL_E_USAGE, "null argument");
  CK(cudaSetDevice(ctx->device));
  // host buffers in, like gerbil_count_host_packed
  const uint64_t nb = rstart[n_reads];
  CK(ctx->in_codes.ensure(std::max<uint64_t>((nb + 31) / 32, 1) * 8));
  CK(ctx->in_nmask.ensure(std::max<uint64_t>((nb + 63) / 64, 1) * 8));
  CK(ctx->in_rstart.ensure((n_reads + 1) * 8));
  CK(cudaMemcpy(ctx->in_codes.p, codes, ((nb + 31) / 32) * 8, cudaMemcpyHostToDevice));
  if (nmask) CK(cudaMemcpy(ctx->in_nmask.p, nmask, ((nb + 63) / 64) * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ctx->in_rstart.p, rstart, (n_reads + 1) * 8, cudaMemcpyHostToDevice));
  const uint32_t B = ctx->cfg.n_bins ? ctx->cfg.n_bins : 512;
  CK(ctx->counters.ensure(sizeof(Counters)));
  CK(ctx->hist.ensure(3ull * B * 8));
  uint64_t n_sm = 0;
  CKS(run_supermer(ctx, ctx->in_codes.as<uint64_t>(), nmask ? ctx->in_nmask.as<uint64_t>() : nullptr,
                   ctx->in_rstart.as<uint64_t>(), n_reads, nb, k, m, B, true, n_sm));
  *n_out = n_sm;
  if (!pos) return GERBIL_OK;
  if (capacity < n_sm) return fail(ctx, GERBIL_E_USAGE, "capacity too small");
  std::vector<uint64_t> d(n_sm);
  CK(cudaMemcpy(d.data(), ctx->desc_pre.p, n_sm * 8, cudaMemcpyDeviceToHost));
  if (bin) CK(cudaMemcpy(bin, ctx->bin_pre.p, n_sm * 4, cudaMemcpyDeviceToHost));
  if (mu) CK(cudaMemcpy(mu, ctx->mu_dbg.p, n_sm * 4, cudaMemcpyDeviceToHost));
  for (uint64_t i = 0; i < n_sm; ++i) {
    pos[i] = d[i] >> kNwinBits;
    if (nwin) nwin[i] = (uint32_t)(d[i] & ((1u << kNwinBits) - 1)) + 1;
  }
  return GERBIL_OK;
}

}  // extern "C"
