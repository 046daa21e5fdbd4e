// waves.cu — steps (c)-(e) after step (b): the bin plans (host and device), the shared-memory /
// reference-table passes, the L2 wave tables with their emergency pass, and the multi-rank
// exchange of bin groups (documentation: DESIGN.md §4, api.cu header).
#include "api_internal.h"

namespace gerbil_api {

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
    // sized for at most an eighth of the device memory and grown between waves when the bound of
    // the next wave might not fit (a sync reads how many results the earlier waves kept).
    uint64_t out_chunk = out_bound;
    {
      // a fixed share of the device memory (not of what is free right now: a budget that moved
      // between calls would re-allocate — and copy — the result buffer every call)
      const uint64_t fit = result_budget_entries(ctx, W, 8);
      uint64_t big_wave = 0;
      for (const Wave& wv : waves) big_wave = std::max(big_wave, std::min<uint64_t>(wv.nb * kSlotsPerBucket, wv.windows));
      out_chunk = std::min(out_bound, std::max(fit, 2 * big_wave));
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
    CK(ctx->counters.ensure(sizeof(Counters)));  // a rank that ran no step (b) (empty spill) has none yet
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
    if (observed > 0) {
      ctx->rho = std::min(1.0, std::max(observed * 1.15 + 0.01, 0.02));
      ctx->rho_seen = true;
    }
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

int ref_tier1_ctas() {
  static const int c = [] {
    const char* e = getenv("GERBIL_REF_CTAS");
    return e && atoi(e) == 1 ? 1 : 2;
  }();
  return c;
}

// Shared-memory table slots per warp for this k (0 = shared-memory path off).
uint32_t smem_slots_for(gerbil_ctx* ctx, uint32_t k) {
  if (ctx->cfg.count_mode == 1) return 0;
  if (!ctx->smem_optin &&
      cudaDeviceGetAttribute(&ctx->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  // W >= 4, or mostly distinct k-mers: one CTA-wide table of occurrence references per bin
  // (count_ref.cu); else per-warp tables of whole keys (count_smem.cu)
  const uint32_t cap = ref_tier1(ctx, k) ? ref_table_slots((size_t)ctx->smem_optin - 1024, ref_tier1_ctas())
                                         : smem_table_slots(k, (size_t)ctx->smem_optin - 1024);
  return cap >= 128 ? cap : 0;
}

// Abandonment threshold of the shared-memory tables: a round inserts <= 32 k-mers per warp, so
// a table never fills.
uint32_t smem_max_fill(const gerbil_ctx* ctx, uint32_t cap, uint32_t k) {
  return ref_tier1(ctx, k) ? ref_max_fill(cap) : cap - std::max<uint32_t>(64u, cap / 4);
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
  // input (C4) that bound can exceed device memory: the buffer is capped at a fifth of the device
  // memory and, if the kept results do not fit, the pass is rerun once with the exact size
  uint64_t out_cap = std::min<uint64_t>(std::max<uint64_t>(out_bound, 1), result_budget_entries(ctx, W, 5));
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
  a.warps = ref_tier1(ctx, k) ? -ref_tier1_ctas() : 0;  // -1 / -2: CTA-wide reference tables (1 / 2 per SM)
  a.out_n = &dc->out_n;
  a.sum_counts = &dc->sum_counts;
  a.distinct = &dc->distinct;
  a.failed = ctx->smem_failed.as<unsigned long long>();
  a.n_failed = &dc->read_work;
  Counters& hc = *ctx->h_counters;
  // Streaming call (gerbil_count_host_stream): the shared-memory pass runs in slices of the bin
  // list; after each slice its results are encoded as App. C records (encode_records on the lane
  // stream, while the next slice counts) and copied to the caller's page-locked buffer on the copy
  // stream — the D2H of slice s overlaps the counting of slices s+1.. .
  const bool streaming = ctx->rec_out != nullptr;
  const uint64_t rec_max = 5 + (k + 3) / 4;
  uint64_t host_off = ctx->rec_base, rec_done = 0;
  int n_slices = 0;
  auto stream_slices = [&](const SmemCountArgs& as, uint32_t list_n, int S) -> gerbil_status {
    CK(ctx->rec_snap_d.ensure((size_t)(S + 1) * 8));
    unsigned long long* snap = ctx->rec_snap_d.as<unsigned long long>();
    CK(cudaMemcpyAsync(snap, &dc->out_n, 8, cudaMemcpyDeviceToDevice, ctx->stream));  // slice 0 start
    if (ctx->h_snap_n < (size_t)S) {
      if (ctx->h_snap) cudaFreeHost(ctx->h_snap);
      ctx->h_snap = nullptr;
      ctx->h_snap_n = 0;
      CK(cudaMallocHost((void**)&ctx->h_snap, (size_t)S * 8));
      ctx->h_snap_n = S;
    }
    while (ctx->wave_ev.size() < (size_t)2 * S) {
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ctx->wave_ev.push_back(ev);
    }
    unsigned long long* rec_ctr = ctx->rec_meta.as<unsigned long long>();
    for (int q = 0; q < S; ++q) {
      const uint32_t i0 = (uint32_t)((uint64_t)list_n * q / S), i1 = (uint32_t)((uint64_t)list_n * (q + 1) / S);
      SmemCountArgs sl = as;
      sl.range = as.range + 2 * (size_t)i0;
      sl.n_list = i1 - i0;
      {
        Timer tm(ctx, K_SMEM);
        CK(launch_count_smem(sl, ctx->sms, ctx->stream));
      }
      CK(cudaMemcpyAsync(snap + q + 1, &dc->out_n, 8, cudaMemcpyDeviceToDevice, ctx->stream));
      CK(cudaEventRecord(ctx->wave_ev[2 * q], ctx->stream));
      CK(cudaStreamWaitEvent(ctx->lane_stream, ctx->wave_ev[2 * q], 0));
      CK(launch_encode_records(as.out_keys, as.out_counts, snap + q, snap + q + 1, as.out_cap, k,
                               ctx->rec_stage2.as<uint8_t>(), ctx->rec_stage2.bytes, rec_ctr, ctx->sms,
                               ctx->lane_stream));
      unsigned long long* hs = nullptr;
      CK(cudaHostGetDevicePointer((void**)&hs, ctx->h_snap + q, 0));
      CK(launch_store_u64(hs, rec_ctr, ctx->lane_stream));
      CK(cudaEventRecord(ctx->wave_ev[2 * q + 1], ctx->lane_stream));
    }
    for (int q = 0; q < S; ++q) {  // copy each slice's records once they exist
      CK(cudaEventSynchronize(ctx->wave_ev[2 * q + 1]));
      const uint64_t end = ctx->h_snap[q], len = end - rec_done;
      if (end < rec_done || end > ctx->rec_stage2.bytes)
        return fail(ctx, GERBIL_E_INTERNAL, "record stream: slice " + std::to_string(q) + "/" + std::to_string(S) +
                                                " end " + std::to_string(end) + " < done " + std::to_string(rec_done) +
                                                " or > staging " + std::to_string(ctx->rec_stage2.bytes));
      if (len && host_off + len <= ctx->rec_cap)
        CK(cudaMemcpyAsync(ctx->rec_out + host_off, ctx->rec_stage2.as<uint8_t>() + rec_done, len,
                           cudaMemcpyDeviceToHost, ctx->pcie_stream));
      rec_done = end;
      host_off += len;
    }
    n_slices += S;
    return GERBIL_OK;
  };
  if (streaming) {
    CK(ctx->rec_stage2.ensure(std::max<uint64_t>(out_cap, 1) * rec_max + 64));
    CK(ctx->rec_meta.ensure(2 * 8));
    CK(cudaMemsetAsync(ctx->rec_meta.p, 0, 2 * 8, ctx->stream));
    CK(cudaStreamSynchronize(ctx->pcie_stream));  // the staging buffer's previous readers are done
  }
  for (int attempt = 0;; ++attempt) {
    a.out_keys = ctx->out_keys.as<uint64_t>();
    a.out_counts = ctx->out_counts.as<uint32_t>();
    a.out_cap = out_cap;
    if (streaming) {
      CKS(stream_slices(a, n, 16));
    } else {
      Timer tm(ctx, K_SMEM);
      CK(launch_count_smem(a, ctx->sms, ctx->stream));
    }
    trace("smem count issued");
    CK(d2h_small(ctx, ctx->h_counters, dc, sizeof(Counters)));
    CK(cudaStreamSynchronize(ctx->stream));
    trace("smem count done (synced)");
    if (hc.out_n > out_bound) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory result bound violated");
    if (hc.out_n <= out_cap) break;
    if (attempt > 0) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory pass: result size changed on rerun");
    out_cap = hc.out_n;  // exact: the rerun keeps the same k-mers
    CK(ctx->out_keys.ensure(out_cap * W * 8));
    CK(ctx->out_counts.ensure(out_cap * 4));
    if (streaming) {  // the records of the first attempt are incomplete: stream them again
      CK(cudaStreamSynchronize(ctx->pcie_stream));
      host_off = ctx->rec_base;
      rec_done = 0;
      CK(ctx->rec_stage2.ensure(out_cap * rec_max + 64));
      CK(cudaMemsetAsync(ctx->rec_meta.p, 0, 2 * 8, ctx->stream));
    }
    CK(cudaMemsetAsync(&dc->ovf_n, 0, sizeof(Counters) - offsetof(Counters, ovf_n), ctx->stream));
  }
  const uint64_t n_failed = hc.read_work;
  Preset pre;
  pre.out_n = hc.out_n;
  pre.sum_counts = hc.sum_counts;
  pre.distinct = hc.distinct;
  uint64_t failed_windows = 0;
  if (n_failed) {
    CK(ctx->h_fail.ensure(2 * n_failed * 8));
    CK(d2h_small(ctx, ctx->h_fail.p, ctx->smem_failed.p, 2 * n_failed * 8));
    CK(cudaStreamSynchronize(ctx->stream));
    const unsigned long long* fr = ctx->h_fail.as<unsigned long long>();
    for (uint64_t i = 0; i < n_failed; ++i) {
      const uint64_t w = fr[2 * i + 1] >> kRangeWinShift;
      rest.push_back({fr[2 * i], fr[2 * i + 1] & kRangeEndMask, w});
      failed_windows += w;
    }
  }
  ctx->stats.smem_bins += n;
  ctx->stats.smem_failed += n_failed;
  uint64_t smem_windows = elig_windows - std::min(elig_windows, failed_windows);
  // A later pass (tier 2, hash-class passes) appends after base.out_n: the result buffer grows by
  // at most `bound` entries but never past the result budget (with min_count > 1 on singleton-rich
  // input the bound is far larger than what is kept); if the kept results do not fit, the pass is
  // rerun once with the exact size after the counters are restored to `base`.
  auto run_pass = [&](const Preset& base, uint64_t bound, auto&& issue) -> gerbil_status {
    // the buffers' present capacity (no reallocation in steady state: a grown buffer is kept), or
    // room for a budget's worth of results after base; a first call that outgrows it reruns once
    const uint64_t have = std::min<uint64_t>(ctx->out_keys.bytes / (W * 8ull), ctx->out_counts.bytes / 4ull);
    const uint64_t budget = std::max<uint64_t>(result_budget_entries(ctx, W, 5), 1);
    uint64_t cap_n = std::max<uint64_t>(have, base.out_n + std::min<uint64_t>(std::max<uint64_t>(bound, 1), budget));
    const uint64_t host_start = host_off;
    for (int attempt = 0;; ++attempt) {
      CK(ensure_keep(ctx->out_keys, cap_n * W * 8, base.out_n * W * 8, ctx->stream));
      CK(ensure_keep(ctx->out_counts, cap_n * 4, base.out_n * 4, ctx->stream));
      if (streaming) {  // the previous pass's records are copied out: this pass starts a fresh staging area
        CK(cudaStreamSynchronize(ctx->pcie_stream));
        rec_done = 0;
        CK(cudaMemsetAsync(ctx->rec_meta.p, 0, 2 * 8, ctx->stream));
        CK(ctx->rec_stage2.ensure(std::min<uint64_t>(cap_n - base.out_n, std::max<uint64_t>(bound, 1)) * rec_max + 64));
      }
      CKS(issue(ctx->out_keys.as<uint64_t>(), ctx->out_counts.as<uint32_t>(), cap_n));
      CK(d2h_small(ctx, ctx->h_counters, dc, sizeof(Counters)));
      CK(cudaStreamSynchronize(ctx->stream));
      if (hc.out_n > base.out_n + bound) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory result bound violated");
      if (hc.out_n <= cap_n) return GERBIL_OK;
      if (attempt > 0) return fail(ctx, GERBIL_E_INTERNAL, "shared-memory pass: result size changed on rerun");
      cap_n = hc.out_n;  // exact: the rerun keeps the same k-mers
      host_off = host_start;
      Counters r = hc;
      r.ovf_n = 0;
      r.read_work = 0;
      r.out_n = base.out_n;
      r.sum_counts = base.sum_counts;
      r.distinct = base.distinct;
      CK(cudaMemcpyAsync(dc, &r, sizeof(Counters), cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
  };
  // Tier 2 (W <= 3): bins too large for the per-warp tables get a second launch — with mostly
  // repeated k-mers (rho < 0.35, e.g. C1) on half as many warps (twice the slots per warp),
  // with mostly distinct ones (C2/C3 shards) on one CTA-wide table of occurrence references per
  // bin (count_ref.cu, ~16K slots: verification re-reads cost little when repeats are rare);
  // what still does not fit goes to the wave tables. (W >= 4: tier 1 already is that table.)
  const bool tier1_ref = ref_tier1(ctx, k);
  const bool tier2_ref = !tier1_ref && W <= 3 && ctx->rho > 0.35;
  const int w1 = a.warps > 0 ? a.warps : smem_count_warps(k);
  const int w2n = std::max(1, w1 / 2);
  // the full-size reference table: tier 2 after half tables in tier 1 (W >= 4, two CTAs per SM),
  // tier 2 for mostly distinct short keys, and the hash-class passes below
  const uint32_t cap_full = ref_table_slots((size_t)ctx->smem_optin - 1024, 1);
  // the tier-2 passes, in order: (table slots, warps per CTA; -1 / -2 = reference tables with
  // one / two CTAs per SM). Mostly distinct short keys first try two half-size reference tables
  // per SM (bins of the C2/C3 shards hold ~10^3 windows: half tables take nearly all of them,
  // and two bins in flight per SM hide the per-bin barriers), then one full-size table per SM.
  std::vector<std::pair<uint32_t, int>> tiers;
  if (tier1_ref && a.warps == -2) {
    tiers.push_back({cap_full, -1});
  } else if (tier2_ref) {
    if (ref_tier1_ctas() == 2) tiers.push_back({ref_table_slots((size_t)ctx->smem_optin - 1024, 2), -2});
    tiers.push_back({cap_full, -1});
  } else if (!tier1_ref && w1 > 4) {
    tiers.push_back({smem_table_slots(k, (size_t)ctx->smem_optin - 1024, w2n), w2n});
  }
  auto tier_pass = [&](uint32_t cap2, int warps2) -> gerbil_status {
    const bool ref2 = warps2 < 0;
    const uint32_t mf2 = ref2 ? ref_max_fill(cap2) : cap2 - std::max<uint32_t>(64u, cap2 / 4);
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
      CK(ctx->smem_range.ensure(n2 * 16));
      CK(ctx->smem_failed.ensure(n2 * 16 + 16));
      CK(cudaMemcpyAsync(ctx->smem_range.p, r2, n2 * 16, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemsetAsync(&dc->read_work, 0, 8, ctx->stream));
      SmemCountArgs a2 = a;
      a2.range = ctx->smem_range.as<unsigned long long>();
      a2.n_list = (uint32_t)n2;
      a2.cap = cap2;
      a2.max_fill = mf2;
      a2.warps = warps2;  // -1 / -2: the CTA-wide reference tables, one / two per SM
      a2.failed = ctx->smem_failed.as<unsigned long long>();
      CKS(run_pass(pre, ob2, [&](uint64_t* ok, uint32_t* oc, uint64_t cap_n) -> gerbil_status {
        a2.out_keys = ok;
        a2.out_counts = oc;
        a2.out_cap = cap_n;
        if (streaming) {
          CKS(stream_slices(a2, (uint32_t)n2, 1));
        } else {
          Timer tm(ctx, K_SMEM);
          CK(launch_count_smem(a2, ctx->sms, ctx->stream));
        }
        return GERBIL_OK;
      }));
      pre.out_n = hc.out_n;
      pre.sum_counts = hc.sum_counts;
      pre.distinct = hc.distinct;
      const uint64_t nf2 = hc.read_work;
      uint64_t fw2 = 0;
      if (nf2) {
        CK(ctx->h_fail.ensure(2 * nf2 * 8));
        CK(d2h_small(ctx, ctx->h_fail.p, ctx->smem_failed.p, 2 * nf2 * 8));
        CK(cudaStreamSynchronize(ctx->stream));
        const unsigned long long* fr = ctx->h_fail.as<unsigned long long>();
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
      trace("smem tier 2 pass done (synced)");
    }
    return GERBIL_OK;
  };
  for (const auto& t : tiers)
    if (!rest.empty() && (t.second < 0 || t.first > cap)) CKS(tier_pass(t.first, t.second));
  // Long keys (reference tables in tier 1): a bin too large for one CTA table is counted in P
  // passes over its super-mers, pass p keeping the k-mers whose hash class is p (distinct k-mers
  // spread evenly over the classes: P = 1.5 x windows / max_fill (distinct <= windows) leaves each
  // pass at most 2/3 of max_fill on average — an overflow would need a deviation of dozens of
  // standard deviations over thousands of keys; it fails the call loudly rather than recount a bin
  // whose other classes are already output). Bins beyond 128 classes stay with the wave tables.
  if (!rest.empty() && ref_tier1(ctx, k) && ctx->cfg.count_mode != 1) {
    std::vector<RestBin> keep;
    std::vector<std::vector<RestBin>> by_p(7);  // P = 2, 4, ..., 128
    const uint32_t mf_full = ref_max_fill(cap_full);  // the passes use full-size tables
    for (const RestBin& rb : rest) {
      const uint64_t want = (3 * rb.win + 2 * (uint64_t)mf_full - 1) / (2 * (uint64_t)std::max<uint32_t>(mf_full, 1));
      int e = 1;
      while (e < 7 && (1ull << e) < want) ++e;
      if ((1ull << e) >= want && rb.win < (1ull << 24)) by_p[e - 1].push_back(rb);
      else keep.push_back(rb);
    }
    for (int e = 1; e <= 7; ++e) {
      const std::vector<RestBin>& L = by_p[e - 1];
      if (L.empty()) continue;
      const uint32_t P = 1u << e;
      uint64_t wsum = 0;
      CK(ctx->h_rng.ensure(L.size() * 16));
      unsigned long long* r2 = ctx->h_rng.as<unsigned long long>();
      for (size_t i = 0; i < L.size(); ++i) {
        r2[2 * i] = L[i].d0;
        r2[2 * i + 1] = L[i].d1 | (L[i].win << kRangeWinShift);
        wsum += L[i].win;
      }
      CK(ctx->smem_range.ensure(L.size() * 16));
      CK(ctx->smem_failed.ensure(L.size() * 16 + 16));
      CK(cudaMemcpyAsync(ctx->smem_range.p, r2, L.size() * 16, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemsetAsync(&dc->read_work, 0, 8, ctx->stream));
      SmemCountArgs a3 = a;
      a3.range = ctx->smem_range.as<unsigned long long>();
      a3.n_list = (uint32_t)L.size();
      a3.failed = ctx->smem_failed.as<unsigned long long>();
      a3.parts = P;
      a3.cap = cap_full;
      a3.max_fill = mf_full;
      a3.warps = -1;
      CKS(run_pass(pre, wsum, [&](uint64_t* ok, uint32_t* oc, uint64_t cap_n) -> gerbil_status {
        a3.out_keys = ok;
        a3.out_counts = oc;
        a3.out_cap = cap_n;
        for (uint32_t q = 0; q < P; ++q) {
          a3.part = q;
          if (streaming) {
            CKS(stream_slices(a3, (uint32_t)L.size(), 1));
          } else {
            Timer tm(ctx, K_SMEM);
            CK(launch_count_smem(a3, ctx->sms, ctx->stream));
          }
        }
        return GERBIL_OK;
      }));
      if (hc.read_work) return fail(ctx, GERBIL_E_INTERNAL, "hash-class pass overflowed a reference table");
      pre.out_n = hc.out_n;
      pre.sum_counts = hc.sum_counts;
      pre.distinct = hc.distinct;
      ctx->stats.smem_bins += L.size();
      smem_windows += wsum;
    }
    rest.swap(keep);
    trace("hash-class passes done (synced)");
  }
  ctx->stats.smem_windows += smem_windows;
  const double smem_obs = smem_windows ? (double)pre.distinct / (double)smem_windows : 0.0;
  gerbil_status st = GERBIL_OK;
  if (streaming) {
    ctx->rec_base = host_off;  // the L2 waves append their records after the shared-memory pass's
    if (rest.empty()) {
      CK(cudaStreamSynchronize(ctx->pcie_stream));
      ctx->rec_bytes = host_off;
    }
  }
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
  if (smem_obs > 0) {
    ctx->rho = std::min(1.0, std::max(rest.empty() ? 0.0 : ctx->rho, std::max(smem_obs * 1.15 + 0.01, 0.02)));
    ctx->rho_seen = true;
  }
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
  const uint32_t cap = smem_slots_for(ctx, k);
  ctx->stats.smem_slots = cap;
  if (cap == 0) return count_waves_l2(ctx, stream_codes, desc, bin_off, bin_win, bins, k, min_count,
                                      total_windows, Preset{});
  const uint32_t max_fill = smem_max_fill(ctx, cap, k);
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
                            uint64_t* tmp_desc, uint32_t* tmp_bin, uint64_t* desc_alt, uint64_t max_windows) {
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
  gs.max_windows = max_windows;
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
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->desc_pre.as<uint64_t>(), windows));
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
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->desc_pre.as<uint64_t>(),
                    ctx->stats.valid_windows));
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
                    ctx->send_desc.as<uint64_t>(), ctx->send_bin.as<uint32_t>(), ctx->recv_desc.as<uint64_t>(),
                    owned_windows));
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
  const uint32_t max_fill = smem_max_fill(ctx, cap, k);
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

}  // namespace gerbil_api
