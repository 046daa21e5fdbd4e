// spill.cu — out-of-core jobs (gerbil_spill_*): phase one to page-locked host memory, phase two
// bin group by bin group.
#include "api_internal.h"

namespace {

struct SpillAcc {
  uint64_t distinct = 0, kept = 0, count_sum = 0, waves = 0, ovf = 0, owned = 0, sent = 0, recv = 0, groups = 0;
  uint64_t max_bin = 0;  // windows of the largest bin (global)
};

// Steps (d)+(e) on one bin group already regrouped in ctx->desc_sorted over `payload`; the
// records stream on from ctx->rec_base.
gerbil_status spill_count_group(gerbil_ctx* ctx, const uint64_t* payload, const std::vector<uint64_t>& bin_off,
                                const std::vector<uint64_t>& bin_win, const std::vector<uint32_t>& owned,
                                uint32_t min_count, uint64_t g_windows, SpillAcc& acc) {
  const gerbil_status st = count_waves(ctx, payload, ctx->desc_sorted.as<uint64_t>(), bin_off, bin_win, owned,
                                       ctx->spill.k, min_count, g_windows);
  trace("spill group counted");
  if (st != GERBIL_OK) return st;
  if (ctx->stats.count_sum != g_windows)
    return fail(ctx, GERBIL_E_INTERNAL, "invariant violated in a spill group: sum of counts != windows");
  acc.distinct += ctx->stats.distinct;
  acc.kept += ctx->stats.kept;
  acc.count_sum += ctx->stats.count_sum;
  acc.waves += ctx->stats.waves;
  acc.ovf += ctx->stats.overflow_kmers;
  acc.owned += g_windows;
  ++acc.groups;
  ctx->rec_base = ctx->rec_bytes;
  return GERBIL_OK;
}

// Blocking all-gather of n host words through the device (comm buffers are device memory).
gerbil_status allgather_host(gerbil_ctx* ctx, const unsigned long long* mine, size_t n,
                             std::vector<unsigned long long>& all) {
  CK(ctx->hist.ensure(n * 8));
  CK(ctx->hist_all.ensure(n * 8 * ctx->world));
  CK(cudaMemcpyAsync(ctx->hist.p, mine, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (!ctx->comm->allgather(ctx->hist.p, ctx->hist_all.p, n * 8, ctx->stream))
    return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
  all.assign(n * ctx->world, 0);
  CK(cudaMemcpyAsync(all.data(), ctx->hist_all.p, n * 8 * ctx->world, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return GERBIL_OK;
}

// world > 1 (PAPER.md:200-210 with the temporary files of :97): every rank spilled its own
// batches; the ranks all-gather their per-bin histograms, split the bins into contiguous
// ranges of about equal global windows (one range per rank: a rank's spilled super-mers of a
// range are one contiguous run per batch), cut every range into groups that fit the device
// budget, and then proceed in rounds: in round t every rank uploads its share of each rank's
// t-th group, rebased into one send segment per destination, one grouped all-to-all
// (descriptors, bins, payload) delivers them, and each rank regroups what it received by bin
// and counts its group.
gerbil_status spill_finish_ranks(gerbil_ctx* ctx, uint32_t min_count, uint64_t budget, SpillAcc& acc) {
  SpillState& sp = ctx->spill;
  const int P = ctx->world, r = ctx->rank;
  const uint32_t B = sp.B;
  {  // the job must be the same on every rank
    const unsigned long long hdr[4] = {B, sp.k, sp.m,
                                       (unsigned long long)ctx->cfg.ordering |
                                           ((unsigned long long)(ctx->cfg.disable_normalization != 0) << 8)};
    std::vector<unsigned long long> all;
    CKS(allgather_host(ctx, hdr, 4, all));
    for (int s = 0; s < P; ++s)
      for (int i = 0; i < 4; ++i)
        if (all[(size_t)s * 4 + i] != hdr[i])
          return fail(ctx, GERBIL_E_USAGE, "out-of-core job differs between ranks (bins, k, m, ordering or -d)");
  }
  std::vector<unsigned long long> mine(3ull * B), H;
  for (uint32_t b = 0; b < B; ++b) {
    mine[b] = sp.win[b];
    mine[B + b] = sp.cnt[b];
    mine[2 * B + b] = sp.words[b];
  }
  CKS(allgather_host(ctx, mine.data(), mine.size(), H));
  auto Hw = [&](int s, uint32_t b) { return (uint64_t)H[(size_t)s * 3 * B + b]; };
  auto Hc = [&](int s, uint32_t b) { return (uint64_t)H[(size_t)s * 3 * B + B + b]; };
  auto Hp = [&](int s, uint32_t b) { return (uint64_t)H[(size_t)s * 3 * B + 2 * B + b]; };
  std::vector<uint64_t> gw(B, 0), gc(B, 0), gp(B, 0);
  uint64_t tot = 0;
  for (int s = 0; s < P; ++s)
    for (uint32_t b = 0; b < B; ++b) {
      gw[b] += Hw(s, b);
      gc[b] += Hc(s, b);
      gp[b] += Hp(s, b);
    }
  for (uint32_t b = 0; b < B; ++b) tot += gw[b];
  acc.max_bin = *std::max_element(gw.begin(), gw.end());
  // owner ranges [lo[d], lo[d+1]): rank d starts at the first bin whose preceding windows reach d/P
  std::vector<uint32_t> lo(P + 1, B);
  lo[0] = 0;
  {
    int d = 1;
    unsigned __int128 cum = 0;
    for (uint32_t b = 0; b < B && d < P; ++b) {
      while (d < P && cum * (unsigned)P >= (unsigned __int128)d * tot) lo[d++] = b;
      cum += gw[b];
    }
  }
  // groups of each range that fit the device budget (receive side: 8 + 4 + 8 B per super-mer)
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> groups(P);
  size_t rounds = 0;
  for (int d = 0; d < P; ++d) {
    for (uint32_t b = lo[d]; b < lo[d + 1];) {
      const uint32_t a = b;
      uint64_t bytes = 0, n = 0;
      while (b < lo[d + 1]) {
        const uint64_t add = gc[b] * 20 + gp[b] * 8;
        if (b > a && bytes + add > budget) break;
        bytes += add;
        n += gc[b];
        ++b;
      }
      if (n) groups[d].push_back({a, b});
    }
    rounds = std::max(rounds, groups[d].size());
  }
  for (size_t t = 0; t < rounds; ++t) {
    auto grp = [&](int d) {
      return t < groups[d].size() ? groups[d][t] : std::pair<uint32_t, uint32_t>(0, 0);
    };
    std::vector<uint64_t> sd(P + 1, 0), sw(P + 1, 0), rd(P + 1, 0), rw(P + 1, 0);
    for (int d = 0; d < P; ++d) {
      const auto g = grp(d);
      for (uint32_t b = g.first; b < g.second; ++b) {
        sd[d + 1] += sp.cnt[b];
        sw[d + 1] += sp.words[b];
      }
      sd[d + 1] += sd[d];
      sw[d + 1] += sw[d];
    }
    const auto my = grp(r);
    for (int s = 0; s < P; ++s) {
      uint64_t c = 0, w = 0;
      for (uint32_t b = my.first; b < my.second; ++b) {
        c += Hc(s, b);
        w += Hp(s, b);
      }
      rd[s + 1] = rd[s] + c;
      rw[s + 1] = rw[s] + w;
    }
    CK(ctx->send_desc.ensure(std::max<uint64_t>(sd[P], 1) * 8));
    CK(ctx->send_bin.ensure(std::max<uint64_t>(sd[P], 1) * 4));
    CK(ctx->send_payload.ensure(std::max<uint64_t>(sw[P], 1) * 8));
    CK(ctx->recv_desc.ensure(std::max<uint64_t>(rd[P], 1) * 8));
    CK(ctx->recv_bin.ensure(std::max<uint64_t>(rd[P], 1) * 4));
    CK(ctx->recv_payload.ensure(std::max<uint64_t>(rw[P], 1) * 8));
    CK(ctx->desc_sorted.ensure(std::max<uint64_t>(rd[P], 1) * 8));
    CK(ctx->cursor.ensure((size_t)B * 8));
    // this rank's share of every destination's group: one run per batch, rebased into the
    // destination's segment (positions relative to the segment start)
    for (int d = 0; d < P; ++d) {
      const auto g = grp(d);
      if (g.first == g.second) continue;
      uint64_t cd = sd[d], cw = sw[d];
      for (const SpillBatch& bt : sp.batches) {
        const uint64_t d0 = bt.d_off[g.first], d1 = bt.d_off[g.second];
        const uint64_t w0 = bt.w_off[g.first], w1 = bt.w_off[g.second];
        if (d1 == d0) continue;
        CK(cudaMemcpyAsync(ctx->send_desc.as<uint64_t>() + cd, bt.desc + d0, (d1 - d0) * 8, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->send_bin.as<uint32_t>() + cd, bt.bin + d0, (d1 - d0) * 4, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaMemcpyAsync(ctx->send_payload.as<uint64_t>() + cw, bt.payload + w0, (w1 - w0) * 8,
                           cudaMemcpyHostToDevice, ctx->stream));
        {
          Timer tm(ctx, K_SHUFFLE);
          CK(launch_rebase_desc(ctx->send_desc.as<uint64_t>() + cd, d1 - d0, (cw - sw[d] - w0) * 32, ctx->sms,
                                ctx->stream));
        }
        cd += d1 - d0;
        cw += w1 - w0;
      }
      if (cd != sd[d + 1] || cw != sw[d + 1]) return fail(ctx, GERBIL_E_INTERNAL, "spill: send layout mismatch");
    }
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<size_t> so[3], sbytes[3], ro[3], rbytes[3];
    const std::vector<uint64_t>* soff[3] = {&sd, &sd, &sw};
    const std::vector<uint64_t>* roff[3] = {&rd, &rd, &rw};
    const size_t elem[3] = {8, 4, 8};
    void* sbuf[3] = {ctx->send_desc.p, ctx->send_bin.p, ctx->send_payload.p};
    void* rbuf[3] = {ctx->recv_desc.p, ctx->recv_bin.p, ctx->recv_payload.p};
    Comm::Xfer x[3];
    for (int b = 0; b < 3; ++b) {
      so[b].resize(P);
      sbytes[b].resize(P);
      ro[b].resize(P);
      rbytes[b].resize(P);
      for (int p = 0; p < P; ++p) {
        so[b][p] = (*soff[b])[p] * elem[b];
        sbytes[b][p] = ((*soff[b])[p + 1] - (*soff[b])[p]) * elem[b];
        ro[b][p] = (*roff[b])[p] * elem[b];
        rbytes[b][p] = ((*roff[b])[p + 1] - (*roff[b])[p]) * elem[b];
      }
      x[b] = Comm::Xfer{sbuf[b], so[b].data(), sbytes[b].data(), rbuf[b], ro[b].data(), rbytes[b].data()};
    }
    {
      Timer tm(ctx, K_SHUFFLE);
      if (!ctx->comm->alltoallv_multi(x, 3, ctx->stream)) return fail(ctx, GERBIL_E_NCCL, ctx->comm->err);
    }
    acc.sent += (sd[P] - (sd[r + 1] - sd[r])) * 12 + (sw[P] - (sw[r + 1] - sw[r])) * 8;
    acc.recv += (rd[P] - (rd[r + 1] - rd[r])) * 12 + (rw[P] - (rw[r + 1] - rw[r])) * 8;
    trace("spill round exchanged");
    if (rd[P] == 0) continue;
    // regroup this rank's group by bin (positions rebased into recv_payload) and count it
    std::vector<uint64_t> bin_off(B + 1, 0), bin_win(B, 0);
    std::vector<uint32_t> owned;
    uint64_t g_windows = 0;
    for (uint32_t b = 0; b < B; ++b) {
      const bool in = b >= my.first && b < my.second;
      bin_off[b + 1] = bin_off[b] + (in ? gc[b] : 0);
      if (in) {
        bin_win[b] = gw[b];
        g_windows += gw[b];
        owned.push_back(b);
      }
    }
    if (bin_off[B] != rd[P]) return fail(ctx, GERBIL_E_INTERNAL, "spill: receive layout mismatch");
    CK(cudaMemcpyAsync(ctx->cursor.p, bin_off.data(), (size_t)B * 8, cudaMemcpyHostToDevice, ctx->stream));
    for (int s = 0; s < P; ++s) {
      ScatterArgs sa{};
      sa.desc_in = ctx->recv_desc.as<uint64_t>() + rd[s];
      sa.bin_in = ctx->recv_bin.as<uint32_t>() + rd[s];
      sa.n = rd[s + 1] - rd[s];
      sa.n_bins = B;
      sa.cursor = ctx->cursor.as<unsigned long long>();
      sa.desc_out = ctx->desc_sorted.as<uint64_t>();
      sa.pos_add = rw[s] * 32;
      Timer tm(ctx, K_SHUFFLE);
      CK(launch_scatter(sa, ctx->sms, ctx->stream));
    }
    CKS(spill_count_group(ctx, ctx->recv_payload.as<uint64_t>(), bin_off, bin_win, owned, min_count, g_windows,
                          acc));
  }
  return GERBIL_OK;
}

}  // namespace

extern "C" {


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
  if (ctx->cfg.force_exchange)
    return fail(ctx, GERBIL_E_USAGE, "out-of-core counting: force_exchange is not supported (use world > 1)");
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
  SpillAcc acc;
  CK(ctx->counters.ensure(sizeof(Counters)));  // a rank that spilled nothing ran no step (b)
  gerbil_status st = GERBIL_OK;
  if (ctx->world > 1) st = spill_finish_ranks(ctx, min_count, budget, acc);
  for (uint32_t b = 0; b < B && ctx->world == 1; ++b) acc.max_bin = std::max<uint64_t>(acc.max_bin, sp.win[b]);
  for (uint32_t b_lo = 0; b_lo < B && st == GERBIL_OK && ctx->world == 1;) {
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
    st = spill_count_group(ctx, ctx->recv_payload.as<uint64_t>(), bin_off, bin_win, owned, min_count, g_windows, acc);
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
  ctx->stats.distinct = acc.distinct;
  ctx->stats.kept = acc.kept;
  ctx->stats.count_sum = acc.count_sum;
  ctx->stats.owned_windows = ctx->world > 1 ? acc.owned : sp.windows;
  ctx->stats.waves = (uint32_t)acc.waves;
  ctx->stats.overflow_kmers = acc.ovf;
  ctx->stats.n_bins = B;
  ctx->stats.W = ctx->W;
  ctx->stats.max_bin_windows = acc.max_bin;
  ctx->stats.bytes_sent = acc.sent;
  ctx->stats.bytes_recv = acc.recv;
  *n_bytes = total;
  if (acc.count_sum != ctx->stats.owned_windows) {
    sp.release();
    return fail(ctx, GERBIL_E_INTERNAL, "invariant violated: sum of counts != valid windows");
  }
  // a sizing call (capacity 0) or a too-small buffer keeps the spilled job: call again with
  // a buffer of *n_bytes (phase one is not repeated). With world > 1 the ranks agree (one
  // all-gather): the job is kept on every rank unless every rank's records fit.
  bool all_fit = total <= capacity;
  if (ctx->world > 1) {
    const unsigned long long fit = all_fit ? 1 : 0;
    std::vector<unsigned long long> fits;
    CKS(allgather_host(ctx, &fit, 1, fits));
    for (unsigned long long f : fits) all_fit = all_fit && f;
  }
  if (total > capacity)
    return fail(ctx, GERBIL_E_USAGE, "output capacity " + std::to_string(capacity) + " < " +
                                         std::to_string(total) + " record bytes");
  if (!all_fit)  // every rank repeats the call (the sizing protocol stays collective)
    return fail(ctx, GERBIL_E_USAGE, "another rank's output buffer is too small: call again on every rank");
  sp.release();
  return GERBIL_OK;
}

}  // extern "C"
