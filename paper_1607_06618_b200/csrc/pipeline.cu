// pipeline.cu — one call of the counting path on this rank: step (b) (run_supermer, the dfp(p)
// table) and the orchestration of steps (c)-(e) with the Σ-count invariant (count_device_impl).
#include "api_internal.h"

namespace gerbil_api {

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
                           uint32_t m, uint32_t B, bool want_mu, uint64_t& n_sm, bool want_hist) {
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
                                uint32_t min_count, bool fresh) {
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
  const uint32_t smem_cap = (B >= kDevicePlanBins && B <= (1u << 22) && n_bases < pos_lim &&
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

}  // namespace gerbil_api
