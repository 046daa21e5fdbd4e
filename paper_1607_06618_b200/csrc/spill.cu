// spill.cu — out-of-core jobs (gerbil_spill_*): phase one to page-locked host memory, phase two
// bin group by bin group.
#include "api_internal.h"

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

}  // extern "C"
