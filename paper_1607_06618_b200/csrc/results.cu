// results.cu — results: minimizer statistics, device-resident results, sorted fetch (device radix
// sort), the paper's encodings, k-way merge, debug super-mers.
#include "api_internal.h"

extern "C" {

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
