// io.cu — host batches (chunked pinned uploads, the streaming record sink) and step (a) on the
// device (gerbil_parse_text / gerbil_count_text).
#include "api_internal.h"

extern "C" {

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
}  // extern "C"
