// api.cu — C ABI (include/gerbil.h): context life cycle, configuration, statistics and the
// count entry points. The host orchestration lives in the other units (api_internal.h):
//   pipeline.cu  one call: (b) super-mers → (c) bin shuffle → (d)+(e) counting, invariant check
//   waves.cu     bin plans (device for many bins, host otherwise), shared-memory / reference
//                table passes, L2 wave tables + emergency pass, the multi-rank group exchange
//   io.cu        host batches (chunked pinned uploads, streamed App. C records), device parsing
//   spill.cu     out-of-core jobs;  results.cu  fetch (device sort), encodings, k-way merge
// One context = one rank = one GPU; everything runs on the context's stream.
#include "api_internal.h"

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
  ctx->rho_seen = cfg.distinct_ratio > 0;
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

}  // extern "C"
