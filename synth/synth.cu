/*
 * synth.cu — host ASCII emitters and the bit-identical device twin of the
 * synthetic read generator (synth_core.h). Test/bench infrastructure: it
 * writes inputs, it never counts anything.
 *
 *  - synth_fastx: FASTA/FASTQ/raw text of the batch (the oracle's input, and
 *    the host reader's input for end-to-end runs).
 *  - synth_packed_host / synth_packed_device: the same reads written straight
 *    into the library's device input layout (2-bit codes, N-mask,
 *    read_start; include/gerbil.h), so that large batches can be created in
 *    HBM without a host round trip.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <thread>
#include <vector>

#include "synth_core.h"

static const char kLetters[5] = {'A', 'C', 'G', 'T', 'N'};

/* Record geometry: fixed-width headers so that record i starts at i*rec. */
static uint64_t rec_size(const synth_params* p, int format, uint32_t lw) {
  const uint64_t L = p->read_len;
  const uint64_t hdr = 1 + 1 + 12 + 1; /* '>'/'@' 'r' 12 digits '\n' */
  if (format == 0) return L + 1;
  if (format == 1) {
    uint64_t lines = (lw == 0 || L == 0) ? 1 : (L + lw - 1) / lw;
    return hdr + L + lines;
  }
  return hdr + L + 1 + 2 + L + 1; /* seq\n +\n qual\n */
}

static void emit_range(const synth_params* p, int format, uint32_t lw, char* out,
                       uint64_t r0, uint64_t r1) {
  const uint64_t L = p->read_len, rs = rec_size(p, format, lw);
  for (uint64_t r = r0; r < r1; ++r) {
    char* o = out + r * rs;
    uint64_t gi = p->first_read + r;
    if (format != 0) {
      *o++ = format == 1 ? '>' : '@';
      *o++ = 'r';
      char d[13];
      snprintf(d, sizeof d, "%012llu", (unsigned long long)(gi % 1000000000000ull));
      memcpy(o, d, 12);
      o += 12;
      *o++ = '\n';
    }
    for (uint64_t j = 0; j < L; ++j) {
      *o++ = kLetters[synth_read_base(p, gi, j)];
      if (format == 1 && lw && (j + 1) % lw == 0 && j + 1 < L) *o++ = '\n';
    }
    *o++ = '\n';
    if (format == 2) {
      *o++ = '+';
      *o++ = '\n';
      memset(o, 'I', L);
      o += L;
      *o++ = '\n';
    }
  }
}

static int pick_threads(int threads) {
  if (threads > 0) return threads;
  unsigned h = std::thread::hardware_concurrency();
  return h ? (int)h : 1;
}

template <class F>
static void parallel_for(uint64_t n, int threads, F f) {
  threads = pick_threads(threads);
  if (threads <= 1 || n < 1024) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  uint64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    uint64_t a = t * per, b = a + per < n ? a + per : n;
    if (a >= b) break;
    ts.emplace_back([=] { f(a, b); });
  }
  for (auto& t : ts) t.join();
}

extern "C" {

/* format: 0 = raw (one read per line), 1 = FASTA (lines wrapped at
 * line_width, 0 = one line), 2 = FASTQ. Returns bytes needed; writes only if
 * out != NULL and cap is large enough. */
uint64_t synth_fastx(const synth_params* p, int format, uint32_t line_width,
                     char* out, uint64_t cap, int threads) {
  uint64_t need = rec_size(p, format, line_width) * p->n_reads;
  if (!out || cap < need) return need;
  parallel_for(p->n_reads, threads, [&](uint64_t a, uint64_t b) {
    emit_range(p, format, line_width, out, a, b);
  });
  return need;
}

/* Host twin of the device packer: codes[ceil(n*L/32)], nmask[ceil(n*L/64)],
 * read_start[n+1]. */
void synth_packed_host(const synth_params* p, uint64_t* codes, uint64_t* nmask,
                       uint64_t* read_start, int threads) {
  const uint64_t L = p->read_len, nb = p->n_reads * L;
  const uint64_t groups = (nb + 63) / 64;
  parallel_for(groups, threads, [&](uint64_t a, uint64_t b) {
    for (uint64_t g = a; g < b; ++g) {
      uint64_t c0 = 0, c1 = 0, nm = 0;
      for (uint32_t t = 0; t < 64; ++t) {
        uint64_t base = g * 64 + t;
        uint32_t c = 0;
        if (base < nb) c = synth_read_base(p, p->first_read + base / L, base % L);
        uint64_t code = c == 4u ? 0u : c;
        if (c == 4u) nm |= 1ull << (63 - t);
        if (t < 32) c0 |= code << (62 - 2 * t);
        else c1 |= code << (62 - 2 * (t - 32));
      }
      codes[2 * g] = c0;
      if (2 * g + 1 < (nb + 31) / 32) codes[2 * g + 1] = c1;
      nmask[g] = nm;
    }
  });
  for (uint64_t r = 0; r <= p->n_reads; ++r) read_start[r] = r * L;
}

} /* extern "C" */

__global__ void synth_packed_kernel(synth_params p, uint64_t* codes, uint64_t* nmask,
                                    uint64_t* read_start) {
  const uint64_t L = p.read_len, nb = p.n_reads * L;
  const uint64_t groups = (nb + 63) / 64, ncw = (nb + 31) / 32;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
       g += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c0 = 0, c1 = 0, nm = 0;
    uint64_t base0 = g * 64;
    uint64_t r = base0 / L, j = base0 % L;
    for (uint32_t t = 0; t < 64; ++t) {
      uint64_t base = base0 + t;
      uint32_t c = 0;
      if (base < nb) c = synth_read_base(&p, p.first_read + r, j);
      if (++j == L) { j = 0; ++r; }
      uint64_t code = c == 4u ? 0u : c;
      if (c == 4u) nm |= 1ull << (63 - t);
      if (t < 32) c0 |= code << (62 - 2 * t);
      else c1 |= code << (62 - 2 * (t - 32));
    }
    codes[2 * g] = c0;
    if (2 * g + 1 < ncw) codes[2 * g + 1] = c1;
    nmask[g] = nm;
  }
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= p.n_reads;
       r += (uint64_t)gridDim.x * blockDim.x)
    read_start[r] = r * L;
}

extern "C" int synth_packed_device(const synth_params* p, uint64_t* d_codes,
                                   uint64_t* d_nmask, uint64_t* d_read_start,
                                   void* stream) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  synth_packed_kernel<<<sms * 8, 256, 0, (cudaStream_t)stream>>>(*p, d_codes, d_nmask,
                                                                  d_read_start);
  return (int)cudaGetLastError();
}
