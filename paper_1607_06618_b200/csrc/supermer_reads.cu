// supermer_reads.cu — step (b), read-per-lane variant (w = k-m+1 <= 64).
//
// Same definitions as supermer.cu (§2.1; strand-symmetric
// minimizers, Q7; value-based runs, Q8; windows never span an N or a
// read boundary), computed by streaming each read through one
// lane — no block barriers, everything in registers except two small per-lane
// shared-memory rings (bank-interleaved: entry t of lane l at [t%64][l]).
//
// Window minimum (sliding minimum over w ordering keys, van Herk / Gil-Werman
// in streaming form): the m-mer positions q of a read are cut into blocks of w
// (q / w); `pre` is the running minimum of the current block; when a block
// completes, a backward pass writes its suffix minima to the ring `suf`. The
// window [p, p+w-1] = [p, q] then has μ_p = min(suf[p], pre) (or pre when p
// starts a block). Every lane starts its read at step j = 0, so block ends
// coincide across the warp and the backward pass is warp-uniform.
// Runs of equal μ become super-mers (cut every kRunCap windows); runs are
// buffered per lane and flushed warp-cooperatively (one global atomic per
// flush). Long reads (> 4096 bases on average) use the tile kernel.
#include "common.cuh"
#include "kernels.h"
#include "ordering.cuh"

namespace gerbil {
namespace {

constexpr int kLanes = 32;
constexpr int kWarpsPerCta = 2;
constexpr int kRing = 64;           // >= w
constexpr int kBuf = 8;             // runs buffered per lane
constexpr uint32_t kRunCap = 2048;  // windows per descriptor (11-bit length field)

struct WarpShared {
  uint32_t key[kRing][kLanes];
  uint32_t suf[kRing][kLanes];
  uint64_t bdesc[kBuf][kLanes];
  uint32_t bmu[kBuf][kLanes];
};

__global__ void __launch_bounds__(kLanes * kWarpsPerCta)
supermer_reads_kernel(SupermerArgs a, unsigned long long* work) {
  __shared__ WarpShared s_w[kWarpsPerCta];
  const uint32_t lane = lane_id();
  WarpShared& S = s_w[threadIdx.x >> 5];
  const uint32_t k = a.k, m = a.m, w = k - m + 1, B = a.n_bins;
  const uint32_t mmask = (uint32_t)((1ull << (2 * m)) - 1);
  const OrderCtx ord = make_order(a.ordering, m, a.order_rank);
  const uint32_t top = 2 * m - 2;
  const uint64_t n_code_words = (a.n_bases + 31) / 32, n_mask_words = (a.n_bases + 63) / 64;
  uint64_t my_windows = 0;
  uint32_t nbuf = 0;  // this lane's buffered runs

  // flush every lane's buffer: one atomic per warp, then each lane writes its runs
  auto flush = [&]() {
    uint32_t incl = nbuf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(a.n_supermers, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 31);
    uint64_t idx = base + incl - nbuf;
    for (uint32_t e = 0; e < nbuf; ++e, ++idx) {
      const uint64_t d = S.bdesc[e][lane];
      const uint32_t key = S.bmu[e][lane];
      const uint32_t b = (uint32_t)(((uint64_t)fmix32(key) * B) >> 32);
      const uint32_t nwin = (uint32_t)(d & ((1u << kNwinBits) - 1)) + 1;
      if (idx < a.cap) {
        a.desc[idx] = d;
        a.bin[idx] = b;
        if (a.mu) a.mu[idx] = key;
      }
      if (a.bin_windows) {
        atomicAdd(&a.bin_windows[b], (unsigned long long)nwin);
        atomicAdd(&a.bin_supermers[b], 1ull);
      }
      if (a.bin_words) atomicAdd(&a.bin_words[b], (unsigned long long)((nwin + k - 1 + 31) / 32));
    }
    nbuf = 0;
    __syncwarp();
  };
  auto push_run = [&](uint64_t s, uint32_t start, uint32_t end, uint32_t mu) {  // windows [start, end)
    S.bdesc[nbuf][lane] = ((s + start) << kNwinBits) | (end - start - 1);
    S.bmu[nbuf][lane] = mu;
    ++nbuf;
    my_windows += end - start;
  };

  for (;;) {
    unsigned long long r0 = 0;
    if (lane == 0) r0 = atomicAdd(work, 32ull);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    if (r0 >= a.n_reads) break;
    const uint64_t r = r0 + lane;
    uint64_t s = 0, len = 0;
    if (r < a.n_reads) {
      s = __ldg(a.read_start + r);
      len = __ldg(a.read_start + r + 1) - s;
    }
    uint64_t cw = 0, nw = 0, cn = 0, nn = 0;  // current and next code / N words
    uint32_t f = 0, rc = 0, fill = 0;         // rolling m-mer, bases since the last N
    uint32_t pre = 0xffffffffu, bpos = 0;     // prefix min of the current key block, q % w
    bool run = false;
    uint32_t run_start = 0, run_mu = 0;
    uint64_t lmax = len;  // the warp walks its longest read; shorter reads idle at the end
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    for (uint64_t j = 0; j < lmax; ++j) {
      const bool act = j < len;
      uint32_t c = 0xffffffffu;  // ordering key of the m-mer ending at j (∞ if invalid)
      bool isn = false;
      if (act) {
        const uint64_t g = s + j;
        if (j == 0) {  // code / N words with one word of prefetch
          cw = __ldg(a.codes + (g >> 5));
          cn = ((g >> 5) + 1 < n_code_words) ? __ldg(a.codes + (g >> 5) + 1) : 0ull;
          if (a.nmask) {
            nw = __ldg(a.nmask + (g >> 6));
            nn = ((g >> 6) + 1 < n_mask_words) ? __ldg(a.nmask + (g >> 6) + 1) : 0ull;
          }
        } else {
          if ((g & 31) == 0) {
            cw = cn;
            cn = ((g >> 5) + 1 < n_code_words) ? __ldg(a.codes + (g >> 5) + 1) : 0ull;
          }
          if (a.nmask && (g & 63) == 0) {
            nw = nn;
            nn = ((g >> 6) + 1 < n_mask_words) ? __ldg(a.nmask + (g >> 6) + 1) : 0ull;
          }
        }
        const uint32_t b = (uint32_t)(cw >> (62 - 2 * (g & 31))) & 3u;
        isn = a.nmask && ((nw >> (63 - (g & 63))) & 1ull);
        if (isn) {
          fill = 0;
        } else {
          ++fill;
          f = ((f << 2) | b) & mmask;
          rc = (rc >> 2) | ((3u - b) << top);
          if (fill >= m) {
            const uint32_t kf = order_key(f, ord), kr = order_key(rc, ord);
            c = kf < kr ? kf : kr;
          }
        }
      }
      // key block bookkeeping for q = j-m+1 (warp-uniform: every lane is at the same j)
      if (j + 1 >= m) {
        const uint32_t q = (uint32_t)(j + 1 - m);
        pre = (bpos == 0) ? c : min(pre, c);
        S.key[q & (kRing - 1)][lane] = c;
        if (act && fill >= k) {  // window p = j-k+1 = q-w+1, all of it N-free and in this read
          const uint32_t p = q - w + 1;
          const uint32_t mu = (bpos == w - 1) ? pre : min(S.suf[p & (kRing - 1)][lane], pre);
          if (!(run && mu == run_mu && p - run_start < kRunCap)) {  // value-based runs
            if (run) push_run(s, run_start, p, run_mu);
            run = true;
            run_start = p;
            run_mu = mu;
          }
        }
        if (bpos == w - 1) {  // block [q-w+1, q] complete: its suffix minima
          uint32_t sm = 0xffffffffu;
          for (uint32_t t = 0; t < w; ++t) {
            const uint32_t qq = q - t;
            sm = min(sm, S.key[qq & (kRing - 1)][lane]);
            S.suf[qq & (kRing - 1)][lane] = sm;
          }
          bpos = 0;
        } else {
          ++bpos;
        }
      }
      if (act && isn && run) {  // an N ends the open run: windows up to j-k are in it
        push_run(s, run_start, (uint32_t)(j + 1 - k), run_mu);
        run = false;
      }
      if (__any_sync(0xffffffffu, nbuf >= kBuf - 1)) flush();
    }
    if (run) push_run(s, run_start, (uint32_t)(len - k + 1), run_mu);  // read end closes the run
    if (__any_sync(0xffffffffu, nbuf >= kBuf - 1)) flush();
  }
  flush();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_windows += __shfl_down_sync(0xffffffffu, my_windows, o);
  if (lane == 0 && my_windows) atomicAdd(a.n_windows, (unsigned long long)my_windows);
}

}  // namespace

bool supermer_reads_applicable(uint32_t k, uint32_t m, uint64_t n_bases, uint64_t n_reads) {
  return n_reads > 0 && k - m + 1 <= (uint32_t)kRing && n_bases / n_reads <= 4096;
}

cudaError_t launch_supermer_reads(const SupermerArgs& a, unsigned long long* work, int sms, cudaStream_t st) {
  if (a.n_reads == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(work, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, supermer_reads_kernel, kLanes * kWarpsPerCta, 0);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * per_sm;
  const uint64_t need = (a.n_reads + kLanes * kWarpsPerCta - 1) / (kLanes * kWarpsPerCta);
  if (grid > need) grid = need;
  supermer_reads_kernel<<<(unsigned)grid, kLanes * kWarpsPerCta, 0, st>>>(a, work);
  return cudaGetLastError();
}

}  // namespace gerbil
