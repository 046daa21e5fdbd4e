// ordering.cu — data-dependent pieces of the minimizer orderings
// (§3.1).
//
//  - dfp_sample_kernel: m-mer frequencies for dfp(p) ("we approximate them by
//    taking samples during runtime"). Sample = every m-mer
//    occurrence starting in a 1024-position tile t ≡ 0 (mod stride) of the
//    batch, inside one read and free of undetermined bases; each occurrence
//    counts for f and rc(f) (reading Q23). The host turns the
//    histogram into the key table (api.cu, build_dfp_table).
//  - minimizer_hist_kernel + hist_max_kernel: the Fig. Minimizer metric
//     — distinct k-mers per strand-symmetric minimizer
//    over a count's results, and its maximum.
#include "common.cuh"
#include "kernels.h"
#include "ordering.cuh"

namespace gerbil {
namespace {

// any set bit among positions [a, b] (b - a < 64) of an MSB-first bitmap
__device__ __forceinline__ bool any_bit(const uint64_t* bm, uint64_t a, uint64_t b) {
  const uint64_t wa = a >> 6, wb = b >> 6;
  const uint32_t oa = (uint32_t)(a & 63), ob = (uint32_t)(b & 63);
  if (wa == wb) return (bm[wa] & ((~0ull >> oa) & (~0ull << (63 - ob)))) != 0;
  return (bm[wa] & (~0ull >> oa)) != 0 || (bm[wb] & (~0ull << (63 - ob))) != 0;
}

__global__ void dfp_sample_kernel(const uint64_t* __restrict__ codes, const uint64_t* __restrict__ nmask,
                                  const uint64_t* __restrict__ rs, uint64_t n_bases, uint32_t m, uint32_t stride,
                                  uint32_t* freq, int smem_hist) {
  extern __shared__ uint32_t s_f[];
  const uint32_t M = 1u << (2 * m), mask = M - 1;
  if (smem_hist) {
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) s_f[i] = 0;
    __syncthreads();
  }
  const uint64_t n_tiles = (n_bases + 1023) / 1024, n_samp = (n_tiles + stride - 1) / stride;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_samp * 1024;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = (i >> 10) * stride * 1024 + (i & 1023);
    if (j + m > n_bases) continue;
    if (nmask && any_bit(nmask, j, j + m - 1)) continue;  // undetermined base
    if (m > 1 && any_bit(rs, j + 1, j + m - 1)) continue;  // a read starts inside
    const uint32_t w = (uint32_t)(j & 31) * 2;
    const uint64_t c0 = codes[j >> 5];
    const uint64_t v = w ? (c0 << w) | ((j >> 5) + 1 < (n_bases + 31) / 32 ? codes[(j >> 5) + 1] >> (64 - w) : 0ull)
                         : c0;
    const uint32_t f = (uint32_t)(v >> (64 - 2 * m));
    const uint32_t rc = (uint32_t)(rev_pairs(~v & (~0ull << (64 - 2 * m))) & mask);
    if (smem_hist) {
      atomicAdd(&s_f[f], 1u);
      atomicAdd(&s_f[rc], 1u);
    } else {
      atomicAdd(&freq[f], 1u);
      atomicAdd(&freq[rc], 1u);
    }
  }
  if (smem_hist) {
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < M; x += blockDim.x)
      if (s_f[x]) atomicAdd(&freq[x], s_f[x]);
  }
}

// one result k-mer per thread: μ = min over its m-mers f of min(key f, key rc f)
__global__ void minimizer_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t W, uint32_t k,
                                      OrderCtx ord, uint32_t* hist) {
  const uint32_t m = ord.m;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t* x = keys + i * W;
    uint32_t f = 0, rc = 0, mu = 0xffffffffu;
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t b = (uint32_t)(x[j >> 5] >> (62 - 2 * (j & 31))) & 3u;
      f = ((f << 2) | b) & ord.mask;
      rc = (rc >> 2) | ((3u - b) << (2 * m - 2));
      if (j + 1 >= m) mu = min(mu, min(order_key(f, ord), order_key(rc, ord)));
    }
    atomicAdd(&hist[mu], 1u);
  }
}

__global__ void hist_max_kernel(const uint32_t* __restrict__ hist, uint64_t n, unsigned long long* out) {
  uint32_t mx = 0, nz = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    mx = max(mx, hist[i]);
    nz += hist[i] != 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
    nz += __shfl_down_sync(0xffffffffu, nz, o);
  }
  if (lane_id() == 0) {
    atomicMax(out, (unsigned long long)mx);
    atomicAdd(out + 1, (unsigned long long)nz);
  }
}

}  // namespace

cudaError_t launch_dfp_sample(const uint64_t* codes, const uint64_t* nmask, const uint64_t* rs_bits,
                              uint64_t n_bases, uint32_t m, uint32_t stride, uint32_t* freq, int sms,
                              cudaStream_t st) {
  const uint32_t M = 1u << (2 * m);
  const int smem_hist = M <= 16384;  // m <= 7: a 64 KB per-CTA histogram
  const size_t dyn = smem_hist ? (size_t)M * 4 : 0;
  cudaError_t e = cudaFuncSetAttribute(dfp_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  dfp_sample_kernel<<<sms * 2, 512, dyn, st>>>(codes, nmask, rs_bits, n_bases, m, stride, freq, smem_hist);
  return cudaGetLastError();
}

cudaError_t launch_minimizer_hist(const uint64_t* keys, uint64_t n, uint32_t W, uint32_t k, uint32_t m,
                                  uint32_t ordering, const uint32_t* rank, uint32_t* hist, uint64_t hist_n,
                                  unsigned long long* out2, int sms, cudaStream_t st) {
  if (n) {
    uint64_t g = (n + 255) / 256;
    if (g > (uint64_t)sms * 8) g = (uint64_t)sms * 8;
    minimizer_hist_kernel<<<(unsigned)g, 256, 0, st>>>(keys, n, W, k, make_order(ordering, m, rank), hist);
  }
  hist_max_kernel<<<sms * 4, 256, 0, st>>>(hist, hist_n, out2);
  return cudaGetLastError();
}

}  // namespace gerbil
