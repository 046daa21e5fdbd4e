// pcie_micro.cu — host<->device transfer rates on one B200 (measurement tool):
// cudaMemcpyAsync H2D / D2H from pinned memory, and kernel stores straight
// into mapped pinned host memory (16-byte coalesced, grid of G CTAs).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void store_host(uint4* dst, const uint4* src, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// compaction-like pattern: each CTA iteration writes its own contiguous chunk of
// `chunk` bytes (16-byte stores) at a position taken from a global counter
__global__ void chunks_to_host(uint8_t* dst, const uint8_t* src, uint64_t total, uint32_t chunk,
                               unsigned long long* ctr) {
  __shared__ unsigned long long base;
  for (;;) {
    if (threadIdx.x == 0) base = atomicAdd(ctr, (unsigned long long)chunk);
    __syncthreads();
    const unsigned long long b0 = base;
    __syncthreads();
    if (b0 >= total) return;
    const uint32_t n = (uint32_t)((total - b0 < chunk ? total - b0 : chunk) / 16);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
      reinterpret_cast<uint4*>(dst + b0)[i] = reinterpret_cast<const uint4*>(src + b0)[i];
  }
}

// L2 atomic load (like the count kernel): random REDs on a 64 MiB table
__global__ void red_storm(unsigned* t, uint64_t n, int iters) {
  uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 6364136223846793005ULL + 1442695040888963407ULL;
    atomicAdd(t + ((x >> 20) % n), 1u);
  }
}

int main() {
  const uint64_t bytes = 1ull << 30;
  void *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  cudaMalloc(&d, bytes);
  cudaMemset(d, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int dir = 0; dir < 2; ++dir) {
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      if (dir == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
      else cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("memcpy %s  %.1f GB/s\n", dir == 0 ? "H2D" : "D2H", bytes / (best * 1e-3) / 1e9);
  }
  void* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  for (int g : {8, 16, 32, 64, 148, 296}) {
    float best = 1e9f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      store_host<<<g, 256>>>((uint4*)hd, (const uint4*)d, bytes / 16);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("kernel stores to mapped host, %3d CTAs x 256: %.1f GB/s\n", g, bytes / (best * 1e-3) / 1e9);
  }
  {
    unsigned long long* ctr;
    cudaMalloc(&ctr, 8);
    for (uint32_t chunk : {4096u, 16384u, 65536u}) {
      for (int g : {64, 148, 592}) {
        float best = 1e9f;
        for (int r = 0; r < 3; ++r) {
          cudaMemset(ctr, 0, 8);
          cudaEventRecord(a);
          chunks_to_host<<<g, 256>>>((uint8_t*)hd, (const uint8_t*)d, bytes, chunk, ctr);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf("chunked stores to host, chunk %6u B, %3d CTAs: %.1f GB/s\n", chunk, g, bytes / (best * 1e-3) / 1e9);
      }
    }
    // the same while an L2-RED storm runs on another stream
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    unsigned* tab;
    const uint64_t tn = (64ull << 20) / 4;
    cudaMalloc(&tab, tn * 4);
    cudaEvent_t c, e2;
    cudaEventCreate(&c);
    cudaEventCreate(&e2);
    cudaMemset(ctr, 0, 8);
    red_storm<<<148 * 4, 256, 0, s2>>>(tab, tn, 4000);
    cudaEventRecord(c, s1);
    chunks_to_host<<<148, 256, 0, s1>>>((uint8_t*)hd, (const uint8_t*)d, bytes, 16384, ctr);
    cudaEventRecord(e2, s1);
    cudaEventSynchronize(e2);
    cudaEventElapsedTime(&ms, c, e2);
    printf("chunked stores to host (16 KB, 148 CTAs) during an L2 RED storm: %.1f GB/s\n", bytes / (ms * 1e-3) / 1e9);
    cudaDeviceSynchronize();
    cudaEventRecord(c, s2);
    red_storm<<<148 * 4, 256, 0, s2>>>(tab, tn, 4000);
    cudaEventRecord(e2, s2);
    cudaEventSynchronize(e2);
    cudaEventElapsedTime(&ms, c, e2);
    printf("RED storm alone: %.2f ms\n", ms);
  }
  // concurrent H2D + D2H
  {
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    void *h2, *d2;
    cudaHostAlloc(&h2, bytes, 0);
    cudaMalloc(&d2, bytes);
    cudaEventRecord(a);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2);
    cudaStreamSynchronize(s1);
    cudaStreamSynchronize(s2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("concurrent H2D + D2H (1 GiB each): %.1f ms (%.1f GB/s aggregate)\n", ms, 2 * bytes / (ms * 1e-3) / 1e9);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
