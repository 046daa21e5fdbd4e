// l2_micro.cu — B200 L2 random-access rates for the count kernel's access mix
// (a measurement tool, not part of the library). A table of T MiB (default
// 64, L2-resident) is hit at hashed random 64-byte buckets by a full grid:
//   load64   two 256-bit relaxed.gpu loads per op (the bucket view)
//   load32   one 256-bit load per op
//   red      one RED.ADD.32 per op
//   load+red bucket load, then RED into that bucket (the hit path)
//   cas128   one 128-bit CAS per op (compare 0, mostly failing)
//   load+cas bucket load, then CAS into that bucket (the claim path)
// Prints ops/s and sectors/s. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t (&w)[4]) {
  asm volatile("ld.global.relaxed.gpu.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld256cg(const uint64_t* p, uint64_t (&w)[4]) {
  asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld256w(const uint64_t* p, uint64_t (&w)[4]) {
  asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ uint64_t cas128(uint64_t* p, uint64_t s0, uint64_t s1) {
  uint64_t r0, r1;
  asm volatile("{ .reg .b128 t, c, s;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 s, {%4, %5};\n\t"
               "atom.global.cas.b128 t, [%6], c, s;\n\tmov.b128 {%0, %1}, t; }"
               : "=l"(r0), "=l"(r1) : "l"(0ull), "l"(0ull), "l"(s0), "l"(s1), "l"(p) : "memory");
  return r0 ^ r1;
}

template <int MODE>
__global__ void __launch_bounds__(128) kern(uint64_t* t, uint64_t nb, int iters, uint64_t* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint64_t h = mix(tid * 0x9E3779B97F4A7C15ULL + i);
    const uint64_t b = (uint64_t)(((unsigned __int128)h * nb) >> 64);
    uint64_t* bk = t + b * 8;
    if (MODE == 0 || MODE == 3 || MODE == 5) {
      uint64_t w[4], v[4];
      ld256(bk, w);
      ld256(bk + 4, v);
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
      if (MODE == 3) atomicAdd(reinterpret_cast<unsigned*>(bk + 1 + 2 * (acc & 3)), 1u);
      if (MODE == 5) acc += cas128(bk + 2 * (acc & 3), h, h | 1);
    } else if (MODE == 1) {
      uint64_t w[4];
      ld256(bk, w);
      acc += w[0] ^ w[3];
    } else if (MODE == 2) {
      atomicAdd(reinterpret_cast<unsigned*>(bk + 1 + 2 * (h & 3)), 1u);
    } else if (MODE == 4) {
      acc += cas128(bk + 2 * (h & 3), h, h | 1);
    } else if (MODE == 6 || MODE == 7) {  // weak (cg / default) bucket load + RED into it
      uint64_t w[4], v[4];
      if (MODE == 6) { ld256cg(bk, w); ld256cg(bk + 4, v); } else { ld256w(bk, w); ld256w(bk + 4, v); }
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
      atomicAdd(reinterpret_cast<unsigned*>(bk + 1 + 2 * (acc & 3)), 1u);
    } else if (MODE == 8) {  // strong bucket load + RED into an unrelated bucket
      uint64_t w[4], v[4];
      ld256(bk, w);
      ld256(bk + 4, v);
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
      const uint64_t b2 = (uint64_t)(((unsigned __int128)mix(h + 1) * nb) >> 64);
      atomicAdd(reinterpret_cast<unsigned*>(t + b2 * 8 + 1 + 2 * (acc & 3)), 1u);
    } else if (MODE == 9) {  // load + RED, loads and REDs on disjoint halves of the table
      const uint64_t half = nb / 2;
      const uint64_t bl = b % half, br = half + (uint64_t)(((unsigned __int128)mix(h + 1) * half) >> 64);
      uint64_t w[4], v[4];
      ld256(t + bl * 8, w);
      ld256(t + bl * 8 + 4, v);
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
      atomicAdd(reinterpret_cast<unsigned*>(t + br * 8 + 1 + 2 * (acc & 3)), 1u);
    } else if (MODE == 10) {  // RED then load of the same bucket
      atomicAdd(reinterpret_cast<unsigned*>(bk + 1 + 2 * (h & 3)), 1u);
      uint64_t w[4], v[4];
      ld256(bk, w);
      ld256(bk + 4, v);
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
    } else if (MODE == 12 || MODE == 13) {  // key bucket load + RED into a separate counts array
      uint64_t w[4], v[4];
      ld256(bk, w);
      ld256(bk + 4, v);
      acc += w[0] ^ v[1] ^ w[2] ^ v[3];
      unsigned* cnt = reinterpret_cast<unsigned*>(t + nb * 8);  // 16 B of counts per bucket after the keys
      if (MODE == 12) atomicAdd(cnt + b * 4 + (acc & 3), 1u);
      else asm volatile("red.global.add.u32 [%0], 1;" ::"l"(cnt + b * 4 + (acc & 3)) : "memory");
    } else if (MODE == 11) {  // independent pair: load of one bucket, RED into another, both random
      uint64_t w[4];
      ld256(bk, w);
      acc += w[0] ^ w[3];
      const uint64_t b2 = (uint64_t)(((unsigned __int128)mix(h + 7) * nb) >> 64);
      atomicAdd(reinterpret_cast<unsigned*>(t + b2 * 8 + 1), 1u);
    }
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

int main(int argc, char** argv) {
  const double mib = argc > 1 ? atof(argv[1]) : 64;
  const int bpsm = argc > 2 ? atoi(argv[2]) : 8;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t nb = (uint64_t)(mib * 1048576.0 / 64);
  uint64_t *t, *sink;
  cudaMalloc(&t, nb * 64 + nb * 16);
  cudaMalloc(&sink, 8);
  cudaMemset(t, 0x11, nb * 64 + nb * 16);  // non-zero: CAS(0 → x) fails, the table stays fixed
  const int grid = sms * bpsm, iters = 256;
  const double ops = (double)grid * 128 * iters;
  const char* names[] = {"load64", "load32", "red", "load+red", "cas128", "load+cas", "cg+red", "weak+red",
                         "load+redX", "ld|red", "red+load", "ld32+redX", "ld+redC", "ld+redC2"};
  const double sectors[] = {2, 1, 1, 3, 1, 3, 3, 3, 3, 3, 3, 2, 3, 3};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 14; ++mode) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      switch (mode) {
        case 0: kern<0><<<grid, 128>>>(t, nb, iters, sink); break;
        case 1: kern<1><<<grid, 128>>>(t, nb, iters, sink); break;
        case 2: kern<2><<<grid, 128>>>(t, nb, iters, sink); break;
        case 3: kern<3><<<grid, 128>>>(t, nb, iters, sink); break;
        case 4: kern<4><<<grid, 128>>>(t, nb, iters, sink); break;
        case 5: kern<5><<<grid, 128>>>(t, nb, iters, sink); break;
        case 6: kern<6><<<grid, 128>>>(t, nb, iters, sink); break;
        case 7: kern<7><<<grid, 128>>>(t, nb, iters, sink); break;
        case 8: kern<8><<<grid, 128>>>(t, nb, iters, sink); break;
        case 9: kern<9><<<grid, 128>>>(t, nb, iters, sink); break;
        case 10: kern<10><<<grid, 128>>>(t, nb, iters, sink); break;
        case 11: kern<11><<<grid, 128>>>(t, nb, iters, sink); break;
        case 12: kern<12><<<grid, 128>>>(t, nb, iters, sink); break;
        case 13: kern<13><<<grid, 128>>>(t, nb, iters, sink); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (rep > 0 && ms < best) best = ms;
    }
    const double gops = ops / (best * 1e-3) / 1e9;
    printf("table=%.0fMiB ctas/sm=%d %-9s %8.2f Gop/s %8.1f Gsector/s  (%.3f ms)\n", mib, bpsm, names[mode], gops,
           gops * sectors[mode], best);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
