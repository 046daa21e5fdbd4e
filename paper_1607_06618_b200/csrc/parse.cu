// parse.cu — step (a) on the device: FASTA / FASTQ / raw text → packed batch
// ("phase one on the GPU" is the paper's future
// work). Same result, bit for bit, as the host reader
// (reader.cpp, readings Q3/Q4): lines end at '\n'; every '\r' is dropped;
// the kind is set by the first non-empty line ('>' FASTA, '@' FASTQ, else
// one read per line); empty lines are skipped (inside a FASTQ record an empty
// sequence is a read of length 0); A/C/G/T (either case) → 2-bit codes, every
// other byte → an undetermined (N) base.
//
// Passes (all integer; one read of the text per pass):
//  1. count '\n' and '\r' per 16 KiB block, scan, write their positions;
//  2. per line: length without CRs (binary search in the CR list — CRs are
//     rare) and first non-CR byte;
//  3. per line: role (FASTA header / sequence, FASTQ by line index mod 4,
//     raw), validation (FASTQ '@' / '+' / quality length / truncation), the
//     sequence length and the read-start flag;
//  4. exclusive scans → base offset of every sequence line, index of every read;
//  5. read starts; then one warp per sequence line packs its bytes: 32 bytes
//     per step, CRs squeezed out with a ballot, codes and N bits assembled by
//     warp OR-reductions and merged into the zeroed batch with atomic ORs
//     (only words shared with a neighbouring line are really contended).
// The device parser needs FASTQ without empty lines between records (the
// host reader skips those); such input is reported, not guessed.
#include "common.cuh"
#include "kernels.h"

namespace gerbil {
namespace {

constexpr int kPT = 256;                 // threads per block
constexpr uint64_t kBlk = kPT * 64ull;   // bytes per block (64 per thread)

__device__ __forceinline__ void load64(const uint8_t* t, uint64_t len, uint64_t i0, uint8_t (&b)[64]) {
  if (i0 + 64 <= len) {
    const uint4* p = reinterpret_cast<const uint4*>(t + i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = p[q];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) b[16 * q + j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 64; ++j) b[j] = i0 + j < len ? t[i0 + j] : 0;
  }
}

// exclusive scan across a block of kPT threads (returns the block total in *tot)
__device__ __forceinline__ uint32_t block_excl(uint32_t v, uint32_t* sh, uint32_t* tot) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t s = threadIdx.x < kPT / 32 ? sh[threadIdx.x] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= (uint32_t)o) s += y;
    }
    if (threadIdx.x < kPT / 32) sh[threadIdx.x] = s;
  }
  __syncthreads();
  const uint32_t before = (w ? sh[w - 1] : 0) + x - v;
  *tot = sh[kPT / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kPT) count_nl_cr_kernel(const uint8_t* t, uint64_t len, uint32_t* cnt_nl,
                                                          uint32_t* cnt_cr) {
  __shared__ uint32_t sh[kPT / 32];
  const uint64_t i0 = blockIdx.x * kBlk + threadIdx.x * 64ull;
  uint8_t b[64];
  load64(t, len, i0, b);
  uint32_t nl = 0, cr = 0;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    nl += b[j] == '\n';
    cr += b[j] == '\r';
  }
  uint32_t tot;
  block_excl(nl, sh, &tot);
  if (threadIdx.x == 0) cnt_nl[blockIdx.x] = tot;
  block_excl(cr, sh, &tot);
  if (threadIdx.x == 0) cnt_cr[blockIdx.x] = tot;
}

// line_start[1 + r] = position after the r-th '\n'; cr_pos[r] = position of the r-th '\r'
__global__ void __launch_bounds__(kPT) write_nl_cr_kernel(const uint8_t* t, uint64_t len, const uint64_t* off_nl,
                                                          const uint64_t* off_cr, uint64_t* line_start,
                                                          uint64_t* cr_pos) {
  __shared__ uint32_t sh[kPT / 32];
  const uint64_t i0 = blockIdx.x * kBlk + threadIdx.x * 64ull;
  uint8_t b[64];
  load64(t, len, i0, b);
  uint32_t nl = 0, cr = 0;
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    nl += b[j] == '\n';
    cr += b[j] == '\r';
  }
  uint32_t tot;
  uint64_t o_nl = off_nl[blockIdx.x] + block_excl(nl, sh, &tot);
  uint64_t o_cr = off_cr[blockIdx.x] + block_excl(cr, sh, &tot);
#pragma unroll
  for (int j = 0; j < 64; ++j) {
    if (b[j] == '\n') line_start[1 + o_nl++] = i0 + j + 1;
    if (b[j] == '\r') cr_pos[o_cr++] = i0 + j;
  }
}

// ---- exclusive scan of u64 arrays: block sums → one-block scan of the sums → apply
constexpr int kSPer = 8;                     // elements per thread
constexpr uint64_t kSBlk = kPT * kSPer;      // elements per block

__device__ __forceinline__ uint64_t block_excl64(uint64_t v, uint64_t* sh, uint64_t* tot) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t z = threadIdx.x < kPT / 32 ? sh[threadIdx.x] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= (uint32_t)o) z += y;
    }
    if (threadIdx.x < kPT / 32) sh[threadIdx.x] = z;
  }
  __syncthreads();
  const uint64_t before = (w ? sh[w - 1] : 0) + x - v;
  *tot = sh[kPT / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kPT) scan_sums_kernel(const uint64_t* in, uint64_t n, uint64_t* sums) {
  __shared__ uint64_t sh[kPT / 32];
  const uint64_t i0 = blockIdx.x * kSBlk + threadIdx.x * (uint64_t)kSPer;
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kSPer; ++j) s += i0 + j < n ? in[i0 + j] : 0;
  uint64_t tot;
  block_excl64(s, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kPT) scan_apply_kernel(const uint64_t* in, uint64_t n, const uint64_t* sums,
                                                         uint64_t* out) {
  __shared__ uint64_t sh[kPT / 32];
  const uint64_t i0 = blockIdx.x * kSBlk + threadIdx.x * (uint64_t)kSPer;
  uint64_t x[kSPer], s = 0;
#pragma unroll
  for (int j = 0; j < kSPer; ++j) {
    x[j] = i0 + j < n ? in[i0 + j] : 0;
    s += x[j];
  }
  uint64_t tot;
  uint64_t run = sums[blockIdx.x] + block_excl64(s, sh, &tot);
#pragma unroll
  for (int j = 0; j < kSPer; ++j)
    if (i0 + j < n) {
      out[i0 + j] = run;
      run += x[j];
    }
}

// exclusive scan in place by one block (block sums; a few hundred thousand entries at most)
__global__ void __launch_bounds__(1024) scan_small_kernel(uint64_t* v, uint64_t n, uint64_t* total) {
  __shared__ uint64_t carry;
  __shared__ uint64_t ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t x = i < n ? v[i] : 0;
    uint64_t s = x;
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= (uint32_t)o) s += y;
    }
    if (lane == 31) ws[w] = s;
    __syncthreads();
    if (w == 0) {
      uint64_t z = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= (uint32_t)o) z += y;
      }
      ws[lane] = z;
    }
    __syncthreads();
    const uint64_t incl = s + (w ? ws[w - 1] : 0);
    if (i < n) v[i] = carry + incl - x;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void widen_kernel(const uint32_t* a, uint64_t* b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// number of CR positions in [a, b)
__device__ __forceinline__ uint64_t cr_in(const uint64_t* cr, uint64_t n_cr, uint64_t a, uint64_t b) {
  uint64_t lo = 0, hi = n_cr;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cr[mid] < a) lo = mid + 1;
    else hi = mid;
  }
  const uint64_t first = lo;
  hi = n_cr;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cr[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo - first;
}

// line i spans [ls[i], ls[i+1] - 1): eff = bytes without CR, first = first non-CR byte (0 if none)
__global__ void line_info_kernel(const uint8_t* t, const uint64_t* ls, uint64_t n_lines, const uint64_t* cr,
                                 uint64_t n_cr, uint32_t* eff, uint8_t* first, unsigned long long* first_nonempty) {
  unsigned long long lo = ~0ull, hi = 0;  // this thread's first / last non-empty line
  bool any = false;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_lines;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = ls[i], b = ls[i + 1] - 1;
    const uint64_t c = n_cr ? cr_in(cr, n_cr, a, b) : 0;
    const uint32_t e = (uint32_t)(b - a - c);
    eff[i] = e;
    uint8_t f = 0;
    for (uint64_t p = a; p < b; ++p)
      if (t[p] != '\r') {
        f = t[p];
        break;
      }
    first[i] = f;
    if (e) {
      lo = min(lo, (unsigned long long)i);
      hi = max(hi, (unsigned long long)i);
      any = true;
    }
  }
  // first_nonempty[0] = min, [1] = max index of a non-empty line: one atomic pair per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) {
    atomicMin(first_nonempty, lo);
    atomicMax(first_nonempty + 1, hi);
  }
}

enum : uint32_t { kErrNone = 0, kErrAt = 1, kErrPlus = 2, kErrQual = 3, kErrTrunc = 4, kErrIrregular = 5 };

// roles; seq_len[i] (u64) = bases the line contributes; rflag[i] = 1 if line i starts a read
__global__ void classify_kernel(const uint32_t* eff, const uint8_t* first, uint64_t n_lines, uint64_t f0,
                                uint64_t n_eff, int kind, uint64_t* seq_len, uint64_t* rflag,
                                unsigned long long* err) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_lines;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = eff[i];
    uint64_t sl = 0, rf = 0;
    if (i >= f0 && i < n_eff) {  // lines before the first / after the last non-empty one are skipped
      if (kind == 0) {  // FASTA
        if (e && first[i] == '>') rf = 1;
        else sl = e;
      } else if (kind == 1) {  // FASTQ, 4 physical lines per record
        const uint32_t role = (uint32_t)((i - f0) & 3);
        unsigned long long code = kErrNone;
        if (role == 0) {
          if (e == 0) code = kErrIrregular;
          else if (first[i] != '@') code = kErrAt;
        } else if (role == 1) {
          sl = e;
          rf = 1;
        } else if (role == 2) {
          if (first[i] != '+') code = kErrPlus;
        } else if (e != eff[i - 2]) {
          code = kErrQual;
        }
        if (i + 1 == n_eff && role != 3 && code == kErrNone) code = kErrTrunc;
        if (code != kErrNone) atomicMin(err, ((unsigned long long)i << 8) | code);
      } else {  // raw: one read per non-empty line
        if (e) {
          sl = e;
          rf = 1;
        }
      }
    }
    seq_len[i] = sl;
    rflag[i] = rf;
  }
}

// read_start[ridx[i]] = pos[i] for every read-start line
__global__ void read_starts_kernel(const uint64_t* pos, const uint64_t* rflag, const uint64_t* ridx, uint64_t n_lines,
                                   uint64_t* read_start) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_lines;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (rflag[i]) read_start[ridx[i]] = pos[i];
}

// one warp per line with bases: 32 bytes per step → codes / N bits at pos[i]...
__global__ void pack_lines_kernel(const uint8_t* t, const uint64_t* ls, const uint64_t* seq_len, const uint64_t* pos,
                                  uint64_t n_lines, unsigned long long* codes, unsigned long long* nmask) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n_lines; i += n_warps) {
    if (seq_len[i] == 0) continue;  // warp-uniform
    const uint64_t a = ls[i], b = ls[i + 1] - 1;
    uint64_t q = pos[i];  // global base position of the next base
    uint32_t pre = 0;     // bytes of the next four 32-byte steps (one per byte lane), loaded together
    for (uint64_t p0 = a; p0 < b; p0 += 32) {
      const uint32_t st = (uint32_t)((p0 - a) >> 5) & 3;
      if (st == 0) {
        pre = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t pu = p0 + 32 * u + lane;
          pre |= (uint32_t)(pu < b ? t[pu] : (uint8_t)'\r') << (8 * u);
        }
      }
      const uint8_t ch = (uint8_t)(pre >> (8 * st));
      const bool valid = ch != '\r';
      const uint32_t vm = __ballot_sync(0xffffffffu, valid);
      const uint32_t j = __popc(vm & ((1u << lane) - 1u));  // base index inside this step
      uint32_t code = 0, isn = 1;
      switch (ch) {
        case 'A': case 'a': code = 0; isn = 0; break;
        case 'C': case 'c': code = 1; isn = 0; break;
        case 'G': case 'g': code = 2; isn = 0; break;
        case 'T': case 't': code = 3; isn = 0; break;
        default: break;
      }
      // 32 bases → 64 code bits, MSB first: base j in bits [63-2j, 62-2j]
      const uint32_t hi = __reduce_or_sync(0xffffffffu, valid && j < 16 ? code << (30 - 2 * j) : 0u);
      const uint32_t lo = __reduce_or_sync(0xffffffffu, valid && j >= 16 ? code << (30 - 2 * (j - 16)) : 0u);
      const uint32_t nb = __reduce_or_sync(0xffffffffu, valid && isn ? 1u << (31 - j) : 0u);
      const uint32_t n = __popc(vm);
      if (lane == 0 && n) {
        const uint64_t w = ((uint64_t)hi << 32) | lo;  // bases q .. q+n-1, left-aligned
        const uint32_t s = (uint32_t)(q & 31) * 2;
        atomicOr(codes + (q >> 5), (unsigned long long)(w >> s));
        if (s && (q & 31) + n > 32) atomicOr(codes + (q >> 5) + 1, (unsigned long long)(w << (64 - s)));
        if (nb) {
          const uint64_t nw = (uint64_t)nb << 32;  // bits q .. q+n-1, left-aligned
          const uint32_t sn = (uint32_t)(q & 63);
          atomicOr(nmask + (q >> 6), (unsigned long long)(nw >> sn));
          if (sn && sn + n > 64) atomicOr(nmask + (q >> 6) + 1, (unsigned long long)(nw << (64 - sn)));
        }
      }
      q += n;
    }
  }
}

}  // namespace

// ---- launchers (api.cu orchestrates, include/gerbil.h gerbil_parse_text) -----------------

uint64_t parse_blocks(uint64_t len) { return (len + kBlk - 1) / kBlk; }

cudaError_t launch_parse_count(const uint8_t* t, uint64_t len, uint32_t* cnt_nl, uint32_t* cnt_cr, cudaStream_t st) {
  const uint64_t nb = parse_blocks(len);
  if (nb) count_nl_cr_kernel<<<(unsigned)nb, kPT, 0, st>>>(t, len, cnt_nl, cnt_cr);
  return cudaGetLastError();
}

cudaError_t launch_widen(const uint32_t* a, uint64_t* b, uint64_t n, int sms, cudaStream_t st) {
  if (n) widen_kernel<<<sms * 4, 256, 0, st>>>(a, b, n);
  return cudaGetLastError();
}

uint64_t scan_tmp_words(uint64_t n) { return (n + kSBlk - 1) / kSBlk + 1; }

cudaError_t launch_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* tmp, uint64_t* total,
                            cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t nb = (n + kSBlk - 1) / kSBlk;
  scan_sums_kernel<<<(unsigned)nb, kPT, 0, st>>>(in, n, tmp);
  scan_small_kernel<<<1, 1024, 0, st>>>(tmp, nb, total);
  scan_apply_kernel<<<(unsigned)nb, kPT, 0, st>>>(in, n, tmp, out);
  return cudaGetLastError();
}

cudaError_t launch_parse_write(const uint8_t* t, uint64_t len, const uint64_t* off_nl, const uint64_t* off_cr,
                               uint64_t* line_start, uint64_t* cr_pos, cudaStream_t st) {
  const uint64_t nb = parse_blocks(len);
  if (nb) write_nl_cr_kernel<<<(unsigned)nb, kPT, 0, st>>>(t, len, off_nl, off_cr, line_start, cr_pos);
  return cudaGetLastError();
}

cudaError_t launch_parse_lines(const uint8_t* t, const uint64_t* ls, uint64_t n_lines, const uint64_t* cr,
                               uint64_t n_cr, uint32_t* eff, uint8_t* first, unsigned long long* first_nonempty,
                               int sms, cudaStream_t st) {
  if (n_lines) line_info_kernel<<<sms * 8, 256, 0, st>>>(t, ls, n_lines, cr, n_cr, eff, first, first_nonempty);
  return cudaGetLastError();
}

cudaError_t launch_parse_classify(const uint32_t* eff, const uint8_t* first, uint64_t n_lines, uint64_t f0,
                                  uint64_t n_eff, int kind, uint64_t* seq_len, uint64_t* rflag,
                                  unsigned long long* err, int sms, cudaStream_t st) {
  if (n_lines) classify_kernel<<<sms * 8, 256, 0, st>>>(eff, first, n_lines, f0, n_eff, kind, seq_len, rflag, err);
  return cudaGetLastError();
}

cudaError_t launch_parse_read_starts(const uint64_t* pos, const uint64_t* rflag, const uint64_t* ridx,
                                     uint64_t n_lines, uint64_t* read_start, int sms, cudaStream_t st) {
  if (n_lines) read_starts_kernel<<<sms * 8, 256, 0, st>>>(pos, rflag, ridx, n_lines, read_start);
  return cudaGetLastError();
}

cudaError_t launch_parse_pack(const uint8_t* t, const uint64_t* ls, const uint64_t* seq_len, const uint64_t* pos,
                              uint64_t n_lines, uint64_t* codes, uint64_t* nmask, int sms, cudaStream_t st) {
  if (n_lines)
    pack_lines_kernel<<<sms * 16, 256, 0, st>>>(t, ls, seq_len, pos, n_lines,
                                                reinterpret_cast<unsigned long long*>(codes),
                                                reinterpret_cast<unsigned long long*>(nmask));
  return cudaGetLastError();
}

}  // namespace gerbil
