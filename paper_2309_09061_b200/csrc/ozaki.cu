// EXPERIMENTAL (H2G_GRAM_OZ=1; the default is gram.cu's double-double FP64 kernel): Gram matrices of
// the wide SVD inputs and the R-only QR stacks on the INTEGER tensor cores (Ozaki-style slicing).
// Status: 1.9x slower than the double-double kernel at c4 (the row-maximum pass and the digit
// extraction are not overlapped with the IMMA work, 1 CTA / SM at 252 registers) and one golden
// per-cluster rank differs at c2 -- kept for the next round, not on the product path.
//
// What is computed: the same partial Grams G_chunk = C_chunk C_chunk^T (C = hstack / vstack of the
// item's segments, m rows, the chunk's lines summed) as gram_dd_partial_kernel, to ~2^-83 relative
// to |row_i|_max |row_j|_max -- far below what the truncation needs (the smallest singular value a
// truncation keeps satisfies sigma^2 >= 5e-15 sigma_1^2 on every config, so 1e-23 sigma_1^2 of Gram
// error moves it by < 1e-9 relative), and written as {hi, lo} double-double partial slices that
// gram_chol_kernel sums and factors exactly as before.
//
// How: per CTA (item, line chunk <= 2048 lines, 64 x 32 output tile of the upper triangle)
//   1. each tile row i gets the exponent e_i of its largest entry over the chunk (|c| < 2^e_i);
//   2. every entry x = c 2^-e_i in (-1, 1) is split into 14 sign-magnitude 7-bit digits,
//      x = sum_p d_p 2^{-7(p+1)} + r, |r| < 2^-98 (exact for entries within 2^-45 of the row
//      maximum), by integer shifts of its mantissa; the digits go to shared memory as int8;
//   3. for the 105 digit pairs p + q <= 13 the products D_p D_q^T run on mma.sync m16n8k32 s8 -> s32
//      (measured 1.14 POPS on this B200, 31x the FP64 tensor pipe), accumulated per weight class
//      s = p + q in int32 -- exact: |sum| <= 14 x 2048 x 127^2 < 2^31;
//   4. G_ij = 2^{e_i + e_j} sum_s 2^{-7(s+2)} acc_s: each term is an exact double, summed as a
//      double-double (two_sum) and scaled by an exact power of two.
// Dropped pairs (p + q > 13) and the digit remainders contribute < 2^-83 relative to 2^{e_i + e_j}
// (N <= 2048 lines per partial).
#include <cuda_runtime.h>

#include <mutex>

#include "h2g_types.h"

namespace h2g {

cudaError_t launch_gram_chol(const GramItem* items, int nitems, int mmax, cudaStream_t st);

namespace {

constexpr int kOzS = 14;       // digits (7 bits each) per entry
constexpr int kOzTM = 64;      // output tile rows (A side)
constexpr int kOzTN = 32;      // output tile columns (B side)
constexpr int kOzKC = 64;      // lines per shared-memory sub-chunk
constexpr int kOzLd = 80;      // bytes per digit row (64 + 16 padding: conflict-free fragment loads)
constexpr int kOzThr = 256;    // 8 warps: 4 (rows) x 2 (columns), each 16 x 16
constexpr int kOzRows = kOzTM + kOzTN;
constexpr size_t kOzSmem = (size_t)kOzS * kOzRows * kOzLd;  // 99,840 bytes

struct LineRef {
  const double* p;  // entry of tile row 0 ... use p + i * rs for row i (gram index)
  long long rs;
  double sc;
};

__device__ __forceinline__ void two_sum_oz(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

__device__ __forceinline__ int oz_find_seg(const Seg* __restrict__ segs, int s0, int s1, long long line) {
  int lo = s0, hi = s1 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].off <= line) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ double oz_scale(const Seg& sg) {
  if (!sg.sdiv) return sg.scale;
  const double d = *sg.sdiv;
  return d > 0.0 ? sg.scale / d : sg.scale;
}

__device__ __forceinline__ void imma(int (&c)[4], const int (&a)[4], int b0, int b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

}  // namespace

__global__ void __launch_bounds__(kOzThr, 1) gram_oz_partial_kernel(const GramItem* __restrict__ items,
                                                                    const Seg* __restrict__ segs,
                                                                    const GramWork* __restrict__ work) {
  extern __shared__ __align__(16) signed char dig[];  // [kOzS][kOzRows][kOzLd]
  __shared__ LineRef lines[kOzKC];
  __shared__ int rexp[kOzRows];
  __shared__ double rmax_w[kOzThr / 32][kOzRows];
  const GramWork w = work[blockIdx.x];
  const GramItem it = items[w.item];
  const int m = it.m;
  const int ia = w.ti * kOzTM, jb = w.tj * kOzTN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // tile row r (0..95) -> gram index: A rows ia + r (r < 64), B rows jb + (r - 64)
  auto gidx = [&](int r) { return r < kOzTM ? ia + r : jb + (r - kOzTM); };
  auto load_lines = [&](long long l0) {
    if (tid < kOzKC) {
      const long long c = l0 + tid;
      LineRef L{nullptr, 0, 0.0};
      if (c < w.c1) {
        const Seg sg = segs[oz_find_seg(segs, it.s0, it.s1, c)];
        L.p = sg.a.p + (c - sg.off) * (it.hcols ? sg.a.cs : sg.a.rs);
        L.rs = it.hcols ? sg.a.rs : sg.a.cs;
        L.sc = oz_scale(sg);
      }
      lines[tid] = L;
    }
  };
  // element of tile row r at sub-chunk line l (0 outside the item / chunk)
  auto elem = [&](int r, int l) -> double {
    const LineRef L = lines[l];
    const int g = gidx(r);
    if (!L.p || g >= m) return 0.0;
    return L.sc * L.p[(long long)g * L.rs];
  };
  // mapping of the 96 x 64 sub-chunk onto the threads: lines fastest when a line's entries are
  // strided (row-major sources, hcols), rows fastest otherwise (vstack of row-major stacks)
  const bool lines_fast = it.hcols != 0;

  // ---- pass 1: per tile row, the largest |c| over the chunk
  double mx[kOzRows * kOzKC / kOzThr];
#pragma unroll
  for (int q = 0; q < kOzRows * kOzKC / kOzThr; ++q) mx[q] = 0.0;
  for (long long l0 = w.c0; l0 < w.c1; l0 += kOzKC) {
    __syncthreads();
    load_lines(l0);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kOzRows * kOzKC / kOzThr; ++q) {
      const int e = tid + q * kOzThr;
      const int r = lines_fast ? e / kOzKC : e % kOzRows;
      const int l = lines_fast ? e % kOzKC : e / kOzRows;
      mx[q] = fmax(mx[q], fabs(elem(r, l)));
    }
  }
  // reduce to one maximum per tile row: in lines_fast mode a row's entries sit in 64 consecutive
  // threads (two warps); otherwise each thread owns fixed rows
  for (int r = tid; r < kOzRows; r += kOzThr) rexp[r] = 0;
  __syncthreads();
  {
    // per-thread partial maxima are for fixed (row) pairs: write them to a per-warp scratch, then fold
    for (int r = lane; r < kOzRows; r += 32) rmax_w[warp][r] = 0.0;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kOzRows * kOzKC / kOzThr; ++q) {
      const int e = tid + q * kOzThr;
      const int r = lines_fast ? e / kOzKC : e % kOzRows;
      // several lanes of the warp may own the same row: combine with an atomic on the bit pattern
      // (non-negative doubles order like their int64 bits)
      atomicMax(reinterpret_cast<unsigned long long*>(&rmax_w[warp][r]), __double_as_longlong(mx[q]));
    }
    __syncthreads();
    for (int r = tid; r < kOzRows; r += kOzThr) {
      double v = 0.0;
      for (int w2 = 0; w2 < kOzThr / 32; ++w2) v = fmax(v, rmax_w[w2][r]);
      int e = 0;
      if (v > 0.0) frexp(v, &e);  // v = f 2^e, f in [0.5, 1): |c| <= v < 2^e
      rexp[r] = e;
    }
  }
  __syncthreads();

  // ---- pass 2: digits + integer tensor-core products
  const int g8 = lane >> 2, t4 = lane & 3;
  const int wr = (warp >> 1) * 16;  // warp's 16 tile rows (A side)
  const int wc = (warp & 1) * 16;   // warp's 16 tile columns (B side), two n8 tiles
  int acc[kOzS][2][4];
#pragma unroll
  for (int s = 0; s < kOzS; ++s)
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[s][n][v] = 0;
  for (long long l0 = w.c0; l0 < w.c1; l0 += kOzKC) {
    __syncthreads();
    load_lines(l0);
    __syncthreads();
#pragma unroll 4
    for (int q = 0; q < kOzRows * kOzKC / kOzThr; ++q) {
      const int e = tid + q * kOzThr;
      const int r = lines_fast ? e / kOzKC : e % kOzRows;
      const int l = lines_fast ? e % kOzKC : e / kOzRows;
      // |x| = |c| 2^-e_r < 1 as a 98-bit fixed-point integer F (exact for every entry within 2^-45
      // of the row maximum, truncated below 2^-98 otherwise), then 14 sign-magnitude 7-bit digits:
      // integer pipe only
      const double c = elem(r, l);
      const unsigned long long bits = (unsigned long long)__double_as_longlong(c);
      const int E = (int)((bits >> 52) & 0x7ff);
      unsigned long long M = bits & ((1ull << 52) - 1);
      int Eu = E;
      if (E == 0) Eu = 1; else M |= 1ull << 52;
      const int sh = Eu - 977 - rexp[r];  // F = M 2^sh, sh <= 45
      unsigned __int128 F = 0;
      if (M != 0) {
        if (sh >= 0) F = (unsigned __int128)M << sh;
        else if (sh > -64) F = (unsigned __int128)(M >> (-sh));
      }
      const bool neg = (bits >> 63) != 0;
      signed char* dst = dig + (size_t)r * kOzLd + l;
#pragma unroll
      for (int p = 0; p < kOzS; ++p) {
        const int d = (int)((unsigned long long)(F >> (98 - 7 * (p + 1))) & 127u);
        dst[(size_t)p * kOzRows * kOzLd] = (signed char)(neg ? -d : d);
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < kOzKC; ks += 32) {
      int a[kOzS][4];
#pragma unroll
      for (int p = 0; p < kOzS; ++p) {
        const signed char* A = dig + (size_t)p * kOzRows * kOzLd + ks;
        a[p][0] = *reinterpret_cast<const int*>(A + (size_t)(wr + g8) * kOzLd + 4 * t4);
        a[p][1] = *reinterpret_cast<const int*>(A + (size_t)(wr + g8 + 8) * kOzLd + 4 * t4);
        a[p][2] = *reinterpret_cast<const int*>(A + (size_t)(wr + g8) * kOzLd + 16 + 4 * t4);
        a[p][3] = *reinterpret_cast<const int*>(A + (size_t)(wr + g8 + 8) * kOzLd + 16 + 4 * t4);
      }
#pragma unroll
      for (int qd = 0; qd < kOzS; ++qd) {
        const signed char* B = dig + (size_t)qd * kOzRows * kOzLd + (size_t)kOzTM * kOzLd + ks;
        int b[2][2];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          b[n][0] = *reinterpret_cast<const int*>(B + (size_t)(wc + 8 * n + g8) * kOzLd + 4 * t4);
          b[n][1] = *reinterpret_cast<const int*>(B + (size_t)(wc + 8 * n + g8) * kOzLd + 16 + 4 * t4);
        }
#pragma unroll
        for (int p = 0; p + qd < kOzS; ++p)
#pragma unroll
          for (int n = 0; n < 2; ++n) imma(acc[p + qd][n], a[p], b[n][0], b[n][1]);
      }
    }
  }
  // ---- combine the weight classes exactly, scale, write the upper triangle of this partial slice
  double* gh = it.gpart + (size_t)w.chunk * 2 * m * m;
  double* gl = gh + (size_t)m * m;
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int ri = wr + g8 + (v >= 2 ? 8 : 0);       // tile row (A side)
      const int cj = wc + 8 * n + 2 * t4 + (v & 1);    // tile column (B side)
      const int i = ia + ri, j = jb + cj;
      if (i >= m || j >= m || i > j) continue;
      double hi = 0.0, lo = 0.0;
#pragma unroll
      for (int s = kOzS - 1; s >= 0; --s) {  // smallest weights first
        const double term = ldexp((double)acc[s][n][v], -7 * (s + 2));
        double sum, err;
        two_sum_oz(hi, term, sum, err);
        hi = sum;
        lo += err;
      }
      const double h2 = hi + lo;
      const double l2 = lo - (h2 - hi);
      const int sh = rexp[ri] + rexp[kOzTM + cj];
      gh[(size_t)i * m + j] = ldexp(h2, sh);
      gl[(size_t)i * m + j] = ldexp(l2, sh);
    }
}

// Work of one item: line chunks of <= 2048 (int32-exact accumulation) x the 64 x 32 tiles that meet
// the upper triangle.
int gram_oz_chunk_lines() { return 2048; }
bool gram_oz_tile_needed(int ti, int tj) { return ti * kOzTM <= tj * kOzTN + kOzTN - 1; }
int gram_oz_tiles_m(int m) { return (m + kOzTM - 1) / kOzTM; }
int gram_oz_tiles_n(int m) { return (m + kOzTN - 1) / kOzTN; }

cudaError_t launch_gram_oz(const GramItem* items, const Seg* segs, const GramWork* work, int nwork, int nitems,
                           int mmax, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute((const void*)gram_oz_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kOzSmem);
  });
  if (nwork > 0) gram_oz_partial_kernel<<<nwork, kOzThr, kOzSmem, st>>>(items, segs, work);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nitems == 0) return e;
  return launch_gram_chol(items, nitems, mmax, st);
}

}  // namespace h2g
