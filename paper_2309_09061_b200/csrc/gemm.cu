// Grouped FP64 chain-GEMM on the tensor pipe (DMMA, mma.sync m8n8k4 f64) for sm_100a.
//
// Same contract as kernels.cu's gsum_kernel (GOut / GTerm / GTile): one CTA per 64x64 output
// tile, 4 warps each owning a 32x32 quadrant (4x4 DMMA tiles, 32 accumulators per lane).  The k
// dimension streams through shared memory in 16-wide chunks with a register prefetch of the next
// chunk, so global loads overlap the tensor work.  3-factor terms first form T = A*B (64 x k2) in
// shared memory, then T*D.
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#ifndef GSUM_WARPS  // warps per 64 x 64 output tile: 8 (16 x 32 each) or 4 (32 x 32 each)
#define GSUM_WARPS 8
#endif
#ifndef GSUM_UNROLL  // full k chunks run an unrolled inner loop (A/B: 980.7 -> 974.0 ms per c4 product)
#define GSUM_UNROLL 1
#endif
#ifndef GSUM_PIPE_MINB
#define GSUM_PIPE_MINB (GSUM_WARPS == 4 ? 3 : 2)
#endif

#include "h2g_types.h"

namespace h2g {

namespace {

constexpr int kT = 64;            // output tile
constexpr int kKC = 16;           // k chunk
constexpr int kLdA = kKC + 4;     // As[64][20]
constexpr int kLdB = kT + 8;      // Bs[16][72]
constexpr int kThr = 32 * GSUM_WARPS;  // 8 warps of 16 x 32 (2 x 4 DMMA tiles) or 4 of 32 x 32 (4 x 4)
constexpr int kPerA = kT * kKC / kThr;  // 4 elements per thread per chunk
constexpr int kPerB = kKC * kT / kThr;  // 4

__device__ __forceinline__ double ld(const MatRef& a, long long i, long long j) {
  return a.p[i * a.rs + j * a.cs];
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

constexpr int kRT = GSUM_WARPS == 4 ? 4 : 2, kCT = 4;  // DMMA tiles per warp (rows x cols)

struct Acc {
  double v[kRT][kCT][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < kRT; ++r)
#pragma unroll
      for (int c = 0; c < kCT; ++c) v[r][c][0] = v[r][c][1] = 0.0;
  }
};

__device__ __forceinline__ int warp_row0() { return (threadIdx.x >> 6) * 8 * kRT; }
__device__ __forceinline__ int warp_col0() { return ((threadIdx.x >> 5) & 1) * 32; }

// chunk loads: A rows i0..i0+63 (only < mt valid), k cols kk..kk+15 (only < kc); B likewise
__device__ __forceinline__ void fetch_chunk(double (&ra)[kPerA], double (&rb)[kPerB], const MatRef& A, int ai0,
                                            int mt, const MatRef& B, int bj0, int nt, int kk, int kc, double alpha) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < kPerA; ++q) {
    const int e = tid + q * kThr;
    const int i = e / kKC, l = e % kKC;
    ra[q] = (i < mt && l < kc) ? ld(A, ai0 + i, kk + l) : 0.0;
  }
  if (alpha != 1.0) {  // uniform per term; most terms have alpha = 1
#pragma unroll
    for (int q = 0; q < kPerA; ++q) ra[q] *= alpha;
  }
#pragma unroll
  for (int q = 0; q < kPerB; ++q) {
    const int e = tid + q * kThr;
    const int l = e / kT, j = e % kT;
    rb[q] = (j < nt && l < kc) ? ld(B, kk + l, bj0 + j) : 0.0;
  }
}

__device__ __forceinline__ void store_chunk(const double (&ra)[kPerA], const double (&rb)[kPerB], double* As,
                                            double* Bs) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int q = 0; q < kPerA; ++q) {
    const int e = tid + q * kThr;
    As[(e / kKC) * kLdA + e % kKC] = ra[q];
  }
#pragma unroll
  for (int q = 0; q < kPerB; ++q) {
    const int e = tid + q * kThr;
    Bs[(e / kT) * kLdB + e % kT] = rb[q];
  }
}

// mt / nt: valid rows / columns of the tile; a warp whose 16 x 32 quadrant lies wholly outside
// skips its DMMAs (its accumulators stay zero and are never stored) -- partial edge tiles of
// k x k outputs (e.g. 78 x 78 in 64 x 64 tiles) otherwise spend the tensor pipe on padding.
__device__ __forceinline__ void mma_chunk(Acc& acc, const double* As, const double* Bs, int kc, int mt, int nt) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
  if (wr >= mt || wc >= nt) return;
  for (int kk = 0; kk < kc; kk += 4) {
    double a[kRT], b[kCT];
#pragma unroll
    for (int r = 0; r < kRT; ++r) a[r] = As[(wr + r * 8 + g) * kLdA + kk + t4];
#pragma unroll
    for (int c = 0; c < kCT; ++c) b[c] = Bs[(kk + t4) * kLdB + wc + c * 8 + g];
#pragma unroll
    for (int r = 0; r < kRT; ++r)
#pragma unroll
      for (int c = 0; c < kCT; ++c) dmma(acc.v[r][c], a[r], b[c]);
  }
}

// acc += alpha * A[ai0:ai0+mt, 0:k] * B[0:k, bj0:bj0+nt]
__device__ void tile_gemm(Acc& acc, const MatRef& A, int ai0, int mt, const MatRef& B, int bj0, int nt, int k,
                          double alpha, double* As, double* Bs) {
  double ra[kPerA], rb[kPerB];
  if (k <= 0) return;
  fetch_chunk(ra, rb, A, ai0, mt, B, bj0, nt, 0, min(kKC, k), alpha);
  for (int kk = 0; kk < k; kk += kKC) {
    const int kc = min(kKC, k - kk);
    __syncthreads();  // previous chunk's readers are done
    store_chunk(ra, rb, As, Bs);
    __syncthreads();
    if (kk + kKC < k) fetch_chunk(ra, rb, A, ai0, mt, B, bj0, nt, kk + kKC, min(kKC, k - kk - kKC), alpha);
    mma_chunk(acc, As, Bs, (kc + 3) & ~3, mt, nt);
  }
}

}  // namespace

// Spill an accumulator into shared memory (rows < nr, cols < nc) with leading dimension ld.
__device__ __forceinline__ void acc_to_smem(const Acc& a, double* S, int ld, int nr, int nc) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
#pragma unroll
  for (int r = 0; r < kRT; ++r)
#pragma unroll
    for (int c = 0; c < kCT; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
        if (i < nr && j < nc) S[i * ld + j] = a.v[r][c][h];
      }
}

// Tag: 0 = every batch, 1 = the dense-target assembly (same code; its own symbol so profilers can
// select that launch by name)
template <int Tag>
__global__ void __launch_bounds__(kThr, 2) gsum_mma_kernel(const GOut* __restrict__ outs,
                                                         const GTerm* __restrict__ terms,
                                                         const GTile* __restrict__ tiles, int k2max) {
  extern __shared__ double smem[];
  double* As = smem;                 // 64 x kLdA
  double* Bs = As + kT * kLdA;       // 16 x kLdB
  double* Ts = Bs + kKC * kLdB;      // 64 x ldT
  const int ldT = k2max + 4;
  const GTile tl = tiles[blockIdx.x];
  const GOut o = outs[tl.out];
  const int i0 = (tl.tij & 0xffff) * kT, j0 = (tl.tij >> 16) * kT;
  const int mt = min(kT, o.m - i0), nt = min(kT, o.n - j0);
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
  Acc acc, aux;  // aux: 3-factor intermediate, or the open nf = 4 / 5 group sum
  acc.zero();
  int grp = 0;
  auto flush = [&]() {
    __syncthreads();  // Ts may still be read by an earlier product
    if (grp == 4) {   // C += T (mt x ka) * da
      acc_to_smem(aux, Ts, ldT, kT, o.ka);
      __syncthreads();
      tile_gemm(acc, MatRef{Ts, ldT, 1}, 0, mt, o.da, j0, nt, o.ka, 1.0, As, Bs);
    } else {          // C += ab (mt x kb) * U
      acc_to_smem(aux, Ts, ldT, o.kb, kT);
      __syncthreads();
      tile_gemm(acc, o.ab, i0, mt, MatRef{Ts, ldT, 1}, 0, nt, o.kb, 1.0, As, Bs);
    }
    __syncthreads();
    grp = 0;
  };
  for (int ti = o.t0; ti < o.t1; ++ti) {
    const GTerm t = terms[ti];
    if (t.nf == 0) continue;  // no-op (triple assembled by another launch)
    if (grp && t.nf != grp) flush();
    if (t.nf == 1) {
#pragma unroll
      for (int r = 0; r < kRT; ++r)
#pragma unroll
        for (int c = 0; c < kCT; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
            if (i < mt && j < nt) acc.v[r][c][h] += t.alpha * ld(t.a, i0 + i, j0 + j);
          }
    } else if (t.nf == 2) {
      tile_gemm(acc, t.a, i0, mt, t.b, j0, nt, t.k, t.alpha, As, Bs);
    } else if (t.nf == 4) {
      if (!grp) { aux.zero(); grp = 4; }
      tile_gemm(aux, t.a, i0, mt, t.b, 0, o.ka, t.k, t.alpha, As, Bs);
    } else if (t.nf == 5) {
      if (!grp) { aux.zero(); grp = 5; }
      tile_gemm(aux, t.a, 0, o.kb, t.b, j0, nt, t.k, t.alpha, As, Bs);
    } else {
      // T = alpha * A[i0:i0+mt, :] * B (mt x k2) into shared memory, 64 columns at a time
      for (int js = 0; js < t.k2; js += kT) {
        aux.zero();
        const int ns = min(kT, t.k2 - js);
        tile_gemm(aux, t.a, i0, mt, t.b, js, ns, t.k, t.alpha, As, Bs);
        acc_to_smem(aux, Ts + js, ldT, kT, ns);
      }
      __syncthreads();
      const MatRef T{Ts, ldT, 1};
      tile_gemm(acc, T, 0, mt, t.d, j0, nt, t.k2, 1.0, As, Bs);
      __syncthreads();  // Ts is rewritten by the next 3-factor term
    }
  }
  if (grp) flush();
#pragma unroll
  for (int r = 0; r < kRT; ++r)
#pragma unroll
    for (int c = 0; c < kCT; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
        if (i < mt && j < nt) {
          double* dst = o.c + (long long)(i0 + i) * o.ldc + (j0 + j);
          *dst = (o.beta ? *dst : 0.0) + acc.v[r][c][h];
        }
      }
}


// ================================================================================================
// gsum_pipe_kernel: the same contract, restructured for the FP64 tensor pipe's latency.
//   * operands stream through a 3-stage shared-memory ring filled by cp.async (8-byte copies along
//     the operand's contiguous dimension, zero-fill outside the tile), so two 16-wide k chunks are
//     in flight while the third is multiplied -- no register prefetch, no spills;
//   * the ring runs across the terms of a run (consecutive 2-factor terms into C, or the grouped
//     nf = 4 / 5 terms into their intermediate), so the pipeline does not drain at term boundaries;
//   * each operand keeps its memory order in shared memory ([i][k] for k-contiguous, [k][i] for
//     i-contiguous views, strides == 4 mod 16 doubles: conflict-free DMMA fragment loads), so
//     transposed views (column passes) load coalesced too;
//   * intermediates (3-factor T, grouped T / U) are read by the fragment loads in place from Ts.
// ================================================================================================
namespace {

constexpr int kPS = 3;                 // pipeline stages
constexpr int kLdKc = kKC + 4;         // [i][k] stride (20)
constexpr int kLdIc = kT + 4;          // [k][i] stride (68)
constexpr int kStg = kT * kLdKc;       // doubles per operand stage (>= kKC * kLdIc)
static_assert(kStg >= kKC * kLdIc, "stage size");

struct StageMeta {
  int aI, aK, bK, bJ;  // fragment strides of the staged (or direct) operands
  int kc4;             // k steps of 4 in this chunk
  int skipA, skipB;    // operand read directly from smem (offset in doubles into Ts), else -1
  int pad_;
  double alpha;
};

// One product of a run: acc += alpha * A[ai0 .. ai0+mr, 0:k] * B[0:k, bj0 .. bj0+nc]
struct Job {
  MatRef a, b;
  int k;
  double alpha;
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Issue the copies of one chunk (k columns kk .. kk+kc of A's rows ai0.., rows kk.. of B's columns
// bj0..) into one stage; `direct` operands (Ts) are not copied.
__device__ __forceinline__ void issue_chunk(const Job& J, int ai0, int mr, int bj0, int nc, int kk, double* sA,
                                            double* sB, bool dirA, bool dirB, StageMeta* meta,
                                            int offA, int offB, int ldDA, int ldDB) {
  const int tid = threadIdx.x;
  const int kc = min(kKC, J.k - kk);
  const bool aK = J.a.cs == 1;  // A row-major (k contiguous)
  const bool bN = J.b.cs == 1;  // B row-major (j contiguous)
  if (!dirA) {
    if (aK) {
#pragma unroll
      for (int q = 0; q < kT * kKC / kThr; ++q) {
        const int e = tid + q * kThr, i = e / kKC, l = e % kKC;
        const bool v = i < mr && l < kc;
        cp_async8(sA + i * kLdKc + l, v ? J.a.p + (long long)(ai0 + i) * J.a.rs + (kk + l) : J.a.p, v);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kT * kKC / kThr; ++q) {
        const int e = tid + q * kThr, l = e / kT, i = e % kT;
        const bool v = i < mr && l < kc;
        cp_async8(sA + l * kLdIc + i,
                  v ? J.a.p + (long long)(ai0 + i) * J.a.rs + (long long)(kk + l) * J.a.cs : J.a.p, v);
      }
    }
  }
  if (!dirB) {
    if (bN) {
#pragma unroll
      for (int q = 0; q < kT * kKC / kThr; ++q) {
        const int e = tid + q * kThr, l = e / kT, j = e % kT;
        const bool v = j < nc && l < kc;
        cp_async8(sB + l * kLdIc + j, v ? J.b.p + (long long)(kk + l) * J.b.rs + (bj0 + j) : J.b.p, v);
      }
    } else {
#pragma unroll
      for (int q = 0; q < kT * kKC / kThr; ++q) {
        const int e = tid + q * kThr, j = e / kKC, l = e % kKC;
        const bool v = j < nc && l < kc;
        cp_async8(sB + j * kLdKc + l,
                  v ? J.b.p + (long long)(kk + l) * J.b.rs + (long long)(bj0 + j) * J.b.cs : J.b.p, v);
      }
    }
  }
  if (tid == 0) {
    StageMeta m;
    if (dirA) { m.aI = ldDA; m.aK = 1; m.skipA = offA + kk; } else { m.aI = aK ? kLdKc : 1; m.aK = aK ? 1 : kLdIc; m.skipA = -1; }
    if (dirB) { m.bK = ldDB; m.bJ = 1; m.skipB = offB + kk * ldDB; } else { m.bK = bN ? kLdIc : 1; m.bJ = bN ? 1 : kLdKc; m.skipB = -1; }
    m.kc4 = (kc + 3) >> 2;
    m.pad_ = 0;
    m.alpha = J.alpha;
    *meta = m;
  }
}

// One run of products into one accumulator, pipelined across all chunks of all its jobs.
// getjob(j) returns job j (k = 0 jobs are skipped); rows ai0.. (mr valid) of every A, columns
// bj0.. (nc valid) of every B; dirA / dirB: A / B read in place from Ts (+offA / +offB).
template <class GetJob>
__device__ void run_stream(Acc& acc, int njobs, GetJob getjob, int ai0, int mr, int bj0, int nc, bool dirA,
                           bool dirB, int offA, int offB, double* ring, StageMeta* metas, const double* Ts,
                           int ldDA, int ldDB) {
  // chunk count
  int total = 0;
  for (int j = 0; j < njobs; ++j) total += (getjob(j).k + kKC - 1) / kKC;
  if (total == 0) return;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
  const bool live = wr < mr && wc < nc;
  // producer cursor
  int pj = 0, pk = 0;
  Job PJ = getjob(0);
  while (PJ.k == 0) PJ = getjob(++pj);
  auto produce = [&](int c) {
    if (c < total) {
      const int s = c % kPS;
      issue_chunk(PJ, ai0, mr, bj0, nc, pk, ring + s * 2 * kStg, ring + s * 2 * kStg + kStg, dirA, dirB, metas + s,
                  offA, offB, ldDA, ldDB);
      pk += kKC;
      if (pk >= PJ.k) {
        pk = 0;
        if (c + 1 < total) {
          do { PJ = getjob(++pj); } while (PJ.k == 0);
        }
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int c = 0; c < kPS - 1; ++c) produce(c);
  for (int c = 0; c < total; ++c) {
    cp_wait<kPS - 2>();
    __syncthreads();
    produce(c + kPS - 1);
    const int s = c % kPS;
    const StageMeta m = metas[s];
    if (live) {
      const double* sA = m.skipA >= 0 ? Ts + m.skipA : ring + s * 2 * kStg;
      const double* sB = m.skipB >= 0 ? Ts + m.skipB : ring + s * 2 * kStg + kStg;
      const bool scale = m.alpha != 1.0;
      auto kstep = [&](int q) {
        const int k = 4 * q + t4;
        double a[kRT], b[kCT];
#pragma unroll
        for (int r = 0; r < kRT; ++r) a[r] = sA[(wr + r * 8 + g) * m.aI + k * m.aK];
#pragma unroll
        for (int cc = 0; cc < kCT; ++cc) b[cc] = sB[k * m.bK + (wc + cc * 8 + g) * m.bJ];
        if (scale) {
#pragma unroll
          for (int r = 0; r < kRT; ++r) a[r] *= m.alpha;
        }
#pragma unroll
        for (int r = 0; r < kRT; ++r)
#pragma unroll
          for (int cc = 0; cc < kCT; ++cc) dmma(acc.v[r][cc], a[r], b[cc]);
      };
#if GSUM_UNROLL
      if (m.kc4 == kKC / 4) {  // full chunk: unrolled, so the fragment loads of step q + 1 are
                               // scheduled under the DMMAs of step q
#pragma unroll
        for (int q = 0; q < kKC / 4; ++q) kstep(q);
      } else
#endif
        for (int q = 0; q < m.kc4; ++q) kstep(q);
    }
  }
  cp_wait<0>();
  __syncthreads();  // the ring (and metas) are reused by the next run
}

}  // namespace

template <int Tag>
__global__ void __launch_bounds__(kThr, GSUM_PIPE_MINB) gsum_pipe_kernel(const GOut* __restrict__ outs,
                                                          const GTerm* __restrict__ terms,
                                                          const GTile* __restrict__ tiles, int k2max) {
  extern __shared__ __align__(16) double smem[];
  __shared__ StageMeta metas[kPS];
  double* ring = smem;                       // kPS x (A stage | B stage)
  double* Ts = ring + kPS * 2 * kStg;        // 64 x ldT
  const int ldT = k2max + 4;
  const GTile tl = tiles[blockIdx.x];
  const GOut o = outs[tl.out];
  // the output's term descriptors are read one dependent load at a time (13 % of gsum_whole's warp
  // samples waited on them): request their lines up front
  for (const char* q = (const char*)(terms + o.t0) + threadIdx.x * 128; q < (const char*)(terms + o.t1);
       q += kThr * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));

  const int i0 = (tl.tij & 0xffff) * kT, j0 = (tl.tij >> 16) * kT;
  const int mt = min(kT, o.m - i0), nt = min(kT, o.n - j0);
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
  if (k2max > 0)  // intermediates are read in place: keep their unwritten padding finite
    for (int e = threadIdx.x; e < kT * ldT; e += kThr) Ts[e] = 0.0;
  if (o.beta) {  // accumulating output: request C's lines now, the epilogue reads them (see gemm_lean.cu)
#pragma unroll
    for (int r = 0; r < kRT; ++r)
#pragma unroll
      for (int c = 0; c < kCT; ++c) {
        const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4;
        if (i < mt && j < nt) {
          const double* q = o.c + (long long)(i0 + i) * o.ldc + (j0 + j);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
        }
      }
  }
  Acc acc, aux;
  acc.zero();
  auto single = [](Job J) { return [J](int) { return J; }; };
  int ti = o.t0;
  while (ti < o.t1) {
    const GTerm t = terms[ti];
    if (t.nf == 0) { ++ti; continue; }  // no-op (triple assembled by another launch)
    // the run of consecutive terms with this nf (2, 4 and 5 accumulate into one target)
    int te = ti + 1;
    if (t.nf == 2 || t.nf == 4 || t.nf == 5)
      while (te < o.t1 && (terms[te].nf == t.nf || terms[te].nf == 0)) ++te;
    const int nrun = te - ti;
    const GTerm* run = terms + ti;
    auto getjob = [run](int j) {
      const GTerm u = run[j];
      return Job{u.a, u.b, u.nf == 0 ? 0 : u.k, u.alpha};
    };
    if (t.nf == 1) {
#pragma unroll
      for (int r = 0; r < kRT; ++r)
#pragma unroll
        for (int c = 0; c < kCT; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
            if (i < mt && j < nt) acc.v[r][c][h] += t.alpha * ld(t.a, i0 + i, j0 + j);
          }
    } else if (t.nf == 2) {
      run_stream(acc, nrun, getjob, i0, mt, j0, nt, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
    } else if (t.nf == 4) {  // T (mt x ka) = sum A B, then C += T * da
      aux.zero();
      run_stream(aux, nrun, getjob, i0, mt, 0, o.ka, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
      acc_to_smem(aux, Ts, ldT, kT, o.ka);
      __syncthreads();
      run_stream(acc, 1, single(Job{MatRef{Ts, ldT, 1}, o.da, o.ka, 1.0}), 0, mt, j0, nt, true, false, 0, 0, ring,
                 metas, Ts, ldT, ldT);
    } else if (t.nf == 5) {  // U (kb x nt) = sum A B, then C += ab * U
      aux.zero();
      run_stream(aux, nrun, getjob, 0, o.kb, j0, nt, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
      acc_to_smem(aux, Ts, ldT, o.kb, kT);
      __syncthreads();
      run_stream(acc, 1, single(Job{o.ab, MatRef{Ts, ldT, 1}, o.kb, 1.0}), i0, mt, 0, nt, false, true, 0, 0, ring,
                 metas, Ts, ldT, ldT);
    } else {  // nf = 3: T = alpha A[i0.., :] B (mt x k2) in Ts, 64 columns at a time, then C += T D
      for (int js = 0; js < t.k2; js += kT) {
        aux.zero();
        const int ns = min(kT, t.k2 - js);
        run_stream(aux, 1, single(Job{t.a, MatRef{t.b.p + (long long)js * t.b.cs, t.b.rs, t.b.cs}, t.k, t.alpha}),
                   i0, mt, 0, ns, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
        acc_to_smem(aux, Ts + js, ldT, kT, ns);
      }
      __syncthreads();
      run_stream(acc, 1, single(Job{MatRef{Ts, ldT, 1}, t.d, t.k2, 1.0}), 0, mt, j0, nt, true, false, 0, 0, ring,
                 metas, Ts, ldT, ldT);
    }
    ti = te;
  }
#pragma unroll
  for (int r = 0; r < kRT; ++r)
#pragma unroll
    for (int c = 0; c < kCT; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
        if (i < mt && j < nt) {
          double* dst = o.c + (long long)(i0 + i) * o.ldc + (j0 + j);
          *dst = (o.beta ? *dst : 0.0) + acc.v[r][c][h];
        }
      }
}

// Whole-output variant for the coupling targets of the assembly (outputs up to 128 x 128: k~ x k~
// couplings, k~ <= 128): ONE CTA walks the (<= 2 x 2) 64 x 64 sub-tiles of its output and keeps the
// grouped intermediates of the first kind-a run (T = sum A S, per row strip, 64 x ka) and kind-b run
// (U = sum S B^T, all columns, kb x n) in shared memory across the sub-tiles -- the tile kernel
// recomputes T for every column tile and U for every row tile of the same output.
constexpr int kLdU = 2 * kT + 4;  // cached U: kb (<= 64) x 128 columns

template <int Tag>
__global__ void __launch_bounds__(kThr, 1) gsum_whole_kernel(const GOut* __restrict__ outs,
                                                           const GTerm* __restrict__ terms,
                                                           const GTile* __restrict__ tiles, int k2max) {
  extern __shared__ __align__(16) double smem[];
  __shared__ StageMeta metas[kPS];
  double* ring = smem;
  double* Ts = ring + kPS * 2 * kStg;  // 64 x ldT (3-factor intermediates, not cached)
  const int ldT = k2max + 4;
  double* Tc = Ts + (size_t)kT * ldT;  // 64 x kLdTc: cached T of the current row strip
  constexpr int kLdTc = kT + 4;
  double* Uc = Tc + (size_t)kT * kLdTc;  // 64 x kLdU: cached U, all columns
  const GOut o = outs[tiles[blockIdx.x].out];
  // the output's term descriptors are read one dependent load at a time (13 % of gsum_whole's warp
  // samples waited on them): request their lines up front
  for (const char* q = (const char*)(terms + o.t0) + threadIdx.x * 128; q < (const char*)(terms + o.t1);
       q += kThr * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = warp_row0(), wc = warp_col0();
  for (int e = threadIdx.x; e < kT * ldT; e += kThr) Ts[e] = 0.0;
  for (int e = threadIdx.x; e < kT * kLdTc; e += kThr) Tc[e] = 0.0;
  for (int e = threadIdx.x; e < kT * kLdU; e += kThr) Uc[e] = 0.0;
  __syncthreads();
  const int tm = (o.m + kT - 1) / kT, tn = (o.n + kT - 1) / kT;
  auto single = [](Job J) { return [J](int) { return J; }; };
  // offsets of the cached intermediates as direct operands (relative to Ts)
  const int offTc = (int)(Tc - Ts), offUc = (int)(Uc - Ts);
  bool u_cached = false;
  for (int ti = 0; ti < tm; ++ti) {
    bool t_cached = false;
    for (int tj = 0; tj < tn; ++tj) {
      const int i0 = ti * kT, j0 = tj * kT;
      const int mt = min(kT, o.m - i0), nt = min(kT, o.n - j0);
      Acc acc, aux;
      acc.zero();
      bool first4 = true, first5 = true;
      int ti2 = o.t0;
      while (ti2 < o.t1) {
        const GTerm t = terms[ti2];
        if (t.nf == 0) { ++ti2; continue; }
        int te = ti2 + 1;
        if (t.nf == 2 || t.nf == 4 || t.nf == 5)
          while (te < o.t1 && (terms[te].nf == t.nf || terms[te].nf == 0)) ++te;
        const int nrun = te - ti2;
        const GTerm* run = terms + ti2;
        auto getjob = [run](int j) {
          const GTerm u = run[j];
          return Job{u.a, u.b, u.nf == 0 ? 0 : u.k, u.alpha};
        };
        if (t.nf == 1) {
#pragma unroll
          for (int r = 0; r < kRT; ++r)
#pragma unroll
            for (int c = 0; c < kCT; ++c)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
                if (i < mt && j < nt) acc.v[r][c][h] += t.alpha * ld(t.a, i0 + i, j0 + j);
              }
        } else if (t.nf == 2) {
          run_stream(acc, nrun, getjob, i0, mt, j0, nt, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
        } else if (t.nf == 4) {  // T (rows of this strip x ka) = sum A B, then C += T * da
          const bool cache = first4;
          first4 = false;
          if (!(cache && t_cached)) {
            aux.zero();
            run_stream(aux, nrun, getjob, i0, mt, 0, o.ka, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
            acc_to_smem(aux, cache ? Tc : Ts, cache ? kLdTc : ldT, kT, o.ka);
            __syncthreads();
            if (cache) t_cached = true;
          }
          run_stream(acc, 1, single(Job{MatRef{cache ? Tc : Ts, cache ? kLdTc : ldT, 1}, o.da, o.ka, 1.0}), 0, mt,
                     j0, nt, true, false, cache ? offTc : 0, 0, ring, metas, Ts, cache ? kLdTc : ldT, ldT);
        } else if (t.nf == 5) {  // U (kb x all columns) = sum A B, then C += ab * U
          const bool cache = first5;
          first5 = false;
          if (cache && !u_cached) {
            for (int uj = 0; uj < tn; ++uj) {  // every column strip once, for all row strips
              aux.zero();
              const int ju = uj * kT, nu = min(kT, o.n - ju);
              run_stream(aux, nrun, getjob, 0, o.kb, ju, nu, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
              acc_to_smem(aux, Uc + ju, kLdU, o.kb, kT);
            }
            __syncthreads();
            u_cached = true;
          } else if (!cache) {
            aux.zero();
            run_stream(aux, nrun, getjob, 0, o.kb, j0, nt, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
            acc_to_smem(aux, Ts, ldT, o.kb, kT);
            __syncthreads();
          }
          run_stream(acc, 1, single(Job{o.ab, MatRef{cache ? Uc + j0 : Ts, cache ? kLdU : ldT, 1}, o.kb, 1.0}), i0,
                     mt, 0, nt, false, true, 0, cache ? offUc + j0 : 0, ring, metas, Ts, ldT, cache ? kLdU : ldT);
        } else {  // nf = 3
          for (int js = 0; js < t.k2; js += kT) {
            aux.zero();
            const int ns = min(kT, t.k2 - js);
            run_stream(aux, 1, single(Job{t.a, MatRef{t.b.p + (long long)js * t.b.cs, t.b.rs, t.b.cs}, t.k, t.alpha}),
                       i0, mt, 0, ns, false, false, 0, 0, ring, metas, Ts, ldT, ldT);
            acc_to_smem(aux, Ts + js, ldT, kT, ns);
          }
          __syncthreads();
          run_stream(acc, 1, single(Job{MatRef{Ts, ldT, 1}, t.d, t.k2, 1.0}), 0, mt, j0, nt, true, false, 0, 0, ring,
                     metas, Ts, ldT, ldT);
        }
        ti2 = te;
      }
#pragma unroll
      for (int r = 0; r < kRT; ++r)
#pragma unroll
        for (int c = 0; c < kCT; ++c)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
            if (i < mt && j < nt) {
              double* dst = o.c + (long long)(i0 + i) * o.ldc + (j0 + j);
              *dst = (o.beta ? *dst : 0.0) + acc.v[r][c][h];
            }
          }
      __syncthreads();  // Ts / ring reuse by the next sub-tile
    }
  }
}

size_t gsum_whole_smem(int k2max) {
  return sizeof(double) * ((size_t)kPS * 2 * kStg + (size_t)kT * (k2max + 4) + (size_t)kT * (kT + 4) +
                           (size_t)kT * kLdU);
}

size_t gsum_pipe_smem(int k2max) {
  return sizeof(double) * ((size_t)kPS * 2 * kStg + (k2max > 0 ? (size_t)kT * (k2max + 4) : 0));
}

size_t gsum_mma_smem(int k2max) {
  return sizeof(double) * ((size_t)kT * kLdA + (size_t)kKC * kLdB + (k2max > 0 ? (size_t)kT * (k2max + 4) : 0));
}

cudaError_t launch_gsum_whole(const GOut* outs, const GTerm* terms, const GTile* tiles, int ntiles, int k2max,
                              cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute((const void*)gsum_whole_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - 1024);
  });
  if (ntiles == 0) return cudaSuccess;
  gsum_whole_kernel<0><<<ntiles, kThr, gsum_whole_smem(k2max), st>>>(outs, terms, tiles, k2max);
  return cudaGetLastError();
}

cudaError_t launch_gsum_mma(const GOut* outs, const GTerm* terms, const GTile* tiles, int ntiles, int k2max,
                            cudaStream_t st, int tag) {
  static std::once_flag once;
  std::call_once(once, [] {
    for (const void* fn : {(const void*)gsum_mma_kernel<0>, (const void*)gsum_mma_kernel<1>,
                           (const void*)gsum_pipe_kernel<0>, (const void*)gsum_pipe_kernel<1>}) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fn);
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
  });
  static const bool v1 = getenv("H2G_GSUM_V1") != nullptr;  // previous kernel, for A/B
  if (ntiles == 0) return cudaSuccess;
  if (!v1) {
    if (tag == 1) gsum_pipe_kernel<1><<<ntiles, kThr, gsum_pipe_smem(k2max), st>>>(outs, terms, tiles, k2max);
    else gsum_pipe_kernel<0><<<ntiles, kThr, gsum_pipe_smem(k2max), st>>>(outs, terms, tiles, k2max);
    return cudaGetLastError();
  }
  if (tag == 1) gsum_mma_kernel<1><<<ntiles, kThr, gsum_mma_smem(k2max), st>>>(outs, terms, tiles, k2max);
  else gsum_mma_kernel<0><<<ntiles, kThr, gsum_mma_smem(k2max), st>>>(outs, terms, tiles, k2max);
  return cudaGetLastError();
}

}  // namespace h2g
