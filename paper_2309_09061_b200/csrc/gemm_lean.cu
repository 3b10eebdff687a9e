// Lean grouped FP64 GEMM (DMMA m8n8k4) for batches whose terms are plain sums and 2-factor
// products (nf <= 2): the push-down, the expansions, the induced / coarse basis stacks.
//
// Those batches' outputs are k~ x k~-sized (33 .. 128 per side): in 64 x 64 tiles of 8 warps only
// ~4 of 8 warps own a live 16 x 32 quadrant (H2G_DEBUG_GSUM), and the idle ones hold a CTA slot
// for the whole latency-bound k loop.  Here a CTA is 4 warps, each owning one 16 x 32 quadrant,
// arranged per tile as 2 x 2 (32 x 64), 4 x 1 (64 x 32) or 1 x 4 (16 x 128) -- the host picks the
// arrangement per output that needs the fewest CTAs -- and, without the 3-factor machinery (second
// accumulator, intermediates in shared memory), four CTAs fit per SM.
//
// Per output element the k order is the one gsum_pipe_kernel uses (16-wide chunks, 4 per DMMA, terms in
// list order), so results are bitwise equal to the 64 x 64 path's.
#include <cuda_runtime.h>

#include <mutex>

#include "h2g_types.h"

namespace h2g {

namespace {

constexpr int kW = 4;         // warps per CTA
constexpr int kThr = 32 * kW;
constexpr int kKC = 16;       // k chunk
constexpr int kLdK = kKC + 4; // [line][k] stride
constexpr int kPS = 3;        // pipeline stages

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

}  // namespace

__global__ void __launch_bounds__(kThr, 4) gsum_lean_kernel(const GOut* __restrict__ outs,
                                                            const GTerm* __restrict__ terms,
                                                            const GLTile* __restrict__ tiles) {
  extern __shared__ __align__(16) double ring[];
  const GLTile tl = tiles[blockIdx.x];
  const GOut o = outs[tl.out];
  const int WC = tl.lay == 0 ? 2 : (tl.lay == 1 ? 1 : 4);  // warp columns
  const int lgTM = tl.lay == 0 ? 5 : (tl.lay == 1 ? 6 : 4), lgTN = tl.lay == 0 ? 6 : (tl.lay == 1 ? 5 : 7);
  const int TM = 1 << lgTM, TN = 1 << lgTN;
  const int szA = TM * kLdK, stg = (TM + TN) * kLdK;  // doubles per stage (A | B), either layout fits
  const int ldAk = TM + 4, ldBk = TN + 4;              // [k][line] strides
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int wr = (w / WC) * 16, wc = (w % WC) * 32;
  const int i0 = tl.i0, j0 = tl.j0;
  const int mt = min(TM, o.m - i0), nt = min(TN, o.n - j0);
  const bool live = wr < mt && wc < nt;
  double acc[2][4][2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c][0] = acc[r][c][1] = 0.0;

  // accumulating outputs (beta): the epilogue's read of C was the kernel's largest stall (28 % of the
  // warp samples on the DADDs behind those loads, push-down launch, ncu) -- request the lines now
  if (o.beta && live) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4;
        if (i < mt && j < nt) {
          const double* q = o.c + (long long)(i0 + i) * o.ldc + (j0 + j);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
        }
      }
  }
  int ti = o.t0;
  while (ti < o.t1) {
    const int nf0 = terms[ti].nf;
    if (nf0 == 0) { ++ti; continue; }
    if (nf0 == 1) {
      const MatRef a = terms[ti].a;
      const double al = terms[ti].alpha;
      if (live) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
              if (i < mt && j < nt) acc[r][c][h] += al * a.p[(long long)(i0 + i) * a.rs + (long long)(j0 + j) * a.cs];
            }
      }
      ++ti;
      continue;
    }
    // run of consecutive 2-factor terms (no-ops skipped), one pipeline across all their chunks
    int te = ti + 1;
    while (te < o.t1 && (terms[te].nf == 2 || terms[te].nf == 0)) ++te;
    int total = 0;
    for (int j = ti; j < te; ++j)
      if (terms[j].nf == 2) total += (terms[j].k + kKC - 1) / kKC;
    if (total > 0) {
      // producer cursor: term pj, k offset pk
      int pj = ti, pk = 0;
      while (terms[pj].nf != 2 || terms[pj].k <= 0) ++pj;
      MatRef PA = terms[pj].a, PB = terms[pj].b;
      int Pk = terms[pj].k;
      auto produce = [&](int c) {
        if (c < total) {
          double* sA = ring + (c % kPS) * stg;
          double* sB = sA + szA;
          const int kc = min(kKC, Pk - pk);
          // each thread copies a fixed fast-dimension line, stepping over the slow dimension
          // (no per-element index arithmetic: the tile extents are powers of two)
          {
            const bool aK = PA.cs == 1;  // k contiguous: [i][k], else [k][i]
            const int lg = aK ? 4 : lgTM;
            const int f = tid & ((1 << lg) - 1), step = kThr >> lg, S = aK ? TM : kKC;
            const bool fv = f < (aK ? kc : mt);
            const int lim = aK ? mt : kc, dS = aK ? kLdK : ldAk;
            const long long gS = aK ? (long long)PA.rs : (long long)PA.cs;
            const double* src = aK ? PA.p + (long long)i0 * PA.rs + (pk + f)
                                   : PA.p + (long long)(i0 + f) * PA.rs + (long long)pk * PA.cs;
            for (int q = tid >> lg; q < S; q += step) {
              const bool v = fv && q < lim;
              cp_async8(sA + q * dS + f, v ? src + q * gS : PA.p, v);
            }
          }
          {
            const bool bN = PB.cs == 1;  // j contiguous: [k][j], else [j][k]
            const int lg = bN ? lgTN : 4;
            const int f = tid & ((1 << lg) - 1), step = kThr >> lg, S = bN ? kKC : TN;
            const bool fv = f < (bN ? nt : kc);
            const int lim = bN ? kc : nt, dS = bN ? ldBk : kLdK;
            const long long gS = bN ? (long long)PB.rs : (long long)PB.cs;
            const double* src = bN ? PB.p + (long long)pk * PB.rs + (j0 + f)
                                   : PB.p + (long long)(pk + f) * PB.rs + (long long)j0 * PB.cs;
            for (int q = tid >> lg; q < S; q += step) {
              const bool v = fv && q < lim;
              cp_async8(sB + q * dS + f, v ? src + q * gS : PB.p, v);
            }
          }
          pk += kKC;
          if (pk >= Pk && c + 1 < total) {
            pk = 0;
            do { ++pj; } while (terms[pj].nf != 2 || terms[pj].k <= 0);
            PA = terms[pj].a;
            PB = terms[pj].b;
            Pk = terms[pj].k;
          }
        }
        cp_commit();
      };
      // consumer cursor
      int cj = ti, ck = 0;
      while (terms[cj].nf != 2 || terms[cj].k <= 0) ++cj;
      int Ck = terms[cj].k;
      double Cal = terms[cj].alpha;
      bool CaK = terms[cj].a.cs == 1, CbN = terms[cj].b.cs == 1;
#pragma unroll
      for (int c = 0; c < kPS - 1; ++c) produce(c);
      for (int c = 0; c < total; ++c) {
        cp_wait<kPS - 2>();
        __syncthreads();
        produce(c + kPS - 1);
        if (live) {
          const double* sA = ring + (c % kPS) * stg;
          const double* sB = sA + szA;
          const int aI = CaK ? kLdK : 1, aK = CaK ? 1 : ldAk;
          const int bK = CbN ? ldBk : 1, bJ = CbN ? 1 : kLdK;
          const int kc4 = (min(kKC, Ck - ck) + 3) >> 2;
          const bool scale = Cal != 1.0;
          const double* pa = sA + (wr + g) * aI + t4 * aK;
          const double* pb = sB + t4 * bK + (wc + g) * bJ;
          auto kstep = [&](int q) {
            double a[2], b[4];
#pragma unroll
            for (int r = 0; r < 2; ++r) a[r] = pa[r * 8 * aI + 4 * q * aK];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) b[cc] = pb[4 * q * bK + cc * 8 * bJ];
            if (scale) {
#pragma unroll
              for (int r = 0; r < 2; ++r) a[r] *= Cal;
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) dmma(acc[r][cc], a[r], b[cc]);
          };
          if (kc4 == kKC / 4) {
#pragma unroll
            for (int q = 0; q < kKC / 4; ++q) kstep(q);
          } else {
            for (int q = 0; q < kc4; ++q) kstep(q);
          }
        }
        ck += kKC;
        if (ck >= Ck && c + 1 < total) {
          ck = 0;
          do { ++cj; } while (terms[cj].nf != 2 || terms[cj].k <= 0);
          Ck = terms[cj].k;
          Cal = terms[cj].alpha;
          CaK = terms[cj].a.cs == 1;
          CbN = terms[cj].b.cs == 1;
        }
      }
      cp_wait<0>();
      __syncthreads();  // the ring is reused by the next run
    }
    ti = te;
  }
  if (live) {
    // accumulating outputs: read all 16 entries of C first, then add and store.  In a single loop the
    // compiler must keep each store ahead of the next load (C is not restrict-qualified), which
    // serialises 16 L2 round trips: 40 % of the warp samples of an expansion launch sat on these adds.
    double cv[2][4][2];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
          cv[r][c][h] = (o.beta && i < mt && j < nt) ? o.c[(long long)(i0 + i) * o.ldc + (j0 + j)] : 0.0;
        }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = wr + r * 8 + g, j = wc + c * 8 + 2 * t4 + h;
          if (i < mt && j < nt) o.c[(long long)(i0 + i) * o.ldc + (j0 + j)] = cv[r][c][h] + acc[r][c][h];
        }
  }
}


// Outputs that are plain sums (every term nf <= 1: the gathers of phase 2's column-tree representatives
// and of the basis stacks are one-term copies) need no tensor work: one CTA per 1024 consecutive
// elements of the row-major output, 8 per thread with consecutive lanes on consecutive columns, the
// term loop outermost so that a term's 8 loads are in flight together.  The lean / tile kernels spend
// four dependent global round trips per CTA on such an output at 12-16 warps per SM.
// Same expression per element as the GEMM kernels' nf = 1 path (bitwise equal).
constexpr int kSumThr = 128, kSumPer = 8;

__global__ void __launch_bounds__(kSumThr, 8) gsum_sum_kernel(const GOut* __restrict__ outs,
                                                          const GTerm* __restrict__ terms,
                                                          const GLTile* __restrict__ tiles) {
  const GLTile tl = tiles[blockIdx.x];
  const GOut o = outs[tl.out];
  const long long total = (long long)o.m * o.n;
  const long long e0 = (long long)tl.i0 * (kSumThr * kSumPer) + threadIdx.x;
  int ii[kSumPer], jj[kSumPer];
  double acc[kSumPer];
#pragma unroll
  for (int q = 0; q < kSumPer; ++q) {
    const long long e = e0 + (long long)q * kSumThr;
    const bool v = e < total;
    ii[q] = v ? (int)(e / o.n) : -1;
    jj[q] = v ? (int)(e - (long long)ii[q] * o.n) : 0;
    acc[q] = 0.0;
  }
  for (int ti = o.t0; ti < o.t1; ++ti) {
    if (terms[ti].nf != 1) continue;
    const MatRef a = terms[ti].a;
    const double al = terms[ti].alpha;
#pragma unroll
    for (int q = 0; q < kSumPer; ++q)
      if (ii[q] >= 0) acc[q] += al * a.p[(long long)ii[q] * a.rs + (long long)jj[q] * a.cs];
  }
  double cv[kSumPer];  // all reads of C before the first store (see gsum_lean_kernel's epilogue)
#pragma unroll
  for (int q = 0; q < kSumPer; ++q) cv[q] = (o.beta && ii[q] >= 0) ? o.c[(long long)ii[q] * o.ldc + jj[q]] : 0.0;
#pragma unroll
  for (int q = 0; q < kSumPer; ++q)
    if (ii[q] >= 0) o.c[(long long)ii[q] * o.ldc + jj[q]] = cv[q] + acc[q];
}

cudaError_t launch_gsum_sum(const GOut* outs, const GTerm* terms, const GLTile* tiles, int ntiles, cudaStream_t st) {
  if (ntiles == 0) return cudaSuccess;
  gsum_sum_kernel<<<ntiles, kSumThr, 0, st>>>(outs, terms, tiles);
  return cudaGetLastError();
}

int gsum_sum_chunk() { return kSumThr * kSumPer; }

// `wide`: the batch holds 1 x 4 tiles (16 x 128: the larger stage)
cudaError_t launch_gsum_lean(const GOut* outs, const GTerm* terms, const GLTile* tiles, int ntiles, bool wide,
                             cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute((const void*)gsum_lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute((const void*)gsum_lean_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  });
  if (ntiles == 0) return cudaSuccess;
  const size_t smem = sizeof(double) * kPS * (size_t)((wide ? 16 + 128 : 96) * kLdK);
  gsum_lean_kernel<<<ntiles, kThr, smem, st>>>(outs, terms, tiles);
  return cudaGetLastError();
}

}  // namespace h2g
