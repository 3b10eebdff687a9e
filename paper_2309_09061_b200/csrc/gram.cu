// Wide truncated SVD inputs without a protected basis (phase-2 C_t = [V_t Z_t^T | N / ||N|| ...],
// reference coarsening.py:294-326, and the orthogonalisations of h2.py:79-113): the n x n triangular
// factor the one-sided Jacobi needs is formed from the Gram matrix G = C C^T in double-double
// arithmetic instead of a Householder TSQR of C^T.
//
//   gram_dd_partial_kernel  one CTA per (item, column chunk, 64 x 64 tile of G's upper triangle):
//                           G_tile += sum over the chunk's columns of c_i c_j, each product exact
//                           (two_prod) and accumulated as a double-double -- no sequential chain,
//                           every item and chunk independent
//   gram_chol_kernel        one CTA per item: sums the chunk partials (fixed order), then a
//                           pivoted Cholesky of G in double-double (pivot = largest remaining
//                           diagonal = QRCP's largest trailing column norm), one barrier per step.
//                           Row j of the factor is written as doubles at the original column
//                           positions (no physical pivoting: the row-Jacobi that follows is
//                           invariant under column permutations).
//
// Why this is as accurate as the Householder path: the double-double Gram carries ~1e-32 relative
// error against ||C||^2, and so does its Cholesky factor R (R^T R = G + E, ||E|| ~ 1e-32
// sigma_1^2), hence sigma_i(R)^2 = sigma_i(C)^2 + O(1e-32 sigma_1^2) -- far below the FP64 SVD's
// own eps sigma_1 for every singular value the truncation can keep (sigma_1 / thr <= 1e7).  The
// factor is rounded to doubles once (backward error eps ||R||, the same as Householder's).  The
// pivoted Cholesky stops under the same rule as the QRCP preconditioner (trailing mass below
// kDeflate thr_lo), so the rows it drops cannot change a truncation decision.
#include <cuda_runtime.h>

#include <mutex>

#include "h2g_types.h"

namespace h2g {

namespace {

constexpr int kGT = 64;    // Gram tile
constexpr int kGP = 32;    // panel columns
constexpr int kGThr = 256;
static_assert(kGramFlatThreads <= kGThr && kGramFlatThreads % 32 == 0, "flat Gram CTA size");
constexpr int kGSeg = 64;  // staged segment descriptors per Gram CTA
constexpr int kCThr = 512;
constexpr double kEpsG = 2.220446049250313e-16;
constexpr double kDeflateG = 1e-5;

struct dd {
  double hi, lo;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  const double s = a + b;
  return dd{s, b - (s - a)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  double s, e;
  two_sum(a.hi, b.hi, s, e);
  e += a.lo + b.lo;
  return fast_two_sum(s, e);
}
__device__ __forceinline__ dd dd_neg(dd a) { return dd{-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return fast_two_sum(p, e);
}
__device__ __forceinline__ dd dd_recip(dd b) {  // 1 / b, two Newton-style corrections
  const double q1 = __drcp_rn(b.hi);
  // r = 1 - b q1
  dd r = dd_add(dd{1.0, 0.0}, dd_neg(dd_mul(b, dd{q1, 0.0})));
  const double q2 = r.hi * q1;
  dd q = fast_two_sum(q1, q2);
  r = dd_add(dd{1.0, 0.0}, dd_neg(dd_mul(b, q)));
  return dd_add(q, dd{r.hi * q1, 0.0});
}
__device__ __forceinline__ dd dd_sqrt(dd a) {  // a > 0
  const double x = sqrt(a.hi);
  const double p = x * x;
  const double pe = fma(x, x, -p);
  const dd r = dd_add(a, dd{-p, -pe});
  return fast_two_sum(x, r.hi * (0.5 * __drcp_rn(x)));
}

__device__ __forceinline__ double gseg_scale(const Seg& sg) {
  if (!sg.sdiv) return sg.scale;
  const double d = *sg.sdiv;
  return d > 0.0 ? sg.scale / d : sg.scale;
}

__device__ __forceinline__ int gfind_seg(const Seg* __restrict__ segs, int s0, int s1, long long line) {
  int lo = s0, hi = s1 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].off <= line) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ long long pidx(int i, int j, int m) {  // packed upper triangle, i <= j
  return (long long)i * (2 * m - i + 1) / 2 + (j - i);
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// Panels stream through a kGStages-deep shared-memory ring filled by cp.async (8-byte copies,
// consecutive lanes = consecutive panel columns, zero-fill outside the tile / chunk): while a panel
// is multiplied the next ones are in flight, so the FP64 pipe does not wait at the panel barrier
// for the global loads.  Each thread scales the entries it copied (fl(sc * x), as the staged
// values were formed before) once its copies have landed.
constexpr int kGStages = 3;
constexpr int kGLd = kGT + 2;
__host__ __device__ constexpr size_t gram_partial_smem() {
  return sizeof(double) * (size_t)kGStages * 2 * kGP * kGLd;
}

__device__ __forceinline__ void g_cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}

// FLAT: the 64 < m <= 128 block-list work units (own instantiation: separate registers), NT threads
template <bool FLAT, int NT = FLAT ? kGramFlatThreads : kGThr>
__global__ void __launch_bounds__(NT, 2) gram_dd_partial_kernel(const GramItem* __restrict__ items,
                                                                   const Seg* __restrict__ segs,
                                                                   const GramWork* __restrict__ work) {
  extern __shared__ __align__(16) double gring[];  // kGStages x {Pa, Pb} x [kGP][kGLd]
  __shared__ long long s_off[kGSeg];
  __shared__ const double* s_p[kGSeg];
  __shared__ int s_rs[kGSeg], s_cs[kGSeg];
  __shared__ double s_sc[kGSeg];
  __shared__ int s_first, s_n;
  const GramWork w = work[blockIdx.x];
  const GramItem it = items[w.item];
  const int m = it.m;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = NT / 32;
  double hi[16], lo[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) hi[q] = lo[q] = 0.0;
  if (tid == 0) {
    const int a = gfind_seg(segs, it.s0, it.s1, w.c0);
    const int b = gfind_seg(segs, it.s0, it.s1, w.c1 - 1);
    s_first = a;
    s_n = b - a + 1;
  }
  __syncthreads();
  const int sfirst = s_first, ns = s_n;
  const bool staged = ns <= kGSeg;
  if (staged)
    for (int q = tid; q < ns; q += NT) {
      const Seg sg = segs[sfirst + q];
      s_off[q] = sg.off;
      s_p[q] = sg.a.p;
      s_rs[q] = it.hcols ? sg.a.rs : sg.a.cs;  // element stride along a line
      s_cs[q] = it.hcols ? sg.a.cs : sg.a.rs;  // line stride
      s_sc[q] = gseg_scale(sg);
    }
  __syncthreads();
  const long long npan = (w.c1 - w.c0 + kGP - 1) / kGP;
  // segment of line c: its column pointer, element stride and scale
  auto line = [&](long long c, const double*& col, long long& rs, double& sc) {
    if (staged) {
      int lo2 = 0, hi2 = ns - 1;
      while (lo2 < hi2) {
        const int mid = (lo2 + hi2 + 1) >> 1;
        if (s_off[mid] <= c) lo2 = mid; else hi2 = mid - 1;
      }
      col = s_p[lo2] + (c - s_off[lo2]) * s_cs[lo2];
      rs = s_rs[lo2];
      sc = s_sc[lo2];
    } else {
      const Seg sg = segs[gfind_seg(segs, it.s0, it.s1, c)];
      col = sg.a.p + (c - sg.off) * (it.hcols ? sg.a.cs : sg.a.rs);
      rs = it.hcols ? sg.a.rs : sg.a.cs;
      sc = gseg_scale(sg);
    }
  };
  const double* dummy = segs[it.s0].a.p;
  if (FLAT) {
    // ---- flat path (m <= 128): this CTA owns the 4 x 4 blocks b0 .. b0 + nbw - 1 of the upper
    // triangle (row-major order), `reps` threads per block splitting each panel's lines; every
    // panel stages all m rows (zero-padded to a multiple of 4), the replicas are summed in shared
    // memory at the end (one partial slice per column chunk)
    const int reps = w.tj >> 16, nbw = w.tj & 0xffff, b0 = w.ti;
    const int nb = (m + 3) / 4, mp = 4 * nb, ldf = mp + 2;
    const int bpc = reps > 1 ? NT / reps : NT;
    const int lb = tid % bpc, rep = tid / bpc;
    const bool act = lb < nbw;
    int bi = 0, bj = 0;
    {
      int rem = b0 + (act ? lb : 0);
      while (bi < nb && rem >= nb - bi) { rem -= nb - bi; ++bi; }
      bj = bi + rem;
    }
    auto stage_f = [&](int s) { return gring + (size_t)s * kGP * ldf; };
    double scf0 = 0.0, scf1 = 0.0, scf2 = 0.0;
    auto issue_f = [&](long long p) {
      if (p < npan) {
        const int s = (int)(p % kGStages);
        const long long c = w.c0 + p * kGP + lane;
        const double* col = nullptr;
        long long rs = 0;
        double sc = 0.0;
        if (c < w.c1) line(c, col, rs, sc);
        if (s == 0) scf0 = sc; else if (s == 1) scf1 = sc; else scf2 = sc;
        double* P = stage_f(s);
        for (int r = warp; r < mp; r += nw) {
          const bool v = col && r < m;
          g_cp_async8(&P[lane * ldf + r], v ? col + (long long)r * rs : dummy, v);
        }
      }
      asm volatile("cp.async.commit_group;");
    };
#pragma unroll
    for (int p = 0; p < kGStages - 1; ++p) issue_f(p);
    for (long long p = 0; p < npan; ++p) {
      asm volatile("cp.async.wait_group %0;" ::"n"(kGStages - 2));
      {
        const int s = (int)(p % kGStages);
        const double sc = s == 0 ? scf0 : (s == 1 ? scf1 : scf2);
        double* P = stage_f(s);
        for (int r = warp; r < mp; r += nw) P[lane * ldf + r] *= sc;
      }
      __syncthreads();
      issue_f(p + kGStages - 1);
      if (act) {
        const double* P = stage_f((int)(p % kGStages));
#pragma unroll 2
        for (int q0 = rep; q0 < kGP; q0 += reps) {
          const double2 a01 = *reinterpret_cast<const double2*>(&P[q0 * ldf + 4 * bi]);
          const double2 a23 = *reinterpret_cast<const double2*>(&P[q0 * ldf + 4 * bi + 2]);
          const double2 b01 = *reinterpret_cast<const double2*>(&P[q0 * ldf + 4 * bj]);
          const double2 b23 = *reinterpret_cast<const double2*>(&P[q0 * ldf + 4 * bj + 2]);
          const double a[4] = {a01.x, a01.y, a23.x, a23.y};
          const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int q = 4 * u + v;
              const double pr = a[u] * b[v];
              const double pe = fma(a[u], b[v], -pr);
              double s2, e;
              two_sum(hi[q], pr, s2, e);
              hi[q] = s2;
              lo[q] += e + pe;
            }
        }
      }
    }
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();  // the ring is free: replicas' partial sums go there
    double* rb = gring;
    if (act && rep > 0)
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        rb[(size_t)tid * 32 + q] = hi[q];
        rb[(size_t)tid * 32 + 16 + q] = lo[q];
      }
    __syncthreads();
    if (!act || rep > 0) return;
    double* gh = it.gpart + (size_t)w.chunk * 2 * m * m;
    double* gl = gh + (size_t)m * m;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int q = 4 * u + v;
        dd acc = fast_two_sum(hi[q], lo[q]);
        for (int r2 = 1; r2 < reps; ++r2) {  // fixed order: the result does not depend on scheduling
          const size_t o = (size_t)(r2 * bpc + lb) * 32;
          acc = dd_add(acc, dd{rb[o + q], rb[o + 16 + q]});
        }
        const int i = 4 * bi + u, j = 4 * bj + v;
        if (i < m && j < m && i <= j) {
          gh[(size_t)i * m + j] = acc.hi;
          gl[(size_t)i * m + j] = acc.lo;
        }
      }
    return;
  }
  // ---- tiled path: one 64 x 64 tile (ti, tj) of G's upper triangle
  const int ia = w.ti * kGT, jb = w.tj * kGT;
  const bool diag = w.ti == w.tj;
  const int nbi = (min(kGT, m - ia) + 3) / 4, nbj = (min(kGT, m - jb) + 3) / 4;
  const int nblk = diag ? nbi * (nbi + 1) / 2 : nbi * nbj;
  const int reps = gram_reps(m), span = (nblk + 31) / 32 * 32;
  const int rep = tid / span, blk = tid % span;
  const bool act = rep < reps && blk < nblk;
  int bi = 0, bj = 0;
  if (diag) {
    int rem = blk;
    while (bi < nbi && rem >= nbi - bi) { rem -= nbi - bi; ++bi; }
    bj = bi + rem;
  } else {
    bi = blk / nbj;
    bj = blk % nbj;
  }
  // this thread's copies: column `lane` of the panel, rows warp, warp + nw, ...
  auto stage_a = [&](int s) { return gring + (size_t)s * 2 * kGP * kGLd; };
  auto stage_b = [&](int s) { return gring + (size_t)s * 2 * kGP * kGLd + kGP * kGLd; };
  static_assert(kGStages == 3, "scale registers");
  double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0;  // scale of this thread's column per stage (registers)
  auto issue = [&](long long p) {
    if (p < npan) {
      const int s = (int)(p % kGStages);
      const long long c = w.c0 + p * kGP + lane;
      const double* col = nullptr;
      long long rs = 0;
      double sc = 0.0;
      if (c < w.c1) {
        if (staged) {
          int lo2 = 0, hi2 = ns - 1;
          while (lo2 < hi2) {
            const int mid = (lo2 + hi2 + 1) >> 1;
            if (s_off[mid] <= c) lo2 = mid; else hi2 = mid - 1;
          }
          col = s_p[lo2] + (c - s_off[lo2]) * s_cs[lo2];
          rs = s_rs[lo2];
          sc = s_sc[lo2];
        } else {
          const Seg sg = segs[gfind_seg(segs, it.s0, it.s1, c)];
          col = sg.a.p + (c - sg.off) * (it.hcols ? sg.a.cs : sg.a.rs);
          rs = it.hcols ? sg.a.rs : sg.a.cs;
          sc = gseg_scale(sg);
        }
      }
      if (s == 0) sc0 = sc; else if (s == 1) sc1 = sc; else sc2 = sc;
      double* Pa = stage_a(s);
      double* Pb = stage_b(s);
      for (int r = warp; r < kGT; r += nw) {
        const int ra = ia + r, rb = jb + r;
        const bool va = col && ra < m;
        g_cp_async8(&Pa[lane * kGLd + r], va ? col + (long long)ra * rs : dummy, va);
        if (!diag) {
          const bool vb = col && rb < m;
          g_cp_async8(&Pb[lane * kGLd + r], vb ? col + (long long)rb * rs : dummy, vb);
        }
      }
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int p = 0; p < kGStages - 1; ++p) issue(p);
  for (long long p = 0; p < npan; ++p) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kGStages - 2));
    {  // scale the entries this thread copied: fl(sc * x)
      const int s = (int)(p % kGStages);
      const double sc = s == 0 ? sc0 : (s == 1 ? sc1 : sc2);
      double* Pa = stage_a(s);
      double* Pb = stage_b(s);
      for (int r = warp; r < kGT; r += nw) {
        Pa[lane * kGLd + r] *= sc;
        if (!diag) Pb[lane * kGLd + r] *= sc;
      }
    }
    __syncthreads();  // panel p visible to all; every thread is past panel p - 1
    issue(p + kGStages - 1);
    if (act) {
      const int s = (int)(p % kGStages);
      const double* Pa = stage_a(s);
      const double* Pbb = diag ? Pa : stage_b(s);
#pragma unroll 2
      for (int q0 = rep; q0 < kGP; q0 += reps) {
        const double2 a01 = *reinterpret_cast<const double2*>(&Pa[q0 * kGLd + 4 * bi]);
        const double2 a23 = *reinterpret_cast<const double2*>(&Pa[q0 * kGLd + 4 * bi + 2]);
        const double* pb = Pbb + q0 * kGLd;
        const double2 b01 = *reinterpret_cast<const double2*>(pb + 4 * bj);
        const double2 b23 = *reinterpret_cast<const double2*>(pb + 4 * bj + 2);
        const double a[4] = {a01.x, a01.y, a23.x, a23.y};
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int q = 4 * u + v;
            const double pr = a[u] * b[v];
            const double pe = fma(a[u], b[v], -pr);
            double s2, e;
            two_sum(hi[q], pr, s2, e);
            hi[q] = s2;
            lo[q] += e + pe;
          }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;");
  if (!act) return;
  double* gh = it.gpart + (size_t)(w.chunk * reps + rep) * 2 * m * m;
  double* gl = gh + (size_t)m * m;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = ia + 4 * bi + u, j = jb + 4 * bj + v;
      if (i < m && j < m && i <= j) {
        const dd r = fast_two_sum(hi[4 * u + v], lo[4 * u + v]);
        gh[(size_t)i * m + j] = r.hi;
        gl[(size_t)i * m + j] = r.lo;
      }
    }
}

// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void argmax_pair_g(double& best, int& bi, int width) {
  for (int o = width >> 1; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
}

__global__ void __launch_bounds__(kCThr, 1) gram_chol_kernel(const GramItem* __restrict__ items) {
  extern __shared__ __align__(16) double gsm[];
  __shared__ double red[2 * (kCThr / 32)];
  __shared__ int ired[2 * (kCThr / 32)];
  const GramItem it = items[blockIdx.x];
  const int m = it.m;
  const long long np = (long long)m * (m + 1) / 2;
  double* Gh = gsm;
  double* Gl = Gh + np;
  int* roff = reinterpret_cast<int*>(Gl + np);  // packed offset of (i, i)
  int* act = roff + m;                      // two sorted lists of the not-yet-pivoted indices (m each)
  unsigned char* done = reinterpret_cast<unsigned char*>(act + 2 * m);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5, nt = blockDim.x;
  double* R = it.rbuf;  // m x m, row-major
  for (int i = tid; i < m; i += blockDim.x) roff[i] = (int)pidx(i, i, m);
  __syncthreads();
#define PX(i, j) (roff[(i)] + ((j) - (i)))
  // 1. sum the chunk partials in a fixed order
  for (int i = warp; i < m; i += nw)
    for (int j = i + lane; j < m; j += 32) {
      dd acc{0.0, 0.0};
      for (int ch = 0; ch < it.nslice; ++ch) {
        const double* gh = it.gpart + (size_t)ch * 2 * m * m;
        acc = dd_add(acc, dd{gh[(size_t)i * m + j], gh[(size_t)m * m + (size_t)i * m + j]});
      }
      const long long e = PX(i, j);
      Gh[e] = acc.hi;
      Gl[e] = acc.lo;
    }
  for (int c = tid; c < m; c += nt) {
    done[c] = 0;
    act[c] = c;
  }
  __syncthreads();
  // argmax partials of the diagonal (buffer 0)
  {
    double best = -1.0;
    int bi = m;
    for (int i = warp; i < m; i += nw) {
      if (lane == 0) {
        const double d = Gh[PX(i, i)];
        if (d > best || (d == best && i < bi)) { best = d; bi = i; }
      }
    }
    argmax_pair_g(best, bi, 32);
    if (lane == 0) { red[warp] = best; ired[warp] = bi; }
  }
  __syncthreads();
  const long long bigc = (long long)m > it.N ? (long long)m : it.N;
  double stop2 = 0.0;
  int j = 0;
  for (; j < m; ++j) {
    const int buf = (j & 1) * nw, nbuf = ((j + 1) & 1) * nw;
    double best = lane < nw ? red[buf + lane] : -1.0;
    int p = lane < nw ? ired[buf + lane] : m;
    argmax_pair_g(best, p, 32);
    if (p >= m) break;
    const dd gpp{Gh[PX(p, p)], Gl[PX(p, p)]};
    const double bst = gpp.hi + gpp.lo;
    if (!(bst > 0.0)) break;
    if (j == 0) {
      const double thr_lo = fmax(it.tol, (double)bigc * kEpsG * sqrt(bst));
      stop2 = fmax(kEpsG * kEpsG * bst * 0.25, kDeflateG * kDeflateG * thr_lo * thr_lo);
    } else if ((double)(m - j) * bst <= stop2) {
      break;
    }
    // done[p] is read this step only behind explicit `== p` tests (short-circuit), so it is set now
    if (tid == 0) done[p] = 1;
    const dd inv = dd_recip(gpp);
    // row j of the factor: r_c = G_pc / r_pp at the original column positions
    if (warp == (j % nw)) {
      const dd rpp = dd_sqrt(gpp);
      const dd irpp = dd_recip(rpp);
      for (int c = lane; c < m; c += 32) {
        double v;
        if (c == p) {
          v = rpp.hi + rpp.lo;
        } else if (done[c]) {
          v = 0.0;
        } else {
          const long long e = c < p ? PX(c, p) : PX(p, c);
          const dd r = dd_mul(dd{Gh[e], Gl[e]}, irpp);
          v = r.hi + r.lo;
        }
        R[(size_t)j * m + c] = v;
      }
    }
    // Schur complement of the remaining rows / columns over the compact sorted list of the indices
    // not pivoted yet (r = m - j of them, p among them): (m - j)^2 / 2 entries per step instead of a
    // sweep over all m^2 / 2 behind per-entry `done` tests; the list without p (still sorted) is
    // written for step j + 1.  Diagonal argmax partials for step j + 1 as the diagonal is updated.
    const int r = m - j;
    const int* ac = act + (j & 1) * m;
    int* an = act + ((j + 1) & 1) * m;
    for (int t = tid; t < r; t += nt) {
      const int a = ac[t];
      if (a != p) an[a < p ? t : t - 1] = a;
    }
    double cbest = -1.0;
    int cbi = m;
    // two rows per warp iteration: their double-double chains are independent and interleave
    for (int i0 = warp; i0 < r; i0 += 2 * nw) {
      const int i1 = i0 + nw;
      const int a0 = ac[i0], a1 = i1 < r ? ac[i1] : m;
      const bool v0 = a0 != p;
      const bool v1 = i1 < r && a1 != p;
      dd g0{0.0, 0.0}, g1{0.0, 0.0};
      if (v0) {
        const long long e = a0 < p ? PX(a0, p) : PX(p, a0);
        g0 = dd_mul(dd{Gh[e], Gl[e]}, inv);
      }
      if (v1) {
        const long long e = a1 < p ? PX(a1, p) : PX(p, a1);
        g1 = dd_mul(dd{Gh[e], Gl[e]}, inv);
      }
      if (!v0 && !v1) continue;
      for (int k = lane; i0 + k < r; k += 32) {
        const int b0 = ac[i0 + k];
        const int b1 = i1 + k < r ? ac[i1 + k] : m;
        const bool w0 = v0 && b0 != p;
        const bool w1 = v1 && i1 + k < r && b1 != p;
        dd x0{0.0, 0.0}, y0{0.0, 0.0}, x1{0.0, 0.0}, y1{0.0, 0.0};
        long long e0 = 0, e1 = 0;
        if (w0) {
          const long long eb = b0 < p ? PX(b0, p) : PX(p, b0);
          e0 = PX(a0, b0);
          x0 = dd{Gh[eb], Gl[eb]};
          y0 = dd{Gh[e0], Gl[e0]};
        }
        if (w1) {
          const long long eb = b1 < p ? PX(b1, p) : PX(p, b1);
          e1 = PX(a1, b1);
          x1 = dd{Gh[eb], Gl[eb]};
          y1 = dd{Gh[e1], Gl[e1]};
        }
        const dd n0 = dd_add(y0, dd_neg(dd_mul(g0, x0)));
        const dd n1 = dd_add(y1, dd_neg(dd_mul(g1, x1)));
        if (w0) {
          Gh[e0] = n0.hi;
          Gl[e0] = n0.lo;
          if (k == 0) {
            const double d = n0.hi + n0.lo;
            if (d > cbest || (d == cbest && a0 < cbi)) { cbest = d; cbi = a0; }
          }
        }
        if (w1) {
          Gh[e1] = n1.hi;
          Gl[e1] = n1.lo;
          if (k == 0) {
            const double d = n1.hi + n1.lo;
            if (d > cbest || (d == cbest && a1 < cbi)) { cbest = d; cbi = a1; }
          }
        }
      }
    }
    argmax_pair_g(cbest, cbi, 32);
    if (lane == 0) { red[nbuf + warp] = cbest; ired[nbuf + warp] = cbi; }
    __syncthreads();  // Schur complement, partials and done[p] complete
  }
  // rows below the numerical rank: zero (they are deflated, see kDeflateG)
  for (long long e = (long long)j * m + tid; e < (long long)m * m; e += nt) R[e] = 0.0;
  if (tid == 0) *it.nr = j;
#undef PX
}

size_t gram_chol_smem(int m) {
  const size_t np = (size_t)m * (m + 1) / 2;
  return sizeof(double) * 2 * np + sizeof(int) * 3 * (size_t)m + (size_t)m + 16;
}

cudaError_t launch_gram_chol(const GramItem* items, int nitems, int mmax, cudaStream_t st);

cudaError_t launch_gram(const GramItem* items, const Seg* segs, const GramWork* work, int nwork, int nflat,
                        int nitems, int mmax, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)gram_chol_kernel);
    cudaFuncSetAttribute((const void*)gram_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - (int)fa.sharedSizeBytes);
    for (const void* fn : {(const void*)gram_dd_partial_kernel<true>, (const void*)gram_dd_partial_kernel<false>})
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_partial_smem());
  });
  // work units: the flat ones (m <= 128) first, then the tiled ones
  if (nflat > 0) gram_dd_partial_kernel<true><<<nflat, kGramFlatThreads, gram_partial_smem(), st>>>(items, segs, work);
  if (nwork > nflat)
    gram_dd_partial_kernel<false><<<nwork - nflat, kGThr, gram_partial_smem(), st>>>(items, segs, work + nflat);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || nitems == 0) return e;
  return launch_gram_chol(items, nitems, mmax, st);
}

cudaError_t launch_gram_chol(const GramItem* items, int nitems, int mmax, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)gram_chol_kernel);
    cudaFuncSetAttribute((const void*)gram_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024 - (int)fa.sharedSizeBytes);
  });
  if (nitems == 0) return cudaSuccess;
  gram_chol_kernel<<<nitems, mmax <= 64 ? 256 : kCThr, gram_chol_smem(mmax), st>>>(items);
  return cudaGetLastError();
}

}  // namespace h2g
