// Batched FP64 kernels for the adaptive H^2 product on sm_100a.
//
//   (grouped chain products C (+)= sum alpha * A*B(*D): gemm.cu, DMMA)
//   qr_r_kernel  : R factor of a stacked tall matrix, streamed in 32-row panels    (dense.py:145-150)
//   svd_*_kernel : protected, QR-preconditioned one-sided Jacobi truncated SVD    (dense.py:77-101,
//                  induced.py:115-146, coarsening.py:294-326)
//   norm_kernel  : sigma_1 via a streamed Gram matrix, Householder tridiagonalisation
//                  and Sturm bisection                                            (dense.py:104-142)
//
// FP64 has no tcgen05 kind; B200's FP64 pipe (DFMA and legacy DMMA measured at the same
// ~37 TFLOP/s, profiles/r01_fp64_peak.json) is fed from shared-memory tiles.  One CTA per
// output tile (gsum) or per matrix (factorisations); grids are sized by the batch.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>
#include <mutex>

#include "h2g_types.h"

namespace h2g {

static void init_attributes();

static constexpr int kThreads = 256;
static constexpr int kPanel = 32;  // TSQR / Gram panel rows (one per lane)
static constexpr int kRawLd = kPanel + 1;  // odd stride of the m x 32 protect panel
static constexpr double kEps = 2.220446049250313e-16;

__device__ __forceinline__ double mref(const MatRef& a, long long i, long long j) {
  return a.p[i * a.rs + j * a.cs];
}

// effective scale of a segment: host factor times 1 / (device norm) when given and positive
// (reference coarsening.py:247-252 `scaled`: divide only when nrm > 0)
__device__ __forceinline__ double seg_scale(const Seg& sg) {
  if (!sg.sdiv) return sg.scale;
  const double d = *sg.sdiv;
  return d > 0.0 ? sg.scale / d : sg.scale;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------------------------
// Streamed structured Householder update (TSQR step): [R; P] -> R', R (n x n upper triangular),
// P (32 x n) the next rows.
// ---------------------------------------------------------------------------------------------

// [R; P] -> R' (structured TSQR step).  A quad of lanes owns one trailing column (lane q of the
// quad holds panel rows 8q..8q+7): reflector j is applied with an 8-term partial dot product, a
// 2-step quad reduction and an 8-term update.  Column j+1 is always the first column of quad 0,
// which right after its update builds reflector j+1 from the same registers' rows (norm, beta,
// tau, v) -- the per-column critical path is a handful of dependent FMAs.  One barrier per
// column; columns < jstart of P are known to be zero (triangular panels in merges).
__device__ void tsqr_absorb(double* R, int n, double* P, int ldp, double* vb /*64*/, double* tb /*2*/,
                            int jstart = 0) {
  const int tid = threadIdx.x;
  const int quad = tid >> 2, q = tid & 3, r0 = q * 8;
  constexpr int kQuads = kThreads / 4;
  if (jstart >= n) return;
  auto make = [&](int j, double* v, double* t) {  // quad 0 only
    double x[8], s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i] = P[(r0 + i) * ldp + j];
      s = fma(x[i], x[i], s);
    }
    s += __shfl_xor_sync(0x0000000fu, s, 1);
    s += __shfl_xor_sync(0x0000000fu, s, 2);
    const double alpha = R[(long long)j * n + j];
    double tau = 0.0, scale = 0.0;
    if (s != 0.0) {
      const double nrm = sqrt(alpha * alpha + s);
      const double beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
      if (q == 0) R[(long long)j * n + j] = beta;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) v[r0 + i] = x[i] * scale;
    if (q == 0) *t = tau;
  };
  if (quad == 0) make(jstart, vb + (jstart & 1) * 32, tb + (jstart & 1));
  __syncthreads();
  for (int j = jstart; j < n; ++j) {
    const int cur = j & 1;
    const double tau = tb[cur];
    const double* v = vb + cur * 32;
    if (tau != 0.0) {
      double vr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) vr[i] = v[r0 + i];
      const int wq = quad & 7;  // quad within the warp: all lanes of a warp iterate together
      for (int cb = j + 1 + (quad - wq); cb < n; cb += kQuads) {
        const int c = cb + wq;
        const bool act = c < n;
        double w = 0.0;
        if (act) {
#pragma unroll
          for (int i = 0; i < 8; ++i) w = fma(vr[i], P[(r0 + i) * ldp + c], w);
        }
        w += __shfl_xor_sync(0xffffffffu, w, 1);
        w += __shfl_xor_sync(0xffffffffu, w, 2);
        if (act) {
          const double tw = tau * (w + R[(long long)j * n + c]);
          if (q == 0) R[(long long)j * n + c] -= tw;
#pragma unroll
          for (int i = 0; i < 8; ++i) P[(r0 + i) * ldp + c] -= tw * vr[i];
        }
      }
    }
    if (quad == 0 && j + 1 < n) {
      __syncwarp(0x0000000fu);
      make(j + 1, vb + (cur ^ 1) * 32, tb + (cur ^ 1));
    }
    __syncthreads();
  }
}

// Locate element col `c` of an hstack of segments: returns the segment index (linear scan cursor).
struct SegCursor {
  int s;          // current segment
  long long off;  // first global column of segment s
};

// Fill P (32 x nrows) with P[p][i] = scale * A(i, col0 + p) for an hstack of segments (A: m x N).
// With `raw` non-null, writes raw[i * 32 + p] instead (m x 32 panel, column p).
__device__ void load_hpanel(const Seg* segs, int s0, int s1, int m, long long N, long long col0,
                            double* dst, bool transpose_rows, int ldd) {
  // each warp handles a set of panel columns; lanes run over rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int p = warp; p < kPanel; p += nw) {
    const long long c = col0 + p;
    if (c >= N) {
      for (int i = lane; i < m; i += 32) {
        if (transpose_rows) dst[p * ldd + i] = 0.0; else dst[i * ldd + p] = 0.0;
      }
      continue;
    }
    // find the segment containing column c
    long long off = 0;
    int s = s0;
    for (; s < s1; ++s) {
      if (c < off + segs[s].w) break;
      off += segs[s].w;
    }
    const Seg sg = segs[s];
    const long long lc = c - off;
    for (int i = lane; i < m; i += 32) {
      const double val = seg_scale(sg) * mref(sg.a, i, lc);
      if (transpose_rows) dst[p * ldd + i] = val; else dst[i * ldd + p] = val;
    }
  }
}

// Fill P (32 x n) with rows row0.. of vstack(segs) (M x n), zero beyond M.
__device__ void load_vpanel(const Seg* segs, int s0, int s1, int n, long long M, long long row0, double* P,
                            int ldp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int p = warp; p < kPanel; p += nw) {
    const long long r = row0 + p;
    if (r >= M) {
      for (int j = lane; j < n; j += 32) P[p * ldp + j] = 0.0;
      continue;
    }
    long long off = 0;
    int s = s0;
    for (; s < s1; ++s) {
      if (r < off + segs[s].w) break;
      off += segs[s].w;
    }
    const Seg sg = segs[s];
    const long long lr = r - off;
    const double ssc = seg_scale(sg);
    for (int j = lane; j < n; j += 32) P[p * ldp + j] = ssc * mref(sg.a, lr, j);
  }
}

// Register-staged panel fetch: every thread holds up to kFetch elements of the NEXT 32-line panel,
// so its global loads are in flight while the current panel is absorbed (the absorb loop is
// latency bound; without the prefetch each panel waited on a chain of dependent HBM loads).
static constexpr int kFetch = 16;  // 32 lines x 128 entries / 256 threads

struct PanelFetch {
  double v[kFetch];
};

__device__ __forceinline__ int find_seg(const Seg* __restrict__ segs, int s0, int s1, long long line) {
  int lo = s0, hi = s1 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].off <= line) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// rows r0..r0+31 of vstack(segs) (M x n): element e -> (p = e / n, j = e % n), row-coalesced
__device__ __forceinline__ void fetch_vrows(PanelFetch& f, const Seg* __restrict__ segs, int s0, int s1, int n,
                                            long long M, long long r0) {
  const int tot = kPanel * n;
  int cur_p = -1;
  MatRef a{nullptr, 0, 0};
  double sc = 0.0;
  long long off = 0;
#pragma unroll
  for (int q = 0; q < kFetch; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    double val = 0.0;
    if (e < tot) {
      const int p = e / n, j = e - p * n;
      const long long r = r0 + p;
      if (r < M) {
        if (p != cur_p) {
          const Seg& sg = segs[find_seg(segs, s0, s1, r)];
          a = sg.a;
          sc = seg_scale(sg);
          off = sg.off;
          cur_p = p;
        }
        val = sc * mref(a, r - off, j);
      }
    }
    f.v[q] = val;
  }
}

__device__ __forceinline__ void store_vrows(const PanelFetch& f, double* P, int ldp, int n) {
  const int tot = kPanel * n;
#pragma unroll
  for (int q = 0; q < kFetch; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    if (e < tot) {
      const int p = e / n, j = e - p * n;
      P[p * ldp + j] = f.v[q];
    }
  }
}

// columns c0..c0+31 of hstack(segs) (m x N): element e -> (i = e / 32, p = e % 32); a thread keeps
// one column p for all its elements (blockDim is a multiple of 32), so one segment lookup per panel
__device__ __forceinline__ void fetch_hcols(PanelFetch& f, const Seg* __restrict__ segs, int s0, int s1, int m,
                                            long long N, long long c0) {
  const int p = threadIdx.x & 31;
  const long long c = c0 + p;
  MatRef a{nullptr, 0, 0};
  double sc = 0.0;
  long long lc = 0;
  const bool live = c < N;
  if (live) {
    const Seg& sg = segs[find_seg(segs, s0, s1, c)];
    a = sg.a;
    sc = seg_scale(sg);
    lc = c - sg.off;
  }
  const int tot = kPanel * m;
#pragma unroll
  for (int q = 0; q < kFetch; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    f.v[q] = (live && e < tot) ? sc * mref(a, e >> 5, lc) : 0.0;
  }
}

// store as P[p * ld + i] (transposed: panel rows are the stack's columns) or raw[i * ld + p]
__device__ __forceinline__ void store_hcols(const PanelFetch& f, double* dst, int ld, int m, bool transpose) {
  const int tot = kPanel * m;
#pragma unroll
  for (int q = 0; q < kFetch; ++q) {
    const int e = threadIdx.x + q * blockDim.x;
    if (e < tot) {
      const int i = e >> 5, p = e & 31;
      if (transpose) dst[p * ld + i] = f.v[q]; else dst[i * ld + p] = f.v[q];
    }
  }
}

// ---------------------------------------------------------------------------------------------
// qr_r: R factor of vstack(segs) (reference dense.py:145-150 / numpy qr mode="r"), as a chunked
// TSQR: qr_chunk_kernel reduces 256-row chunks (one CTA each) to partial R factors,
// tsqr_merge_kernel combines them pairwise, qr_out_kernel writes the first min(M, n) rows.
// ---------------------------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads, 3) qr_chunk_kernel(const QrItem* __restrict__ items,
                                                             const Seg* __restrict__ segs,
                                                             const SvdWork* __restrict__ work, int rsmem) {
  extern __shared__ double smem[];
  const SvdWork w = work[blockIdx.x];
  const QrItem it = items[w.item];
  const int n = it.n;
  const int ldp = n | 1;               // odd row stride: conflict-free column access
  double* P = smem;                    // 32 x ldp
  double* vb = P + kPanel * ldp;       // 64
  double* tb = vb + 64;                // 2 (+pad)
  double* R = rsmem ? tb + 4 : it.rbuf + (long long)w.a * n * n;
  const long long nn = (long long)n * n;
  for (long long e = threadIdx.x; e < nn; e += blockDim.x) R[e] = 0.0;
  __syncthreads();
  const long long per = (it.M + it.nchunk - 1) / it.nchunk;
  const long long rbeg = w.a * per, rend = min(it.M, rbeg + per);
  const bool pre = kPanel * n <= kFetch * (int)blockDim.x;
  PanelFetch f;
  if (pre && rbeg < rend) fetch_vrows(f, segs, it.s0, it.s1, n, rend, rbeg);
  for (long long r0 = rbeg; r0 < rend; r0 += kPanel) {
    if (pre) store_vrows(f, P, ldp, n);
    else load_vpanel(segs, it.s0, it.s1, n, rend, r0, P, ldp);
    __syncthreads();
    if (pre && r0 + kPanel < rend) fetch_vrows(f, segs, it.s0, it.s1, n, rend, r0 + kPanel);
    tsqr_absorb(R, n, P, ldp, vb, tb);
  }
  if (rsmem) {
    double* dst = it.rbuf + (long long)w.a * n * n;
    for (long long e = threadIdx.x; e < nn; e += blockDim.x) dst[e] = R[e];
  }
}

__global__ void __launch_bounds__(kThreads, 3) tsqr_merge_kernel(const MergeWork* __restrict__ work, int rsmem) {
  extern __shared__ double smem[];
  const MergeWork w = work[blockIdx.x];
  const int n = w.n;
  const int ldp = n | 1;
  double* P = smem;               // 32 x ldp
  double* vb = P + kPanel * ldp;  // 64
  double* tb = vb + 64;           // 4
  double* Ra = w.rbuf + (long long)w.a * n * n;
  const double* Rb = w.rbuf + (long long)w.b * n * n;
  double* R = rsmem ? tb + 4 : Ra;
  if (rsmem)
    for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) R[e] = Ra[e];
  for (int r0 = 0; r0 < n; r0 += kPanel) {
    for (int e = threadIdx.x; e < kPanel * n; e += blockDim.x) {
      const int p = e / n, j = e % n;
      P[p * ldp + j] = (r0 + p < n) ? Rb[(long long)(r0 + p) * n + j] : 0.0;
    }
    __syncthreads();
    tsqr_absorb(R, n, P, ldp, vb, tb, r0);
  }
  if (rsmem) {
    __syncthreads();
    for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) Ra[e] = R[e];
  }
}

__global__ void qr_out_kernel(const QrItem* __restrict__ items) {
  const QrItem it = items[blockIdx.x];
  const int n = it.n;
  const long long rows = it.M < n ? it.M : n;
  for (long long e = threadIdx.x; e < rows * n; e += blockDim.x) {
    const long long i = e / n, j = e % n;
    it.out[e] = (it.full || j >= i) ? it.rbuf[i * n + j] : 0.0;
  }
}

// ---------------------------------------------------------------------------------------------
// One-sided Jacobi on the ROWS of W (n x n, row-major): afterwards the rows are mutually
// orthogonal to working precision (relative cosine criterion), so normalised rows are
// orthonormal regardless of the row norms.  Round-robin pairing, one pair per warp at a time.
// ---------------------------------------------------------------------------------------------

// Rotation of the row pair (a, b) with Gram entries al = |a|^2, be = |b|^2, ga = a.b:
// t = sign(d) 2ga / (|d| + hypot(d, 2ga)), d = be - al (the smaller root of t^2 + 2 zeta t - 1,
// zeta = d / 2ga; Rutishauser), c = 1 / sqrt(1 + t^2), s = c t.  One sqrt, one division, one rsqrt.
// Row stride of R in the finish kernel's shared memory: >= n and == 4 (mod 16) -- even (double2
// rows) and 8 banks between consecutive rows.
__host__ __device__ inline int fin_ld(int n) { return n + (20 - n % 16) % 16; }

__device__ __forceinline__ void jacobi_rotation(double al, double be, double ga, double& c, double& sn) {
  const double d = be - al, g2 = 2.0 * ga;
  const double ad = fabs(d), ag = fabs(g2);
  double t;
  const double mx = fmax(ad, ag);
  if (mx > 1e150 || mx < 1e-150) {  // far from 1: scale-free form (no over/underflow of d^2 + g2^2)
    const double zeta = d / g2, az = fabs(zeta);
    const double t0 = az > 1e150 ? 0.5 / az : 1.0 / (az + sqrt(fma(az, az, 1.0)));
    t = zeta >= 0.0 ? t0 : -t0;
  } else {
    // r = |(d, g2)| and 1 / (|d| + r) by reciprocal square root / reciprocal (short dependent
    // chains); t only steers the rotation, its orthogonality comes from c = 1 / sqrt(1 + t^2)
    const double r2 = fma(d, d, g2 * g2);
    const double r = r2 * rsqrt(r2);
    t = g2 * __drcp_rn(ad + r);
    if (d < 0.0) t = -t;
  }
  c = rsqrt(fma(t, t, 1.0));
  sn = c * t;
}

// NPL > 0: rows of length n <= 16 NPL held in registers per half-warp (unrolled); NPL = 0: loops.
template <int NPL>
__device__ int jacobi_rows(double* W, int nr, int n, int ld, int* flag, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // Rows whose norm is below eps * (largest row norm) can never pass the truncation threshold
  // (thr >= max(rows, cols) eps sigma_1); rotating against them moves the other row by less than
  // eps relative, so they are frozen.  Without this the numerically-null rows of rank-deficient
  // inputs keep the sweep loop busy orthogonalising rounding noise.
  {
    double mx = 0.0;
    for (int i = warp; i < nr; i += nw) {
      double s = 0.0;
      for (int j = lane; j < n; j += 32) s = fma(W[(long long)i * ld + j], W[(long long)i * ld + j], s);
      s = warp_sum(s);
      mx = fmax(mx, s);
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < nw; ++w) m = fmax(m, red[w]);
      red[nw] = m * kEps * kEps;
    }
    __syncthreads();
  }
  const double frozen = red[nw];
  const int np = (nr + 1) & ~1;  // even number of players, player nr (if odd) is a bye
  const int npairs = np / 2, m1 = np - 1;
  // convergence threshold sqrt(n) eps (LAPACK dgesvj); tested squared to avoid square roots
  const double tol2 = kEps * kEps * (double)n;
  // one row pair per half-warp (16 lanes, 4-step butterflies)
  const int half = lane >> 4, hl = lane & 15;
  const int slot = 2 * warp + half, nslots = 2 * nw;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < m1; ++step) {
      for (int q = slot; q < npairs; q += nslots) {
        // circle method: player 0 fixed, players 1..np-1 rotate by `step` (no integer division)
        int xa = q + step;
        if (xa >= m1) xa -= m1;
        int xb = (q == 0 ? 0 : m1 - q) + step;
        if (xb >= m1) xb -= m1;
        if (xb >= m1) xb -= m1;
        const int a = (q == 0) ? 0 : 1 + xa;
        const int b = 1 + xb;
        if (a >= nr || b >= nr) continue;  // bye (odd nr): uniform per half-warp
        double* ra = W + (long long)a * ld;
        double* rb = W + (long long)b * ld;
        double al = 0.0, be = 0.0, ga = 0.0;
        double xav[NPL > 0 ? NPL : 1], xbv[NPL > 0 ? NPL : 1];
        if (NPL > 0) {
#pragma unroll
          for (int k = 0; k < NPL; ++k) {
            const int j = hl + 16 * k;
            xav[k] = j < n ? ra[j] : 0.0;
            xbv[k] = j < n ? rb[j] : 0.0;
          }
#pragma unroll
          for (int k = 0; k < NPL; ++k) {
            al = fma(xav[k], xav[k], al);
            be = fma(xbv[k], xbv[k], be);
            ga = fma(xav[k], xbv[k], ga);
          }
        } else {
          for (int j = hl; j < n; j += 16) {
            const double x = ra[j], y = rb[j];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
        }
        const unsigned hmask = 0xffffu << (16 * half);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {  // three independent butterflies within the half-warp
          al += __shfl_xor_sync(hmask, al, o);
          be += __shfl_xor_sync(hmask, be, o);
          ga += __shfl_xor_sync(hmask, ga, o);
        }
        if (ga != 0.0 && al > frozen && be > frozen && ga * ga > tol2 * al * be) {
          double c, sn;
          jacobi_rotation(al, be, ga, c, sn);
          if (NPL > 0) {
#pragma unroll
            for (int k = 0; k < NPL; ++k) {
              const int j = hl + 16 * k;
              if (j < n) {
                ra[j] = c * xav[k] - sn * xbv[k];
                rb[j] = sn * xav[k] + c * xbv[k];
              }
            }
          } else {
            for (int j = hl; j < n; j += 16) {
              const double x = ra[j], y = rb[j];
              ra[j] = c * x - sn * y;
              rb[j] = sn * x + c * y;
            }
          }
          if (hl == 0) *flag = 1;
        }
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) return sweep + 1;
  }
  return 40;
}

// Octet variant: one row pair per 8 lanes (64 pairs per 512-thread CTA, i.e. n <= 128), NPL =
// ceil(n / 8) entries per lane.  Against the half-warp version it halves the lanes per pair, so
// every step is one round and the three butterflies cost 3 levels per 4 pairs instead of 4 levels
// per 2 -- the step is then bound by the FP64 pipe rather than by shuffles and issue overhead.
// V2 (R in shared memory, ld even and the padding columns zero): lane ol of an octet owns the
// double2 pairs (2 ol, 2 ol + 1) + 16 k, so each octet's LDS.128 / STS.128 covers 128 contiguous
// bytes -- one conflict-free quarter-warp wavefront whatever the two rows are (the scalar mapping
// ol + 8 k put two rows' 64-byte windows in one half-warp, two-way conflicts for most pairs).
// Stop after a sweep whose rotations all had |cos angle| = |gamma| / sqrt(alpha beta) <= 1e-9:
// cyclic Jacobi converges quadratically, so the rows are then orthogonal to ~1e-18 and the
// confirming sweep (which would find nothing above the sqrt(n) eps threshold) is skipped.
static constexpr double kQuad = 1e-18;
template <int NPL, bool V2>
__device__ int jacobi_rows_oct(double* W, int nr, int n, int ld, int* flag, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  {
    double mx = 0.0;
    for (int i = warp; i < nr; i += nw) {
      double s = 0.0;
      for (int j = lane; j < n; j += 32) s = fma(W[(long long)i * ld + j], W[(long long)i * ld + j], s);
      s = warp_sum(s);
      mx = fmax(mx, s);
    }
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = 0.0;
      for (int w = 0; w < nw; ++w) m = fmax(m, red[w]);
      red[nw] = m * kEps * kEps;
    }
    __syncthreads();
  }
  const double frozen = red[nw];
  const int np = (nr + 1) & ~1;
  const int npairs = np / 2, m1 = np - 1;
  const double tol2 = kEps * kEps * (double)n;
  const int q0 = threadIdx.x >> 3, ol = lane & 7, nq = blockDim.x >> 3;
  const unsigned omask = 0xffu << (lane & 24);
  // circle method positions of this octet's pairs (q0 and q0 + nq: n <= 192 with 64 octets),
  // advanced by one per step (no divisions)
  int xa0 = q0 < m1 ? q0 : 0, xb0 = q0 == 0 ? 0 : (q0 < m1 ? m1 - q0 : 0);
  if (xb0 >= m1) xb0 -= m1;
  int xa1 = q0 + nq < m1 ? q0 + nq : 0, xb1 = q0 + nq < m1 ? m1 - q0 - nq : 0;
  if (xb1 >= m1) xb1 -= m1;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) flag[0] = flag[1] = 0;
    __syncthreads();
    for (int step = 0; step < m1; ++step) {
     constexpr int kReps = NPL > 16 ? 2 : 1;  // n <= 128: one pair per octet suffices
#pragma unroll
     for (int r = 0; r < kReps; ++r) {
      const int q = q0 + r * nq;
      const int a = (q == 0) ? 0 : 1 + (r ? xa1 : xa0);
      const int b = 1 + (r ? xb1 : xb0);
      if (q < npairs && a < nr && b < nr) {
        double* ra = W + a * ld;
        double* rb = W + b * ld;
        double x[NPL], y[NPL];
        if (V2) {
#pragma unroll
          for (int k = 0; k < NPL; k += 2) {
            const int j = 2 * ol + 8 * k;
            double2 u = make_double2(0.0, 0.0), v = make_double2(0.0, 0.0);
            if (j < n) {
              u = *reinterpret_cast<const double2*>(ra + j);
              v = *reinterpret_cast<const double2*>(rb + j);
            }
            x[k] = u.x; x[k + 1] = u.y;
            y[k] = v.x; y[k + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int k = 0; k < NPL; ++k) {
            const int j = ol + 8 * k;
            x[k] = j < n ? ra[j] : 0.0;
            y[k] = j < n ? rb[j] : 0.0;
          }
        }
        double al0 = 0.0, be0 = 0.0, ga0 = 0.0, al1 = 0.0, be1 = 0.0, ga1 = 0.0;
#pragma unroll
        for (int k = 0; k < NPL; k += 2) {
          al0 = fma(x[k], x[k], al0);
          be0 = fma(y[k], y[k], be0);
          ga0 = fma(x[k], y[k], ga0);
          if (k + 1 < NPL) {
            al1 = fma(x[k + 1], x[k + 1], al1);
            be1 = fma(y[k + 1], y[k + 1], be1);
            ga1 = fma(x[k + 1], y[k + 1], ga1);
          }
        }
        double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          al += __shfl_xor_sync(omask, al, o);
          be += __shfl_xor_sync(omask, be, o);
          ga += __shfl_xor_sync(omask, ga, o);
        }
        if (ga != 0.0 && al > frozen && be > frozen && ga * ga > tol2 * al * be) {
          double c, sn;
          jacobi_rotation(al, be, ga, c, sn);
          if (V2) {
#pragma unroll
            for (int k = 0; k < NPL; k += 2) {
              const int j = 2 * ol + 8 * k;
              if (j < n) {
                *reinterpret_cast<double2*>(ra + j) = make_double2(c * x[k] - sn * y[k], c * x[k + 1] - sn * y[k + 1]);
                *reinterpret_cast<double2*>(rb + j) = make_double2(sn * x[k] + c * y[k], sn * x[k + 1] + c * y[k + 1]);
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < NPL; ++k) {
              const int j = ol + 8 * k;
              if (j < n) {
                ra[j] = c * x[k] - sn * y[k];
                rb[j] = sn * x[k] + c * y[k];
              }
            }
          }
          if (ol == 0) {
            flag[0] = 1;
            if (ga * ga > kQuad * al * be) flag[1] = 1;
          }
        }
      }
     }
      if (++xa0 == m1) xa0 = 0;
      if (++xb0 == m1) xb0 = 0;
      if (++xa1 == m1) xa1 = 0;
      if (++xb1 == m1) xb1 = 0;
      __syncthreads();
    }
    const int any = flag[0], large = flag[1];
    __syncthreads();
    if (!any || !large) return sweep + 1;
  }
  return 40;
}

// ---------------------------------------------------------------------------------------------
// Truncated SVD pipeline (see SvdItem), split so one wide matrix spreads over many CTAs:
//   svd_tsqr_kernel   one CTA per (item, column chunk): Householder QR of the protected V,
//                     Q^T applied to each 32-column panel, structured TSQR into R_chunk
//   svd_merge_kernel  one CTA per tree merge: R_a <- R([R_a; R_b]) (triangular panels skip
//                     their known-zero columns)
//   svd_finish_kernel one CTA per item: one-sided Jacobi on the rows of R, rank rule, outputs
// ---------------------------------------------------------------------------------------------

__device__ void householder_qr_cols(double* V, int m, int kx, int ldv, int k1, double* tv, double* red) {
  // In-place Householder QR of V (m x kx, row-major): reflector j stored below the diagonal
  // (implicit 1 on the diagonal), R on and above.  LAPACK dgeqrf sign convention.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = 0; j < k1; ++j) {
    // norm of V[j+1:, j]
    double part = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) part += V[i * ldv + j] * V[i * ldv + j];
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w];
      const double alpha = V[j * ldv + j];
      double tau = 0.0, scale = 0.0;
      if (s != 0.0) {
        const double nrm = sqrt(alpha * alpha + s);
        const double beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
        V[j * ldv + j] = beta;
      }
      tv[j] = tau;
      red[nw] = scale;
    }
    __syncthreads();
    const double scale = red[nw];
    const double tau = tv[j];
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) V[i * ldv + j] *= scale;
    __syncthreads();
    if (tau != 0.0) {
      for (int c = j + 1 + warp; c < kx; c += nw) {
        double w = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w += V[i * ldv + j] * V[i * ldv + c];
        w = warp_sum(w) + V[j * ldv + c];
        __syncwarp();
        if (lane == 0) V[j * ldv + c] -= tau * w;
        for (int i = j + 1 + lane; i < m; i += 32) V[i * ldv + c] -= tau * w * V[i * ldv + j];
      }
    }
    __syncthreads();
  }
}

// Apply H_j (j in [jb, je) in the given direction) to column c of X (rows m, ld ldx) by one warp.
__device__ __forceinline__ void apply_reflector_col(const double* V, int ldv, int m, int j, double tau,
                                                    double* X, int ldx, int c) {
  const int lane = threadIdx.x & 31;
  double w = X[(long long)j * ldx + c];
  double part = 0.0;
  for (int i = j + 1 + lane; i < m; i += 32) part += V[i * ldv + j] * X[(long long)i * ldx + c];
  w += warp_sum(part);
  __syncwarp();
  if (lane == 0) X[(long long)j * ldx + c] -= tau * w;
  for (int i = j + 1 + lane; i < m; i += 32) X[(long long)i * ldx + c] -= tau * w * V[i * ldv + j];
  __syncwarp();
}


__device__ __forceinline__ int svd_n(const SvdItem& it) { return it.m - min(it.m, it.kx); }

__device__ void load_v_factor(const SvdItem& it, double* V, int ldv, double* tv, double* red) {
  const int m = it.m, kx = it.kx, k1 = min(m, kx);
  for (int e = threadIdx.x; e < m * kx; e += blockDim.x) V[(e / kx) * ldv + e % kx] = mref(it.v, e / kx, e % kx);
  __syncthreads();
  householder_qr_cols(V, m, kx, ldv, k1, tv, red);
}

__global__ void __launch_bounds__(kThreads, 3) svd_tsqr_kernel(const SvdItem* __restrict__ items,
                                                            const Seg* __restrict__ segs,
                                                            const SvdWork* __restrict__ work, int rsmem) {
  extern __shared__ double smem[];
  __shared__ double red[40];
  const SvdWork w = work[blockIdx.x];
  const SvdItem it = items[w.item];
  const int m = it.m, kx = it.kx, k1 = min(m, kx), n = svd_n(it);
  const long long N = it.N;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ldv = kx | 1, ldp = n | 1;            // odd strides: conflict-free lane-per-row access
  double* V = smem;                                // m x ldv
  double* tv = V + (long long)m * ldv;             // kx + 1
  double* raw = tv + kx + 1;                       // m x kRawLd (protect case)
  double* P = raw + (kx > 0 ? m * kRawLd : 0);     // 32 x ldp
  double* vb = P + kPanel * ldp;                   // 64
  double* tb = vb + 64;                            // 4
  double* R = rsmem ? tb + 4 : it.rbuf + (long long)w.a * n * n;
  if (kx > 0) {
    load_v_factor(it, V, ldv, tv, red);
    if (w.a == 0) {
      for (int e = threadIdx.x; e < m * ldv; e += blockDim.x) it.vws[e] = V[e];
      for (int e = threadIdx.x; e < kx; e += blockDim.x) it.vws[m * ldv + e] = tv[e];
    }
  }
  if (n == 0) return;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) R[e] = 0.0;
  __syncthreads();
  const long long per = (N + it.nchunk - 1) / it.nchunk;
  const long long cbeg = w.a * per, cend = min(N, cbeg + per);
  const bool pre = kPanel * m <= kFetch * (int)blockDim.x;
  PanelFetch f;
  if (pre && cbeg < cend) fetch_hcols(f, segs, it.s0, it.s1, m, min(cend, cbeg + kPanel), cbeg);
  for (long long c0 = cbeg; c0 < cend; c0 += kPanel) {
    const long long lim = min(cend, c0 + kPanel);  // columns beyond this chunk load as zero
    if (kx > 0) {
      if (pre) store_hcols(f, raw, kRawLd, m, false);
      else load_hpanel(segs, it.s0, it.s1, m, lim, c0, raw, false, kRawLd);
      __syncthreads();
      if (pre && c0 + kPanel < cend) fetch_hcols(f, segs, it.s0, it.s1, m, min(cend, c0 + 2 * kPanel), c0 + kPanel);
      for (int p = warp; p < kPanel; p += nw)
        for (int j = 0; j < k1; ++j)
          if (tv[j] != 0.0) apply_reflector_col(V, ldv, m, j, tv[j], raw, kRawLd, p);
      __syncthreads();
      for (int e = threadIdx.x; e < kPanel * n; e += blockDim.x) {
        const int p = e / n, i = e % n;
        P[p * ldp + i] = raw[(k1 + i) * kRawLd + p];
      }
    } else {
      if (pre) store_hcols(f, P, ldp, m, true);
      else load_hpanel(segs, it.s0, it.s1, m, lim, c0, P, true, ldp);
      __syncthreads();
      if (pre && c0 + kPanel < cend) fetch_hcols(f, segs, it.s0, it.s1, m, min(cend, c0 + 2 * kPanel), c0 + kPanel);
    }
    __syncthreads();
    tsqr_absorb(R, n, P, ldp, vb, tb);
  }
  if (rsmem) {
    double* dst = it.rbuf + (long long)w.a * n * n;
    for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) dst[e] = R[e];
  }
}

// Householder QR with column pivoting of W (n x n, row-major), in place; only the triangular factor
// is kept.  perm[c] = original column of column c.  Used as the Jacobi preconditioner
// (Drmac-Veselic): W Pi = Q1 R1, and the rows of R1 are graded by the pivoting, so one-sided Jacobi
// on them needs a few sweeps instead of ~15.  Left singular vectors of W^T = Pi x those of R1^T.
// Truncation-aware deflation (stop_scale > 0): the threshold is thr = max(tol, big eps sigma_1) >=
// thr_lo = max(tol, big eps |r_00|) (|r_00| = largest column norm <= sigma_1).  Once the trailing
// block's Frobenius norm is <= kDeflate thr_lo, dropping its rows moves every singular value by at
// most kDeflate^2 thr / 2 relative to thr (sigma_i(A)^2 - sigma_i(B)^2 in [0, ||C||^2] for A =
// [B; C]) -- below the FP64 SVD's own absolute error eps sigma_1 (sigma_1 / thr <= 1e7 on every
// config), so no truncation decision changes, and the kept rows' Jacobi runs on fewer rows.
static constexpr double kDeflate = 1e-5;

__device__ __forceinline__ void argmax_pair(double& best, int& bi, unsigned mask, int width) {
  // (value, index) maximum over `width` lanes, ties to the smaller index
  for (int o = width >> 1; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(mask, best, o);
    const int oi = __shfl_xor_sync(mask, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
}

// One barrier per pivot step.  Columns never move: the pivot p of step j is recorded (pst[p] = j)
// and its entries stay untouched until the loop ends (every warp reads them to form the same
// reflector redundantly), then row j of it becomes beta and the rows below zero.  The rows of R1
// are therefore the rows of (R1 in pivoted column order) with the columns back in original order --
// row-Jacobi is invariant under column permutations, so perm = identity.  Thread groups of four own
// columns (rows split by residue mod 4) and publish per-warp argmax partials of the updated column
// norms into a double-buffered slot for the next step.
__device__ int qrcp_rows_precondition(double* W, int n, int ld, int* perm, double* cn, double* cn0, double* beta_s,
                                      int* pst, double* red, int* ired, double tol = 0.0, double big_eps = 0.0) {
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int grp = tid >> 2, sub = tid & 3, ngrp = nt >> 2;
  const unsigned qmask = 0xfu << (lane & ~3);
  for (int c = tid; c < n; c += nt) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = fma(W[(long long)i * ld + c], W[(long long)i * ld + c], s);
    cn[c] = cn0[c] = s;
    perm[c] = c;
    pst[c] = -1;
  }
  __syncthreads();
  // argmax partials of step 0 (buffer 0)
  {
    double best = -1.0;
    int bi = n;
    if (sub == 0)
      for (int c = grp; c < n; c += ngrp)
        if (cn[c] > best) { best = cn[c]; bi = c; }
    argmax_pair(best, bi, 0xffffffffu, 32);
    if (lane == 0) { red[warp] = best; ired[warp] = bi; }
  }
  __syncthreads();
  double stop2 = 0.0;
  int j = 0;
  for (; j < n; ++j) {
    const int buf = (j & 1) * nw, nbuf = ((j + 1) & 1) * nw;
    // every warp reduces the partials itself (no second barrier)
    double best = lane < nw ? red[buf + lane] : -1.0;
    int p = lane < nw ? ired[buf + lane] : n;
    argmax_pair(best, p, 0xffffffffu, 32);
    const double bst = cn[p];
    if (j == 0) {
      const double thr_lo = fmax(tol, big_eps * sqrt(bst));
      stop2 = fmax(kEps * kEps * bst * 0.25, kDeflate * kDeflate * thr_lo * thr_lo);
    } else if ((double)(n - j) * bst <= stop2) {
      break;
    }
    // reflector of column p, rows j.. (LAPACK dlarfg sign convention), formed by every warp
    double ss = 0.0;
    for (int i = j + 1 + lane; i < n; i += 32) ss = fma(W[(long long)i * ld + p], W[(long long)i * ld + p], ss);
    ss = warp_sum(ss);
    const double alpha = W[(long long)j * ld + p];
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (ss != 0.0) {
      const double nrm = sqrt(alpha * alpha + ss);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) * __drcp_rn(beta);
      scale = __drcp_rn(alpha - beta);
    }
    if (tid == 0) beta_s[j] = beta;
    // trailing update of the remaining columns: v = [1; W(j+1:, p) scale]
    double cbest = -1.0;
    int cbi = n;
    for (int cb = 0; cb < n; cb += ngrp) {
      const int c = cb + grp;
      const bool act = c < n && c != p && pst[c] < 0;
      if (act && tau != 0.0) {
        double w0 = 0.0, w1 = 0.0;
        int i = j + 1 + sub;
        for (; i + 4 < n; i += 8) {
          w0 = fma(W[(long long)i * ld + p], W[(long long)i * ld + c], w0);
          w1 = fma(W[(long long)(i + 4) * ld + p], W[(long long)(i + 4) * ld + c], w1);
        }
        if (i < n) w0 = fma(W[(long long)i * ld + p], W[(long long)i * ld + c], w0);
        double wv = w0 + w1;
        wv += __shfl_xor_sync(qmask, wv, 1);
        wv += __shfl_xor_sync(qmask, wv, 2);
        const double rj0 = W[(long long)j * ld + c];
        const double tw = tau * fma(wv, scale, rj0);
        const double tws = tw * scale;
        for (int i2 = j + 1 + sub; i2 < n; i2 += 4) W[(long long)i2 * ld + c] -= tws * W[(long long)i2 * ld + p];
        __syncwarp(qmask);  // row j of column c read by all four before it changes
        if (sub == 0) W[(long long)j * ld + c] = rj0 - tw;
        __syncwarp(qmask);
      } else if (c == p && sub == 0) {
        pst[c] = j;
      }
      if (act) {
        const double rj = W[(long long)j * ld + c];
        const bool recompute = cn[c] - rj * rj <= 1e-2 * cn0[c];
        __syncwarp(qmask);
        double nc = cn[c] - rj * rj;
        if (recompute) {  // cancellation: recompute the trailing norm exactly
          double s2 = 0.0;
          for (int i2 = j + 1 + sub; i2 < n; i2 += 4) s2 = fma(W[(long long)i2 * ld + c], W[(long long)i2 * ld + c], s2);
          s2 += __shfl_xor_sync(qmask, s2, 1);
          s2 += __shfl_xor_sync(qmask, s2, 2);
          nc = s2;
          if (sub == 0) cn0[c] = s2;
        }
        if (sub == 0) cn[c] = nc;
        if (nc > cbest) { cbest = nc; cbi = c; }
      }
    }
    if (sub != 0) { cbest = -1.0; cbi = n; }
    argmax_pair(cbest, cbi, 0xffffffffu, 32);
    if (lane == 0) { red[nbuf + warp] = cbest; ired[nbuf + warp] = cbi; }
    __syncthreads();
  }
  // pivot columns: beta on their step's row, zeros below
  for (int c = grp; c < n; c += ngrp) {
    const int sj = pst[c];
    if (sj < 0) continue;
    if (sub == 0) W[(long long)sj * ld + c] = beta_s[sj];
    for (int i = sj + 1 + sub; i < n; i += 4) W[(long long)i * ld + c] = 0.0;
  }
  __syncthreads();
  return j;
}

// NPLO: octet-Jacobi entries per lane (8: n <= 64, 16: n <= 128, 24: n <= 192), 0: half-warp loop
static constexpr int NT = 512;
// RS: R in shared memory (compile-time, so every access to it is an LDS/STS rather than a generic
// load), else R is worked on in place in global memory (items too large for shared memory).
template <int NPLO, bool RS>
__global__ void __launch_bounds__(NT, (NPLO >= 16 || NPLO == 0) ? 1 : 2) svd_finish_kernel(const SvdItem* __restrict__ items,
                                                                             const Seg* __restrict__ segs,
                                                                             int vsm, long long smem_doubles) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int flag[2];
  __shared__ int s_k2;
  __shared__ double jred[2 * (NT / 32) + 2];
  const SvdItem it = items[blockIdx.x];
  const int m = it.m, kx = it.kx, k1 = min(m, kx), n = svd_n(it);
  long long N = it.N;
  if (it.zskip)  // blocks of exactly zero norm are not columns of the reference's stack (induced.py:121-125)
    for (int q = it.s0; q < it.s1; ++q) {
      const Seg sg = segs[q];
      if (sg.sdiv && *sg.sdiv == 0.0) N -= sg.w;
    }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ldv = kx | 1;
  // vsm bit 1: "tight" layout -- R at the unpadded stride n (rounded up to even) and the QRCP work
  // vectors in global memory (the R input buffer, free once R is in shared memory), for n up to
  // ~168 where the padded layout misses the 227 KB by a few KB (the top-level clusters of c4's
  // row pass: shared memory instead of the global-memory fallback, ~3.5x on those launches)
  const bool tight = RS && (vsm & 2);
  vsm &= 1;
  double* sig = smem;                        // n
  int* ord = (int*)(sig + n);                // n ints
  double *cn, *cn0, *vh, *R;
  int *perm, *iperm;
  int ld;
  if (tight) {
    perm = (int*)(sig + n + (n / 2 + 1));    // n ints
    iperm = perm + n;                        // n ints
    ld = n + (n & 1);
    R = smem + ((n + (n / 2 + 1) + n + 1) & ~1);
    cn = it.rbuf;                            // QRCP column norms, reference norms, reflector
    cn0 = cn + n;
    vh = cn0 + n;
  } else {
    cn = sig + n + (n / 2 + 1);              // QRCP column norms (n), reference norms (n), reflector (n)
    cn0 = cn + n;
    vh = cn0 + n;
    perm = (int*)(vh + n);                   // n ints
    iperm = perm + n;                        // n ints
    // R in shared memory: 16-byte aligned rows of stride ld = fin_ld(n) (padding columns zero), so
    // the octet Jacobi moves double2 and the QRCP trailing update's 4 x 4 (rows x columns) half-warp
    // accesses fall in distinct banks; in global memory (the merge output) the stride stays n
    ld = RS ? fin_ld(n) : n;
    R = RS ? smem + (((int)(vh + 2 * n + 1 - smem) + 1) & ~1) : it.rbuf;
  }
  // V (m x ldv, reflectors of the protected basis) and tv (kx + 1): staged in shared memory after
  // the rest when they fit (vsm), else read where the tsqr stage left them
  double* V = vsm ? (RS ? R + (long long)n * ld : vh + n + n + 1) : it.vws;
  double* tv = V + (long long)m * ldv;
  __shared__ int ired[2 * (NT / 32) + 2];
  if (kx > 0 && vsm) {
    for (int e = threadIdx.x; e < m * ldv; e += blockDim.x) V[e] = it.vws[e];
    for (int e = threadIdx.x; e < kx; e += blockDim.x) tv[e] = it.vws[m * ldv + e];
  }
  int k2 = 0;
  long long tk[5] = {clock64(), 0, 0, 0, 0};  // phase timestamps (diagnostic output only)
  if (n > 0 && N > 0) {
    if (RS)
      for (long long e = threadIdx.x; e < (long long)n * ld; e += blockDim.x) {
        const int i = (int)(e / ld), j = (int)(e % ld);
        R[e] = j < n ? it.rbuf[(long long)i * n + j] : 0.0;
      }
    __syncthreads();
    tk[1] = clock64();
    // B = R^T Q_B^T: left singular vectors of B = those of R^T.  QRCP preconditioning R Pi = Q1 R1,
    // then the left singular vectors of R^T are Pi x the normalised rows of R1 after row Jacobi.
    const long long bigc = (long long)n > N ? (long long)n : N;
    int nr;
    if (it.pre_nr) {  // Gram path: R is already the pivoted (double-double) Cholesky factor
      nr = *it.pre_nr;
      for (int c = threadIdx.x; c < n; c += blockDim.x) perm[c] = c;
      __syncthreads();
    } else {
      nr = qrcp_rows_precondition(R, n, ld, perm, cn, cn0, vh, iperm, jred, ired, it.tol, (double)bigc * kEps);
    }
    for (int c = threadIdx.x; c < n; c += blockDim.x) iperm[perm[c]] = c;
    __syncthreads();
    tk[2] = clock64();
    const int sw = (NPLO > 0 && n <= 8 * NPLO)
                       ? jacobi_rows_oct<(NPLO > 0 ? NPLO : 2), RS>(R, nr, n, ld, flag, jred)
                       : (NPLO == 0 && n <= 256)
                       ? jacobi_rows<(NPLO == 0 ? 16 : 1)>(R, nr, n, ld, flag, jred)  // rows cached in registers
                       : jacobi_rows<0>(R, nr, n, ld, flag, jred);
    tk[3] = clock64();
    if (it.sweeps_out && threadIdx.x == 0) {
      it.sweeps_out[0] = sw;
      it.sweeps_out[1] = n;
      it.sweeps_out[2] = nr;
    }
    for (int i = warp; i < n; i += nw) {
      double s = 0.0;
      for (int j = lane; j < n; j += 32) s = fma(R[(long long)i * ld + j], R[(long long)i * ld + j], s);
      s = warp_sum(s);
      if (lane == 0) sig[i] = sqrt(s);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      int pos = 0;
      const double si = sig[i];
      for (int j = 0; j < n; ++j) {
        const double sj = sig[j];
        pos += (sj > si) || (sj == si && j < i);
      }
      ord[pos] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double s1 = sig[ord[0]];
      const long long big = (long long)n > N ? (long long)n : N;
      const double thr = fmax(it.tol, (double)big * kEps * s1);
      int k = 0;
      while (k < n && sig[ord[k]] > thr) ++k;
      if (it.cap >= 0 && k > it.cap) k = it.cap;
      s_k2 = k;
    }
    __syncthreads();
    k2 = s_k2;
    if (it.sig_out)
      for (int i = threadIdx.x; i < n; i += blockDim.x) it.sig_out[i] = sig[ord[i]];
    if (it.sweeps_out && threadIdx.x == 0) it.sweeps_out[3] = k2;
  }
  __syncthreads();
  const int kt = k1 + k2;
  double* Q = it.q_out;  // m x kt
  if (it.u_out && k1 > 0 && n > 0) {
    // deferred output: U = normalised rows of R1 in singular order, mapped back through the column
    // pivoting; Q_t = Q_V [[I, 0], [0, U]] is one batched GEMM on the host's next launch
    for (long long e = threadIdx.x; e < (long long)n * k2; e += blockDim.x) {
      const int l = (int)(e / k2), j = (int)(e % k2);
      const int src = ord[j];
      it.u_out[(long long)l * n + j] = R[(long long)src * ld + iperm[l]] / sig[src];
    }
  } else if (it.q2) {
    // explicit Q_V from svd_prep_kernel: Q_t = [Q_V[:, :k1] | Q_V[:, k1:] U], U = normalised rows of
    // R1 (singular order) mapped back through the column pivoting -- one small product instead of
    // k1 sequential reflector applications per column
    for (long long e = threadIdx.x; e < (long long)m * kt; e += blockDim.x) {
      const int i = (int)(e / kt), j = (int)(e % kt);
      const double* qrow = it.q2 + (long long)i * m;
      double val;
      if (j < k1) {
        val = qrow[j];
      } else {
        const int src = ord[j - k1];
        const double* rr = R + (long long)src * ld;
        double s0 = 0.0, s1 = 0.0;
        int l = 0;
        for (; l + 1 < n; l += 2) {
          s0 = fma(qrow[k1 + l], rr[iperm[l]], s0);
          s1 = fma(qrow[k1 + l + 1], rr[iperm[l + 1]], s1);
        }
        if (l < n) s0 = fma(qrow[k1 + l], rr[iperm[l]], s0);
        val = (s0 + s1) / sig[src];
      }
      Q[e] = val;
    }
  } else {
  for (long long e = threadIdx.x; e < (long long)m * kt; e += blockDim.x) {
    const int i = (int)(e / kt), j = (int)(e % kt);
    double val;
    if (j < k1) {
      val = (i == j) ? 1.0 : 0.0;
    } else {
      const int src = ord[j - k1];
      val = (i < k1) ? 0.0 : R[(long long)src * ld + iperm[i - k1]] / sig[src];
    }
    Q[e] = val;
  }
  __syncthreads();
  if (k1 > 0) {
    // Q = H_0 H_1 ... H_{k1-1} Y: reflectors in reverse order.  With R in shared memory its space is
    // free now: Q is staged there in column blocks (column-major, each warp owning whole columns, so
    // the k1 reflectors need no barrier), V beside it -- the global-memory version re-reads every
    // column of Q (stride kt) for every reflector and thrashes L1 at m ~ 200.
    int CB = 0;
    const int ldq = m | 1;
    double* Qs = nullptr;
    const double* Vs = V;
    const double* tvs = tv;
    if (RS) {
      const long long room_r = (long long)n * ld;  // R's region (doubles)
      const long long avail = (long long)smem_doubles - (long long)(R - smem);
      if (vsm) {  // V and tv are already in shared memory, after R
        CB = (int)min((long long)kt, room_r / ldq);
        Qs = R;
      } else {
        const long long vneed = (((long long)m * ldv + kx + 1) + 1) & ~1LL;
        if (vneed + (long long)ldq < avail) {
          double* Vd = R;
          for (long long e = threadIdx.x; e < (long long)m * ldv + kx; e += blockDim.x) Vd[e] = it.vws[e];
          Vs = Vd;
          tvs = Vd + (long long)m * ldv;
          Qs = Vd + vneed;
          CB = (int)min((long long)kt, (avail - vneed) / ldq);
        }
      }
    }
    if (CB >= 4 || (CB > 0 && CB == kt)) {
      __syncthreads();
      for (int c0 = 0; c0 < kt; c0 += CB) {
        const int cb = min(CB, kt - c0);
        for (long long e = threadIdx.x; e < (long long)m * cb; e += blockDim.x) {
          const int i = (int)(e / cb), c = (int)(e % cb);
          Qs[(long long)c * ldq + i] = Q[(long long)i * kt + c0 + c];
        }
        __syncthreads();
        for (int c = warp; c < cb; c += nw) {
          double* qc = Qs + (long long)c * ldq;
          for (int j = k1 - 1; j >= 0; --j) {
            const double tau = tvs[j];
            if (tau == 0.0) continue;
            double part = 0.0;
            for (int i = j + 1 + lane; i < m; i += 32) part = fma(Vs[(long long)i * ldv + j], qc[i], part);
            const double wv = qc[j] + warp_sum(part);
            __syncwarp();
            if (lane == 0) qc[j] -= tau * wv;
            for (int i = j + 1 + lane; i < m; i += 32) qc[i] -= tau * wv * Vs[(long long)i * ldv + j];
            __syncwarp();
          }
        }
        __syncthreads();
        for (long long e = threadIdx.x; e < (long long)m * cb; e += blockDim.x) {
          const int i = (int)(e / cb), c = (int)(e % cb);
          Q[(long long)i * kt + c0 + c] = Qs[(long long)c * ldq + i];
        }
        __syncthreads();
      }
    } else {
      for (int c = warp; c < kt; c += nw)
        for (int j = k1 - 1; j >= 0; --j)
          if (tv[j] != 0.0) apply_reflector_col(V, ldv, m, j, tv[j], Q, kt, c);
    }
  }
  }
  if (it.bc_out) {
    for (int e = threadIdx.x; e < kt * kx; e += blockDim.x) {
      const int i = e / kx, j = e % kx;
      it.bc_out[e] = (i < k1 && j >= i) ? V[i * ldv + j] : 0.0;
    }
  }
  if (threadIdx.x == 0) *it.rank_out = kt;
  if (it.sweeps_out && threadIdx.x == 0 && tk[3] > 0) {
    tk[4] = clock64();
    for (int q = 1; q < 5; ++q) it.sweeps_out[3 + q] = (int)((tk[q] - tk[q - 1]) / 1000);
  }
}

// ---------------------------------------------------------------------------------------------
// norm_kernel: sigma_1 of hstack(segs) (m x N).  Gram on the row side (m <= N), else on the column
// side; Lanczos on the Gram with Sturm multisection on its tridiagonal for lambda_max.
// ---------------------------------------------------------------------------------------------

__device__ double sturm_lambda_max(const double* d, const double* e, int g, double* red) {
  // all threads call; warp 0 computes
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) == 0) {
    double lo = 1e300, hi = -1e300;
    for (int i = lane; i < g; i += 32) {
      const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < g ? fabs(e[i]) : 0.0);
      lo = fmin(lo, d[i] - r);
      hi = fmax(hi, d[i] + r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const double span = fmax(fabs(lo), fabs(hi));
    if (span == 0.0) {  // exactly zero Gram: sigma_1 == 0 exactly (zero-norm skips are exact tests)
      if (lane == 0) red[0] = 0.0;
      lo = hi = 0.0;
    }
    hi += 2.0 * kEps * span + 1e-300;
    lo -= 2.0 * kEps * span + 1e-300;
    for (int round = 0; round < 64 && span != 0.0; ++round) {
      if (hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
      const double x = lo + (hi - lo) * (double)(lane + 1) / 33.0;
      int cnt = 0;
      double q = d[0] - x;
      if (q < 0.0) ++cnt;
      for (int i = 1; i < g; ++i) {
        if (q == 0.0) q = -1e-300;
        q = (d[i] - x) - e[i - 1] * e[i - 1] / q;
        if (q < 0.0) ++cnt;
      }
      // first lane whose point has all g eigenvalues below it
      const unsigned full = __ballot_sync(0xffffffffu, cnt >= g);
      double nlo = lo, nhi = hi;
      if (full) {
        const int f = __ffs(full) - 1;
        nhi = lo + (hi - lo) * (double)(f + 1) / 33.0;
        nlo = f > 0 ? lo + (hi - lo) * (double)f / 33.0 : lo;
      } else {
        nlo = lo + (hi - lo) * 32.0 / 33.0;
      }
      if (nlo == lo && nhi == hi) break;  // a few ulps wide: no further progress possible
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) red[0] = span == 0.0 ? 0.0 : 0.5 * (lo + hi);
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ double warp_lambda_max(const double* d, const double* e, int g);

__global__ void __launch_bounds__(kThreads) norm_kernel(const NormItem* __restrict__ items,
                                                        const Seg* __restrict__ segs) {
  extern __shared__ double smem[];
  __shared__ double red[40];
  const NormItem it = items[blockIdx.x];
  const int m = it.m;
  const long long N = it.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (m == 0 || N == 0) {
    if (threadIdx.x == 0) *it.out = 0.0;
    return;
  }
  const bool rowside = m <= N;  // Gram on the smaller side
  const int g = rowside ? m : (int)N;
  double* G = it.gbuf ? it.gbuf : smem;                  // g x g (global scratch for large items)
  double* Pn = it.gbuf ? smem : G + (long long)g * g;    // 32 x max(m, N) panel
  double* d = Pn + kPanel * (rowside ? m : (int)N);
  double* e = d + g;
  double* v = e + g;
  double* p = v + g;
  for (int q = threadIdx.x; q < g * g; q += blockDim.x) G[q] = 0.0;
  __syncthreads();
  if (rowside) {
    // G = sum over column panels of A_panel A_panel^T, panel stored transposed (32 x m)
    for (long long c0 = 0; c0 < N; c0 += kPanel) {
      load_hpanel(segs, it.s0, it.s1, m, N, c0, Pn, true, m);
      __syncthreads();
      for (int q = threadIdx.x; q < g * g; q += blockDim.x) {
        const int i = q / g, j = q % g;
        if (j < i) continue;
        double s = 0.0;
#pragma unroll 8
        for (int c = 0; c < kPanel; ++c) s = fma(Pn[c * m + i], Pn[c * m + j], s);
        G[i * g + j] += s;
      }
      __syncthreads();
    }
  } else {
    // G = sum over row panels of P^T P (P: 32 x N from an hstack of column segments)
    for (long long r0 = 0; r0 < m; r0 += kPanel) {
      for (int pr = warp; pr < kPanel; pr += nw) {
        const long long r = r0 + pr;
        long long off = 0;
        for (int s = it.s0; s < it.s1; ++s) {
          const Seg sg = segs[s];
          for (int c = lane; c < sg.w; c += 32)
            Pn[pr * N + off + c] = (r < m) ? seg_scale(sg) * mref(sg.a, r, c) : 0.0;
          off += sg.w;
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < g * g; q += blockDim.x) {
        const int i = q / g, j = q % g;
        if (j < i) continue;
        double s = 0.0;
#pragma unroll 8
        for (int c = 0; c < kPanel; ++c) s = fma(Pn[c * N + i], Pn[c * N + j], s);
        G[i * g + j] += s;
      }
      __syncthreads();
    }
  }
  for (int q = threadIdx.x; q < g * g; q += blockDim.x) {
    const int i = q / g, j = q % g;
    if (j < i) G[q] = G[j * g + i];
  }
  __syncthreads();
  // Lanczos on the symmetric Gram (sigma_1^2 = lambda_max(G)) with the early exit of the Lanczos
  // kernels -- a few block-wide G v products instead of g Householder steps of five barriers each
  // (the tridiagonalisation was the bulk of this kernel on phase 2's merged representations)
  const int tid = threadIdx.x, nt = blockDim.x;
  double* al = d;      // Lanczos diagonal (g)
  double* be = e;      // off-diagonal (g)
  double* q = p + g;   // previous Lanczos vector (g); p holds w
  auto block_sum = [&](double x) -> double {
    x = warp_sum(x);
    __syncthreads();
    if (lane == 0) red[warp] = x;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
  };
  double part = 0.0;
  for (int i = tid; i < g; i += nt) {
    unsigned x = 2654435761u * (i + 1) ^ (i < 32 ? 0x9e3779b9u : 0x85ebca6bu);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    v[i] = 0.5 + (double)(x & 0xffff) / 65536.0;
    q[i] = 0.0;
    part += v[i] * v[i];
  }
  const double nv = sqrt(block_sum(part));
  for (int i = tid; i < g; i += nt) v[i] /= nv;
  __syncthreads();
  double bprev = 0.0, theta = 0.0, done = -1.0;
  int k = 0;
  for (; k < g; ++k) {
    double pa = 0.0;
    for (int i = tid; i < g; i += nt) {  // w = G v: column i of the symmetric G (conflict-free)
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 1 < g; j += 2) {
        s0 = fma(G[(long long)j * g + i], v[j], s0);
        s1 = fma(G[(long long)(j + 1) * g + i], v[j + 1], s1);
      }
      if (j < g) s0 = fma(G[(long long)j * g + i], v[j], s0);
      p[i] = s0 + s1;
      pa += p[i] * v[i];
    }
    const double a = block_sum(pa);
    double pb = 0.0;
    for (int i = tid; i < g; i += nt) {
      p[i] -= a * v[i] + bprev * q[i];
      pb += p[i] * p[i];
    }
    const double bb = sqrt(block_sum(pb));
    if (tid == 0) al[k] = a;
    if (k + 1 == g || bb <= 1e-15 * (fabs(a) + bprev)) {
      ++k;
      break;
    }
    if (tid == 0) be[k] = bb;
    if ((k & 1) == 1 && k >= 5) {  // top Ritz value settled to 1e-14 relative: stop
      __syncthreads();
      if (warp == 0) {
        const double th = warp_lambda_max(al, be, k + 1);
        if (lane == 0) red[nw] = th;
      }
      __syncthreads();
      const double th = red[nw];
      if (th - theta <= 1e-14 * th) {
        done = th;
        break;
      }
      theta = th;
    }
    for (int i = tid; i < g; i += nt) {
      q[i] = v[i];
      v[i] = p[i] / bb;
    }
    bprev = bb;
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) {
    const double lam = done >= 0.0 ? done : warp_lambda_max(al, be, k);
    if (lane == 0) *it.out = sqrt(fmax(lam, 0.0));
  }
}

// ---------------------------------------------------------------------------------------------
// norm_warp_kernel: sigma_1 of a single-segment matrix with m, N <= 64, one warp per matrix.
// A lives in shared memory; Lanczos on the smaller Gram side (A^T A or A A^T, never formed) runs
// at most min(m, N) steps, then Sturm multisection on the tridiagonal.  The top Ritz value grows
// monotonically with the step count; from step 6 on it is re-evaluated every 2 steps and the
// iteration stops once it moved by <= 1e-14 relative (the sigma_1 are scale factors and rank
// thresholds: an error of that size cannot move a truncation whose margin is >= 1e-4).
// An exactly zero matrix returns exactly 0 (the reference's zero-norm skips are exact tests).
// ---------------------------------------------------------------------------------------------

static constexpr int kNW = 2;            // warps (matrices) per CTA
static constexpr int kNWMax = 64;        // smaller side (Lanczos vector length) handled here
static constexpr int kNWMaxH = 128;      // larger side
static constexpr int kNWCap = 64 * 65;   // A capacity (doubles): m * (N | 1) <= kNWCap

__device__ double warp_lambda_max(const double* d, const double* e, int g) {
  const int lane = threadIdx.x & 31;
  double lo = 1e300, hi = -1e300;
  for (int i = lane; i < g; i += 32) {
    const double r = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < g ? fabs(e[i]) : 0.0);
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const double span = fmax(fabs(lo), fabs(hi));
  if (span == 0.0) return 0.0;
  hi += 2.0 * kEps * span + 1e-300;
  lo -= 2.0 * kEps * span + 1e-300;
  for (int round = 0; round < 64; ++round) {
    if (hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
    // two points per lane (independent recurrences interleaved): 65-way multisection
    const double w = (hi - lo) / 65.0;
    const double x0 = lo + w * (double)(2 * lane + 1), x1 = lo + w * (double)(2 * lane + 2);
    // Sturm counts without divisions: leading minors p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2},
    // rescaled every 8 steps; #sign changes of (1, p_1, .., p_g) = #eigenvalues below x
    int c0 = 0, c1 = 0;
    double pa0 = 1.0, pb0 = d[0] - x0, pa1 = 1.0, pb1 = d[0] - x1;
    if (pb0 == 0.0) pb0 = -1e-300;
    if (pb1 == 0.0) pb1 = -1e-300;
    c0 += pb0 < 0.0;
    c1 += pb1 < 0.0;
    for (int i = 1; i < g; ++i) {
      const double e2 = e[i - 1] * e[i - 1];
      double n0 = fma(d[i] - x0, pb0, -e2 * pa0);
      double n1 = fma(d[i] - x1, pb1, -e2 * pa1);
      if (n0 == 0.0) n0 = -1e-300 * pb0;
      if (n1 == 0.0) n1 = -1e-300 * pb1;
      c0 += (n0 < 0.0) != (pb0 < 0.0);
      c1 += (n1 < 0.0) != (pb1 < 0.0);
      pa0 = pb0;
      pb0 = n0;
      pa1 = pb1;
      pb1 = n1;
      if ((i & 7) == 0) {
        const double s0 = fabs(pa0) + fabs(pb0), s1 = fabs(pa1) + fabs(pb1);
        if (s0 > 1e150) { pa0 *= 1e-150; pb0 *= 1e-150; }
        else if (s0 < 1e-150) { pa0 *= 1e150; pb0 *= 1e150; }
        if (s1 > 1e150) { pa1 *= 1e-150; pb1 *= 1e-150; }
        else if (s1 < 1e-150) { pa1 *= 1e150; pb1 *= 1e150; }
      }
    }
    // points in increasing order: p = 2*lane+1 (x0), 2*lane+2 (x1); find the first with count == g
    const unsigned f0 = __ballot_sync(0xffffffffu, c0 >= g), f1 = __ballot_sync(0xffffffffu, c1 >= g);
    int first = 65;
    if (f0) first = min(first, 2 * (__ffs(f0) - 1) + 1);
    if (f1) first = min(first, 2 * (__ffs(f1) - 1) + 2);
    const double nhi = first < 65 ? lo + w * first : hi;
    const double nlo = first < 65 ? lo + w * (first - 1) : lo + w * 64.0;
    // a bracket a few ulps wide cannot shrink further (its points round onto its ends): stop there
    // instead of spinning through the remaining rounds
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

__global__ void __launch_bounds__(32 * kNW) norm_warp_kernel(const NormItem* __restrict__ items,
                                                             const Seg* __restrict__ segs, int nitems) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * kNW + warp;
  if (idx >= nitems) return;
  double* A = smem + warp * (kNWCap + 3 * kNWMax + kNWMaxH);
  double* vs = A + kNWCap;          // broadcast vector (length g)
  double* us = vs + kNWMax;         // intermediate (length h)
  double* al = us + kNWMaxH;        // Lanczos diagonal
  double* be = al + kNWMax;         // Lanczos off-diagonal
  const NormItem it = items[idx];
  const Seg sg = segs[it.s0];
  const int m = it.m, N = (int)it.N;
  const int kNWLd = N | 1;          // odd row stride: lane-per-row access without bank conflicts
  double amax = 0.0;
  const double ssc = seg_scale(sg);
  const double* ap = sg.a.p;
  const int ars = sg.a.rs, acs = sg.a.cs;
  for (int i0 = 0; i0 < m; i0 += 4) {  // 4 rows x up to 4 column chunks of loads in flight per lane
    double a[4][4];
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int i = i0 + ii, j = lane + 32 * jj;
        a[ii][jj] = (i < m && j < N) ? ap[i * ars + j * acs] : 0.0;
      }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int i = i0 + ii, j = lane + 32 * jj;
        if (i < m && j < N) {
          const double v = ssc * a[ii][jj];
          A[i * kNWLd + j] = v;
          amax = fmax(amax, fabs(v));
        }
      }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (amax == 0.0) {
    if (lane == 0) *it.out = 0.0;
    return;
  }
  const bool colside = N <= m;  // Lanczos vectors live on the smaller side
  const int g = colside ? N : m, h = colside ? m : N;
  // deterministic pseudo-random start vector
  double v0 = 0.0, v1 = 0.0;
  {
    unsigned s0 = 2654435761u * (lane + 1) ^ 0x9e3779b9u, s1 = 2654435761u * (lane + 33) ^ 0x85ebca6bu;
    s0 ^= s0 >> 13; s0 *= 0x5bd1e995u; s0 ^= s0 >> 15;
    s1 ^= s1 >> 13; s1 *= 0x5bd1e995u; s1 ^= s1 >> 15;
    v0 = lane < g ? 0.5 + (double)(s0 & 0xffff) / 65536.0 : 0.0;
    v1 = lane + 32 < g ? 0.5 + (double)(s1 & 0xffff) / 65536.0 : 0.0;
    const double nv = sqrt(warp_sum(v0 * v0 + v1 * v1));
    v0 /= nv;
    v1 /= nv;
  }
  double p0 = 0.0, p1 = 0.0, bprev = 0.0, theta = 0.0, done = -1.0;
  int k = 0;
  for (; k < g; ++k) {
    // w = op(v): u = B v (length h), w = B^T u (length g), B = A (colside) or A^T
    if (lane < g) vs[lane] = v0;
    if (lane + 32 < g) vs[lane + 32] = v1;
    __syncwarp();
    // B (h x g) = A (colside) or A^T; u = B v (lane per row of B), w = B^T u (lane per column of B)
    double w0 = 0.0, w1 = 0.0;
    if (colside) {
      for (int r = lane; r < h; r += 32) {
        const double* ar = A + r * kNWLd;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 3 < g; j += 4) {
          a0 = fma(ar[j], vs[j], a0);
          a1 = fma(ar[j + 1], vs[j + 1], a1);
          a2 = fma(ar[j + 2], vs[j + 2], a2);
          a3 = fma(ar[j + 3], vs[j + 3], a3);
        }
        for (; j < g; ++j) a0 = fma(ar[j], vs[j], a0);
        us[r] = (a0 + a1) + (a2 + a3);
      }
      __syncwarp();
      double x0 = 0.0, x1 = 0.0;
      const int c0 = lane < g ? lane : 0, c1 = lane + 32 < g ? lane + 32 : 0;
      int i = 0;
      for (; i + 1 < h; i += 2) {
        const double u = us[i], u2 = us[i + 1];
        const double* a0p = A + i * kNWLd;
        w0 = fma(a0p[c0], u, w0);
        w1 = fma(a0p[c1], u, w1);
        x0 = fma(a0p[kNWLd + c0], u2, x0);
        x1 = fma(a0p[kNWLd + c1], u2, x1);
      }
      if (i < h) {
        w0 = fma(A[i * kNWLd + c0], us[i], w0);
        w1 = fma(A[i * kNWLd + c1], us[i], w1);
      }
      w0 += x0;
      w1 += x1;
    } else {
      for (int r = lane; r < h; r += 32) {  // row r of A^T = column r of A
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 3 < g; j += 4) {
          a0 = fma(A[j * kNWLd + r], vs[j], a0);
          a1 = fma(A[(j + 1) * kNWLd + r], vs[j + 1], a1);
          a2 = fma(A[(j + 2) * kNWLd + r], vs[j + 2], a2);
          a3 = fma(A[(j + 3) * kNWLd + r], vs[j + 3], a3);
        }
        for (; j < g; ++j) a0 = fma(A[j * kNWLd + r], vs[j], a0);
        us[r] = (a0 + a1) + (a2 + a3);
      }
      __syncwarp();
      double x0 = 0.0, x1 = 0.0;
      const int c0 = lane < g ? lane : 0, c1 = lane + 32 < g ? lane + 32 : 0;
      const double* r0p = A + c0 * kNWLd;
      const double* r1p = A + c1 * kNWLd;
      int i = 0;
      for (; i + 1 < h; i += 2) {
        const double u = us[i], u2 = us[i + 1];
        w0 = fma(r0p[i], u, w0);
        w1 = fma(r1p[i], u, w1);
        x0 = fma(r0p[i + 1], u2, x0);
        x1 = fma(r1p[i + 1], u2, x1);
      }
      if (i < h) {
        w0 = fma(r0p[i], us[i], w0);
        w1 = fma(r1p[i], us[i], w1);
      }
      w0 += x0;
      w1 += x1;
    }
    w0 = lane < g ? w0 : 0.0;
    w1 = lane + 32 < g ? w1 : 0.0;
    const double a = warp_sum(w0 * v0 + w1 * v1);
    w0 -= a * v0 + bprev * p0;
    w1 -= a * v1 + bprev * p1;
    const double b = sqrt(warp_sum(w0 * w0 + w1 * w1));
    if (lane == 0) al[k] = a;
    if (k + 1 == g || b <= 1e-15 * (fabs(a) + bprev)) {
      ++k;
      break;
    }
    if (lane == 0) be[k] = b;
    if ((k & 1) == 1 && k >= 5) {
      // early exit once the top Ritz value (monotone in k) has settled to ~1e-14 relative
      __syncwarp();
      const double th = warp_lambda_max(al, be, k + 1);
      if (th - theta <= 1e-14 * th) {
        done = th;
        break;
      }
      theta = th;
    }
    p0 = v0;
    p1 = v1;
    v0 = w0 / b;
    v1 = w1 / b;
    bprev = b;
  }
  __syncwarp();
  const double lam = done >= 0.0 ? done : warp_lambda_max(al, be, k);
  if (lane == 0) *it.out = sqrt(fmax(lam, 0.0));
}

size_t norm_warp_smem() { return sizeof(double) * kNW * (kNWCap + 3 * kNWMax + kNWMaxH); }

cudaError_t launch_norm_warp(const NormItem* items, const Seg* segs, int nitems, cudaStream_t st) {
  init_attributes();
  if (nitems == 0) return cudaSuccess;
  const size_t sm = norm_warp_smem();
  norm_warp_kernel<<<(nitems + kNW - 1) / kNW, 32 * kNW, sm, st>>>(items, segs, nitems);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// norm_cta_kernel: sigma_1 of a single-segment matrix with m, N <= 128 (e.g. 128 x 128 nearfield
// blocks): one CTA per matrix, A in shared memory, Lanczos on the smaller Gram side with the same
// early exit as the warp version.  Matvecs: thread per row (u = B v) and thread per column
// (w = B^T u), each split over two thread halves; odd row stride keeps both conflict-free.
// ---------------------------------------------------------------------------------------------

static constexpr int kNC = 128;  // max side
static constexpr int kNCThreads = 256;

__global__ void __launch_bounds__(kNCThreads) norm_cta_kernel(const NormItem* __restrict__ items,
                                                              const Seg* __restrict__ segs) {
  extern __shared__ double smem[];
  __shared__ double red[kNCThreads / 32 + 2];
  __shared__ double lam_s;
  __shared__ int stop_s;
  const NormItem it = items[blockIdx.x];
  const Seg sg = segs[it.s0];
  const int m = it.m, N = (int)it.N, ld = N | 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  double* A = smem;                  // m x ld
  double* v = A + (size_t)m * ld;    // g
  double* u = v + kNC;               // h
  double* part = u + kNC;            // 2 x kNC partial sums
  double* al = part + 2 * kNC;       // Lanczos diagonal
  double* be = al + kNC;             // off-diagonal
  const double ssc = seg_scale(sg);
  double amax = 0.0;
  for (int e = tid; e < m * N; e += blockDim.x) {
    const int i = e / N, j = e % N;
    const double x = ssc * mref(sg.a, i, j);
    A[i * ld + j] = x;
    amax = fmax(amax, fabs(x));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) red[warp] = amax;
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < nw; ++w) a = fmax(a, red[w]);
    red[nw] = a;
  }
  __syncthreads();
  if (red[nw] == 0.0) {
    if (tid == 0) *it.out = 0.0;
    return;
  }
  const bool colside = N <= m;  // Lanczos vectors on the smaller side
  const int g = colside ? N : m, h = colside ? m : N;
  // deterministic pseudo-random positive start vector (as norm_warp_kernel)
  for (int i = tid; i < g; i += blockDim.x) {
    unsigned x = 2654435761u * (i + 1) ^ (i < 32 ? 0x9e3779b9u : 0x85ebca6bu);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    v[i] = 0.5 + (double)(x & 0xffff) / 65536.0;
  }
  __syncthreads();
  auto block_sum = [&](double x) -> double {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane == 0) red[warp] = x;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
  };
  {
    const double nv = sqrt(block_sum(tid < g ? v[tid] * v[tid] : 0.0));
    if (tid < g) v[tid] /= nv;
    __syncthreads();
  }
  const int half = tid >> 7, hi = tid & 127;  // two halves of 128 threads
  double vprev = 0.0, bprev = 0.0, theta = 0.0, done = -1.0;
  int k = 0;
  for (; k < g; ++k) {
    // u = B v (length h), B = A (colside) or A^T: thread per entry, k-range split in halves
    if (hi < h) {
      double s0 = 0.0, s1 = 0.0;
      const int j0 = half ? g / 2 : 0, j1 = half ? g : g / 2;
      int j = j0;
      if (colside) {
        const double* ar = A + hi * ld;
        for (; j + 1 < j1; j += 2) { s0 = fma(ar[j], v[j], s0); s1 = fma(ar[j + 1], v[j + 1], s1); }
        if (j < j1) s0 = fma(ar[j], v[j], s0);
      } else {
        for (; j + 1 < j1; j += 2) { s0 = fma(A[j * ld + hi], v[j], s0); s1 = fma(A[(j + 1) * ld + hi], v[j + 1], s1); }
        if (j < j1) s0 = fma(A[j * ld + hi], v[j], s0);
      }
      part[half * kNC + hi] = s0 + s1;
    }
    __syncthreads();
    if (tid < h) u[tid] = part[tid] + part[kNC + tid];
    __syncthreads();
    // w = B^T u (length g)
    double wv = 0.0;
    if (hi < g) {
      double s0 = 0.0, s1 = 0.0;
      const int i0 = half ? h / 2 : 0, i1 = half ? h : h / 2;
      int i = i0;
      if (colside) {
        for (; i + 1 < i1; i += 2) { s0 = fma(A[i * ld + hi], u[i], s0); s1 = fma(A[(i + 1) * ld + hi], u[i + 1], s1); }
        if (i < i1) s0 = fma(A[i * ld + hi], u[i], s0);
      } else {
        const double* ar = A + hi * ld;
        for (; i + 1 < i1; i += 2) { s0 = fma(ar[i], u[i], s0); s1 = fma(ar[i + 1], u[i + 1], s1); }
        if (i < i1) s0 = fma(ar[i], u[i], s0);
      }
      part[half * kNC + hi] = s0 + s1;
    }
    __syncthreads();
    const double vi = tid < g ? v[tid] : 0.0;
    if (tid < g) wv = part[tid] + part[kNC + tid];
    const double a = block_sum(wv * vi);
    if (tid < g) wv -= a * vi + bprev * vprev;
    const double b = sqrt(block_sum(tid < g ? wv * wv : 0.0));
    if (tid == 0) al[k] = a;
    if (k + 1 == g || b <= 1e-15 * (fabs(a) + bprev)) {
      ++k;
      break;
    }
    if (tid == 0) be[k] = b;
    if ((k & 1) == 1 && k >= 5) {  // top Ritz value settled to 1e-14 relative: stop
      __syncthreads();
      if (warp == 0) {
        const double th = warp_lambda_max(al, be, k + 1);
        if (lane == 0) {
          lam_s = th;
          stop_s = th - theta <= 1e-14 * th;
        }
      }
      __syncthreads();
      if (stop_s) {
        done = lam_s;
        break;
      }
      theta = lam_s;
    }
    vprev = vi;
    bprev = b;
    __syncthreads();
    if (tid < g) v[tid] = wv / b;
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) {
    const double lam = done >= 0.0 ? done : warp_lambda_max(al, be, k);
    if (lane == 0) *it.out = sqrt(fmax(lam, 0.0));
  }
}

size_t norm_cta_smem(int m, int N) {
  return sizeof(double) * ((size_t)m * (N | 1) + 6 * (size_t)kNC);
}

cudaError_t launch_norm_cta(const NormItem* items, const Seg* segs, int nitems, size_t smem, cudaStream_t st) {
  init_attributes();
  if (nitems == 0) return cudaSuccess;
  norm_cta_kernel<<<nitems, kNCThreads, smem, st>>>(items, segs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// norm_lz_kernel: sigma_1 of a single-segment matrix with m, N <= 128 (the product's nearfield blocks
// and k~ x k~ couplings, phase 2's block norms), replacing norm_cta_kernel for them.  The matrix lives
// in REGISTERS: 512 threads, thread (rg, cg) holds A[rg + 32p][cg + 16q] (p < 4, q < 8; lanes 0-15 of
// a warp cover 16 consecutive columns, so every load instruction reads full lines), so the Lanczos
// matvecs u = A v, w = A^T u never touch shared memory for A (the shared-memory version moved
// 2 x 128 KB per iteration through 128 B/clk and held one CTA per SM for its A).  u is reduced over
// the 16 column lanes by shuffles, w over the 32 row groups by one shuffle step and a 16-way
// shared-memory sum.  Lanczos on A^T A with the same start vector, early exit and exact-zero rule as
// norm_cta_kernel; the top Ritz value is re-evaluated every 2 steps from step 5.
// ---------------------------------------------------------------------------------------------

// NW warps (2 NW row groups) x P rows x Q column groups of 16: up to 2 NW P rows and 16 Q columns
template <int NW, int P, int Q>
__global__ void __launch_bounds__(32 * NW, NW >= 16 ? 1 : (NW >= 12 ? 2 : 3))
    norm_lz_kernel(const NormItem* __restrict__ items, const Seg* __restrict__ segs) {
  constexpr int RG = 2 * NW, NCOL = 16 * Q;
  __shared__ double part[NW][NCOL];  // w partials per warp
  __shared__ double vs[NCOL];        // current Lanczos vector
  __shared__ double red[2][4];
  __shared__ double al[kNC], be[kNC];
  __shared__ double amax_s[NW];
  __shared__ double lam_s;
  __shared__ int stop_s;
  const NormItem it = items[blockIdx.x];
  const Seg sg = segs[it.s0];
  const int m = it.m, N = (int)it.N;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cg = lane & 15, rg = 2 * warp + (lane >> 4);
  const double ssc = seg_scale(sg);
  double a[P][Q];
  double amax = 0.0;
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = rg + RG * p, j = cg + 16 * q;
      const double x = (i < m && j < N) ? ssc * __ldg(sg.a.p + (long long)i * sg.a.rs + (long long)j * sg.a.cs) : 0.0;
      a[p][q] = x;
      amax = fmax(amax, fabs(x));
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) amax_s[warp] = amax;
  // deterministic pseudo-random positive start vector (as norm_cta_kernel), length N
  double vt = 0.0;
  if (tid < N) {
    unsigned x = 2654435761u * (tid + 1) ^ (tid < 32 ? 0x9e3779b9u : 0x85ebca6bu);
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    vt = 0.5 + (double)(x & 0xffff) / 65536.0;
  }
  auto sum4 = [&](double x, int slot) -> double {  // sum over threads 0..127 (warps 0-3); all call
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (warp < 4 && lane == 0) red[slot][warp] = x;
    __syncthreads();
    return (red[slot][0] + red[slot][1]) + (red[slot][2] + red[slot][3]);
  };
  {
    const double nv = sqrt(sum4(tid < N ? vt * vt : 0.0, 0));
    double mx = 0.0;
    for (int w = 0; w < NW; ++w) mx = fmax(mx, amax_s[w]);
    if (mx == 0.0) {
      if (tid == 0) *it.out = 0.0;
      return;
    }
    vt = tid < N ? vt / nv : 0.0;
    if (tid < NCOL) vs[tid] = vt;  // zero past N: the matvec reads all columns (0 * uninitialised may be NaN)
  }
  __syncthreads();
  const int g = min(m, N);
  double vprev = 0.0, bprev = 0.0, theta = 0.0, done = -1.0;
  int k = 0;
  for (; k < g; ++k) {
    // u = A v over this thread's 4 rows, reduced over the 16 column lanes
    double vq[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) vq[q] = vs[cg + 16 * q];
    double u[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; q += 2) {
        s0 = fma(a[p][q], vq[q], s0);
        if (q + 1 < Q) s1 = fma(a[p][q + 1], vq[q + 1], s1);
      }
      u[p] = s0 + s1;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
      for (int p = 0; p < P; ++p) u[p] += __shfl_xor_sync(0xffffffffu, u[p], o);
    // w = A^T u over this thread's 8 columns, reduced over the two row groups of the warp, then
    // over the 16 warps in shared memory (fixed order)
    double w[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      double s = 0.0;
#pragma unroll
      for (int p = 0; p < P; ++p) s = fma(a[p][q], u[p], s);
      w[q] = s + __shfl_xor_sync(0xffffffffu, s, 16);
    }
    if (lane < 16)
#pragma unroll
      for (int q = 0; q < Q; ++q) part[warp][cg + 16 * q] = w[q];
    __syncthreads();
    double wt = 0.0;
    if (tid < N) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int ww = 0; ww < NW; ww += 2) {
        s0 += part[ww][tid];
        s1 += part[ww + 1][tid];
      }
      wt = s0 + s1;
    }
    const double alpha = sum4(wt * vt, 0);
    if (tid < N) wt -= alpha * vt + bprev * vprev;
    const double b = sqrt(sum4(tid < N ? wt * wt : 0.0, 1));
    if (tid == 0) al[k] = alpha;
    if (k + 1 == g || b <= 1e-15 * (fabs(alpha) + bprev)) {
      ++k;
      break;
    }
    if (tid == 0) be[k] = b;
    if ((k & 1) == 1 && k >= 5) {  // top Ritz value settled to 1e-14 relative: stop
      __syncthreads();
      if (warp == 0) {
        const double th = warp_lambda_max(al, be, k + 1);
        if (lane == 0) {
          lam_s = th;
          stop_s = th - theta <= 1e-14 * th;
        }
      }
      __syncthreads();
      if (stop_s) {
        done = lam_s;
        break;
      }
      theta = lam_s;
    }
    vprev = vt;
    bprev = b;
    vt = tid < N ? wt / b : 0.0;
    if (tid < NCOL) vs[tid] = vt;
    __syncthreads();
  }
  __syncthreads();
  if (warp == 0) {
    const double lam = done >= 0.0 ? done : warp_lambda_max(al, be, k);
    if (lane == 0) *it.out = sqrt(fmax(lam, 0.0));
  }
}

cudaError_t launch_norm_lz(const NormItem* items, const Seg* segs, int nitems, int mmax, int nmax, cudaStream_t st) {
  if (nitems == 0) return cudaSuccess;
  if (mmax <= 64 && nmax <= 64) norm_lz_kernel<8, 4, 4><<<nitems, 256, 0, st>>>(items, segs);
  else if (mmax <= 96 && nmax <= 96) norm_lz_kernel<12, 4, 6><<<nitems, 384, 0, st>>>(items, segs);
  else norm_lz_kernel<16, 4, 8><<<nitems, 512, 0, st>>>(items, segs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// gather: items (src, count, dst) as int64 triples; one CTA per item (packing for download)
// ---------------------------------------------------------------------------------------------

__global__ void gather_kernel(const long long* __restrict__ items) {
  const long long* it = items + 3 * blockIdx.x;
  const double* src = (const double*)it[0];
  const long long n = it[1];
  double* dst = (double*)it[2];
  for (long long i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------------------------------------
// asm_expand_kernel: one thread per terminal triple writes its GTerm (see AsmTables)
// ---------------------------------------------------------------------------------------------

__device__ __forceinline__ MatRef mt(MatRef m) { return MatRef{m.p, m.cs, m.rs}; }

__global__ void asm_expand_kernel(AsmTables T, int ntrip, GTerm* __restrict__ terms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntrip) return;
  const int b = T.tnode[i];
  const int t = T.node_row[b], r = T.node_col[b];
  const bool dense = T.node_dense[b] != 0;
  const int s = T.ts[i], bts = T.tbx[i], bsr = T.tby[i];
  const char k = T.tk[i];
  GTerm g;
  g.alpha = 1.0;
  g.pad_ = 0;
  g.d = MatRef{nullptr, 0, 0};
  if ((T.only == 1 && !dense) || (T.only == 2 && dense)) {  // handled by another launch
    g.nf = 0;
    g.k = g.k2 = 0;
    g.a = g.b = g.d;
  } else if (k == 'a' && T.grouped && T.kwy_col[r] <= 64) {  // T += (xv | row factor) S_Y; flushed * D_r
    g.nf = 4;
    g.k = T.ky_mid[s];
    g.k2 = 0;
    g.b = T.ycoup[bsr];
    g.a = dense ? T.xv[bts] : (T.xadm[bts] ? T.rf[bts] : T.rproj[bts]);
  } else if (k == 'b' && T.grouped && T.kx_row[t] <= 64) {  // U += S_X (W_X,s-side)^T; flushed A_t *
    g.nf = 5;
    g.k = T.kwx_mid[s];
    g.k2 = 0;
    g.a = T.xcoup[bts];
    g.b = dense ? mt(T.wyl[bsr]) : mt(T.cproj[bsr]);
  } else if (k == 'a') {  // Y|sr admissible: S_Y, (xv | row factor), (W_Y leaf | Y's basis change)^T
    g.nf = 3;
    g.k = T.ky_mid[s];
    g.k2 = T.kwy_col[r];
    g.b = T.ycoup[bsr];
    if (dense) {
      g.a = T.xv[bts];
      g.d = mt(T.wyleaf[r]);
    } else {
      g.a = T.xadm[bts] ? T.rf[bts] : T.rproj[bts];
      g.d = mt(T.bcc[r]);
    }
  } else if (k == 'b') {  // X|ts admissible
    g.nf = 3;
    g.k = T.kx_row[t];
    g.k2 = T.kwx_mid[s];
    g.b = T.xcoup[bts];
    if (dense) {
      g.a = T.vxleaf[t];
      g.d = mt(T.wyl[bsr]);
    } else {
      g.a = T.bcr[t];
      g.d = mt(T.cproj[bsr]);
    }
  } else {  // both dense
    g.nf = 2;
    g.a = T.xnear[bts];
    g.b = T.ynear[bsr];
    g.k = T.size_mid[s];
    g.k2 = 0;
  }
  terms[i] = g;
}

// ---------------------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------------------

// Opt every kernel into the full 227 KB of dynamic shared memory once.  (Setting the attribute per
// launch races when two host threads launch the same kernel with different sizes.)
static void init_attributes() {
  static std::once_flag once;
  std::call_once(once, [] {
    auto opt_in = [](const void* fn) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fn);  // dynamic limit = 227 KB minus the kernel's static shared memory
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
      // prefer the largest shared-memory carveout so several CTAs fit per SM
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    };
    opt_in((const void*)qr_chunk_kernel);
    opt_in((const void*)tsqr_merge_kernel);
    opt_in((const void*)svd_tsqr_kernel);
    opt_in((const void*)svd_finish_kernel<0, true>);
    opt_in((const void*)svd_finish_kernel<8, true>);
    opt_in((const void*)svd_finish_kernel<16, true>);
    opt_in((const void*)svd_finish_kernel<24, true>);
    opt_in((const void*)svd_finish_kernel<24, false>);
    opt_in((const void*)svd_finish_kernel<0, false>);
    opt_in((const void*)svd_finish_kernel<8, false>);
    opt_in((const void*)svd_finish_kernel<16, false>);
    opt_in((const void*)norm_kernel);
    opt_in((const void*)norm_warp_kernel);
    opt_in((const void*)norm_cta_kernel);
  });
}

cudaError_t launch_gsum_mma(const GOut* outs, const GTerm* terms, const GTile* tiles, int ntiles, int k2max,
                            cudaStream_t st, int tag);

cudaError_t launch_gsum(const GOut* outs, const GTerm* terms, const GTile* tiles, int ntiles, int k2max,
                       cudaStream_t st, int tag) {
  return launch_gsum_mma(outs, terms, tiles, ntiles, k2max, st, tag);
}

size_t qr_smem(int n, bool rsmem) {
  return sizeof(double) * ((size_t)kPanel * (n | 1) + 64 + 4 + (rsmem ? (size_t)n * n : 0));
}

cudaError_t launch_qr_chunks(const QrItem* items, const Seg* segs, const SvdWork* work, int nwork, size_t smem,
                             bool rsmem, cudaStream_t st) {
  init_attributes();
  if (nwork == 0) return cudaSuccess;
  qr_chunk_kernel<<<nwork, kThreads, smem, st>>>(items, segs, work, rsmem ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_tsqr_merge(const MergeWork* work, int nwork, size_t smem, bool rsmem, cudaStream_t st) {
  init_attributes();
  if (nwork == 0) return cudaSuccess;
  tsqr_merge_kernel<<<nwork, kThreads, smem, st>>>(work, rsmem ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_qr_out(const QrItem* items, int nitems, cudaStream_t st) {
  if (nitems == 0) return cudaSuccess;
  qr_out_kernel<<<nitems, kThreads, 0, st>>>(items);
  return cudaGetLastError();
}

size_t svd_tsqr_smem(int m, int kx, bool rsmem) {
  const int k1 = m < kx ? m : kx;
  const int n = m - k1;
  size_t d = (size_t)m * (kx | 1) + kx + 1 + (kx > 0 ? (size_t)m * kRawLd : 0) + (size_t)kPanel * (n | 1) + 64 + 4;
  if (rsmem) d += (size_t)n * n;
  return d * sizeof(double);
}

size_t merge_smem(int n, bool rsmem) {
  return sizeof(double) * ((size_t)kPanel * (n | 1) + 68 + (rsmem ? (size_t)n * n : 0));
}

size_t svd_finish_smem(int m, int kx, bool rsmem, bool vsmem, bool tight) {
  const int k1 = m < kx ? m : kx;
  const int n = m - k1;
  if (tight)  // sig, ord, perm, iperm and R at stride n (even); no V
    return sizeof(double) * ((((size_t)n + (n / 2 + 1) + n + 1) & ~size_t(1)) + (size_t)n * (n + (n & 1)));
  return sizeof(double) * ((vsmem ? (size_t)m * (kx | 1) + kx + 1 : 0) + n + (n / 2 + 1) + 4 * (size_t)n + 2 +
                           (rsmem ? (size_t)n * fin_ld(n) : 0));
}

cudaError_t launch_svd_tsqr(const SvdItem* items, const Seg* segs, const SvdWork* work, int nwork, size_t smem,
                            bool rsmem, cudaStream_t st) {
  init_attributes();
  if (nwork == 0) return cudaSuccess;
  svd_tsqr_kernel<<<nwork, kThreads, smem, st>>>(items, segs, work, rsmem ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_svd_finish(const SvdItem* items, const Seg* segs, int nitems, size_t smem, bool rsmem, bool vsmem,
                              int nmax, cudaStream_t st, bool tight) {
  init_attributes();
  if (nitems == 0) return cudaSuccess;
  const int v = (vsmem && !tight ? 1 : 0) | (tight && rsmem ? 2 : 0);
  const long long sd = (long long)(smem / sizeof(double));
  if (rsmem) {
    if (nmax <= 64) svd_finish_kernel<8, true><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else if (nmax <= 128) svd_finish_kernel<16, true><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else if (nmax <= 192) svd_finish_kernel<24, true><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else svd_finish_kernel<0, true><<<nitems, NT, smem, st>>>(items, segs, v, sd);
  } else {
    if (nmax <= 64) svd_finish_kernel<8, false><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else if (nmax <= 128) svd_finish_kernel<16, false><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else if (nmax <= 192) svd_finish_kernel<24, false><<<nitems, NT, smem, st>>>(items, segs, v, sd);
    else svd_finish_kernel<0, false><<<nitems, NT, smem, st>>>(items, segs, v, sd);
  }
  return cudaGetLastError();
}

size_t norm_smem(int m, long long N, bool gram_in_smem) {
  const bool rowside = m <= N;  // Gram on the smaller side
  const int g = rowside ? m : (int)N;
  const int w = rowside ? m : (int)N;
  return sizeof(double) * ((gram_in_smem ? (size_t)g * g : 0) + (size_t)kPanel * w + 5 * (size_t)g);
}

cudaError_t launch_norm(const NormItem* items, const Seg* segs, int nitems, size_t smem, cudaStream_t st) {
  init_attributes();
  if (nitems == 0) return cudaSuccess;
  norm_kernel<<<nitems, kThreads, smem, st>>>(items, segs);
  return cudaGetLastError();
}

cudaError_t launch_asm_expand(const AsmTables& T, int ntrip, GTerm* terms, cudaStream_t st) {
  init_attributes();
  if (ntrip == 0) return cudaSuccess;
  asm_expand_kernel<<<(ntrip + 255) / 256, 256, 0, st>>>(T, ntrip, terms);
  return cudaGetLastError();
}

cudaError_t launch_gather(const long long* items, int nitems, cudaStream_t st) {
  init_attributes();
  if (nitems == 0) return cudaSuccess;
  gather_kernel<<<nitems, kThreads, 0, st>>>(items);
  return cudaGetLastError();
}

}  // namespace h2g
