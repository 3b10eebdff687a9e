// Register-tile Householder TSQR for sm_100a (R factors with n <= 128 columns).
//
// tile_absorb_kernel: one CTA absorbs 128-line tiles of a stacked operand into an n x n R factor
// held in shared memory (reference qr_r / the stacked QRs of weights.py:37-101,
// coarsening.py:231-245 and the wide SVD inputs of induced.py:127-137, coarsening.py:294-326).
// Thread (c, sub) = (threadIdx.x / 4, threadIdx.x % 4) owns column c of the tile, rows
// sub*32 .. sub*32+31, in 32 registers.  Householder step j: the owner group (c == j) forms the
// reflector of [R_jj; tile(:, j)] and publishes it through shared memory; after ONE barrier every
// column c > j updates its own registers and R_jc.  n steps per 128-line tile (the previous
// panel absorb needed n steps per 32 lines).
//
// Sources: lines of vstack(segs) (QrItem), columns of hstack(segs) (SvdItem; optionally
// projected onto Q2 = Q_V[:, k1:], i.e. tile = A_chunk^T Q2, the protected SVD input
// B^T = (Q_V^T A)[k1:]^T), or a second R factor (tree merge R_a <- R([R_a; R_b])).
// Arithmetic: LAPACK dlarfg sign convention, exact-zero columns skip (tau = 0), as the
// reference's numpy/LAPACK QR.
#include <cuda_runtime.h>

#include <mutex>

#include "h2g_types.h"

namespace h2g {

namespace {

constexpr int kRows = 128;          // tile lines
constexpr int kRpt = 32;            // rows per thread
constexpr int kSubLd = 34;          // shared stride per 32-row block (16B aligned, conflict-free)
constexpr int kLineLd = 4 * kSubLd;  // 136: one staged tile column
constexpr int kKs = 16;             // staging depth (source columns per slice)

__device__ __forceinline__ double seg_scale(const Seg& sg) {
  if (!sg.sdiv) return sg.scale;
  const double d = *sg.sdiv;
  return d > 0.0 ? sg.scale / d : sg.scale;
}

__device__ __forceinline__ int find_seg(const Seg* __restrict__ segs, int s0, int s1, long long line) {
  int lo = s0, hi = s1 - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].off <= line) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int lpos(int r) { return r + 2 * (r >> 5); }  // padded line index

struct Layout {
  double* R;        // n x n
  double* vb;       // 2 x kLineLd reflector buffers
  double* As;       // kKs x kLineLd staged source slice (line-major per source column)
  double* Qs;       // kKs x n projection slice
  const double** rp;  // per line: base pointer (null: zero line)
  long long* rst;   // per line: stride along the source columns
  double* rsc;      // per line: scale
};

__device__ __forceinline__ Layout carve(double* smem, int n) {
  Layout L;
  L.R = smem;
  L.vb = L.R + (((size_t)n * n + 1) & ~(size_t)1);  // 16-byte aligned for the double2 accesses
  L.As = L.vb + 2 * kLineLd;
  L.Qs = L.As + kKs * kLineLd;
  L.rp = (const double**)(L.Qs + (size_t)kKs * n);
  L.rst = (long long*)(L.rp + kRows);
  L.rsc = (double*)(L.rst + kRows);
  return L;
}

}  // namespace

size_t tile_absorb_smem(int n) {
  return sizeof(double) * ((size_t)n * n + 1 + 2 * kLineLd + kKs * kLineLd + (size_t)kKs * n + 3 * kRows);
}

// Staged slice element (k, r): source column k0 + k of line r (k < kk_lim), zero beyond.
__device__ __forceinline__ void stage_slice(const Layout& L, int hcols, int k0, int kdim, const double* q2, int q2ld,
                                            int n) {
  const int nt = blockDim.x;
  const int klim = min(kKs, kdim - k0);
  for (int e = threadIdx.x; e < kKs * kRows; e += nt) {
    int k, r;
    if (hcols) { k = e / kRows; r = e % kRows; }   // consecutive lines = consecutive source columns
    else { r = e / kKs; k = e % kKs; }             // consecutive entries of one source row
    const double* p = L.rp[r];
    double v = 0.0;
    if (p && k < klim) v = L.rsc[r] * p[(long long)(k0 + k) * L.rst[r]];
    L.As[k * kLineLd + lpos(r)] = v;
  }
  if (q2)
    for (int e = threadIdx.x; e < kKs * n; e += nt) {
      const int k = e / n, c = e % n;
      L.Qs[e] = k < klim ? q2[(long long)(k0 + k) * q2ld + c] : 0.0;
    }
}

__global__ void __launch_bounds__(512) tile_absorb_kernel(const TileItem* __restrict__ items,
                                                          const Seg* __restrict__ segs,
                                                          const TileWork* __restrict__ work) {
  extern __shared__ double smem[];
  __shared__ double tbuf[2];
  __shared__ int s_sa, s_sb;
  __shared__ long long g_off[kRows];  // staged segments of the current tile
  __shared__ const double* g_p[kRows];
  __shared__ int g_rs[kRows], g_cs[kRows];
  __shared__ double g_sc[kRows];
  const TileWork w = work[blockIdx.x];
  const TileItem it = items[w.item];
  const int n = it.n;
  const Layout L = carve(smem, n);
  const int t = threadIdx.x, c = t >> 2, sub = t & 3, lane = t & 31;
  const unsigned gmask = 0xfu << (lane & ~3);
  const bool live = c < n;
  for (int e = t; e < n * n; e += blockDim.x) L.R[e] = w.rinit ? w.rinit[e] : 0.0;

  double x[kRpt];
  long long l = w.l0;
  for (;;) {
#pragma unroll
    for (int i = 0; i < kRpt; ++i) x[i] = 0.0;
    if (w.rsrc) {
      // merge: the tile is R_b (n x n, upper triangular)
      if (live) {
#pragma unroll
        for (int i = 0; i < kRpt; ++i) {
          const int r = sub * kRpt + i;
          if (r < n) x[i] = w.rsrc[(long long)r * n + c];
        }
      }
      __syncthreads();
    } else {
      // per-line source descriptors: the segments covering this tile's lines are located once
      // (two binary searches in global memory) and staged in shared memory, every line then
      // searches the staged offsets
      const long long llast = min(l + kRows, w.l1) - 1;
      if (t == 0) s_sa = llast >= l ? find_seg(segs, it.s0, it.s1, l) : 0;
      if (t == 32 || (blockDim.x <= 32 && t == 0)) s_sb = llast >= l ? find_seg(segs, it.s0, it.s1, llast) : -1;
      __syncthreads();
      const int sa = s_sa, nseg = s_sb - s_sa + 1;
      const bool staged = nseg <= kRows;
      if (staged)
        for (int i = t; i < nseg; i += blockDim.x) {
          const Seg sg = segs[sa + i];
          g_off[i] = sg.off;
          g_p[i] = sg.a.p;
          g_rs[i] = sg.a.rs;
          g_cs[i] = sg.a.cs;
          g_sc[i] = seg_scale(sg);
        }
      __syncthreads();
      for (int r = t; r < kRows; r += blockDim.x) {
        const long long line = l + r;
        const double* p = nullptr;
        long long st = 0;
        double sc = 0.0;
        if (line < w.l1) {
          if (staged) {
            int lo = 0, hi = nseg - 1;
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (g_off[mid] <= line) lo = mid; else hi = mid - 1;
            }
            const long long loc = line - g_off[lo];
            sc = g_sc[lo];
            if (it.hcols) { p = g_p[lo] + loc * g_cs[lo]; st = g_rs[lo]; }
            else { p = g_p[lo] + loc * g_rs[lo]; st = g_cs[lo]; }
          } else {
            const int sidx = find_seg(segs, it.s0, it.s1, line);
            const Seg sg = segs[sidx];
            const long long loc = line - sg.off;
            sc = seg_scale(sg);
            if (it.hcols) { p = sg.a.p + loc * sg.a.cs; st = sg.a.rs; }
            else { p = sg.a.p + loc * sg.a.rs; st = sg.a.cs; }
          }
        }
        L.rp[r] = p;
        L.rst[r] = st;
        L.rsc[r] = sc;
      }
      __syncthreads();
      for (int k0 = 0; k0 < it.kdim; k0 += kKs) {
        stage_slice(L, it.hcols, k0, it.kdim, it.q2, it.q2ld, n);
        __syncthreads();
        if (live) {
          const double* a = L.As + sub * kSubLd;
          if (it.q2) {
            const int klim = min(kKs, it.kdim - k0);
            for (int k = 0; k < klim; ++k) {
              const double q = L.Qs[k * n + c];
              const double2* ak = reinterpret_cast<const double2*>(a + k * kLineLd);
#pragma unroll
              for (int i = 0; i < kRpt / 2; ++i) {
                const double2 v = ak[i];
                x[2 * i] = fma(v.x, q, x[2 * i]);
                x[2 * i + 1] = fma(v.y, q, x[2 * i + 1]);
              }
            }
          } else if (c >= k0 && c < k0 + kKs) {
            const double2* ak = reinterpret_cast<const double2*>(a + (c - k0) * kLineLd);
#pragma unroll
            for (int i = 0; i < kRpt / 2; ++i) {
              const double2 v = ak[i];
              x[2 * i] = v.x;
              x[2 * i + 1] = v.y;
            }
          }
        }
        __syncthreads();
      }
    }

    // Householder absorb of the tile into R, one barrier per column
    int buf = 0;
    for (int j = 0; j < n; ++j) {
      double* v = L.vb + buf * kLineLd;
      if (c == j) {
        // critical path of the step: four partial sums, reciprocals instead of divisions
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int i = 0; i < kRpt; i += 4) {
          s0 = fma(x[i], x[i], s0);
          s1 = fma(x[i + 1], x[i + 1], s1);
          s2 = fma(x[i + 2], x[i + 2], s2);
          s3 = fma(x[i + 3], x[i + 3], s3);
        }
        double s = (s0 + s1) + (s2 + s3);
        s += __shfl_xor_sync(gmask, s, 1);
        s += __shfl_xor_sync(gmask, s, 2);
        const double alpha = L.R[j * n + j];
        double tau = 0.0, scale = 0.0, beta = alpha;
        if (s != 0.0) {
          const double nrm = sqrt(fma(alpha, alpha, s));
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau = (beta - alpha) * __drcp_rn(beta);
          scale = __drcp_rn(alpha - beta);
        }
        __syncwarp(gmask);  // every lane of the group has read R_jj
        if (sub == 0) L.R[j * n + j] = beta;
        double2* vv = reinterpret_cast<double2*>(v + sub * kSubLd);
#pragma unroll
        for (int i = 0; i < kRpt / 2; ++i) vv[i] = make_double2(x[2 * i] * scale, x[2 * i + 1] * scale);
#pragma unroll
        for (int i = 0; i < kRpt; ++i) x[i] = 0.0;
        if (sub == 0) tbuf[buf] = tau;
      }
      __syncthreads();
      const double tau = tbuf[buf];
      if (tau != 0.0 && c > j && live) {
        const double2* vv = reinterpret_cast<const double2*>(v + sub * kSubLd);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int i = 0; i < kRpt / 4; ++i) {
          const double2 p = vv[2 * i], q = vv[2 * i + 1];
          a0 = fma(p.x, x[4 * i], a0);
          a1 = fma(p.y, x[4 * i + 1], a1);
          a2 = fma(q.x, x[4 * i + 2], a2);
          a3 = fma(q.y, x[4 * i + 3], a3);
        }
        double wv = (a0 + a1) + (a2 + a3);
        const double rj = L.R[j * n + c];
        wv += __shfl_xor_sync(gmask, wv, 1);
        wv += __shfl_xor_sync(gmask, wv, 2);
        __syncwarp(gmask);  // every lane of the group has read R_jc
        const double tw = tau * (wv + rj);
        if (sub == 0) L.R[j * n + c] = rj - tw;
#pragma unroll
        for (int i = 0; i < kRpt / 2; ++i) {
          const double2 p = vv[i];
          x[2 * i] = fma(-tw, p.x, x[2 * i]);
          x[2 * i + 1] = fma(-tw, p.y, x[2 * i + 1]);
        }
      }
      buf ^= 1;
    }
    __syncthreads();
    l += kRows;
    if (w.rsrc || l >= w.l1) break;
  }
  for (int e = t; e < n * n; e += blockDim.x) w.rout[e] = L.R[e];
}

// Protected-SVD preparation, one CTA per item with kx > 0: Householder QR of V (m x kx) into
// it.vws (reflectors + tau) and the explicit Q_V (m x m, row major) into it.q2: its last n
// columns Q2 = Q_V[:, k1:] are the projection the tiles apply (B^T = A^T Q2), its first k1 and
// Q2 U give svd_finish_kernel's output Q_t = Q_V [[I, 0], [0, U]] as one product.
__device__ void prep_qr_cols(double* V, int m, int kx, int ldv, int k1, double* tv, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = 0; j < k1; ++j) {
    double part = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) part = fma(V[i * ldv + j], V[i * ldv + j], part);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < nw; ++q) s += red[q];
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
    if (tau != 0.0)
      for (int c = j + 1 + warp; c < kx; c += nw) {
        double w = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w = fma(V[i * ldv + j], V[i * ldv + c], w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w += V[j * ldv + c];
        __syncwarp();
        if (lane == 0) V[j * ldv + c] -= tau * w;
        for (int i = j + 1 + lane; i < m; i += 32) V[i * ldv + c] -= tau * w * V[i * ldv + j];
      }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) svd_prep_kernel(const SvdItem* __restrict__ items, const int* __restrict__ ids,
                                                       size_t smem_bytes) {
  extern __shared__ double smem[];
  __shared__ double red[20];
  const SvdItem it = items[ids[blockIdx.x]];
  const int m = it.m, kx = it.kx, k1 = min(m, kx);
  const int ldv = kx | 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* V = smem;
  double* tv = V + (size_t)m * ldv;
  // Q_V built in shared memory when it fits, else in place in the output buffer
  const bool xs = sizeof(double) * ((size_t)m * ldv + kx + 1 + (size_t)m * (m | 1)) <= smem_bytes;
  const int ldx = xs ? (m | 1) : m;
  double* X = xs ? tv + kx + 1 : it.q2;
  for (int e = threadIdx.x; e < m * kx; e += blockDim.x) V[(e / kx) * ldv + e % kx] = it.v.p[(long long)(e / kx) * it.v.rs + (long long)(e % kx) * it.v.cs];
  __syncthreads();
  prep_qr_cols(V, m, kx, ldv, k1, tv, red);
  for (int e = threadIdx.x; e < m * ldv; e += blockDim.x) it.vws[e] = V[e];
  for (int e = threadIdx.x; e < kx; e += blockDim.x) it.vws[m * ldv + e] = tv[e];
  if (!it.q2) return;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, j = e % m;
    X[i * ldx + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  // Q_V = H_0 H_1 .. H_{k1-1} I (m x m): reflectors in reverse order, one warp per column
  for (int c = warp; c < m; c += nw)
    for (int j = k1 - 1; j >= 0; --j) {
      const double tau = tv[j];
      if (tau == 0.0) continue;
      double part = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) part = fma(V[i * ldv + j], X[i * ldx + c], part);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      const double wv = part + X[j * ldx + c];
      __syncwarp();
      if (lane == 0) X[j * ldx + c] -= tau * wv;
      for (int i = j + 1 + lane; i < m; i += 32) X[i * ldx + c] -= tau * wv * V[i * ldv + j];
      __syncwarp();
    }
  __syncthreads();
  if (xs)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) it.q2[e] = X[(e / m) * ldx + e % m];
}

size_t svd_prep_smem(int m, int kx, bool with_q) {
  return sizeof(double) * ((size_t)m * (kx | 1) + kx + 1 + (with_q ? (size_t)m * (m | 1) : 0));
}

static void tile_attributes() {
  static std::once_flag once;
  std::call_once(once, [] {
    for (const void* fn : {(const void*)tile_absorb_kernel, (const void*)svd_prep_kernel}) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, fn);
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - (int)fa.sharedSizeBytes);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
  });
}

cudaError_t launch_tile_absorb(const TileItem* items, const Seg* segs, const TileWork* work, int nwork, int nmax,
                               cudaStream_t st) {
  tile_attributes();
  if (nwork == 0) return cudaSuccess;
  const int threads = 32 * ((nmax + 7) / 8);
  tile_absorb_kernel<<<nwork, threads, tile_absorb_smem(nmax), st>>>(items, segs, work);
  return cudaGetLastError();
}

cudaError_t launch_svd_prep(const SvdItem* items, const int* ids, int nids, size_t smem, cudaStream_t st) {
  tile_attributes();
  if (nids == 0) return cudaSuccess;
  svd_prep_kernel<<<nids, 512, smem, st>>>(items, ids, smem);
  return cudaGetLastError();
}

}  // namespace h2g
