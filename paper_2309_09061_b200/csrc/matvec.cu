// H^2 matrix-vector products on the GPU (reference h2.py:197-267 h2_matvec / h2_matvec_adjoint):
// y (+)= alpha * op(G) x in O(n k) operations, the building block of the power-iteration error
// estimate (bench.py:126-174).  Memory bound: every basis, coupling and nearfield entry is read
// once per product.
//
// Stages (each a batch of small GEMVs, one CTA per output segment):
//   forward   xhat_s = W_s^T x|s (leaves), sum_c E_c^T xhat_c (inner), bottom-up by level
//   coupling  yhat_t = sum_{b=(t,s) admissible} S_b xhat_s
//   backward  yhat_c += E_c yhat_t, top-down by level
//   leaves    y|t (+)= alpha V_t yhat_t, then y|t += alpha sum_{b=(t,s) dense} N_b x|s
// The adjoint is the same on the transposed view (bases swapped, blocks transposed).
#include <cuda_runtime.h>

#include <algorithm>

#include "engine.h"

namespace h2g {

namespace {

constexpr int kMvThreads = 256;

// One warp per term (terms of an output are spread over the CTA's warps, no barriers between
// them).  Row-major blocks (k contiguous, the nearfield / coupling blocks of G and Z): 8 lanes per
// row, 4 rows per warp step, each lane striding k by 8 -- every warp load covers four 64-byte row
// segments (full sectors), partial sums joined by 3 butterflies.  Column-major views (transposed
// blocks, adjoint): lanes own rows, so consecutive lanes read consecutive addresses.  Each warp
// accumulates into its own shared-memory row buffer; the buffers are summed in warp order at the
// end, so the result does not depend on scheduling.
__device__ void mv_term_warp(const MvTerm& t, int m, double* acc) {
  const int lane = threadIdx.x & 31;
  const MatRef a = t.a;
  if (a.cs == 1 && t.k >= 8) {
    const int grp = lane >> 3, gl = lane & 7;
    for (int i0 = 0; i0 < m; i0 += 4) {
      const int i = i0 + grp;
      double s0 = 0.0, s1 = 0.0;
      if (i < m) {
        const double* row = a.p + (long long)i * a.rs;
        int j = gl;
        for (; j + 8 < t.k; j += 16) {
          s0 = fma(row[j], t.x[j], s0);
          s1 = fma(row[j + 8], t.x[j + 8], s1);
        }
        if (j < t.k) s0 = fma(row[j], t.x[j], s0);
      }
      double s = s0 + s1;
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (gl == 0 && i < m) acc[i] += t.alpha * s;
    }
    return;
  }
  for (int i = lane; i < m; i += 32) {
    const double* row = a.p + (long long)i * a.rs;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = 0;
    for (; j + 3 < t.k; j += 4) {
      s0 = fma(row[(long long)j * a.cs], t.x[j], s0);
      s1 = fma(row[(long long)(j + 1) * a.cs], t.x[j + 1], s1);
      s2 = fma(row[(long long)(j + 2) * a.cs], t.x[j + 2], s2);
      s3 = fma(row[(long long)(j + 3) * a.cs], t.x[j + 3], s3);
    }
    for (; j < t.k; ++j) s0 = fma(row[(long long)j * a.cs], t.x[j], s0);
    acc[i] += t.alpha * ((s0 + s1) + (s2 + s3));
  }
}

}  // namespace

__global__ void __launch_bounds__(kMvThreads) mv_kernel(const MvOut* __restrict__ outs,
                                                        const MvTerm* __restrict__ terms, int ldacc) {
  extern __shared__ double acc[];  // nwarps x ldacc
  const MvOut o = outs[blockIdx.x];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* mine = acc + warp * ldacc;
  for (int i = threadIdx.x & 31; i < o.m; i += 32) mine[i] = 0.0;
  __syncwarp();
  for (int ti = o.t0 + warp; ti < o.t1; ti += nw) mv_term_warp(terms[ti], o.m, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < o.m; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[w * ldacc + i];
    o.y[i] = (o.beta ? o.y[i] : 0.0) + s;
  }
}

// Term-heavy batches: chunk c of an output (terms [t0, t1)) writes its partial sum to part + poff;
// mv_reduce_kernel then adds the chunks of each output in chunk order (deterministic).
struct MvChunk {
  int out, t0, t1, pad_;
  long long poff;
};

__global__ void __launch_bounds__(kMvThreads) mv_chunk_kernel(const MvOut* __restrict__ outs,
                                                              const MvChunk* __restrict__ chunks,
                                                              const MvTerm* __restrict__ terms, double* part,
                                                              int ldacc) {
  extern __shared__ double acc[];
  const MvChunk ch = chunks[blockIdx.x];
  const int m = outs[ch.out].m;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* mine = acc + warp * ldacc;
  for (int i = threadIdx.x & 31; i < m; i += 32) mine[i] = 0.0;
  __syncwarp();
  for (int ti = ch.t0 + warp; ti < ch.t1; ti += nw) mv_term_warp(terms[ti], m, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[w * ldacc + i];
    part[ch.poff + i] = s;
  }
}

__global__ void mv_reduce_kernel(const MvOut* __restrict__ outs, const int* __restrict__ cptr,
                                 const MvChunk* __restrict__ chunks, const double* __restrict__ part) {
  const MvOut o = outs[blockIdx.x];
  const int c0 = cptr[blockIdx.x], c1 = cptr[blockIdx.x + 1];
  for (int i = threadIdx.x; i < o.m; i += blockDim.x) {
    double s = 0.0;
    for (int c = c0; c < c1; ++c) s += part[chunks[c].poff + i];
    o.y[i] = (o.beta ? o.y[i] : 0.0) + s;
  }
}

void MvBatch::run(Ctx& C) {
  if (outs.empty()) return;
  int mmax = 1;
  for (const MvOut& o : outs) mmax = std::max(mmax, o.m);
  const int ldacc = mmax | 1;
  const size_t smem = sizeof(double) * ldacc * (kMvThreads / 32);
  static constexpr int kChunkTerms = 8;  // one term per warp
  cudaEvent_t ev = nullptr;
  if ((long long)terms.size() > 4LL * (long long)outs.size() && terms.size() > 1024) {
    // term-heavy (dense leaf rows): spread each output over ceil(terms / 8) CTAs
    std::vector<MvChunk> ch;
    std::vector<int> cptr{0};
    long long poff = 0;
    for (int oi = 0; oi < (int)outs.size(); ++oi) {
      const MvOut& o = outs[oi];
      for (int t = o.t0; t < o.t1 || t == o.t0; t += kChunkTerms) {
        ch.push_back(MvChunk{oi, t, std::min(o.t1, t + kChunkTerms), 0, poff});
        poff += o.m;
        if (o.t1 == o.t0) break;
      }
      cptr.push_back((int)ch.size());
    }
    Arena sc(C.st);
    double* part = sc.alloc(std::max<long long>(1, poff));
    MvOut* d_o = C.push(outs);
    MvTerm* d_t = C.push(terms);
    MvChunk* d_c = C.push(ch);
    int* d_p = C.push(cptr);
    C.flush();
    ev = C.prof_begin();
    mv_chunk_kernel<<<(unsigned)ch.size(), kMvThreads, smem, C.st>>>(d_o, d_c, d_t, part, ldacc);
    cuda_check(cudaGetLastError(), "mv_chunk_kernel");
    mv_reduce_kernel<<<(unsigned)outs.size(), 128, 0, C.st>>>(d_o, d_p, d_c, part);
    cuda_check(cudaGetLastError(), "mv_reduce_kernel");
    C.launches += 2;
  } else {
    MvOut* d_o = C.push(outs);
    MvTerm* d_t = terms.empty() ? nullptr : C.push(terms);
    C.flush();
    ev = C.prof_begin();
    mv_kernel<<<(unsigned)outs.size(), kMvThreads, smem, C.st>>>(d_o, d_t, ldacc);
    cuda_check(cudaGetLastError(), "mv_kernel");
    ++C.launches;
  }
  double by = 0.0;
  if (C.prof)
    for (const MvTerm& t : terms) by += 8.0 * t.k;  // vector reads on top of the matrix bytes
  C.prof_end(K_MV, ev, 2.0 * bytes_a / 8.0, bytes_a + by);
  outs.clear();
  terms.clear();
  bytes_a = 0.0;
}

// y (+)= alpha * G x on the view g (rows x cols); x, y device vectors.
void h2_matvec(Ctx& C, HView g, const double* x, double* y, double alpha, bool accumulate) {
  const Tree& rt = g.rows();
  const Tree& ct = g.cols();
  const Basis& RB = g.rb();
  const Basis& CB = g.cb();
  const BView bv = g.bv();
  const Blocks& B = *g.h->bt;
  wait_near(C, *g.h);
  Arena sc(C.st);
  std::vector<long long> xo(ct.n), yo(rt.n);
  long long nx = 0, ny = 0;
  for (int s = 0; s < ct.n; ++s) { xo[s] = nx; nx += CB.rank[s]; }
  for (int t = 0; t < rt.n; ++t) { yo[t] = ny; ny += RB.rank[t]; }
  double* xh = sc.alloc(std::max<long long>(1, nx));
  double* yh = sc.alloc(std::max<long long>(1, ny));
  MvBatch mb;
  // forward transform, bottom-up (h2.py:197-210)
  for (int lev = ct.depth; lev >= 0; --lev) {
    for (int s : ct.by_level[lev]) {
      const int k = CB.rank[s];
      if (k == 0) continue;
      mb.out(xh + xo[s], k, false);
      if (ct.leaf(s)) {
        mb.term(CB.leafm(s).tref(), x + ct.start[s], ct.size(s), 1.0, (double)ct.size(s) * k);
      } else {
        for (int i = 0; i < ct.nkids(s); ++i) {
          const int c = ct.kid(s, i);
          if (CB.rank[c] > 0) mb.term(CB.xferm(c).tref(), xh + xo[c], CB.rank[c], 1.0, (double)CB.rank[c] * k);
        }
      }
    }
    mb.run(C);
  }
  // coupling accumulation (h2.py:229-231)
  {
    std::vector<std::vector<int>> by_row(rt.n);
    for (int b = 0; b < B.nb; ++b)
      if (B.adm_leaf(b)) by_row[bv.row(b)].push_back(b);
    for (int t = 0; t < rt.n; ++t) {
      const int k = RB.rank[t];
      if (k == 0) continue;
      mb.out(yh + yo[t], k, false);
      for (int b : by_row[t]) {
        const int s = bv.col(b);
        if (CB.rank[s] > 0) mb.term(g.coup(b), xh + xo[s], CB.rank[s], 1.0, (double)k * CB.rank[s]);
      }
    }
    mb.run(C);
  }
  // backward transform, top-down (h2.py:213-221)
  for (int lev = 1; lev <= rt.depth; ++lev) {
    for (int t : rt.by_level[lev]) {
      const int p = rt.parent[t];
      if (RB.rank[t] == 0 || RB.rank[p] == 0) continue;
      mb.out(yh + yo[t], RB.rank[t], true);
      mb.term(RB.xferm(t).ref(), yh + yo[p], RB.rank[p], 1.0, (double)RB.rank[t] * RB.rank[p]);
    }
    mb.run(C);
  }
  // leaves: y|t (+)= alpha (V_t yhat_t + sum_{b=(t,s) dense} N_b x|s); dense blocks on inner row
  // clusters (rare) follow in one launch per level so that concurrent outputs never overlap
  std::vector<std::vector<int>> near_by_row(rt.n);
  for (int b = 0; b < B.nb; ++b)
    if (B.near_leaf(b)) near_by_row[bv.row(b)].push_back(b);
  auto near_terms = [&](int t) {
    for (int b : near_by_row[t]) {
      const int s = bv.col(b);
      mb.term(g.near(b), x + ct.start[s], ct.size(s), alpha, (double)rt.size(t) * ct.size(s));
    }
  };
  for (int t = 0; t < rt.n; ++t) {
    if (!rt.leaf(t)) continue;
    mb.out(y + rt.start[t], rt.size(t), accumulate);
    if (RB.rank[t] > 0)
      mb.term(RB.leafm(t).ref(), yh + yo[t], RB.rank[t], alpha, (double)rt.size(t) * RB.rank[t]);
    near_terms(t);
  }
  mb.run(C);
  for (int lev = 0; lev <= rt.depth; ++lev) {
    for (int t : rt.by_level[lev]) {
      if (rt.leaf(t) || near_by_row[t].empty()) continue;
      mb.out(y + rt.start[t], rt.size(t), true);
      near_terms(t);
    }
    mb.run(C);
  }
}

}  // namespace h2g
