// H^2 matrix-vector products on the GPU (reference h2.py:197-267 h2_matvec / h2_matvec_adjoint):
// y (+)= alpha * op(G) x in O(n k) operations, the building block of the power-iteration error
// estimate (bench.py:126-174).  Memory bound: every basis, coupling and nearfield entry is read
// once per product.
//
// Stages (each a batch of small GEMVs):
//   nearfield y|t (+)= alpha sum_{b=(t,s) dense} N_b x|s -- independent of the transforms, so it runs
//             on a second stream concurrently with the latency-bound chain below (the bulk of the
//             bytes against many small dependent launches)
//   forward   xhat_s = W_s^T x|s (leaves), sum_c E_c^T xhat_c (inner), bottom-up by level
//   coupling  yhat_t = sum_{b=(t,s) admissible} S_b xhat_s
//   backward  yhat_c += E_c yhat_t, top-down by level
//   leaves    y|t += alpha V_t yhat_t, once both streams joined
// The adjoint is the same on the transposed view (bases swapped, blocks transposed).  The launches
// of a matrix and orientation are planned once (descriptors uploaded once) and replayed per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.h"

namespace h2g {

// Batched small GEMVs: y (m) = (beta ? y : 0) + sum alpha * A (m x k) x (k).  Vector pointers may be
// tagged (bit 63): offsets into the call's x (bit 62 clear) or y (bit 62 set), so a plan's
// descriptors are built and uploaded once and replayed for every call; a term with flag 1 is
// scaled by the call's alpha, an output with beta 2 takes the call's accumulate flag.
struct MvTerm {
  MatRef a;
  const double* x;
  int k, flags;
  double alpha;
};
struct MvOut {
  double* y;
  int m, t0, t1, beta;
};
struct MvCall {  // per-call arguments of a plan replay
  const double* x;
  double* y;
  double alpha;
  int accumulate;
};

namespace {

constexpr int kMvThreads = 256;
constexpr unsigned long long kTag = 1ull << 63, kTagY = 1ull << 62, kTagOff = kTagY - 1;

inline const double* tag_x(long long off) { return reinterpret_cast<const double*>(kTag | (unsigned long long)off); }
inline double* tag_y(long long off) { return reinterpret_cast<double*>(kTag | kTagY | (unsigned long long)off); }

__device__ __forceinline__ const double* rv(const double* p, const MvCall& A) {
  const unsigned long long u = reinterpret_cast<unsigned long long>(p);
  if (!(u & kTag)) return p;
  return ((u & kTagY) ? A.y : A.x) + (u & kTagOff);
}
__device__ __forceinline__ MvTerm resolve(MvTerm t, const MvCall& A) {
  t.x = rv(t.x, A);
  if (t.flags & 1) t.alpha *= A.alpha;
  return t;
}
__device__ __forceinline__ MvOut resolve(MvOut o, const MvCall& A) {
  o.y = const_cast<double*>(rv(o.y, A));
  if (o.beta == 2) o.beta = A.accumulate;
  return o;
}

// Warp-level GEMV of one term, emitted 32 rows at a time: emit(r0, v) receives, in lane l, alpha
// times row r0 + l of A x (meaningful for r0 + l < m).  Every load is unconditional (row and column
// indices are clamped into the block, the clamped entries meet zero weights or land in lanes whose
// row is discarded), so the compiler keeps many rows' loads in flight per lane.
//
// Row-major blocks, k <= 256 (nearfield / coupling blocks of G and Z): the lane's slice of x stays in
// registers for the whole block (columns 2*lane + 64c as double2 when rows are 16-byte aligned, else
// lane + 32c), each row is read by the whole warp in full-line loads, and the 32 per-lane partials
// of a 32-row group are reduced by a transposing butterfly (31 exchanges for 32 rows, lane l ends
// with row r0 + l) -- no shuffle tree per row, no x re-reads.  Rows r and r + 16 are loaded together
// and the butterfly's first exchange (offset 16) is applied as they arrive, so only 16 partials stay
// live; a group with at most 16 rows left skips the upper half.
template <bool V2, int NC, class Emit>
__device__ __forceinline__ void mv_rm_term(const MvTerm& t, int m, Emit&& emit) {
  const int lane = threadIdx.x & 31;
  const MatRef a = t.a;
  const int k = t.k;
  constexpr int W = V2 ? 64 : 32;  // columns per chunk
  constexpr int X2 = V2 ? 2 : 1;
  double xr[NC][X2];
  int jc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = W * c + X2 * lane;
    xr[c][0] = j < k ? t.x[j] : 0.0;
    if (V2) xr[c][X2 - 1] = j + 1 < k ? t.x[j + 1] : 0.0;
    jc[c] = min(j, k - X2);  // clamped column: its weights are zero beyond k
  }
  auto rowdot = [&](int i) {
    const double* row = a.p + (long long)min(i, m - 1) * a.rs;
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (V2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row + jc[c]));
        s = fma(v.x, xr[c][0], s);
        s = fma(v.y, xr[c][X2 - 1], s);
      } else {
        s = fma(__ldg(row + jc[c]), xr[c][0], s);
      }
    }
    return s;
  };
  const bool up16 = (lane & 16) != 0;
  for (int r0 = 0; r0 < m; r0 += 32) {
    double p[16];
    if (m - r0 > 16) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const double lo = rowdot(r0 + r), hi = rowdot(r0 + 16 + r);
        p[r] = (up16 ? hi : lo) + __shfl_xor_sync(0xffffffffu, up16 ? lo : hi, 16);
      }
    } else {  // at most 16 rows left: the upper half is zero
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const double lo = rowdot(r0 + r);
        p[r] = (up16 ? 0.0 : lo) + __shfl_xor_sync(0xffffffffu, up16 ? lo : 0.0, 16);
      }
    }
    // transposing butterfly: after the step with offset o, lanes with bit o set hold the upper half
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int r = 0; r < o; ++r) {
        const double send = up ? p[r] : p[r + o];
        const double keep = up ? p[r + o] : p[r];
        p[r] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    emit(r0, t.alpha * p[0]);
  }
}

// Any layout (column-major views: the adjoint, transposed leaf bases of the forward transform):
// lanes own rows, so consecutive lanes read consecutive addresses; a 32-column block's loads are all
// issued before they are consumed, x entries broadcast from the warp's registers.
template <class Emit>
__device__ __forceinline__ void mv_cm_term(const MvTerm& t, int m, Emit&& emit) {
  const int lane = threadIdx.x & 31;
  const MatRef a = t.a;
  const int k = t.k;
  for (int r0 = 0; r0 < m; r0 += 32) {
    const double* row = a.p + (long long)min(r0 + lane, m - 1) * a.rs;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int jb = 0; jb < k; jb += 32) {
      const double xv = jb + lane < k ? t.x[jb + lane] : 0.0;
      double v[32];  // clamped into the block: columns past k meet x = 0
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = row[(long long)min(jb + q, k - 1) * a.cs];
#pragma unroll
      for (int q = 0; q < 32; q += 4) {
        s0 = fma(v[q], __shfl_sync(0xffffffffu, xv, q), s0);
        s1 = fma(v[q + 1], __shfl_sync(0xffffffffu, xv, q + 1), s1);
        s2 = fma(v[q + 2], __shfl_sync(0xffffffffu, xv, q + 2), s2);
        s3 = fma(v[q + 3], __shfl_sync(0xffffffffu, xv, q + 3), s3);
      }
    }
    emit(r0, t.alpha * ((s0 + s1) + (s2 + s3)));
  }
}

template <class Emit>
__device__ __forceinline__ void mv_term(const MvTerm& t, int m, Emit&& emit) {
  if (m <= 0 || t.k <= 0) return;
  if (t.a.cs == 1 && t.k <= 256) {
    const bool v2 = ((reinterpret_cast<unsigned long long>(t.a.p) & 15ull) == 0) && (t.a.rs % 2 == 0) &&
                    (t.k % 2 == 0);
    if (v2) {
      if (t.k <= 64) mv_rm_term<true, 1>(t, m, emit);
      else if (t.k <= 128) mv_rm_term<true, 2>(t, m, emit);
      else if (t.k <= 192) mv_rm_term<true, 3>(t, m, emit);
      else mv_rm_term<true, 4>(t, m, emit);
    } else {
      if (t.k <= 32) mv_rm_term<false, 1>(t, m, emit);
      else if (t.k <= 64) mv_rm_term<false, 2>(t, m, emit);
      else if (t.k <= 128) mv_rm_term<false, 4>(t, m, emit);
      else mv_rm_term<false, 8>(t, m, emit);
    }
    return;
  }
  mv_cm_term(t, m, emit);
}

// the terms of one output (m <= 128) into four row registers (row 32g + lane in acc g), in order,
// the next term's descriptor loaded while the current one runs
__device__ __forceinline__ void mv_terms_regs(const MvTerm* __restrict__ terms, int t0, int t1, int m,
                                              double (&acc)[4], const MvCall& A) {
  MvTerm nx;
  if (t0 < t1) nx = terms[t0];
  for (int ti = t0; ti < t1; ++ti) {
    const MvTerm t = resolve(nx, A);
    if (ti + 1 < t1) nx = terms[ti + 1];
    mv_term(t, m, [&](int r0, double v) {
      if (r0 == 0) acc[0] += v;
      else if (r0 == 32) acc[1] += v;
      else if (r0 == 64) acc[2] += v;
      else acc[3] += v;
    });
  }
}

// CTA kernels (m > 128): each warp accumulates its terms into its own shared-memory row buffer; the
// buffers are summed in warp order at the end, so the result does not depend on scheduling.
__device__ __forceinline__ void mv_term_warp(const MvTerm& t, int m, double* acc) {
  const int lane = threadIdx.x & 31;
  mv_term(t, m, [&](int r0, double v) {
    if (r0 + lane < m) acc[r0 + lane] += v;
  });
}

}  // namespace

__global__ void __launch_bounds__(kMvThreads, 2) mv_kernel(const MvOut* __restrict__ outs,
                                                           const MvTerm* __restrict__ terms, int ldacc,
                                                           const MvCall A) {
  extern __shared__ double acc[];  // nwarps x ldacc
  const MvOut o = resolve(outs[blockIdx.x], A);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* mine = acc + warp * ldacc;
  for (int i = threadIdx.x & 31; i < o.m; i += 32) mine[i] = 0.0;
  __syncwarp();
  for (int ti = o.t0 + warp; ti < o.t1; ti += nw) mv_term_warp(resolve(terms[ti], A), o.m, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < o.m; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[w * ldacc + i];
    o.y[i] = (o.beta ? o.y[i] : 0.0) + s;
  }
}

// Chunk c of an output (terms [t0, t1)) writes its partial sum to part + poff (poff < 0: the
// output's only chunk, written to y directly); the reduce kernels then add the chunks of each output
// in chunk order (deterministic).
struct MvChunk {
  int out, t0, t1, pad_;
  long long poff;
};

// Warp per chunk of an output with m <= 128 (the level stages of the basis transforms, the coupling
// stage, c4's nearfield rows): the output rows live in registers, no shared memory and no barriers --
// a CTA per output left 7 of 8 warps idle on one-term outputs, and a CTA per 8 terms made each term
// a latency chain of its own.
__global__ void __launch_bounds__(kMvThreads, 2) mv_warp_kernel(const MvOut* __restrict__ outs,
                                                                const MvChunk* __restrict__ chunks,
                                                                const MvTerm* __restrict__ terms, double* part,
                                                                int nchunks, const MvCall A) {
  const int lane = threadIdx.x & 31;
  const int ci = blockIdx.x * (kMvThreads / 32) + (threadIdx.x >> 5);
  if (ci >= nchunks) return;
  const MvChunk ch = chunks[ci];
  const MvOut o = resolve(outs[ch.out], A);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  mv_terms_regs(terms, ch.t0, ch.t1, o.m, acc, A);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int i = 32 * g + lane;
    if (i < o.m) {
      if (ch.poff < 0) o.y[i] = (o.beta ? o.y[i] : 0.0) + acc[g];
      else part[ch.poff + i] = acc[g];
    }
  }
}

// outputs split over several warp chunks: red = (output, first chunk, end chunk)
__global__ void mv_wreduce_kernel(const MvOut* __restrict__ outs, const int4* __restrict__ red,
                                  const MvChunk* __restrict__ chunks, const double* __restrict__ part,
                                  const MvCall A) {
  const int4 r = red[blockIdx.x];
  const MvOut o = resolve(outs[r.x], A);
  for (int i = threadIdx.x; i < o.m; i += blockDim.x) {
    double s = 0.0;
    for (int c = r.y; c < r.z; ++c) s += part[chunks[c].poff + i];
    o.y[i] = (o.beta ? o.y[i] : 0.0) + s;
  }
}

// Several dependent level batches of few outputs each (the upper levels of the forward / backward
// basis transforms) in ONE single-CTA launch: level l's outputs [lptr[l], lptr[l+1]) are taken by the
// CTA's warps round robin and a barrier separates the levels (global writes of a level are visible to
// the whole CTA after it) -- one launch instead of one per level.
constexpr int kLvThreads = 512;
__global__ void __launch_bounds__(kLvThreads, 1) mv_levels_kernel(const MvOut* __restrict__ outs,
                                                                  const MvTerm* __restrict__ terms,
                                                                  const int* __restrict__ lptr, int nlev,
                                                                  const MvCall A) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kLvThreads / 32;
  for (int l = 0; l < nlev; ++l) {
    for (int oi = lptr[l] + warp; oi < lptr[l + 1]; oi += nw) {
      const MvOut o = resolve(outs[oi], A);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      mv_terms_regs(terms, o.t0, o.t1, o.m, acc, A);
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int i = 32 * g + lane;
        if (i < o.m) o.y[i] = (o.beta ? o.y[i] : 0.0) + acc[g];
      }
    }
    __syncthreads();
  }
}

// Term-heavy batches with m > 128: a CTA per chunk of 8 terms (one per warp).
__global__ void __launch_bounds__(kMvThreads, 2) mv_chunk_kernel(const MvOut* __restrict__ outs,
                                                                 const MvChunk* __restrict__ chunks,
                                                                 const MvTerm* __restrict__ terms, double* part,
                                                                 int ldacc, const MvCall A) {
  extern __shared__ double acc[];
  const MvChunk ch = chunks[blockIdx.x];
  const int m = outs[ch.out].m;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* mine = acc + warp * ldacc;
  for (int i = threadIdx.x & 31; i < m; i += 32) mine[i] = 0.0;
  __syncwarp();
  for (int ti = ch.t0 + warp; ti < ch.t1; ti += nw) mv_term_warp(resolve(terms[ti], A), m, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += acc[w * ldacc + i];
    part[ch.poff + i] = s;
  }
}

__global__ void mv_reduce_kernel(const MvOut* __restrict__ outs, const int* __restrict__ cptr,
                                 const MvChunk* __restrict__ chunks, const double* __restrict__ part,
                                 const MvCall A) {
  const MvOut o = resolve(outs[blockIdx.x], A);
  const int c0 = cptr[blockIdx.x], c1 = cptr[blockIdx.x + 1];
  for (int i = threadIdx.x; i < o.m; i += blockDim.x) {
    double s = 0.0;
    for (int c = c0; c < c1; ++c) s += part[chunks[c].poff + i];
    o.y[i] = (o.beta ? o.y[i] : 0.0) + s;
  }
}

// ------------------------------------------------------------------------------------------------
// Launch plans.  h2_matvec builds, once per matrix and orientation, every stage's descriptors (outs,
// terms, chunks, reduce lists) into one host buffer, uploads it, and records the launches; a call
// replays them with its x, y, alpha and accumulate flag -- ~20 launches of host work per call
// instead of walking every block and re-staging ~100k descriptors (3.4 ms of host time per c4 Z v).
struct MvLaunch {
  int kind;  // 0 warp chunks (+ reduce), 1 fused levels, 2 CTA per output, 3 CTA chunks (+ reduce),
             // 4 fork (the nearfield stream waits for the main stream), 5 join (the reverse)
  int ns;    // on the nearfield stream
  size_t o = 0, t = 0, c = 0, r = 0;  // byte offsets of outs, terms, chunks, reduce / level lists
  int grid = 0, grid2 = 0, ldacc = 0, nlev = 0;
  size_t smem = 0;
  long long part = -1;  // offset of the partial sums (doubles), -1: none
  double bytes = 0.0, flops = 0.0;
};

struct MvPlan {
  std::vector<char> host;
  std::vector<MvLaunch> launches;
  ArenaPtr mem;
  char* dev = nullptr;
  double* part = nullptr;
  long long part_n = 0;
  // what the descriptors point into (a different matrix state means a new plan)
  const void* f[6] = {};
  size_t fn[2] = {};
  bool fdist = false;
  size_t put(const void* p, size_t bytes) {
    const size_t off = host.size();
    host.resize(off + ((bytes + 255) & ~size_t(255)));
    if (bytes) memcpy(host.data() + off, p, bytes);
    return off;
  }
  template <class T> size_t put(const std::vector<T>& v) { return put(v.data(), v.size() * sizeof(T)); }
};

namespace {

void fingerprint(const H2& h, const void* (&f)[6], size_t (&fn)[2], bool& dist) {
  f[0] = h.coup.data();
  f[1] = h.near.data();
  f[2] = h.rb.get();
  f[3] = h.cb.get();
  f[4] = h.rb ? (const void*)h.rb->leaf.data() : nullptr;
  f[5] = h.cb ? (const void*)h.cb->leaf.data() : nullptr;
  fn[0] = h.coup.size();
  fn[1] = h.near.size();
  dist = h.dist_rows;
}

// one batch of outputs and their terms, recorded into a plan
struct MvBatch {
  MvPlan* P = nullptr;
  std::vector<MvOut> outs;
  std::vector<MvTerm> terms;
  std::vector<int> lvl;  // first output of each fused level (run_levels)
  double bytes_a = 0.0, bytes_x = 0.0;  // matrix / vector bytes read (profile ledger)
  void level() { lvl.push_back((int)outs.size()); }
  void out(double* y, int m, int beta) {
    outs.push_back(MvOut{y, m, (int)terms.size(), (int)terms.size(), beta});
  }
  void term(MatRef a, const double* x, int k, bool call_alpha, double elems) {
    terms.push_back(MvTerm{a, x, k, call_alpha ? 1 : 0, 1.0});
    outs.back().t1 = (int)terms.size();
    bytes_a += 8.0 * elems;
    bytes_x += 8.0 * k;
  }
  void clear() {
    outs.clear();
    terms.clear();
    lvl.clear();
    bytes_a = bytes_x = 0.0;
  }
  void run(bool ns = false);
  void run_levels();  // several dependent levels (boundaries in lvl) in one launch
};

void MvBatch::run(bool ns) {
  if (outs.empty()) return;
  int mmax = 1;
  for (const MvOut& o : outs) mmax = std::max(mmax, o.m);
  MvLaunch L;
  L.ns = ns ? 1 : 0;
  L.ldacc = mmax | 1;
  L.smem = sizeof(double) * L.ldacc * (kMvThreads / 32);
  L.bytes = bytes_a + bytes_x;
  L.flops = 2.0 * bytes_a / 8.0;
  static constexpr int kChunkTerms = 8;  // one term per warp
  if (mmax > 128 && (long long)terms.size() > 4LL * (long long)outs.size() && terms.size() > 1024) {
    // term-heavy, large rows: spread each output over ceil(terms / 8) CTAs
    std::vector<MvChunk> ch;
    std::vector<int> cptr{0};
    long long poff = P->part_n;
    for (int oi = 0; oi < (int)outs.size(); ++oi) {
      const MvOut& o = outs[oi];
      for (int t = o.t0; t < o.t1 || t == o.t0; t += kChunkTerms) {
        ch.push_back(MvChunk{oi, t, std::min(o.t1, t + kChunkTerms), 0, poff - P->part_n});
        poff += o.m;
        if (o.t1 == o.t0) break;
      }
      cptr.push_back((int)ch.size());
    }
    L.kind = 3;
    L.part = P->part_n;
    P->part_n = poff;
    L.o = P->put(outs);
    L.t = P->put(terms);
    L.c = P->put(ch);
    L.r = P->put(cptr);
    L.grid = (int)ch.size();
    L.grid2 = (int)outs.size();
  } else if (mmax <= 128) {
    // warp chunks: about kTargetWarps of them (two resident CTAs per SM, twice over), an output's
    // terms split into chunks of at most tpc (one- and two-term outputs, the transform levels, are
    // never split); single-chunk outputs write y directly
    static constexpr long long kTargetWarps = 148LL * 16 * 2;
    const long long nt = (long long)terms.size();
    const int tpc = (int)std::max<long long>(2, (nt + kTargetWarps - 1) / kTargetWarps);
    std::vector<MvChunk> ch;
    std::vector<int4> red;
    long long poff = 0;
    for (int oi = 0; oi < (int)outs.size(); ++oi) {
      const MvOut& o = outs[oi];
      if (o.t1 - o.t0 <= tpc) {
        ch.push_back(MvChunk{oi, o.t0, o.t1, 0, -1});
        continue;
      }
      const int c0 = (int)ch.size();
      for (int t = o.t0; t < o.t1; t += tpc) {
        ch.push_back(MvChunk{oi, t, std::min(o.t1, t + tpc), 0, poff});
        poff += o.m;
      }
      red.push_back(make_int4(oi, c0, (int)ch.size(), 0));
    }
    L.kind = 0;
    if (poff > 0) {
      L.part = P->part_n;
      P->part_n += poff;
    }
    L.o = P->put(outs);
    L.t = P->put(terms);
    L.c = P->put(ch);
    L.r = P->put(red);
    L.grid = (int)ch.size();
    L.grid2 = (int)red.size();
  } else {
    L.kind = 2;
    L.o = P->put(outs);
    L.t = P->put(terms);
    L.grid = (int)outs.size();
  }
  P->launches.push_back(L);
  clear();
}

void MvBatch::run_levels() {
  if (outs.empty()) {
    lvl.clear();
    return;
  }
  int mmax = 1;
  for (const MvOut& o : outs) mmax = std::max(mmax, o.m);
  if (mmax > 128) {  // not expected for transfer levels; one launch per level instead
    std::vector<MvOut> ao;
    std::vector<MvTerm> at;
    std::vector<int> lv;
    ao.swap(outs);
    at.swap(terms);
    lv.swap(lvl);
    lv.push_back((int)ao.size());
    const double ba = bytes_a, bx = bytes_x;
    for (size_t l = 0; l + 1 < lv.size(); ++l) {
      for (int oi = lv[l]; oi < lv[l + 1]; ++oi) {
        const MvOut& o = ao[oi];
        outs.push_back(MvOut{o.y, o.m, (int)terms.size(), (int)terms.size(), o.beta});
        for (int ti = o.t0; ti < o.t1; ++ti) terms.push_back(at[ti]);
        outs.back().t1 = (int)terms.size();
      }
      bytes_a = l == 0 ? ba : 0.0;
      bytes_x = l == 0 ? bx : 0.0;
      run();
    }
    return;
  }
  std::vector<int> lp = lvl;
  lp.push_back((int)outs.size());
  MvLaunch L;
  L.kind = 1;
  L.ns = 0;
  L.bytes = bytes_a + bytes_x;
  L.flops = 2.0 * bytes_a / 8.0;
  L.o = P->put(outs);
  L.t = P->put(terms);
  L.r = P->put(lp);
  L.nlev = (int)lvl.size();
  P->launches.push_back(L);
  clear();
}

std::shared_ptr<MvPlan> build_plan(Ctx& C, HView g) {
  auto P = std::make_shared<MvPlan>();
  fingerprint(*g.h, P->f, P->fn, P->fdist);
  const Tree& rt = g.rows();
  const Tree& ct = g.cols();
  const Basis& RB = g.rb();
  const Basis& CB = g.cb();
  const BView bv = g.bv();
  const Blocks& B = *g.h->bt;
  P->mem = std::make_shared<Arena>(C.st);
  std::vector<long long> xo(ct.n), yo(rt.n);
  long long nx = 0, ny = 0;
  for (int s = 0; s < ct.n; ++s) { xo[s] = nx; nx += CB.rank[s]; }
  for (int t = 0; t < rt.n; ++t) { yo[t] = ny; ny += RB.rank[t]; }
  double* xh = P->mem->alloc(std::max<long long>(1, nx));
  double* yh = P->mem->alloc(std::max<long long>(1, ny));
  MvBatch mb;
  mb.P = P.get();
  // nearfield first, on the second stream (h2.py:244-251): y|t (+)= alpha sum N_b x|s for every leaf
  // row (a leaf without dense blocks is zeroed unless accumulating); dense blocks on inner row
  // clusters (rare) follow in one launch per level, on the same stream, so that outputs never overlap
  P->launches.push_back(MvLaunch{4, 1});
  std::vector<std::vector<int>> near_by_row(rt.n);
  for (int b = 0; b < B.nb; ++b)
    if (B.near_leaf(b)) near_by_row[bv.row(b)].push_back(b);
  auto near_terms = [&](int t) {
    for (int b : near_by_row[t]) {
      const int s = bv.col(b);
      mb.term(g.near(b), tag_x(ct.start[s]), ct.size(s), true, (double)rt.size(t) * ct.size(s));
    }
  };
  for (int t = 0; t < rt.n; ++t) {
    if (!rt.leaf(t)) continue;
    mb.out(tag_y(rt.start[t]), rt.size(t), 2);
    near_terms(t);
  }
  mb.run(true);
  for (int lev = 0; lev <= rt.depth; ++lev) {
    for (int t : rt.by_level[lev]) {
      if (rt.leaf(t) || near_by_row[t].empty()) continue;
      mb.out(tag_y(rt.start[t]), rt.size(t), 1);
      near_terms(t);
    }
    mb.run(true);
  }
  // forward transform, bottom-up (h2.py:197-210); levels with at most kFuse clusters (the upper
  // tree) go into one mv_levels_kernel launch
  static constexpr int kFuse = 32;
  for (int lev = ct.depth; lev >= 0; --lev) {
    const bool fuse = (int)ct.by_level[lev].size() <= kFuse;
    if (fuse) mb.level();
    else if (!mb.lvl.empty()) mb.run_levels();  // fused levels below a large one (unbalanced trees)
    for (int s : ct.by_level[lev]) {
      const int k = CB.rank[s];
      if (k == 0) continue;
      mb.out(xh + xo[s], k, 0);
      if (ct.leaf(s)) {
        mb.term(CB.leafm(s).tref(), tag_x(ct.start[s]), ct.size(s), false, (double)ct.size(s) * k);
      } else {
        for (int i = 0; i < ct.nkids(s); ++i) {
          const int c = ct.kid(s, i);
          if (CB.rank[c] > 0) mb.term(CB.xferm(c).tref(), xh + xo[c], CB.rank[c], false, (double)CB.rank[c] * k);
        }
      }
    }
    if (!fuse) mb.run();
  }
  mb.run_levels();
  // coupling accumulation (h2.py:229-231)
  {
    std::vector<std::vector<int>> by_row(rt.n);
    for (int b = 0; b < B.nb; ++b)
      if (B.adm_leaf(b)) by_row[bv.row(b)].push_back(b);
    for (int t = 0; t < rt.n; ++t) {
      const int k = RB.rank[t];
      if (k == 0) continue;
      mb.out(yh + yo[t], k, 0);
      for (int b : by_row[t]) {
        const int s = bv.col(b);
        if (CB.rank[s] > 0) mb.term(g.coup(b), xh + xo[s], CB.rank[s], false, (double)k * CB.rank[s]);
      }
    }
    mb.run();
  }
  // backward transform, top-down (h2.py:213-221); the fused upper levels precede the first large one
  for (int lev = 1; lev <= rt.depth; ++lev) {
    const bool fuse = (int)rt.by_level[lev].size() <= kFuse;
    if (!fuse) mb.run_levels();
    else mb.level();
    for (int t : rt.by_level[lev]) {
      const int p = rt.parent[t];
      if (RB.rank[t] == 0 || RB.rank[p] == 0) continue;
      mb.out(yh + yo[t], RB.rank[t], 1);
      mb.term(RB.xferm(t).ref(), yh + yo[p], RB.rank[p], false, (double)RB.rank[t] * RB.rank[p]);
    }
    if (!fuse) mb.run();
  }
  mb.run_levels();
  // join the nearfield stream, then y|t += alpha V_t yhat_t on the leaves (h2.py:240-243)
  P->launches.push_back(MvLaunch{5, 0});
  for (int t = 0; t < rt.n; ++t) {
    if (!rt.leaf(t) || RB.rank[t] == 0) continue;
    mb.out(tag_y(rt.start[t]), rt.size(t), 1);
    mb.term(RB.leafm(t).ref(), yh + yo[t], RB.rank[t], true, (double)rt.size(t) * RB.rank[t]);
  }
  mb.run();
  // upload once (synchronously: a plan may be replayed from another context's stream)
  P->dev = (char*)P->mem->alloc_bytes(std::max<size_t>(256, P->host.size()));
  if (P->part_n > 0) P->part = P->mem->alloc(P->part_n);
  cuda_check(cudaMemcpyAsync(P->dev, P->host.data(), P->host.size(), cudaMemcpyHostToDevice, C.st), "plan upload");
  cuda_check(cudaStreamSynchronize(C.st), "plan upload");
  P->host.clear();
  P->host.shrink_to_fit();
  return P;
}

void replay(Ctx& C, const MvPlan& P, const MvCall& A) {
  const cudaStream_t ns = C.prof ? C.st : C.mv_stream();
  auto evwait = [](cudaStream_t from, cudaStream_t to) {
    if (from == to) return;
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(e, from), "event record");
    cuda_check(cudaStreamWaitEvent(to, e, 0), "stream wait");
    cudaEventDestroy(e);
  };
  for (const MvLaunch& L : P.launches) {
    if (L.kind == 4) { evwait(C.st, ns); continue; }
    if (L.kind == 5) { evwait(ns, C.st); continue; }
    const cudaStream_t s = L.ns ? ns : C.st;
    const MvOut* d_o = (const MvOut*)(P.dev + L.o);
    const MvTerm* d_t = (const MvTerm*)(P.dev + L.t);
    double* part = L.part >= 0 ? P.part + L.part : nullptr;
    cudaEvent_t ev = C.prof_begin();
    if (L.kind == 0) {
      const MvChunk* d_c = (const MvChunk*)(P.dev + L.c);
      const int wpc = kMvThreads / 32;
      mv_warp_kernel<<<(unsigned)((L.grid + wpc - 1) / wpc), kMvThreads, 0, s>>>(d_o, d_c, d_t, part, L.grid, A);
      cuda_check(cudaGetLastError(), "mv_warp_kernel");
      ++C.launches;
      if (L.grid2 > 0) {
        mv_wreduce_kernel<<<(unsigned)L.grid2, 128, 0, s>>>(d_o, (const int4*)(P.dev + L.r), d_c, part, A);
        cuda_check(cudaGetLastError(), "mv_wreduce_kernel");
        ++C.launches;
      }
    } else if (L.kind == 1) {
      mv_levels_kernel<<<1, kLvThreads, 0, s>>>(d_o, d_t, (const int*)(P.dev + L.r), L.nlev, A);
      cuda_check(cudaGetLastError(), "mv_levels_kernel");
      ++C.launches;
    } else if (L.kind == 2) {
      mv_kernel<<<(unsigned)L.grid, kMvThreads, L.smem, s>>>(d_o, d_t, L.ldacc, A);
      cuda_check(cudaGetLastError(), "mv_kernel");
      ++C.launches;
    } else {
      const MvChunk* d_c = (const MvChunk*)(P.dev + L.c);
      mv_chunk_kernel<<<(unsigned)L.grid, kMvThreads, L.smem, s>>>(d_o, d_c, d_t, part, L.ldacc, A);
      cuda_check(cudaGetLastError(), "mv_chunk_kernel");
      mv_reduce_kernel<<<(unsigned)L.grid2, 128, 0, s>>>(d_o, (const int*)(P.dev + L.r), d_c, part, A);
      cuda_check(cudaGetLastError(), "mv_reduce_kernel");
      C.launches += 2;
    }
    C.prof_end(K_MV, ev, L.flops, L.bytes);
  }
}

}  // namespace

// y (+)= alpha * G x on the view g (rows x cols); x, y device vectors.
void h2_matvec(Ctx& C, HView g, const double* x, double* y, double alpha, bool accumulate) {
  wait_near(C, *g.h);
  std::shared_ptr<MvPlan>& slot = g.h->mv_plan[g.T ? 1 : 0];
  if (slot) {
    const void* f[6];
    size_t fn[2];
    bool dist;
    fingerprint(*g.h, f, fn, dist);
    if (!std::equal(f, f + 6, slot->f) || fn[0] != slot->fn[0] || fn[1] != slot->fn[1] || dist != slot->fdist)
      slot.reset();
  }
  if (!slot) {
    static const bool dbg = getenv("H2G_DEBUG_MV") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    slot = build_plan(C, g);
    if (dbg)
      fprintf(stderr, "h2g: matvec plan (%s) built in %.2f ms, %zu launches\n", g.T ? "adjoint" : "plain",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
              slot->launches.size());
  }
  replay(C, *slot, MvCall{x, y, alpha, accumulate ? 1 : 0});
}

}  // namespace h2g
