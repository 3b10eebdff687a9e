// Descriptor types shared by the host planner (engine.cu) and the batched kernels (kernels.cu).
// All numerics are FP64, row-major unless a MatRef says otherwise (reference dense.py:3-4).
#pragma once
#include <cstdint>

namespace h2g {

// Strided view of a matrix: element (i, j) lives at p[i * rs + j * cs].
// A transposed view is the same pointer with rs/cs swapped.
struct MatRef {
  const double* p;
  int rs;
  int cs;
};

// One product term accumulated into a GOut:  C += alpha * op
//   nf = 1: A (m x n)
//   nf = 2: A (m x k) * B (k x n)
//   nf = 3: (A (m x k) * B (k x k2)) * D (k2 x n)
struct GTerm {
  MatRef a, b, d;
  int k, k2, nf;
  int pad_;
  double alpha;
};

// One output matrix: C (m x n, row-major, ldc) = (beta ? C : 0) + sum_{t0 <= i < t1} term_i
// Grouped 3-factor terms (product assembly, reference induced.py:286-307 regrouped):
//   nf = 4: T (m x ka) += alpha * A B, consecutive terms, flushed once as C += T * da
//   nf = 5: U (kb x n) += alpha * A B, consecutive terms, flushed once as C += ab * U
// (the kind-a terms of one target share their right factor, the kind-b terms their left one).
struct GOut {
  double* c;
  int ldc, m, n, beta;
  int t0, t1;
  int ka = 0, kb = 0;
  MatRef da = {nullptr, 0, 0};
  MatRef ab = {nullptr, 0, 0};
};

// One 64 x 64 output tile of a GOut.
struct GTile {
  int out;
  int tij;  // ti | (tj << 16)
};

// One tile of a GOut for the lean 2-factor kernel (gemm_lean.cu): origin and warp arrangement
// (lay 0: 2 x 2 warps = 32 x 64, 1: 4 x 1 = 64 x 32, 2: 1 x 4 = 16 x 128; a warp owns 16 x 32).
struct GLTile {
  int out;
  int i0, j0;
  int lay;
};

// Segment of a stacked operand.  hstack: a is (m x w); vstack: a is (w x n).  Scaled by `scale`.
struct Seg {
  MatRef a;
  int w;
  int pad_;
  double scale;
  long long off;       // first stacked line of this segment within its item
  const double* sdiv;  // optional device scalar: the segment is divided by *sdiv when *sdiv > 0
};

// R-only QR of vstack(segs[s0:s1]) (M x n); writes min(M, n) x n rows (ld n) to out.
struct QrItem {
  int s0, s1, n, nchunk;  // nchunk row chunks (>= 1), each reduced by its own CTA
  long long M;
  double* out;
  double* rbuf;  // nchunk x (n x n) partial R factors
  int full;      // 1: rbuf holds a pivoted (Gram) factor, copied whole (not only its upper triangle)
  int pad_;
};

// Tree merge of two partial R factors: rbuf[a] <- R([rbuf[a]; rbuf[b]]) (n x n each).
struct MergeWork {
  double* rbuf;
  int n, a, b, pad_;
};

// Truncated SVD of hstack(segs[s0:s1]) (m x N), optionally protecting range(V) (m x kx)
// first (Fig. 3 of the paper, reference induced.py:127-137):
//   k1 = min(m, kx); B = (Q_V^T A)[k1:]; U, k2 = trunc_svd(B, tol, cap)
//   q_out  (m x (k1 + k2), ld k1 + k2) = Q_V [[I, 0], [0, U]]
//   bc_out ((k1 + k2) x kx, ld kx)    = [R_V[:k1]; 0]
// Without V (kx = 0): q_out = U (m x k2), the reference's truncated_svd(A).u (dense.py:77-101).
// Rank rule: thr = max(tol, max(rows(B), N) * eps * sigma_1); k2 = #{sigma > thr}, min(k2, cap).
struct SvdItem {
  int s0, s1, m, kx;
  long long N;
  MatRef v;
  double tol;
  int cap;  // < 0: no cap
  int nchunk;  // column chunks of the streamed TSQR (>= 1)
  double* q_out;
  double* bc_out;
  int* rank_out;    // k1 + k2
  double* sig_out;  // optional: sorted singular values of B (capacity m)
  double* rbuf;     // nchunk x (n x n) partial R factors, n = m - min(m, kx)
  double* vws;      // m x kx Householder vectors of V + kx coefficients
  int* sweeps_out;  // optional diagnostic: Jacobi sweeps used, n, live rows, k2
  int zskip;        // 1: segments whose device divisor is exactly 0 are absent (their widths leave N)
  double* q2;       // tile path with kx > 0: explicit Q_V (m x m), written by svd_prep_kernel
  double* gpart;    // Gram path (kx = 0): nchunk x {hi, lo} x (m x m) partial double-double Grams
  int* pre_nr;      // Gram path: rows of the pivoted-Cholesky factor in rbuf (the finish skips QRCP)
  double* u_out;    // deferred output (kx > 0, n > 0, q2 set): the finish writes U (n x k2, ld n) and
                    // the host forms Q_t = [Q_V[:, :k1] | Q_V[:, k1:] U] as one batched GEMM afterwards
};

// Gram CTAs of a small item (m <= 64, one 64 x 64 tile) run `reps` replicas of its 4 x 4 block set
// over interleaved panel columns, each replica writing its own partial slice.
__host__ __device__ inline int gram_reps(int m) {
  if (m > 64) return 1;
  const int nb = (m + 3) / 4, nblk = nb * (nb + 1) / 2, span = (nblk + 31) / 32 * 32;
  const int r = 256 / span;
  return r > 1 ? r : 1;
}

// Double-double Gram + pivoted Cholesky item (gram.cu): the lines of hstack(segs) (hcols = 1: the
// columns of an m-row wide matrix) or of vstack(segs) (hcols = 0: the rows of an N x m stack).
struct GramItem {
  int s0, s1, m, nslice;  // nslice partial slices (column chunks x replicas)
  long long N;            // lines
  int hcols, pad_;
  double tol;             // truncation tolerance of the SVD that follows (0: factorisation only)
  double* gpart;          // nslice x {hi, lo} x (m x m)
  double* rbuf;           // m x m factor (rows = pivot steps, columns in original order)
  int* nr;                // rows of the factor
};

// One CTA of the double-double Gram (gram.cu): columns [c0, c1) of item `item`, G tile (ti, tj); for
// m <= kGramFlatMax, ti = first 4 x 4 block (row-major upper triangle) and tj = blocks | reps << 16.
constexpr int kGramFlatMax = 128;
constexpr int kGramFlatThreads = 192;  // CTA size of the flat path (528 blocks of m = 128: 3 x 176)
struct GramWork {
  int item, ti, tj, chunk;
  long long c0, c1;
};

// Register-tile TSQR (tileqr.cu): one item = one stacked operand reduced to an n x n R factor
// (n <= 128).  Lines are rows of vstack(segs) (hcols = 0) or columns of hstack(segs)
// (hcols = 1); each line contributes kdim source entries, projected onto q2 (kdim x n) if given.
struct TileItem {
  int s0, s1, n, kdim, hcols, q2ld;
  const double* q2;  // kdim x n, leading dimension q2ld
};

// One CTA: absorb lines [l0, l1) (128 per tile) into R (starting from rinit, else zero) and
// write R to rout; with rsrc the single tile is the n x n factor rsrc (tree merge).
struct TileWork {
  int item, pad_;
  long long l0, l1;
  const double* rinit;
  const double* rsrc;
  double* rout;
};

// Work units of the SVD pipeline: stage-1 chunk (item, chunk) and tree merges R_a <- [R_a; R_b].
struct SvdWork {
  int item, a, b, pad_;
};

// sigma_1 of hstack(segs[s0:s1]) (m x N) (reference dense.py:104-142).
struct NormItem {
  int s0, s1, m, pad_;
  long long N;
  double* out;
  double* gbuf;  // optional global scratch for the Gram matrix (large items); null: shared memory
};

// Device-side expansion of the product assembly (reference induced.py:286-307): one GTerm per
// terminal triple (node, middle s, kind), operands looked up in per-block / per-cluster tables.
struct AsmTables {
  // per triple
  const int* tnode;
  const int* ts;
  const char* tk;
  const int* tbx;
  const int* tby;
  // per product node
  const int* node_row;
  const int* node_col;
  const unsigned char* node_dense;
  // per X block (row view): coupling, nearfield, admissible-leaf flag, row factor, projection, X|ts V_Y,s
  const MatRef* xcoup;
  const MatRef* xnear;
  const unsigned char* xadm;
  const MatRef* rf;
  const MatRef* rproj;
  const MatRef* xv;
  // per Y block: coupling, nearfield, column projection, Y|sr^T W_X,s
  const MatRef* ycoup;
  const MatRef* ynear;
  const MatRef* cproj;
  const MatRef* wyl;
  // per cluster
  const MatRef* vxleaf;  // row tree: V_X leaf
  const MatRef* bcr;     // row tree: induced basis change
  const MatRef* wyleaf;  // column tree: W_Y leaf
  const MatRef* bcc;     // column tree: induced basis change
  const int* kx_row;     // rank of V_X per row cluster
  const int* kwx_mid;    // rank of W_X per middle cluster
  const int* ky_mid;     // rank of V_Y per middle cluster
  const int* kwy_col;    // rank of W_Y per column cluster
  const int* size_mid;   // middle cluster sizes
  int grouped;           // emit nf = 4 / 5 group terms where the shared factor has rank <= 64
  int only;              // 0: every triple; 1: dense targets only; 2: coupling targets only
                         // (the other triples become nf = 0 no-op terms; their tables are not read)
};

}  // namespace h2g
