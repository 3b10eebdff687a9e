// Input construction on the GPU: kernel evaluation for the coupling matrices
// (kernel at the clusters' Chebyshev grids) and the nearfield blocks (kernel at the points times
// the quadrature weights) of an interpolation H^2 matrix (reference problems.py:295-332).  These
// are the O(n) and O(n k^2) bulk of the input (c4: ~3.2 GB of nearfield); the interpolation bases
// (Lagrange products, problems.py:225-266) are small and come from the host.
//
// Arithmetic follows the host builder (paper_2309_09061_b200/problems.py `_kernel`): r is the
// Euclidean norm summed in axis order without fused multiply-adds, g(0) = 0, value g(r) * (w_i w_j).
#include <cuda_runtime.h>

#include <algorithm>

#include "engine.h"

namespace h2g {

namespace {

struct EvalBlock {
  const double* xr;  // row points (nr x dim)
  const double* xc;  // column points (nc x dim)
  const double* wr;  // optional row weights
  const double* wc;  // optional column weights
  double* out;       // nr x nc row-major
  int nr, nc;
};

__device__ __forceinline__ double kernel_value(int kind, double r) {
  if (!(r > 0.0)) return 0.0;
  switch (kind) {
    case 0: return -log(r);                                   // -log|x - y|
    case 1: return 1.0 / __dmul_rn(12.566370614359172, r);    // 1 / (4 pi |x - y|)
    case 2: return 1.0 / r;                                   // 1 / |x - y|
    default: return exp(-r) / r;                              // exp(-|x - y|) / |x - y|
  }
}

__global__ void eval_blocks_kernel(const EvalBlock* __restrict__ blocks, int kind, int dim) {
  const EvalBlock b = blocks[blockIdx.x];
  const long long tot = (long long)b.nr * b.nc;
  for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
    const int i = (int)(e / b.nc), j = (int)(e % b.nc);
    double s = 0.0;
    for (int a = 0; a < dim; ++a) {
      const double d = __dadd_rn(b.xr[i * dim + a], -b.xc[j * dim + a]);
      s = __dadd_rn(s, __dmul_rn(d, d));
    }
    double v = kernel_value(kind, sqrt(s));
    if (b.wr) v = __dmul_rn(v, __dmul_rn(b.wr[i], b.wc[j]));
    b.out[e] = v;
  }
}

}  // namespace

std::shared_ptr<H2> build_kernel_h2(Ctx& C, std::shared_ptr<const Blocks> bt, int kind, int dim,
                                    const double* points, const double* weights, const long long* rank,
                                    const long long* loff, const long long* xoff, const double* basis,
                                    long long basis_len, const long long* node_off, const double* nodes,
                                    long long nodes_len) {
  if (kind < 0 || kind > 3) throw InvalidInput("unknown kernel id");
  if (dim < 1 || dim > 3) throw InvalidInput("dimension must be 1, 2 or 3");
  const Blocks& B = *bt;
  const Tree& tr = *B.rows;
  if (!B.rows->same(*B.cols)) throw InvalidInput("kernel builder needs identical row and column trees");
  const long long n = tr.stop[0] - tr.start[0];
  auto h = std::make_shared<H2>();
  auto ar = std::make_shared<Arena>(C.st);
  h->owned.push_back(ar);
  h->bt = bt;
  // interpolation basis (shared by rows and columns)
  auto Bs = std::make_shared<Basis>();
  Bs->tree = &tr;
  Bs->rank.assign(rank, rank + tr.n);
  Bs->leaf.assign(tr.n, nullptr);
  Bs->xfer.assign(tr.n, nullptr);
  double* dbasis = ar->alloc(std::max<long long>(1, basis_len));
  if (basis_len > 0)
    cuda_check(cudaMemcpyAsync(dbasis, basis, basis_len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  for (int t = 0; t < tr.n; ++t) {
    if (tr.leaf(t)) {
      if (loff[t] < 0 || loff[t] + (long long)tr.size(t) * rank[t] > basis_len) throw InvalidInput("leaf out of range");
      Bs->leaf[t] = dbasis + loff[t];
    }
    if (tr.parent[t] >= 0) {
      if (xoff[t] < 0 || xoff[t] + rank[t] * rank[tr.parent[t]] > basis_len) throw InvalidInput("transfer out of range");
      Bs->xfer[t] = dbasis + xoff[t];
    }
  }
  h->rb = h->cb = Bs;
  // points, weights, Chebyshev grids
  Arena sc(C.st);
  double* dpts = sc.alloc(std::max<long long>(1, n * dim));
  double* dw = sc.alloc(std::max<long long>(1, n));
  double* dnodes = sc.alloc(std::max<long long>(1, nodes_len));
  cuda_check(cudaMemcpyAsync(dpts, points, n * dim * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  cuda_check(cudaMemcpyAsync(dw, weights, n * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  if (nodes_len > 0)
    cuda_check(cudaMemcpyAsync(dnodes, nodes, nodes_len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  // storage and evaluation lists
  long long ncoup = 0, nnear = 0;
  for (int b = 0; b < B.nb; ++b) {
    if (!B.leaf(b)) continue;
    const int t = B.row[b], s = B.col[b];
    if (B.adm[b]) ncoup += rank[t] * rank[s];
    else nnear += (long long)tr.size(t) * tr.size(s);
  }
  double* dc = ar->alloc(std::max<long long>(1, ncoup));
  double* dn = ar->alloc(std::max<long long>(1, nnear));
  h->coup.assign(B.nb, nullptr);
  h->near.assign(B.nb, nullptr);
  std::vector<EvalBlock> ev;
  long long oc = 0, on = 0;
  for (int b = 0; b < B.nb; ++b) {
    if (!B.leaf(b)) continue;
    const int t = B.row[b], s = B.col[b];
    if (B.adm[b]) {  // S_ts = g(xi_t, xi_s) (problems.py:323-325)
      if (node_off[t] < 0 || node_off[s] < 0) throw InvalidInput("missing interpolation grid");
      h->coup[b] = dc + oc;
      ev.push_back(EvalBlock{dnodes + node_off[t], dnodes + node_off[s], nullptr, nullptr, dc + oc, (int)rank[t],
                             (int)rank[s]});
      oc += rank[t] * rank[s];
    } else {  // N_ts = g(x_i, x_j) w_i w_j (problems.py:326-330)
      h->near[b] = dn + on;
      ev.push_back(EvalBlock{dpts + tr.start[t] * dim, dpts + tr.start[s] * dim, dw + tr.start[t], dw + tr.start[s],
                             dn + on, tr.size(t), tr.size(s)});
      on += (long long)tr.size(t) * tr.size(s);
    }
  }
  if (!ev.empty()) {
    EvalBlock* d_ev = C.push(ev);
    C.flush();
    eval_blocks_kernel<<<(unsigned)ev.size(), 256, 0, C.st>>>(d_ev, kind, dim);
    cuda_check(cudaGetLastError(), "eval_blocks_kernel");
    ++C.launches;
  }
  C.sync();  // host inputs may be released by the caller after return
  return h;
}

}  // namespace h2g
