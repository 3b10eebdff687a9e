// Host engine: structure, staging, batch planning and the stage drivers of the adaptive H^2 product.
//
// Every stage walks the reference recursion (h2mul induced.py / coarsening.py / weights.py) level by
// level over the cluster tree and emits one batched launch per dependency level; the only host
// round trips are the ones the algorithm forces (exact zero-norm skips and the data-dependent ranks
// that size the next level).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>

#include "engine.h"

namespace h2g {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

// ============================================================================ infrastructure

Arena::~Arena() {
  for (void* p : chunks) cudaFreeAsync(p, st);
}

void* Arena::alloc_bytes(size_t nb) {
  nb = (nb + 255) & ~size_t(255);
  if (nb == 0) return nullptr;
  if (nb > left) {
    size_t chunk = std::max(nb, size_t(64) << 20);
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, chunk, st), "cudaMallocAsync");
    chunks.push_back(p);
    cur = (char*)p;
    left = chunk;
  }
  void* r = cur;
  cur += nb;
  left -= nb;
  bytes += nb;
  return r;
}

double* Arena::alloc(size_t n) { return (double*)alloc_bytes(n * sizeof(double)); }

Ctx::Ctx(int dev, cudaStream_t s) : device(dev), st(s) {
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  if (!st) {
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    own_stream = true;
  }
  stage_cap = size_t(64) << 20;
  cuda_check(cudaMallocHost(&hstage, stage_cap), "cudaMallocHost");
  cuda_check(cudaMalloc(&dstage, stage_cap), "cudaMalloc stage");
  ensure_read(1 << 20);
}

Ctx::~Ctx() {
  cudaStreamSynchronize(st);
  for (auto e : evpool) cudaEventDestroy(e);
  cudaFreeHost(hstage);
  cudaFree(dstage);
  if (hread) cudaFreeHost(hread);
  if (own_stream) cudaStreamDestroy(st);
}

void Ctx::ensure_read(size_t bytes) {
  if (bytes <= read_cap) return;
  if (hread) cudaFreeHost(hread);
  read_cap = std::max(bytes, read_cap * 2);
  cuda_check(cudaMallocHost(&hread, read_cap), "cudaMallocHost read");
}

void Ctx::sync() {
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  stage_off = 0;
  ++syncs;
}

void* Ctx::stage(const void* src, size_t bytes) {
  const size_t need = (bytes + 255) & ~size_t(255);
  if (stage_off + need > stage_cap) {
    sync();
    if (need > stage_cap) {
      cudaFreeHost(hstage);
      cudaFree(dstage);
      stage_cap = std::max(need, stage_cap * 2);
      cuda_check(cudaMallocHost(&hstage, stage_cap), "cudaMallocHost");
      cuda_check(cudaMalloc(&dstage, stage_cap), "cudaMalloc stage");
    }
  }
  char* h = hstage + stage_off;
  char* d = dstage + stage_off;
  memcpy(h, src, bytes);
  cuda_check(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st), "stage copy");
  stage_off += need;
  return d;
}

cudaEvent_t Ctx::event() {
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "event");
  evpool.push_back(e);
  return e;
}

void GBatch::t1(MatRef a, double al) {
  terms.push_back(GTerm{a, MatRef{nullptr, 0, 0}, MatRef{nullptr, 0, 0}, 0, 0, 1, 0, al});
  outs.back().t1 = (int)terms.size();
}

void GBatch::t2(MatRef a, MatRef b, int k, double al) {
  if (k == 0) return;
  terms.push_back(GTerm{a, b, MatRef{nullptr, 0, 0}, k, 0, 2, 0, al});
  outs.back().t1 = (int)terms.size();
}

void GBatch::t3(MatRef a, MatRef b, MatRef d, int k, int k2, double al) {
  if (k == 0 || k2 == 0) return;
  if (k2 > 256) throw StructureErr("gsum: 3-factor middle dimension above 256");
  terms.push_back(GTerm{a, b, d, k, k2, 3, 0, al});
  k2max = std::max(k2max, k2);
  outs.back().t1 = (int)terms.size();
}

void GBatch::run(Ctx& C) {
  std::vector<GTile> tiles;
  for (int i = 0; i < (int)outs.size(); ++i) {
    const GOut& o = outs[i];
    if (o.m <= 0 || o.n <= 0) continue;
    const int tm = (o.m + 63) / 64, tn = (o.n + 63) / 64;
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) tiles.push_back(GTile{i, a | (b << 16)});
  }
  if (tiles.empty()) return;
  GOut* d_o = C.push(outs);
  GTerm* d_t = C.push(terms);
  GTile* d_l = C.push(tiles);
  cuda_check(launch_gsum(d_o, d_t, d_l, (int)tiles.size(), k2max, C.st), "gsum");
  ++C.launches;
  outs.clear();
  terms.clear();
  k2max = 0;
}

static constexpr size_t kSmemLimit = 227 * 1024;

void QrBatch::run(Ctx& C, Arena& scratch) {
  std::vector<QrItem> small, big;
  int nsmall = 0, nbig = 0;
  for (auto& it : items) {
    if (it.n == 0 || it.M == 0) continue;
    if (qr_smem(it.n, false) <= kSmemLimit) {
      small.push_back(it);
      nsmall = std::max(nsmall, it.n);
    } else {
      it.ws = scratch.alloc((size_t)it.n * it.n);
      big.push_back(it);
      nbig = std::max(nbig, it.n);
    }
  }
  if (small.empty() && big.empty()) { items.clear(); sl.segs.clear(); return; }
  Seg* d_s = C.push(sl.segs);
  if (!small.empty()) {
    cuda_check(launch_qr(C.push(small), d_s, (int)small.size(), nsmall, false, C.st), "qr_r");
    ++C.launches;
  }
  if (!big.empty()) {
    cuda_check(launch_qr(C.push(big), d_s, (int)big.size(), nbig, true, C.st), "qr_r ws");
    ++C.launches;
  }
  items.clear();
  sl.segs.clear();
}

std::vector<double> NormBatch::run(Ctx& C, Arena& scratch) {
  std::vector<double> res(items.size(), 0.0);
  if (items.empty()) return res;
  double* d_out = scratch.alloc(items.size());
  size_t smem = 0;
  std::vector<NormItem> live;
  std::vector<int> where;
  for (size_t i = 0; i < items.size(); ++i) {
    items[i].out = d_out + i;
    if (items[i].m == 0 || items[i].N == 0) continue;
    const bool rowside = (items[i].m <= items[i].N) || (items[i].m <= 160);
    const long long g = rowside ? items[i].m : items[i].N;
    if (g > 180) throw StructureErr("spectral norm: both sides above 180");
    smem = std::max(smem, norm_smem(items[i].m, items[i].N));
    live.push_back(items[i]);
    where.push_back((int)i);
  }
  if (!live.empty()) {
    cuda_check(launch_norm(C.push(live), C.push(sl.segs), (int)live.size(), smem, C.st), "norm");
    ++C.launches;
    std::vector<double> vals = C.read(d_out, items.size());
    for (int w : where) res[w] = vals[w];
  }
  items.clear();
  sl.segs.clear();
  return res;
}

std::vector<int> SvdBatch::run(Ctx& C, Arena& scratch) {
  std::vector<int> ranks(items.size(), 0);
  if (items.empty()) return ranks;
  int* d_rank = (int*)scratch.alloc_bytes(items.size() * sizeof(int));
  cuda_check(cudaMemsetAsync(d_rank, 0, items.size() * sizeof(int), C.st), "memset");
  std::vector<SvdItem> small, big;
  size_t sm_small = 0, sm_big = 0;
  for (size_t i = 0; i < items.size(); ++i) {
    SvdItem& it = items[i];
    it.rank_out = d_rank + i;
    if (it.m == 0) continue;
    const int k1 = std::min(it.m, it.kx);
    const size_t s1 = svd_smem(it.m, it.kx, false);
    if (s1 <= kSmemLimit) {
      small.push_back(it);
      sm_small = std::max(sm_small, s1);
    } else {
      const size_t s2 = svd_smem(it.m, it.kx, true);
      if (s2 > kSmemLimit) throw StructureErr("svd: item too large for shared memory");
      const int n = it.m - k1;
      it.ws = scratch.alloc((size_t)n * n);
      big.push_back(it);
      sm_big = std::max(sm_big, s2);
    }
  }
  Seg* d_s = C.push(sl.segs);
  if (!small.empty()) {
    cuda_check(launch_svd(C.push(small), d_s, (int)small.size(), sm_small, C.st), "svd");
    ++C.launches;
  }
  if (!big.empty()) {
    cuda_check(launch_svd(C.push(big), d_s, (int)big.size(), sm_big, C.st), "svd ws");
    ++C.launches;
  }
  ranks = C.read(d_rank, items.size());
  items.clear();
  sl.segs.clear();
  return ranks;
}

// ============================================================================ structure

bool Tree::same(const Tree& o) const {
  return this == &o || (n == o.n && start == o.start && stop == o.stop && cptr == o.cptr && cidx == o.cidx);
}

void Tree::finalize() {
  parent.assign(n, -1);
  level.assign(n, 0);
  depth = 0;
  for (int t = 0; t < n; ++t)
    for (int i = cptr[t]; i < cptr[t + 1]; ++i) {
      const int c = cidx[i];
      if (c <= t || c >= n) throw InvalidInput("cluster tree is not in preorder");
      parent[c] = t;
      level[c] = level[t] + 1;
      depth = std::max(depth, level[c]);
    }
  by_level.assign(depth + 1, {});
  for (int t = 0; t < n; ++t) by_level[level[t]].push_back(t);
}

void Blocks::finalize() {
  parent.assign(nb, -1);
  level.assign(nb, 0);
  depth = 0;
  index.clear();
  index.reserve(nb * 2);
  for (int b = 0; b < nb; ++b) {
    index[(long long)row[b] * cols->n + col[b]] = b;
    for (int i = cptr[b]; i < cptr[b + 1]; ++i) {
      const int c = cidx[i];
      if (c <= b || c >= nb) throw InvalidInput("block tree is not in preorder");
      parent[c] = b;
      level[c] = level[b] + 1;
      depth = std::max(depth, level[c]);
    }
  }
  by_level.assign(depth + 1, {});
  for (int b = 0; b < nb; ++b) by_level[level[b]].push_back(b);
}

std::shared_ptr<Tree> make_tree(int n, const long long* start, const long long* stop, const long long* cptr,
                                const long long* cidx) {
  auto t = std::make_shared<Tree>();
  t->n = n;
  t->start.assign(start, start + n);
  t->stop.assign(stop, stop + n);
  t->cptr.assign(cptr, cptr + n + 1);
  t->cidx.assign(cidx, cidx + cptr[n]);
  t->finalize();
  return t;
}

std::shared_ptr<Blocks> make_blocks(const Tree* rows, const Tree* cols, int nb, const long long* row,
                                    const long long* col, const long long* cptr, const long long* cidx,
                                    const unsigned char* adm) {
  auto b = std::make_shared<Blocks>();
  b->rows = rows;
  b->cols = cols;
  b->nb = nb;
  b->row.assign(row, row + nb);
  b->col.assign(col, col + nb);
  b->cptr.assign(cptr, cptr + nb + 1);
  b->cidx.assign(cidx, cidx + cptr[nb]);
  b->adm.assign(adm, adm + nb);
  b->finalize();
  return b;
}

// Triple kind (reference trees.py:288-300): 'a' > 'b' > 'c' > 'n'.
static char classify(BView bx, BView by, int t, int s, int r, int* pts, int* psr) {
  const int bts = bx.find(t, s), bsr = by.find(s, r);
  if (bts < 0 || bsr < 0) throw StructureErr("triple not covered by the factor block trees");
  *pts = bts;
  *psr = bsr;
  if (by.b->adm_leaf(bsr)) return 'a';
  if (bx.b->adm_leaf(bts)) return 'b';
  if (by.b->leaf(bsr) && bx.b->leaf(bts)) return 'c';
  return 'n';
}

// Product block tree T^XY with the per-node terminal triples (trees.py:314-359, induced.py:280-326).
PTree product_tree(BView bx, BView by) {
  const Tree& rows = bx.rows();
  const Tree& mid = bx.cols();
  const Tree& cols = by.cols();
  if (!mid.same(by.rows())) throw InvalidInput("factors do not share the middle cluster tree");
  PTree P;
  auto bt = std::make_shared<Blocks>();
  bt->rows = &rows;
  bt->cols = &cols;
  std::vector<std::vector<int>> kids;
  struct Frame {
    int t, r, parent, slot;
    std::vector<int> mids;
  };
  std::vector<Frame> stack;
  stack.push_back(Frame{0, 0, -1, 0, {0}});
  std::vector<int> pend, open;
  while (!stack.empty()) {
    Frame f = std::move(stack.back());
    stack.pop_back();
    const int b = (int)bt->row.size();
    if (f.parent >= 0) kids[f.parent][f.slot] = b;
    bt->row.push_back(f.t);
    bt->col.push_back(f.r);
    bt->adm.push_back(1);
    kids.emplace_back();
    P.tptr.push_back((int)P.ts.size());
    const bool both_leaf = rows.leaf(f.t) && cols.leaf(f.r);
    pend = f.mids;
    open.clear();
    bool dense = false;
    while (!pend.empty()) {
      const int s = pend.back();
      pend.pop_back();
      int bts, bsr;
      const char k = classify(bx, by, f.t, s, f.r, &bts, &bsr);
      if (k == 'n') {
        if (both_leaf) {
          for (int i = 0; i < mid.nkids(s); ++i) pend.push_back(mid.kid(s, i));
        } else {
          open.push_back(s);
        }
        continue;
      }
      if (k == 'c') dense = true;
      P.ts.push_back(s);
      P.tk.push_back(k);
    }
    if (!open.empty()) {
      std::vector<int> subs;
      for (int s : open) {  // _sub_middles (trees.py:303-311)
        const int bts = bx.find(f.t, s), bsr = by.find(s, f.r);
        if (!bx.b->leaf(bts) && !by.b->leaf(bsr) && mid.nkids(s) > 0) {
          for (int i = 0; i < mid.nkids(s); ++i) subs.push_back(mid.kid(s, i));
        } else {
          subs.push_back(s);
        }
      }
      std::vector<std::pair<int, int>> pairs;
      const int nt = std::max(1, rows.nkids(f.t)), nr = std::max(1, cols.nkids(f.r));
      for (int i = 0; i < nt; ++i)
        for (int j = 0; j < nr; ++j)
          pairs.emplace_back(rows.nkids(f.t) ? rows.kid(f.t, i) : f.t, cols.nkids(f.r) ? cols.kid(f.r, j) : f.r);
      kids[b].assign(pairs.size(), -1);
      for (int i = (int)pairs.size() - 1; i >= 0; --i)
        stack.push_back(Frame{pairs[i].first, pairs[i].second, b, i, subs});
    } else if (dense) {
      bt->adm[b] = 0;
    }
  }
  P.tptr.push_back((int)P.ts.size());
  bt->nb = (int)bt->row.size();
  bt->cptr.assign(bt->nb + 1, 0);
  for (int b = 0; b < bt->nb; ++b) bt->cptr[b + 1] = bt->cptr[b] + (int)kids[b].size();
  for (int b = 0; b < bt->nb; ++b)
    for (int c : kids[b]) bt->cidx.push_back(c);
  bt->finalize();
  P.bt = bt;
  return P;
}

// ============================================================================ setup stages

// P_s = W_s^T V_s bottom-up (reference h2.py:127-145).
MatStore basis_product(Ctx& C, Arena& ar, const Basis& W, const Basis& V) {
  const Tree& tr = *W.tree;
  if (!tr.same(*V.tree)) throw InvalidInput("bases live on different cluster trees");
  MatStore P(tr.n);
  for (int s = 0; s < tr.n; ++s) P[s] = Mat{ar.alloc((size_t)W.rank[s] * V.rank[s]), W.rank[s], V.rank[s]};
  for (int lev = tr.depth; lev >= 0; --lev) {
    GBatch g;
    for (int s : tr.by_level[lev]) {
      g.out(P[s], false);
      if (tr.leaf(s)) {
        g.t2(W.leafm(s).tref(), V.leafm(s).ref(), tr.size(s));
      } else {
        for (int i = 0; i < tr.nkids(s); ++i) {
          const int c = tr.kid(s, i);
          g.t3(W.xferm(c).tref(), P[c].ref(), V.xferm(c).ref(), W.rank[c], V.rank[c]);
        }
      }
    }
    g.run(C);
  }
  return P;
}

// R_r of a bottom-up QR of the basis (reference weights.py:37-57).
MatStore basis_weights(Ctx& C, Arena& ar, const Basis& W) {
  const Tree& tr = *W.tree;
  MatStore R(tr.n);
  for (int lev = tr.depth; lev >= 0; --lev) {
    GBatch g;
    QrBatch q;
    for (int t : tr.by_level[lev]) {
      const int k = W.rank[t];
      QrItem it{};
      it.s0 = q.sl.begin();
      it.n = k;
      if (tr.leaf(t)) {
        q.sl.add(W.leafm(t).ref(), tr.size(t));
        it.M = tr.size(t);
      } else {
        long long M = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {
          const int c = tr.kid(t, i);
          Mat part{ar.alloc((size_t)R[c].r * k), R[c].r, k};
          g.out(part, false);
          g.t2(R[c].ref(), W.xferm(c).ref(), R[c].c);
          q.sl.add(part.ref(), part.r);
          M += part.r;
        }
        it.M = M;
      }
      it.s1 = q.sl.begin();
      const int rows = (int)std::min<long long>(it.M, k);
      R[t] = Mat{ar.alloc((size_t)rows * k), rows, k};
      it.out = R[t].p;
      q.items.push_back(it);
    }
    g.run(C);
    q.run(C, ar);
  }
  return R;
}

// Top-down condensed weights Z_s (reference weights.py:60-101).
MatStore total_weights(Ctx& C, Arena& ar, HView h, const MatStore& rw, bool scaling) {
  const Tree& tr = h.rows();
  const int nb = h.h->bt->nb;
  std::vector<std::vector<int>> adm_of(tr.n);
  for (int b = 0; b < nb; ++b)
    if (h.h->bt->adm_leaf(b)) adm_of[h.row(b)].push_back(b);
  // T_b = R_{col b} S_b^T and their norms
  std::vector<Mat> Tb(nb);
  GBatch g;
  NormBatch nbatch;
  std::vector<int> order;
  for (int t = 0; t < tr.n; ++t)
    for (int b : adm_of[t]) {
      const Mat& R = rw[h.col(b)];
      const int kr = h.rb().rank[t];
      Tb[b] = Mat{ar.alloc((size_t)R.r * kr), R.r, kr};
      g.out(Tb[b], false);
      g.t2(R.ref(), trn(h.coup(b)), R.c);
      if (scaling) {
        NormItem it{};
        it.s0 = nbatch.sl.begin();
        nbatch.sl.add(Tb[b].ref(), kr);
        it.s1 = nbatch.sl.begin();
        it.m = Tb[b].r;
        it.N = kr;
        nbatch.items.push_back(it);
        order.push_back(b);
      }
    }
  g.run(C);
  std::vector<double> nrm(nb, 1.0);
  if (scaling) {
    auto v = nbatch.run(C, ar);
    for (size_t i = 0; i < order.size(); ++i) nrm[order[i]] = v[i];
  }
  MatStore Z(tr.n);
  for (int lev = 0; lev <= tr.depth; ++lev) {
    GBatch ge;
    QrBatch q;
    for (int s : tr.by_level[lev]) {
      const int k = h.rb().rank[s];
      QrItem it{};
      it.s0 = q.sl.begin();
      it.n = k;
      long long M = 0;
      const int p = tr.parent[s];
      if (p >= 0 && Z[p].r > 0) {
        Mat ze{ar.alloc((size_t)Z[p].r * k), Z[p].r, k};
        ge.out(ze, false);
        ge.t2(Z[p].ref(), h.rb().xferm(s).tref(), Z[p].c);
        q.sl.add(ze.ref(), ze.r);
        M += ze.r;
      }
      for (int b : adm_of[s]) {
        if (scaling && nrm[b] == 0.0) continue;
        q.sl.add(Tb[b].ref(), Tb[b].r, scaling ? 1.0 / nrm[b] : 1.0);
        M += Tb[b].r;
      }
      it.s1 = q.sl.begin();
      it.M = M;
      const int rows = (int)std::min<long long>(M, k);
      Z[s] = Mat{ar.alloc((size_t)rows * k), rows, k};
      it.out = Z[s].p;
      q.items.push_back(it);
    }
    ge.run(C);
    q.run(C, ar);
  }
  return Z;
}

}  // namespace h2g
