// Phase 2 of the product: adaptive re-compression onto the prescribed block tree (Figs. 4-5) and
// the final projection (reference coarsening.py:36-445), plus input recompression.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <future>
#include <map>
#include <unordered_map>
#include <thread>

#include "engine.h"

namespace h2g {

// ------------------------------------------------------------------ column trees (trees.py:362-406)
// Flat column tree: children of a node are contiguous (k0[u] .. k0[u] + nk[u] - 1); node 0 is the
// root.  Matrices live on the leaves.  (The reference's ColumnTree objects, built and discarded per
// block, become index arithmetic here.)
struct CT {
  std::vector<int> cl, k0, nk;
  std::vector<char> adm;
  std::vector<Mat> mat;
  int add(int c, bool a, Mat m = Mat{}) {
    cl.push_back(c);
    adm.push_back(a ? 1 : 0);
    k0.push_back(0);
    nk.push_back(0);
    mat.push_back(m);
    return (int)cl.size() - 1;
  }
  void set(int u, int c, bool a, Mat m) {
    cl[u] = c;
    adm[u] = a ? 1 : 0;
    mat[u] = m;
  }
  int reserve_kids(int u, int n) {  // allocates n contiguous child slots of u
    const int base = (int)cl.size();
    for (int i = 0; i < n; ++i) add(-1, true);
    k0[u] = base;
    nk[u] = n;
    return base;
  }
  bool leaf(int u) const { return nk[u] == 0; }
  int kid(int u, int i) const { return k0[u] + i; }
  void clear() {
    cl.clear();
    k0.clear();
    nk.clear();
    adm.clear();
    mat.clear();
  }
  void leaves(int u, std::vector<int>& out) const {
    if (leaf(u)) { out.push_back(u); return; }
    for (int i = 0; i < nk[u]; ++i) leaves(k0[u] + i, out);
  }
};
using CTP = std::shared_ptr<CT>;
struct CTRef {  // a column tree inside a pooled flat tree
  const CT* t = nullptr;
  int root = -1;
};

static int ct_copy(const CT& a, int u, CT& out, bool with_mats, int slot = -1) {
  if (slot < 0) slot = out.add(a.cl[u], a.adm[u], with_mats ? a.mat[u] : Mat{});
  else out.set(slot, a.cl[u], a.adm[u], with_mats ? a.mat[u] : Mat{});
  if (!a.leaf(u)) {
    const int n = a.nk[u];
    const int base = out.reserve_kids(slot, n);
    for (int i = 0; i < n; ++i) ct_copy(a, a.kid(u, i), out, with_mats, base + i);
  }
  return slot;
}

// Structure-only union (coarsening.py:89-105).
static int ct_union(const CT* a, int ua, const CT* b, int ub, CT& out, int slot = -1) {
  if (!a) return ct_copy(*b, ub, out, false, slot);
  if (!b) return ct_copy(*a, ua, out, false, slot);
  if (a->cl[ua] != b->cl[ub]) throw StructureErr("column trees rooted at different clusters");
  const bool ak = !a->leaf(ua), bk = !b->leaf(ub);
  if (ak && bk) {
    if (slot < 0) slot = out.add(a->cl[ua], true);
    else out.set(slot, a->cl[ua], true, Mat{});
    const int n = std::min(a->nk[ua], b->nk[ub]);
    const int base = out.reserve_kids(slot, n);
    for (int i = 0; i < n; ++i) ct_union(a, a->kid(ua, i), b, b->kid(ub, i), out, base + i);
    return slot;
  }
  if (ak) return ct_copy(*a, ua, out, false, slot);
  if (bk) return ct_copy(*b, ub, out, false, slot);
  if (slot < 0) return out.add(a->cl[ua], a->adm[ua] && b->adm[ub]);
  out.set(slot, a->cl[ua], a->adm[ua] && b->adm[ub], Mat{});
  return slot;
}

// Deferred products  dst = src * F_{path[0]}^T * ... * F_{path[-1]}^T (* W_leaf^T)  (match_column,
// coarsening.py:108-136), resolved with memoised prefix products in dependency waves.  Paths live in
// one shared pool.
struct Jobs {
  struct J {
    Mat dst, src;
    int p0, plen;
    bool conv;
    int leafcl;
  };
  std::vector<J> v;
  std::vector<int> pool;
};

static void ct_push_down(const Mat& src, int* path, int depth, const CT& T, int tu, int ro, Jobs& J) {
  if (!T.leaf(tu)) {
    if (depth >= 62) throw StructureErr("column tree deeper than 62 levels");
    for (int i = 0; i < T.nk[tu]; ++i) {
      const int tc = T.kid(tu, i);
      path[depth] = T.cl[tc];
      ct_push_down(src, path, depth + 1, T, tc, ro, J);
    }
    return;
  }
  const int p0 = (int)J.pool.size();
  J.pool.insert(J.pool.end(), path, path + depth);
  J.v.push_back(Jobs::J{T.mat[tu].band(ro, src.r), src, p0, depth, !T.adm[tu], T.cl[tu]});
}

static void ct_match(const CT& P, int pu, const CT& T, int tu, int ro, Jobs& J) {
  if (P.cl[pu] != T.cl[tu]) throw InvalidInput("representation and target roots differ");
  if (!P.leaf(pu)) {
    if (T.leaf(tu)) throw StructureErr("match_column: target coarser than representation");
    for (int i = 0; i < P.nk[pu]; ++i) ct_match(P, P.kid(pu, i), T, T.kid(tu, i), ro, J);
    return;
  }
  const Mat& src = P.mat[pu];
  if (!T.leaf(tu)) {
    int path[64];
    for (int i = 0; i < T.nk[tu]; ++i) {
      const int tc = T.kid(tu, i);
      path[0] = T.cl[tc];
      ct_push_down(src, path, 1, T, tc, ro, J);
    }
    return;
  }
  J.v.push_back(Jobs::J{T.mat[tu].band(ro, src.r), src, 0, 0, P.adm[pu] && !T.adm[tu], T.cl[tu]});
}

struct PtrClusterHash {
  size_t operator()(const std::pair<const double*, int>& k) const {
    return std::hash<const void*>()(k.first) * 1000003u ^ (size_t)k.second;
  }
};

static void resolve_jobs(Ctx& C, Arena& sc, Jobs& J, const Basis& w) {
  HostTimer ht(C, "p2_jobs");
  std::unordered_map<std::pair<const double*, int>, Mat, PtrClusterHash> inter;
  inter.reserve(J.v.size());
  std::vector<std::vector<std::pair<const Jobs::J*, int>>> waves;
  for (const auto& j : J.v) {
    const int* path = J.pool.data() + j.p0;
    const int nf = j.plen + (j.conv ? 1 : 0);
    const int L = nf - 2;
    for (int i = 0; i < L; ++i) {
      auto key = std::make_pair((const double*)j.src.p, path[i]);
      if (inter.count(key)) continue;
      inter[key] = Mat{sc.alloc((size_t)j.src.r * w.rank[path[i]]), j.src.r, w.rank[path[i]]};
      if ((int)waves.size() <= i) waves.resize(i + 1);
      waves[i].emplace_back(&j, i);
    }
  }
  for (auto& wave : waves) {
    GBatch g;
    for (auto& pr : wave) {
      const Jobs::J& j = *pr.first;
      const int* path = J.pool.data() + j.p0;
      const int i = pr.second;
      const Mat in = i == 0 ? j.src : inter[std::make_pair((const double*)j.src.p, path[i - 1])];
      g.out(inter[std::make_pair((const double*)j.src.p, path[i])], false);
      g.t2(in.ref(), w.xferm(path[i]).tref(), in.c);
    }
    g.run(C);
  }
  GBatch g;
  g.outs.reserve(J.v.size());
  g.terms.reserve(J.v.size());
  for (const auto& j : J.v) {
    const int* path = J.pool.data() + j.p0;
    const int nf = j.plen + (j.conv ? 1 : 0);
    const int L = std::max(0, nf - 2);
    const Mat base = L > 0 ? inter[std::make_pair((const double*)j.src.p, path[L - 1])] : j.src;
    MatRef f[2];
    int fc[2], nfac = 0;
    for (int i = L; i < j.plen; ++i) {
      f[nfac] = w.xferm(path[i]).tref();
      fc[nfac++] = w.rank[path[i]];
    }
    if (j.conv) {
      f[nfac] = w.leafm(j.leafcl).tref();
      fc[nfac++] = w.tree->size(j.leafcl);
    }
    g.out(j.dst, false);
    if (nfac == 0) g.t1(base.ref());
    else if (nfac == 1) g.t2(base.ref(), f[0], base.c);
    else g.t3(base.ref(), f[0], f[1], base.c, fc[0]);
  }
  g.run(C);
  J.v.clear();
  J.pool.clear();
}

// ------------------------------------------------------------------ coverage (coarsening.py:160-184)
static void validate_coarse(BView pt, BView coarse) {
  if (!(pt.rows().same(coarse.rows()) && pt.cols().same(coarse.cols())))
    throw InvalidInput("coarse tree lives on different cluster trees");
  for (int b = 0; b < coarse.nb(); ++b)
    if (pt.find(coarse.row(b), coarse.col(b)) < 0)
      throw InvalidInput("coarse block is finer than the product block tree");
}

static std::vector<char> coverage(BView pt, BView coarse) {
  std::vector<char> cov(pt.nb(), 0);
  struct F { int pb, cb, state; };  // state: 0 none, 1 admissible, 2 inadmissible
  std::vector<F> st{{0, 0, 0}};
  while (!st.empty()) {
    F f = st.back();
    st.pop_back();
    if (f.state == 0 && f.cb >= 0 && coarse.b->leaf(f.cb)) f.state = coarse.b->adm[f.cb] ? 1 : 2;
    cov[f.pb] = f.state == 1;
    for (int i = 0; i < pt.b->nkids(f.pb); ++i) {
      const int ch = pt.b->kid(f.pb, i);
      const int cb = f.state == 0 ? coarse.find(pt.row(ch), pt.col(ch)) : -1;
      st.push_back(F{ch, cb, f.state});
    }
  }
  return cov;
}

struct CState {
  std::shared_ptr<Basis> q;
  MatStore r, z;
  std::vector<CTRef> reps;
  std::vector<std::unique_ptr<CT>> pools;  // owners of the stored representations
};

// Structure-only preparation of one pass (runs on a host thread while the norms are computed):
// coverage of T^XY by the coarse tree and the per-row-cluster block lists.
struct CPrep {
  std::vector<std::vector<int>> row_adm, near_cov, sub_cov;
};

static CPrep prep_rows(BView pv, BView coarse) {
  validate_coarse(pv, coarse);
  const std::vector<char> cov = coverage(pv, coarse);
  const Tree& tr = pv.rows();
  const Blocks& pt = *pv.b;
  CPrep P;
  P.row_adm.resize(tr.n);
  P.near_cov.resize(tr.n);
  P.sub_cov.resize(tr.n);
  for (int b = 0; b < pt.nb; ++b) {
    const int t = pv.row(b);
    if (pt.adm_leaf(b)) P.row_adm[t].push_back(b);
    else if (pt.near_leaf(b)) { if (cov[b]) P.near_cov[t].push_back(b); }
    else if (cov[b]) P.sub_cov[t].push_back(b);
  }
  return P;
}

// Fig. 5: adaptive coarse row basis (reference coarsening.py:187-332).
static CState coarse_rows(Ctx& C, Arena& out, HView g, BView coarse, double tol, int max_rank, bool scale,
                          const double* d_cn, const double* d_nn, const CPrep& prep,
                          cudaEvent_t nn_ready = nullptr) {
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  const BView pv = g.bv();
  const Blocks& pt = *g.h->bt;
  const Tree& tr = pv.rows();
  const Basis& v1 = g.rb();
  const Basis& w1 = g.cb();
  const std::vector<std::vector<int>>& row_adm = prep.row_adm;
  const std::vector<std::vector<int>>& near_cov = prep.near_cov;
  const std::vector<std::vector<int>>& sub_cov = prep.sub_cov;
  CState S;
  S.q = std::make_shared<Basis>();
  Basis& q = *S.q;
  q.tree = &tr;
  q.rank.assign(tr.n, 0);
  q.leaf.assign(tr.n, nullptr);
  q.xfer.assign(tr.n, nullptr);
  S.r.assign(tr.n, Mat{});
  S.z.assign(tr.n, Mat{});
  S.reps.assign(pt.nb, CTRef{});
  // multi-GPU: this rank's subtrees of tr. The replicated top levels may not merge representations
  // of partitioned children (those stay on their rank); the BASELINE trees never do -- no product
  // block above the partition level is covered -- and otherwise the pass runs replicated.
  Part part = make_part(tr, C.comm);
  if (part.on())
    for (int l = 0; l < part.level && part.on(); ++l)
      for (int t : tr.by_level[l])
        if (!sub_cov[t].empty()) {
          part = Part{};
          break;
        }
  CT mpool, singles, acc, nxt, tg[8];  // per-level scratch trees (capacity reused)
  std::vector<int> mroot(pt.nb, -1);
  Arena sc(C.st);
  double* d_msc = sc.alloc(std::max(1, pt.nb));  // sigma_1 of merged reps, per block

  // top-down condensation weights Z_t (coarsening.py:231-245).  Exactly-zero couplings are not
  // rows of the reference's stack (coarsening.py:237-241): their norms are read back once so that
  // the factor's row count min(M, k) -- the column count of the SVD inputs built from Z -- matches
  std::vector<double> cn_host;
  // coupling norms (main-stream work); only needed when the SVD floor can bind (kFloorFreeTol)
  const bool exact_rows = scale && tol < kFloorFreeTol;
  if (exact_rows) cn_host = C.read(d_cn, (size_t)std::max(1, pt.nb));
  std::vector<int> Lp;
  for (int lev = 0; lev <= tr.depth; ++lev) {
    StageTag tag(C, "p2.Z.L" + std::to_string(lev));
    GBatch ge;
    QrBatch qb;
    if (part.on()) Lp = part.filter(tr.by_level[lev]);
    for (int t : part.on() ? Lp : tr.by_level[lev]) {
      const int k = v1.rank[t];
      QrItem it{};
      it.s0 = qb.sl.begin();
      it.n = k;
      long long M = 0;
      const int p = tr.parent[t];
      if (p >= 0 && S.z[p].r > 0) {
        Mat ze{sc.alloc((size_t)S.z[p].r * k), S.z[p].r, k};
        ge.out(ze, false);
        ge.t2(S.z[p].ref(), v1.xferm(t).tref(), S.z[p].c);
        qb.sl.add(ze.ref(), ze.r);
        M += ze.r;
      }
      for (int b : row_adm[t]) {
        // S_tr^T / ||S_tr||_2 with the norm as a device divisor
        if (exact_rows && cn_host[b] == 0.0) continue;
        const int kc = w1.rank[pv.col(b)];
        qb.sl.add(trn(g.coup(b)), kc, 1.0, scale ? d_cn + b : nullptr);
        M += kc;
      }
      it.s1 = qb.sl.begin();
      it.M = M;
      const int rows = (int)std::min<long long>(M, k);
      S.z[t] = Mat{sc.alloc((size_t)rows * k), rows, k};
      it.out = S.z[t].p;
      qb.items.push_back(it);
    }
    ge.run(C);
    qb.run(C, sc);
  }

  // the nearfield norms (SVD segment divisors at the leaves) come from the auxiliary stream
  if (nn_ready) cuda_check(cudaStreamWaitEvent(C.st, nn_ready, 0), "wait nearfield norms");
  std::vector<Mat> lm(pt.nb);  // R_t S_b for admissible leaves used inside representations
  for (int lev = tr.depth; lev >= 0; --lev) {
    if (part.on()) Lp = part.filter(tr.by_level[lev]);
    const std::vector<int>& L = part.on() ? Lp : tr.by_level[lev];
    const size_t nl = L.size();
    StageTag tag(C, "p2.B.L" + std::to_string(lev));
    // this level's temporaries (V_t, V_t Z_t^T, merged representations, admissible-leaf products,
    // SVD scratch): freed stream-ordered when the level is done, so the pass's footprint is one
    // level's scratch instead of the sum over levels
    Arena lvl(C.st);
    std::vector<int> lm_level;  // lm entries allocated from lvl (cleared with it)
    HostTimer htv(C, "p2_vz_plan");
    GBatch g1, g2;
    std::vector<Mat> V(nl), VZ(nl);
    for (size_t li = 0; li < nl; ++li) {
      const int t = L[li];
      const Mat& Z = S.z[t];
      if (tr.leaf(t)) {
        V[li] = v1.leafm(t);
      } else {
        int m = 0;
        for (int i = 0; i < tr.nkids(t); ++i) m += q.rank[tr.kid(t, i)];
        V[li] = Mat{lvl.alloc((size_t)m * v1.rank[t]), m, v1.rank[t]};
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {  // vhat = vstack(R_c E_c) (coarsening.py:313-314)
          const int c = tr.kid(t, i);
          g1.out(V[li].band(off, q.rank[c]), false);
          g1.t2(S.r[c].ref(), v1.xferm(c).ref(), S.r[c].c);
          off += q.rank[c];
        }
        for (int b : sub_cov[t])
          for (int i = 0; i < pt.nkids(b); ++i) {  // child_rep of admissible children (coarsening.py:254-258)
            const int b2 = pt.kid(b, i);
            if (!pt.adm_leaf(b2) || lm[b2].p) continue;
            const int t2 = pv.row(b2), r2 = pv.col(b2);
            lm[b2] = Mat{lvl.alloc((size_t)q.rank[t2] * w1.rank[r2]), q.rank[t2], w1.rank[r2]};
            lm_level.push_back(b2);
            g1.out(lm[b2], false);
            g1.t2(S.r[t2].ref(), g.coup(b2), S.r[t2].c);
          }
      }
      VZ[li] = Mat{lvl.alloc((size_t)V[li].r * Z.r), V[li].r, Z.r};
      GBatch& gz = tr.leaf(t) ? g1 : g2;
      gz.out(VZ[li], false);
      gz.t2(V[li].ref(), Z.tref(), Z.c);
    }
    g1.run(C);
    g2.run(C);
    htv.stop();

    // merged representations of subdivided covered blocks (coarsening.py:260-279); all column
    // trees of the level live in pooled flat trees (no per-block allocations)
    mpool.clear();
    std::vector<int> mblocks;
    Jobs J;
    {
    HostTimer htm(C, "p2_merge_plan");
    for (size_t li = 0; li < nl; ++li) {
      const int t = L[li];
      if (tr.leaf(t)) continue;
      for (int b : sub_cov[t]) {
        // children of (t, r) are chil(t) x (chil(r) or {r}): group by column r2, first appearance
        int order[8], ngroup = 0;
        CTRef gpart[8][8];
        int grows[8][8], gcnt[8] = {0};
        singles.clear();  // one-leaf column trees for admissible children (R_t2 S_b2)
        if (pt.nkids(b) > 8) throw StructureErr("product block with more than 8 children");
        for (int i = 0; i < pt.nkids(b); ++i) {
          const int b2 = pt.kid(b, i);
          const int r2 = pv.col(b2);
          CTRef part;
          if (pt.adm_leaf(b2)) {
            part = CTRef{&singles, singles.add(r2, true, lm[b2])};
          } else {
            part = S.reps[b2];
            if (!part.t) throw StructureErr("missing child representation");
          }
          int gi = 0;
          while (gi < ngroup && order[gi] != r2) ++gi;
          if (gi == ngroup) order[ngroup++] = r2;
          gpart[gi][gcnt[gi]] = part;
          grows[gi][gcnt[gi]++] = q.rank[pv.row(b2)];
        }
        for (int gi = 0; gi < ngroup; ++gi) {
          CT& tgt = tg[gi];
          tgt.clear();
          if (gcnt[gi] == 1) {
            ct_copy(*gpart[gi][0].t, gpart[gi][0].root, tgt, false);
          } else {
            acc.clear();
            ct_union(nullptr, 0, gpart[gi][0].t, gpart[gi][0].root, acc);
            for (int i = 1; i < gcnt[gi]; ++i) {
              nxt.clear();
              ct_union(&acc, 0, gpart[gi][i].t, gpart[gi][i].root, nxt);
              std::swap(acc, nxt);
            }
            ct_copy(acc, 0, tgt, false);
          }
          int rows = 0;
          for (int i = 0; i < gcnt[gi]; ++i) rows += grows[gi][i];
          for (int u = 0; u < (int)tgt.cl.size(); ++u) {
            if (!tgt.leaf(u)) continue;
            const int c = tgt.cl[u];
            const int cols = tgt.adm[u] ? w1.rank[c] : w1.tree->size(c);
            tgt.mat[u] = Mat{lvl.alloc((size_t)rows * cols), rows, cols};
          }
          int ro = 0;
          for (int i = 0; i < gcnt[gi]; ++i) {
            ct_match(*gpart[gi][i].t, gpart[gi][i].root, tgt, 0, ro, J);
            ro += grows[gi][i];
          }
        }
        const int r = pv.col(b);
        if (ngroup == 1 && order[0] == r) {
          mroot[b] = ct_copy(tg[0], 0, mpool, true);
        } else {
          const int root = mpool.add(r, true);
          const int base = mpool.reserve_kids(root, ngroup);
          for (int gi = 0; gi < ngroup; ++gi) ct_copy(tg[gi], 0, mpool, true, base + gi);
          mroot[b] = root;
        }
        mblocks.push_back(b);
      }
    }
    static const bool dbg_jobs = getenv("H2G_DEBUG_JOBS") != nullptr;
    if (dbg_jobs)
      fprintf(stderr, "level %d: %zu merged reps, %zu nodes, %zu jobs, path pool %zu\n", lev, mblocks.size(),
              mpool.cl.size(), J.v.size(), J.pool.size());
    htm.next("p2_merge_resolve");
    resolve_jobs(C, lvl, J, w1);
    }
    mem_mark(("p2 L" + std::to_string(lev) + " ch" + std::to_string(C.channel) + " reps").c_str());

    // scales of the flattened merged reps (coarsening.py:316-317), kept on the device
    std::vector<int> lv;
    if (scale && !mblocks.empty()) {
      NormBatch nbat;
      cuda_check(cudaMemsetAsync(d_msc, 0, sizeof(double) * pt.nb, C.st), "memset");
      for (int b : mblocks) {
        lv.clear();
        mpool.leaves(mroot[b], lv);
        NormItem it{};
        it.s0 = nbat.sl.begin();
        long long N = 0;
        for (int u : lv) {
          nbat.sl.add(mpool.mat[u].ref(), mpool.mat[u].c);
          N += mpool.mat[u].c;
        }
        it.s1 = nbat.sl.begin();
        it.m = lv.empty() ? 0 : mpool.mat[lv[0]].r;
        it.N = N;
        it.out = d_msc + b;
        nbat.items.push_back(it);
      }
      nbat.run_async(C);
    }

    // truncated SVDs of C_t = [V Z^T | scaled columns] (coarsening.py:294-326)
    SvdBatch sv;
    std::vector<Mat> qbuf(nl);
    for (size_t li = 0; li < nl; ++li) {
      const int t = L[li];
      const int m = V[li].r;
      SvdItem it{};
      it.s0 = sv.sl.begin();
      sv.sl.add(VZ[li].ref(), VZ[li].c);
      long long N = VZ[li].c;
      if (tr.leaf(t)) {
        for (int b : near_cov[t]) {
          const int w = w1.tree->size(pv.col(b));
          sv.sl.add(g.near(b), w, 1.0, scale ? d_nn + b : nullptr);
          N += w;
        }
      } else {
        for (int b : sub_cov[t]) {
          lv.clear();
          mpool.leaves(mroot[b], lv);
          for (int u : lv) {
            sv.sl.add(mpool.mat[u].ref(), mpool.mat[u].c, 1.0, scale ? d_msc + b : nullptr);
            N += mpool.mat[u].c;
          }
        }
      }
      it.s1 = sv.sl.begin();
      it.m = m;
      it.kx = 0;
      it.N = N;
      it.tol = tol;
      it.cap = max_rank;
      const long long kcap = std::min<long long>(m, N);
      qbuf[li] = Mat{out.alloc((size_t)m * std::max<long long>(kcap, 0)), m, (int)kcap};
      it.q_out = qbuf[li].p;
      sv.items.push_back(it);
    }
    std::vector<int> rk = sv.run(C, lvl);
    mem_mark(("p2 L" + std::to_string(lev) + " ch" + std::to_string(C.channel) + " svd").c_str());

    HostTimer htp(C, "p2_post");
    S.pools.emplace_back(new CT());
    CT& rp = *S.pools.back();  // this level's stored representations
    GBatch gp, gq;
    std::vector<int> lv2;
    for (size_t li = 0; li < nl; ++li) {
      const int t = L[li];
      const int k = rk[li];
      const Mat Q{qbuf[li].p, V[li].r, k};
      q.rank[t] = k;
      S.r[t] = Mat{out.alloc((size_t)k * V[li].c), k, V[li].c};
      gp.out(S.r[t], false);  // R_t = Q_t^T V_t
      gp.t2(Q.tref(), V[li].ref(), Q.r);
      if (tr.leaf(t)) {
        q.leaf[t] = Q.p;
        for (int b : near_cov[t]) {  // reps: Q_t^T N (coarsening.py:306-307)
          const int r = pv.col(b);
          Mat rep{out.alloc((size_t)k * w1.tree->size(r)), k, w1.tree->size(r)};
          gp.out(rep, false);
          gp.t2(Q.tref(), g.near(b), Q.r);
          S.reps[b] = CTRef{&rp, rp.add(r, false, rep)};
        }
      } else {
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {
          const int c = tr.kid(t, i);
          q.xfer[c] = Q.p + (long long)off * k;
          off += q.rank[c];
        }
        for (int b : sub_cov[t]) {  // stored reps are Q^T (unscaled rep) (coarsening.py:327-328)
          const int root = ct_copy(mpool, mroot[b], rp, false);
          lv.clear();
          lv2.clear();
          mpool.leaves(mroot[b], lv);
          rp.leaves(root, lv2);
          for (size_t i = 0; i < lv.size(); ++i) {
            const Mat& src = mpool.mat[lv[i]];
            rp.mat[lv2[i]] = Mat{out.alloc((size_t)k * src.c), k, src.c};
            gp.out(rp.mat[lv2[i]], false);
            gp.t2(Q.tref(), src.ref(), Q.r);
          }
          S.reps[b] = CTRef{&rp, root};
        }
      }
    }
    gp.run(C);
    HostTimer htc(C, "p2_compose");
    // compose_leaf_rep for subdivided covered blocks at leaf row clusters (coarsening.py:281-290)
    for (size_t li = 0; li < nl; ++li) {
      const int t = L[li];
      if (!tr.leaf(t)) continue;
      std::function<int(CT&, int, int)> build = [&](CT& T, int b, int slot) -> int {
        const int r = pv.col(b);
        if (pt.adm_leaf(b)) {
          if (!lm[b].p) {
            lm[b] = Mat{out.alloc((size_t)q.rank[t] * w1.rank[r]), q.rank[t], w1.rank[r]};
            gq.out(lm[b], false);
            gq.t2(S.r[t].ref(), g.coup(b), S.r[t].c);
          }
          if (slot < 0) return T.add(r, true, lm[b]);
          T.set(slot, r, true, lm[b]);
          return slot;
        }
        if (pt.near_leaf(b)) {
          const Mat nm = S.reps[b].t->mat[S.reps[b].root];
          if (slot < 0) return T.add(r, false, nm);
          T.set(slot, r, false, nm);
          return slot;
        }
        if (slot < 0) slot = T.add(r, true);
        else T.set(slot, r, true, Mat{});
        const int base = T.reserve_kids(slot, pt.nkids(b));
        for (int i = 0; i < pt.nkids(b); ++i) build(T, pt.kid(b, i), base + i);
        return slot;
      };
      std::function<void(int)> all = [&](int b) {
        if (pt.leaf(b)) return;
        S.reps[b] = CTRef{&rp, build(rp, b, -1)};
        for (int i = 0; i < pt.nkids(b); ++i) all(pt.kid(b, i));
      };
      for (int b : sub_cov[t]) all(b);
    }
    gq.run(C);
    for (int b : lm_level) lm[b] = Mat{};
    if (part.on() && lev == part.level) {
      // every rank receives the partitioned levels' ranks, Q_t and R_t (the representations stay
      // with their rank: only its own rows' final projection reads them)
      C.gate_enter();
      StageTag tagx(C, "p2.exchange");
      std::vector<int> ids;
      for (int l = part.level; l <= tr.depth; ++l)
        for (int t : tr.by_level[l]) ids.push_back(t);
      exchange_ints(C, part, ids, q.rank);
      std::vector<XItem> items;
      std::vector<double*> qp(tr.n, nullptr);
      for (int t : ids) {
        const int o = part.owner[t], k = q.rank[t];
        int m = tr.size(t);
        if (!tr.leaf(t)) {
          m = 0;
          for (int i = 0; i < tr.nkids(t); ++i) m += q.rank[tr.kid(t, i)];
        }
        if (o == part.me) qp[t] = tr.leaf(t) ? q.leaf[t] : q.xfer[tr.kid(t, 0)];
        else S.r[t] = Mat{nullptr, k, v1.rank[t]};
        items.push_back(XItem{o, (long long)m * k, &qp[t]});
        items.push_back(XItem{o, (long long)k * v1.rank[t], &S.r[t].p});
      }
      exchange(C, out, items);
      for (int t : ids) {
        if (part.owner[t] == part.me) continue;
        if (tr.leaf(t)) {
          q.leaf[t] = qp[t];
        } else {
          int off = 0;
          for (int i = 0; i < tr.nkids(t); ++i) {
            const int c = tr.kid(t, i);
            q.xfer[c] = qp[t] + (long long)off * q.rank[t];
            off += q.rank[c];
          }
        }
      }
      C.gate_leave();
    }
  }
  return S;
}

// Final projection (reference coarsening.py:354-405), in two parts: the structure (product block
// of every coarse leaf, representation leaves of the covered admissible blocks, the transfer chains
// to materialise) needs only the row pass and is planned while the column pass still runs; the
// products need both.
struct ProjLeaf {
  int c;
  bool adm;
  Mat M;
};
struct ProjPlan {
  std::vector<int> pb;          // per coarse block: the product block (leaves only)
  std::vector<int> lptr;        // per coarse block: its representation leaves [lptr[b], lptr[b+1])
  std::vector<ProjLeaf> leaves;
  std::vector<std::vector<std::pair<int, int>>> waves;  // chains (r, c) of depth >= 2, by depth
};

static ProjPlan plan_project(HView g, const CState& rs, const Blocks& cb) {
  const BView pv = g.bv();
  validate_coarse(pv, BView{&cb, false});
  const Blocks& pt = *g.h->bt;
  const Tree& ctree = *cb.cols;
  // multi-GPU: the coarse blocks of this rank's row subtrees
  ProjPlan P;
  P.pb.assign(cb.nb, -1);
  P.lptr.assign(cb.nb + 1, 0);
  std::unordered_map<long long, char> seen;
  seen.reserve(1024);
  std::function<void(int, int)> need = [&](int r, int c) {
    if (ctree.parent[c] == r || c == r) return;
    const long long key = (long long)r * ctree.n + c;
    if (seen.count(key)) return;
    seen[key] = 1;
    need(r, ctree.parent[c]);
    int d = 0;
    for (int u = c; u != r; u = ctree.parent[u]) ++d;
    if ((int)P.waves.size() <= d) P.waves.resize(d + 1);
    P.waves[d].push_back(std::make_pair(r, c));
  };
  std::vector<int> lv;
  for (int b = 0; b < cb.nb; ++b) {
    P.lptr[b + 1] = P.lptr[b];
    if (!cb.leaf(b)) continue;
    const int pb = pt.find(cb.row[b], cb.col[b]);
    P.pb[b] = pb;
    if (!cb.adm[b] || pt.adm_leaf(pb)) continue;
    const CTRef rr = rs.reps[pb];
    if (!rr.t) continue;  // (a partitioned rank holds only its own rows' representations)
    lv.clear();
    rr.t->leaves(rr.root, lv);
    for (int u : lv) {
      P.leaves.push_back(ProjLeaf{rr.t->cl[u], rr.t->adm[u] != 0, rr.t->mat[u]});
      need(cb.col[b], rr.t->cl[u]);
    }
    P.lptr[b + 1] = (int)P.leaves.size();
  }
  return P;
}

static std::shared_ptr<H2> project_final(Ctx& C, HView g, CState& rs, CState& cs,
                                         std::shared_ptr<const Blocks> coarse, ArenaPtr ar, const ProjPlan& plan) {
  HostTimer htp(C, "p2_project_plan");
  auto Z = std::make_shared<H2>();
  Z->bt = coarse;
  Z->rb = rs.q;
  Z->cb = cs.q;
  Z->owned.push_back(ar);
  if (g.h->near_owner) Z->owned.push_back(g.h->near_owner);  // dense blocks shared with the product
  const Blocks& cb = *coarse;
  const Blocks& pt = *g.h->bt;
  const Basis& qr = *rs.q;
  const Basis& qc = *cs.q;
  const Tree& ctree = *cb.cols;
  Z->coup.assign(cb.nb, nullptr);
  Z->near.assign(cb.nb, nullptr);
  Arena sc(C.st);
  // chain(r, c) = F'_c F'_parent ... (k'_c x k'_r), memoised, depth >= 2 materialised in waves
  std::unordered_map<long long, Mat> chain;
  chain.reserve(1024);
  auto ckey = [&](int r, int c) { return (long long)r * ctree.n + c; };
  for (auto& wave : plan.waves)
    for (auto& key : wave)
      chain[ckey(key.first, key.second)] =
          Mat{sc.alloc((size_t)qc.rank[key.second] * qc.rank[key.first]), qc.rank[key.second], qc.rank[key.first]};
  auto chain_ref = [&](int r, int c) -> Mat {
    if (ctree.parent[c] == r) return qc.xferm(c);
    return chain[ckey(r, c)];
  };
  for (auto& wave : plan.waves) {
    GBatch gw;
    for (auto& key : wave) {
      const int r = key.first, c = key.second;
      gw.out(chain[ckey(r, c)], false);
      const Mat up = chain_ref(r, ctree.parent[c]);
      gw.t2(qc.xferm(c).ref(), up.ref(), qc.rank[ctree.parent[c]]);
    }
    gw.run(C);
  }
  const Part part = make_part(*cb.rows, C.comm);
  htp.next("p2_project_blocks");
  GBatch g1;
  std::vector<XItem> items;
  for (int b = 0; b < cb.nb; ++b) {
    if (!cb.leaf(b)) continue;
    const int t = cb.row[b], r = cb.col[b];
    const int pb = plan.pb[b];
    const bool shared = !cb.adm[b] && pt.near_leaf(pb) && !g.T && g.h->near_owner;
    if (!part.mine(t) && !shared) {  // received below
      if (cb.adm[b]) items.push_back(XItem{part.owner[t], (long long)qr.rank[t] * qc.rank[r], &Z->coup[b]});
      else items.push_back(XItem{part.owner[t], (long long)cb.rows->size(t) * ctree.size(r), &Z->near[b]});
      continue;
    }
    if (!part.top(t) && !shared) {
      if (cb.adm[b]) items.push_back(XItem{part.owner[t], (long long)qr.rank[t] * qc.rank[r], &Z->coup[b]});
      else items.push_back(XItem{part.owner[t], (long long)cb.rows->size(t) * ctree.size(r), &Z->near[b]});
    }
    if (cb.adm[b]) {
      Mat S{ar->alloc((size_t)qr.rank[t] * qc.rank[r]), qr.rank[t], qc.rank[r]};
      Z->coup[b] = S.p;
      g1.out(S, false);
      if (pt.adm_leaf(pb)) {
        g1.t3(rs.r[t].ref(), g.coup(pb), cs.r[r].tref(), rs.r[t].c, cs.r[r].c);
      } else {
        if (plan.lptr[b] == plan.lptr[b + 1] && !rs.reps[pb].t)
          throw StructureErr("missing representation of a covered product block");
        for (int li = plan.lptr[b]; li < plan.lptr[b + 1]; ++li) {  // lift (coarsening.py:374-382)
          const ProjLeaf& L = plan.leaves[li];
          const int c = L.c;
          const MatRef X = L.adm ? cs.r[c].tref() : qc.leafm(c).ref();
          if (c == r) g1.t2(L.M.ref(), X, L.M.c);
          else g1.t3(L.M.ref(), X, chain_ref(r, c).ref(), L.M.c, qc.rank[c]);
        }
      }
    } else if (shared) {
      // the reference copies G's dense block (coarsening.py:397-398); device matrices are immutable,
      // so Z shares it (its arena stays alive with Z) instead of copying
      Z->near[b] = g.h->near[pb];
    } else {
      const int nr = cb.rows->size(t), nc = ctree.size(r);
      Mat N{ar->alloc((size_t)nr * nc), nr, nc};
      Z->near[b] = N.p;
      g1.out(N, false);
      if (pt.near_leaf(pb)) g1.t1(g.near(pb));
      else if (pt.adm_leaf(pb)) g1.t3(g.rb().leafm(t).ref(), g.coup(pb), g.cb().leafm(r).tref(), g.rb().rank[t], g.cb().rank[r]);
      else throw StructureErr("inadmissible coarse leaf is subdivided in the product tree");
    }
  }
  g1.run(C);
  // multi-GPU: Z stays distributed by block rows (gather_rows completes it on demand: downloads,
  // matvecs); the items listed above are what such a gather moves
  if (part.on()) Z->dist_rows = true;
  (void)items;
  return Z;
}

// sigma_1 of every coupling (synchronously: their exact zeros skip rows of the Z stacks) and every
// nearfield block of g (asynchronously into a device array: they only scale SVD segments)
// (coarsening.py:342-351)
// The coupling norms are needed first (top-down Z), the nearfield norms only at the leaf SVDs: with
// an auxiliary context the latter run there, under the Z levels, and `nn_ready` completes them.
std::shared_ptr<NormPrep> build_norm_prep(const H2& g, const Comm& comm) {
  const Blocks& B = *g.bt;
  auto np = std::make_shared<NormPrep>();
  HView v{&g, false};
  // multi-GPU: the blocks read by this rank's row or column passes
  const Part pr = make_part(*B.rows, comm), pc = make_part(*B.cols, comm);
  for (int b = 0; b < B.nb; ++b) {
    if (!B.leaf(b)) continue;
    if (!pr.mine(B.row[b]) && !pc.mine(B.col[b])) continue;
    const bool coupling = B.adm[b];
    const int t = B.row[b], s = B.col[b];
    const int m = coupling ? g.rb->rank[t] : B.rows->size(t);
    const int n = coupling ? g.cb->rank[s] : B.cols->size(s);
    NormBatch& nb = coupling ? np->nbc : np->nbn;
    NormItem it{};
    it.s0 = nb.sl.begin();
    nb.sl.add(coupling ? v.coup(b) : v.near(b), n);
    it.s1 = nb.sl.begin();
    it.m = m;
    it.N = n;
    nb.items.push_back(it);
    (coupling ? np->ids : np->nids).push_back(b);
  }
  return np;
}

static void all_norms(Ctx& C, Arena& sc, const H2& g, double* d_cn, double* d_nn, Ctx* A = nullptr,
                      cudaEvent_t* nn_ready = nullptr) {
  const Blocks& B = *g.bt;
  HostTimer ht(C, "p2_norm_build");
  std::shared_ptr<NormPrep> np;
  if (g.norm_prep.valid()) np = g.norm_prep.get();  // built while the assembly ran
  if (!np) np = build_norm_prep(g, C.comm);
  NormBatch nbn = np->nbn, nbc = np->nbc;  // copies: the prepared batches stay reusable
  for (size_t i = 0; i < nbn.items.size(); ++i) nbn.items[i].out = d_nn + np->nids[i];
  const std::vector<int>& ids = np->ids;
  cuda_check(cudaMemsetAsync(d_nn, 0, sizeof(double) * B.nb, C.st), "memset");
  ht.next("p2_norm_launch");
  if (A) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(e, C.st), "event");  // G final, d_nn zero-filled
    cuda_check(cudaStreamWaitEvent(A->st, e, 0), "wait");
    cudaEventDestroy(e);
    if (g.near_ready) cuda_check(cudaStreamWaitEvent(A->st, g.near_ready, 0), "wait nearfield");
    nbn.run_async(*A);
    A->flush();
    cuda_check(cudaEventCreateWithFlags(nn_ready, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(*nn_ready, A->st), "event");
  } else {
    nbn.run_async(C);
  }
  // coupling norms stay on the device too (no host round trip); the passes' streams fork from the
  // main stream after this launch
  cuda_check(cudaMemsetAsync(d_cn, 0, sizeof(double) * std::max(1, B.nb), C.st), "memset");
  for (size_t i = 0; i < nbc.items.size(); ++i) nbc.items[i].out = d_cn + ids[i];
  nbc.scratch = &sc;
  nbc.run_async(C);
}

// Phase-2 driver (reference coarsening.py:408-422).
std::shared_ptr<H2> coarsen(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, double tol, int max_rank,
                            bool scale) {
  return coarsen(C, g, coarse, tol, max_rank, scale, nullptr, 0);
}

// Z's dense blocks that are G's dense blocks (shared in project_final) are final already: with a
// host buffer for Z's packed nearfield, copy them there now on the copy stream, overlapping the
// whole of phase 2; h2g_h2_download then only moves the rest.
struct NearPrefetch {
  std::vector<char> mask;
  ArenaPtr arena;
  cudaEvent_t ev = nullptr;
};

static NearPrefetch prefetch_near(Ctx& C, const H2& g, const Blocks& cbk, double* near_host, long long near_cap) {
  NearPrefetch P;
  const Blocks& pt = *g.bt;
  P.mask.assign(cbk.nb, 0);
  std::vector<long long> items;
  std::vector<long long> zoff(cbk.nb, -1), zlen(cbk.nb, 0);
  long long off = 0, npf = 0;
  for (int b = 0; b < cbk.nb; ++b) {
    if (!cbk.leaf(b) || cbk.adm[b]) continue;
    const int t = cbk.row[b], r = cbk.col[b];
    const long long sz = (long long)cbk.rows->size(t) * cbk.cols->size(r);
    zoff[b] = off;
    zlen[b] = sz;
    const int pb = pt.find(t, r);
    if (pb >= 0 && pt.near_leaf(pb) && sz > 0) {
      P.mask[b] = 1;
      items.push_back((long long)g.near[pb]);
      items.push_back(sz);
      items.push_back(off);  // patched to the staging address below
      ++npf;
    }
    off += sz;
  }
  if (!npf || off > near_cap) {
    P.mask.clear();
    return P;
  }
  if (!C.up_stream) cuda_check(cudaStreamCreateWithFlags(&C.up_stream, cudaStreamNonBlocking), "stream");
  P.arena = std::make_shared<Arena>(C.up_stream);
  double* stage = P.arena->alloc(off);
  for (size_t i = 2; i < items.size(); i += 3) items[i] = (long long)(stage + items[i]);
  // the gather's descriptors live in the prefetch arena (copied on the copy stream, from pageable
  // memory: the call returns once the host vector has been read), not in C's staging buffer that the
  // next host sync recycles -- so the main stream never has to wait for the copy stream
  long long* di = (long long*)P.arena->alloc_bytes(items.size() * sizeof(long long));
  cuda_check(cudaMemcpyAsync(di, items.data(), items.size() * sizeof(long long), cudaMemcpyHostToDevice,
                             C.up_stream),
             "prefetch descriptors");
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(e, C.st), "event");  // G's blocks complete on the main stream
  cuda_check(cudaStreamWaitEvent(C.up_stream, e, 0), "wait");
  cudaEventDestroy(e);
  if (g.near_ready) cuda_check(cudaStreamWaitEvent(C.up_stream, g.near_ready, 0), "wait nearfield");
  cuda_check(launch_gather(di, (int)npf, C.up_stream), "gather(prefetch)");
  ++C.launches;
  for (int b = 0; b < cbk.nb;) {  // one copy per run of consecutive prefetched blocks
    if (!P.mask[b]) { ++b; continue; }
    const long long lo = zoff[b];
    long long hi = lo;
    int e2 = b;
    for (; e2 < cbk.nb; ++e2) {
      if (zoff[e2] < 0) continue;  // not a dense block: does not break the run
      if (!P.mask[e2]) break;
      hi = zoff[e2] + zlen[e2];
    }
    cuda_check(cudaMemcpyAsync(near_host + lo, stage + lo, (hi - lo) * sizeof(double), cudaMemcpyDeviceToHost,
                               C.up_stream),
               "prefetch download");
    b = e2;
  }
  cuda_check(cudaEventCreateWithFlags(&P.ev, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(P.ev, C.up_stream), "event");
  return P;
}

std::shared_ptr<H2> coarsen(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, double tol, int max_rank,
                            bool scale, double* near_host, long long near_cap) {
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
  if (C.timing) { e0 = C.event(); cudaEventRecord(e0, C.st); }
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  HostTimer htpre(C, "p2_pre");
  // g's nearfield may still be in flight on the auxiliary stream (multiply's push-down expansions):
  // with block scaling its readers -- the nearfield norms on that stream, the leaf SVDs behind
  // nn_ready, the prefetch copy -- are ordered after it, so the main stream starts on the couplings
  g.start_near(C);  // a deferred upload (an uploaded matrix coarsened directly)
  const bool near_async = scale && !serial_passes() && g.near_ready;
  if (!near_async) wait_near(C, g);
  NearPrefetch pf;
  if (near_host && g.near_owner) pf = prefetch_near(C, g, *coarse, near_host, near_cap);
  htpre.stop();
  // structure of both passes on host threads while the block norms run on the GPU
  const BView gv{g.bt.get(), false}, gvt{g.bt.get(), true};
  const BView cvw{coarse.get(), false}, cvt{coarse.get(), true};
  auto prep_r = std::async(std::launch::async, [gv, cvw] { return prep_rows(gv, cvw); });
  auto prep_c = std::async(std::launch::async, [gvt, cvt] { return prep_rows(gvt, cvt); });
  Arena sc(C.st);
  cudaEvent_t nn_ready = nullptr;
  struct EvGuard {
    cudaEvent_t& e;
    ~EvGuard() { if (e) cudaEventDestroy(e); }
  } nn_guard{nn_ready};
  double* d_nn = sc.alloc(std::max(1, g.bt->nb));
  double* d_cn = sc.alloc(std::max(1, g.bt->nb));
  if (scale) {
    StageTag tag(C, "p2.norms");
    // the nearfield norms gate the leaf-level SVDs: on a normal-priority auxiliary stream (the
    // low-priority one was starved by the Z levels and made the leaf SVDs wait ~26 ms at c4)
    if (!serial_passes()) all_norms(C, sc, g, d_cn, d_nn, &C.aux(true), &nn_ready);
    else all_norms(C, sc, g, d_cn, d_nn);
  }
  const cudaEvent_t ev_norms = mark_event(C);
  mem_mark("p2 norms");
  prep_r.wait();
  prep_c.wait();
  auto ar = std::make_shared<Arena>(C.st);
  cudaEvent_t ev_r[2] = {}, ev_c[2] = {};  // begin / end of each coarse-basis pass (timing mode)
  // row and column coarse bases are independent until the final projection: concurrent passes
  auto ar2 = std::make_shared<Arena>(C.st);
  CState rs, cs;
  ProjPlan plan;
  if (serial_passes()) {  // profiling aid: deterministic single-stream launch order
    rs = coarse_rows(C, *ar, HView{&g, false}, BView{coarse.get(), false}, tol, max_rank, scale, d_cn, d_nn,
                     prep_r.get());
    cs = coarse_rows(C, *ar2, HView{&g, true}, BView{coarse.get(), true}, tol, max_rank, scale, d_cn, d_nn,
                     prep_c.get());
    plan = plan_project(HView{&g, false}, rs, *coarse);
  } else {
    Ctx& S = C.side();
    ar2->st = S.st;
    C.order_free(*ar2);
    PassGate gate;  // partitioned products: the column pass's collectives follow the row pass's
    C.gate = &gate;
    S.gate = &gate;
    struct GateReset {
      Ctx &a, &b;
      ~GateReset() {
        a.gate_leave();
        a.gate = b.gate = nullptr;
      }
    } gate_reset{C, S};
    std::exception_ptr err;
    std::thread th([&] {
      try {
        ev_c[0] = mark_event(S);
        cs = coarse_rows(S, *ar2, HView{&g, true}, BView{coarse.get(), true}, tol, max_rank, scale, d_cn, d_nn,
                         prep_c.get(), nn_ready);
        ev_c[1] = mark_event(S);
        S.sync();
      } catch (...) {
        err = std::current_exception();
      }
    });
    try {
      ev_r[0] = mark_event(C);
      rs = coarse_rows(C, *ar, HView{&g, false}, BView{coarse.get(), false}, tol, max_rank, scale, d_cn, d_nn,
                       prep_r.get(), nn_ready);
      C.gate_leave();
      ev_r[1] = mark_event(C);
      HostTimer htpp(C, "p2_project_structure");
      plan = plan_project(HView{&g, false}, rs, *coarse);  // while the column pass runs
    } catch (...) {
      C.gate_leave();
      th.join();
      throw;
    }
    th.join();
    if (err) std::rethrow_exception(err);
    C.join_side(S);
  }
  mem_mark("p2 coarse bases");
  if (C.timing) { e1 = C.event(); cudaEventRecord(e1, C.st); }
  e2 = e1;
  StageTag tagp(C, "p2.project");
  auto Z = project_final(C, HView{&g, false}, rs, cs, coarse, ar, plan);
  if (pf.ev) {
    Z->near_on_host = std::move(pf.mask);
    Z->near_host = near_host;
    Z->near_host_ready = pf.ev;
    Z->owned.push_back(pf.arena);
  }
  Z->owned.push_back(ar2);
  if (nn_ready) C.join_side(C.aux(true));  // counters / profile of the auxiliary stream's norms
  Z->own_rows = g.own_rows;
  Z->own_cols = g.own_cols;
  if (C.timing) {
    e3 = C.event();
    cudaEventRecord(e3, C.st);
    C.sync();
    // the reference's t2_row includes the block norms (bench.py:218-224)
    C.times.t2_norms = event_ms(e0, ev_norms);
    C.times.t2_row = ev_r[1] ? event_ms(e0, ev_r[1]) : event_ms(e0, e1);
    C.times.t2_col = event_ms(ev_c[0], ev_c[1]);
    C.times.t2_span = event_ms(e0, e1);
    C.times.t2_mat = event_ms(e2, e3);
  }
  return Z;
}

// Isometric re-factorisation, exact-zero directions dropped (reference h2.py:79-113).
static std::shared_ptr<Basis> orthogonalize(Ctx& C, Arena& out, const Basis& B, MatStore& rmap) {
  const Tree& tr = *B.tree;
  auto q = std::make_shared<Basis>();
  q->tree = &tr;
  q->rank.assign(tr.n, 0);
  q->leaf.assign(tr.n, nullptr);
  q->xfer.assign(tr.n, nullptr);
  rmap.assign(tr.n, Mat{});
  Arena sc(C.st);
  for (int lev = tr.depth; lev >= 0; --lev) {
    const auto& L = tr.by_level[lev];
    GBatch g;
    SvdBatch sv;
    std::vector<Mat> st(L.size()), qb(L.size());
    for (size_t li = 0; li < L.size(); ++li) {
      const int t = L[li];
      if (tr.leaf(t)) {
        st[li] = B.leafm(t);
      } else {
        int m = 0;
        for (int i = 0; i < tr.nkids(t); ++i) m += rmap[tr.kid(t, i)].r;
        st[li] = Mat{sc.alloc((size_t)m * B.rank[t]), m, B.rank[t]};
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {
          const int c = tr.kid(t, i);
          g.out(st[li].band(off, rmap[c].r), false);
          g.t2(rmap[c].ref(), B.xferm(c).ref(), rmap[c].c);
          off += rmap[c].r;
        }
      }
      SvdItem it{};
      it.s0 = sv.sl.begin();
      sv.sl.add(st[li].ref(), st[li].c);
      it.s1 = sv.sl.begin();
      it.m = st[li].r;
      it.N = st[li].c;
      it.tol = 0.0;
      it.cap = -1;
      const int kc = std::min(st[li].r, st[li].c);
      qb[li] = Mat{out.alloc((size_t)st[li].r * kc), st[li].r, kc};
      it.q_out = qb[li].p;
      sv.items.push_back(it);
    }
    g.run(C);
    std::vector<int> rk = sv.run(C, sc);
    mem_mark(("p2 L" + std::to_string(lev) + " ch" + std::to_string(C.channel) + " svd").c_str());
    GBatch g2;
    for (size_t li = 0; li < L.size(); ++li) {
      const int t = L[li];
      const int k = rk[li];
      const Mat Q{qb[li].p, st[li].r, k};
      q->rank[t] = k;
      rmap[t] = Mat{out.alloc((size_t)k * st[li].c), k, st[li].c};  // sigma V^T = U^T stacked
      g2.out(rmap[t], false);
      g2.t2(Q.tref(), st[li].ref(), Q.r);
      if (tr.leaf(t)) {
        q->leaf[t] = Q.p;
      } else {
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {
          const int c = tr.kid(t, i);
          q->xfer[c] = Q.p + (long long)off * k;
          off += q->rank[c];
        }
      }
    }
    g2.run(C);
  }
  return q;
}

// Input preparation: orthogonalise, then coarsen onto the own block tree (coarsening.py:425-445).
std::shared_ptr<H2> recompress(Ctx& C, const H2& g, double tol, int max_rank) {
  g.start_near(C);
  auto ar = std::make_shared<Arena>(C.st);
  MatStore rr, rc;
  auto qr = orthogonalize(C, *ar, *g.rb, rr);
  std::shared_ptr<Basis> qc;
  if (g.cb == g.rb) {
    qc = qr;
    rc = rr;
  } else {
    qc = orthogonalize(C, *ar, *g.cb, rc);
  }
  H2 o;
  o.bt = g.bt;
  o.rb = qr;
  o.cb = qc;
  o.near = g.near;
  o.owned = g.owned;
  o.owned.push_back(ar);
  o.own_rows = g.own_rows;
  o.own_cols = g.own_cols;
  o.coup.assign(g.bt->nb, nullptr);
  GBatch gb;
  HView v{&g, false};
  for (int b = 0; b < g.bt->nb; ++b) {
    if (!g.bt->adm_leaf(b)) continue;
    const int t = g.bt->row[b], s = g.bt->col[b];
    Mat S{ar->alloc((size_t)rr[t].r * rc[s].r), rr[t].r, rc[s].r};
    o.coup[b] = S.p;
    gb.out(S, false);
    gb.t3(rr[t].ref(), v.coup(b), rc[s].tref(), rr[t].c, rc[s].c);
  }
  gb.run(C);
  return coarsen(C, o, g.bt, tol, max_rank, true);
}

// ------------------------------------------------------------------ stage-level entry points
struct CoarseStage {
  CState st;
  ArenaPtr ar;
  bool T = false;
  const H2* g = nullptr;
  std::shared_ptr<const Blocks> coarse;
};

void block_norms_stage(Ctx& C, const H2& g, double* d_cn, double* d_nn) {
  wait_near(C, g);
  Arena sc(C.st);
  all_norms(C, sc, g, d_cn, d_nn);
  C.sync();
}

// build_coarse_row_basis / build_coarse_col_basis (coarsening.py:187-339): one pass, on G (col =
// false) or G^T with the transposed coarse tree (col = true).  Norms: given device arrays (per block
// of G) or, with scale_blocks and none given, computed here (coarsening.py:342-351).
std::shared_ptr<CoarseStage> coarse_basis_stage(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, bool col,
                                                double tol, int max_rank, bool scale, const double* d_cn,
                                                const double* d_nn) {
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  wait_near(C, g);
  auto out = std::make_shared<CoarseStage>();
  out->ar = std::make_shared<Arena>(C.st);
  out->T = col;
  out->g = &g;
  out->coarse = coarse;
  const BView gv{g.bt.get(), col}, cv{coarse.get(), col};
  const CPrep prep = prep_rows(gv, cv);
  Arena sc(C.st);
  if (scale && (!d_cn || !d_nn)) {
    double* cn = sc.alloc(std::max(1, g.bt->nb));
    double* nn = sc.alloc(std::max(1, g.bt->nb));
    all_norms(C, sc, g, cn, nn);
    if (!d_cn) d_cn = cn;
    if (!d_nn) d_nn = nn;
  }
  out->st = coarse_rows(C, *out->ar, HView{&g, col}, cv, tol, max_rank, scale, d_cn, d_nn, prep);
  C.sync();
  return out;
}

// project_final (coarsening.py:354-405) from the two pass states of the same G and coarse tree.
std::shared_ptr<H2> project_final_stage(Ctx& C, const H2& g, const CoarseStage& rs, const CoarseStage& cs,
                                        std::shared_ptr<const Blocks> coarse) {
  if (rs.T || !cs.T) throw InvalidInput("project_final needs a row state and a column state");
  if (rs.g != &g || cs.g != &g) throw InvalidInput("the coarsen states belong to another product");
  if (rs.coarse.get() != coarse.get() || cs.coarse.get() != coarse.get())
    throw InvalidInput("the coarsen states were built for another coarse block tree");
  wait_near(C, g);
  CState& r = const_cast<CState&>(rs.st);  // read only (states stay reusable)
  CState& c = const_cast<CState&>(cs.st);
  const ProjPlan plan = plan_project(HView{&g, false}, r, *coarse);
  auto ar = std::make_shared<Arena>(C.st);
  auto Z = project_final(C, HView{&g, false}, r, c, coarse, ar, plan);
  Z->owned.push_back(rs.ar);
  Z->owned.push_back(cs.ar);
  Z->own_rows = g.own_rows;
  Z->own_cols = g.own_cols;
  C.sync();
  return Z;
}

std::shared_ptr<Basis> coarse_stage_basis(const CoarseStage& s, MatStore* r, MatStore* z, ArenaPtr* ar, int* nreps) {
  if (r) *r = s.st.r;
  if (z) *z = s.st.z;
  if (ar) *ar = s.ar;
  if (nreps) {
    int n = 0;
    for (const auto& rep : s.st.reps) n += rep.t != nullptr;
    *nreps = n;
  }
  return s.st.q;
}

}  // namespace h2g
