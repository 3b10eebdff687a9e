// Phase 1 of the product: compressed induced bases (Fig. 3) and exact-structure assembly over
// the refined product tree (reference induced.py:49-372).
#include <algorithm>
#include <cmath>
#include <functional>
#include <future>
#include <thread>

#include "engine.h"

namespace h2g {

// X|ts V_Y,s for leaf row clusters t by block descent (reference induced.py:59-73).
// Each requested block and every block below it (same row t) is computed once, deepest first;
// `memo` is indexed by block id of the view x.
void xv_compute(Ctx& C, Arena& ar, HView x, HView y, PRef P, const std::vector<int>& want,
                std::vector<Mat>& memo) {
  const Blocks& B = *x.h->bt;
  if ((int)memo.size() < B.nb) memo.resize(B.nb);
  std::vector<std::vector<int>> by_h;   // block ids by height
  std::vector<int> height(B.nb, -2);   // -2: not scheduled by this call
  std::function<int(int)> visit = [&](int b) -> int {
    if (height[b] != -2) return height[b];
    if (memo[b].p || (memo[b].r > 0 && memo[b].c == 0)) return -1;  // computed by an earlier call
    int h = 0;
    for (int i = 0; i < B.nkids(b); ++i) h = std::max(h, visit(B.kid(b, i)) + 1);
    height[b] = h;
    if ((int)by_h.size() <= h) by_h.resize(h + 1);
    by_h[h].push_back(b);
    return h;
  };
  for (int b : want) {
    if (b < 0) throw StructureErr("xv: pair not in the block tree");
    visit(b);
  }
  const Basis& VX = x.rb();
  const Basis& VY = y.rb();
  const Tree& rows = x.rows();
  for (auto& lvl : by_h) {
    GBatch g;
    for (int b : lvl) {
      const int t = x.row(b), s = x.col(b);
      Mat m{ar.alloc((size_t)rows.size(t) * VY.rank[s]), rows.size(t), VY.rank[s]};
      memo[b] = m;
      g.out(m, false);
      if (B.adm_leaf(b)) {
        g.t3(VX.leafm(t).ref(), x.coup(b), P.at(s), VX.rank[t], P.rows(s));
      } else if (B.leaf(b)) {
        g.t2(x.near(b), VY.leafm(s).ref(), VY.tree->size(s));
      } else {
        for (int i = 0; i < B.nkids(b); ++i) {
          const int b2 = B.kid(b, i);
          const int s2 = x.col(b2);
          const Mat part = memo[b2];
          if (s2 != s) g.t2(part.ref(), VY.xferm(s2).ref(), VY.rank[s2]);
          else g.t1(part.ref());
        }
      }
    }
    g.run(C);
  }
}

// Multi-GPU: after the partitioned levels (>= part.level) every rank receives the other ranks'
// results -- ranks, Q_t (leaf basis or the stacked transfers), basis_change and the projections
// A_ts -- so the replicated top levels and the later stages see the full induced basis.
static void exchange_induced(Ctx& C, Arena& out, const Part& part, HView x, HView y,
                             const std::vector<std::vector<int>>& mids, Induced& R, bool row_proj_local) {
  const Tree& tr = x.rows();
  const Basis& VX = x.rb();
  const Basis& VY = y.rb();
  Basis& q = *R.q;
  std::vector<int> ids;
  for (int l = part.level; l <= tr.depth; ++l)
    for (int t : tr.by_level[l]) ids.push_back(t);
  StageTag tag(C, "p1.exchange");
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
    else R.bc[t] = Mat{nullptr, k, VX.rank[t]};
    items.push_back(XItem{o, (long long)m * k, &qp[t]});
    items.push_back(XItem{o, (long long)k * VX.rank[t], &R.bc[t].p});
    // projections A_ts: the assembly reads only its own rows' (and the replicated top's), and the
    // top levels' ahat only those of the partition level's clusters -- the deeper rows stay local
    // for the row pass (row_proj_local); the column pass's are read by every rank's assembly
    // (product blocks of own rows reach columns of every rank), so they are all exchanged
    static const bool proj_all = getenv("H2G_PROJ_ALL") != nullptr;  // A/B: exchange every projection
    if (row_proj_local && !proj_all && tr.level[t] != part.level) continue;
    for (int b : mids[t]) {
      const int ky = VY.rank[x.col(b)];
      if (o != part.me) R.proj[b] = Mat{nullptr, k, ky};
      items.push_back(XItem{o, (long long)k * ky, &R.proj[b].p});
    }
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
}

// Fig. 3: bottom-up compression of the induced row basis (reference induced.py:76-184).
Induced induced_rows(Ctx& C, Arena& out, HView x, HView y, const MatStore& zy, PRef P, double tol,
                     int max_rank, bool scale, double level_decay) {
  if (!x.cols().same(y.rows())) throw InvalidInput("x and y do not share the middle cluster tree");
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  const Blocks& B = *x.h->bt;
  const Tree& tr = x.rows();
  const Basis& VX = x.rb();
  const Basis& VY = y.rb();
  Arena sc(C.st);
  // middles: columns of the non-admissible-leaf blocks per row cluster, block preorder (induced.py:49-56)
  std::vector<std::vector<int>> mids(tr.n);
  for (int b = 0; b < B.nb; ++b)
    if (!B.adm_leaf(b)) mids[x.row(b)].push_back(b);

  wait_near(C, *x.h);  // X|ts and Y|sr dense blocks are read from here on
  wait_near(C, *y.h);
  Induced R;
  R.q = std::make_shared<Basis>();
  Basis& q = *R.q;
  q.tree = &tr;
  q.rank.assign(tr.n, 0);
  q.leaf.assign(tr.n, nullptr);
  q.xfer.assign(tr.n, nullptr);
  R.bc.assign(tr.n, Mat{});

  const Part part = make_part(tr, C.comm);  // multi-GPU: this rank's subtrees (all of tr when P = 1)
  std::vector<int> leaf_blocks;
  for (int t = 0; t < tr.n; ++t)
    if (tr.leaf(t) && part.mine(t))
      for (int b : mids[t]) leaf_blocks.push_back(b);
  R.proj.assign(B.nb, Mat{});
  {
    StageTag tag(C, "p1.xv");
    xv_compute(C, out, x, y, P, leaf_blocks, R.xv);
  }

  std::vector<Mat> blk(B.nb);
  std::vector<Mat> vx(tr.n);
  std::vector<Mat> rfb(B.nb);
  std::vector<int> Lp;
  double* d_nrm = sc.alloc(std::max(1, B.nb));  // sigma_1 per block (0: absent from the SVD stacks)
  cuda_check(cudaMemsetAsync(d_nrm, 0, sizeof(double) * std::max(1, B.nb), C.st), "memset");
  for (int lev = tr.depth; lev >= 0; --lev) {
    if (part.on()) Lp = part.filter(tr.by_level[lev]);
    const std::vector<int>& L = part.on() ? Lp : tr.by_level[lev];
    StageTag tag(C, "p1.L" + std::to_string(lev));
    // this level's temporaries (vhat, projected blocks, ahat, weighted stacks, SVD scratch): freed
    // stream-ordered at the end of the level
    Arena lvl(C.st);
    GBatch g1, g2;
    std::vector<Mat>& rf = rfb;
    for (int t : L) {
      if (tr.leaf(t)) {
        vx[t] = VX.leafm(t);
        for (int b : mids[t]) blk[b] = R.xv[b];
        continue;
      }
      const int kx = VX.rank[t];
      int m = 0;
      for (int i = 0; i < tr.nkids(t); ++i) m += q.rank[tr.kid(t, i)];
      Mat vh{lvl.alloc((size_t)m * kx), m, kx};
      int off = 0;
      for (int i = 0; i < tr.nkids(t); ++i) {  // vhat = vstack(bc_c E_X,c) (induced.py:177-178)
        const int c = tr.kid(t, i);
        g1.out(vh.band(off, q.rank[c]), false);
        g1.t2(R.bc[c].ref(), VX.xferm(c).ref(), R.bc[c].c);
        off += q.rank[c];
      }
      vx[t] = vh;
      for (int b : mids[t])
        for (int i = 0; i < B.nkids(b); ++i) {  // projected_block for admissible children (induced.py:148-153)
          const int b2 = B.kid(b, i);
          if (!B.adm_leaf(b2)) continue;
          const int t2 = x.row(b2), s2 = x.col(b2);
          Mat m2{lvl.alloc((size_t)q.rank[t2] * VY.rank[s2]), q.rank[t2], VY.rank[s2]};
          g1.out(m2, false);
          g1.t3(R.bc[t2].ref(), x.coup(b2), P.at(s2), R.bc[t2].c, P.rows(s2));
          rf[b2] = m2;
        }
    }
    g1.run(C);
    for (int t : L) {  // ahat (induced.py:155-167), one output band per child row cluster
      if (tr.leaf(t)) continue;
      const int m = vx[t].r;
      for (int b : mids[t]) {
        const int s = x.col(b);
        Mat A{lvl.alloc((size_t)m * VY.rank[s]), m, VY.rank[s]};
        blk[b] = A;
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {
          const int c = tr.kid(t, i);
          g2.out(A.band(off, q.rank[c]), false);
          for (int j = 0; j < B.nkids(b); ++j) {
            const int b2 = B.kid(b, j);
            if (x.row(b2) != c) continue;
            const int s2 = x.col(b2);
            const Mat pb = B.adm_leaf(b2) ? rf[b2] : R.proj[b2];
            if (s2 != s) g2.t2(pb.ref(), VY.xferm(s2).ref(), VY.rank[s2]);
            else g2.t1(pb.ref());
          }
          off += q.rank[c];
        }
      }
    }
    g2.run(C);

    // block norms for block-relative scaling (induced.py:121-125), left on the device: they divide
    // the SVD segments there, and the SVD drops the columns of exact-zero blocks (SvdItem::zskip)
    // -- no host synchronisation for them
    if (scale) {
      NormBatch nbat;
      for (int t : L)
        for (int b : mids[t]) {
          NormItem it{};
          it.s0 = nbat.sl.begin();
          nbat.sl.add(blk[b].ref(), blk[b].c);
          it.s1 = nbat.sl.begin();
          it.m = blk[b].r;
          it.N = blk[b].c;
          it.out = d_nrm + b;
          nbat.items.push_back(it);
        }
      nbat.scratch = &lvl;
      nbat.run_async(C);
    }

    // weighted stack w_i = blk_i Z_s^T / ||blk_i|| and the protected truncated SVD (induced.py:115-146)
    GBatch g3;
    SvdBatch sv;
    std::vector<Mat> qbuf(L.size()), bcbuf(L.size());
    for (size_t li = 0; li < L.size(); ++li) {
      const int t = L[li];
      const int m = vx[t].r, kx = vx[t].c, k1 = std::min(m, kx);
      SvdItem it{};
      it.s0 = sv.sl.begin();
      long long N = 0;
      for (int b : mids[t]) {
        const Mat& Z = zy[x.col(b)];
        if (Z.r == 0 || m == 0) continue;
        Mat w{lvl.alloc((size_t)m * Z.r), m, Z.r};
        g3.out(w, false);
        g3.t2(blk[b].ref(), Z.tref(), Z.c);
        sv.sl.add(w.ref(), Z.r, 1.0, scale ? d_nrm + b : nullptr);  // w_i = blk_i Z_s^T / ||blk_i||
        N += Z.r;
      }
      it.s1 = sv.sl.begin();
      it.m = m;
      it.kx = kx;
      it.N = N;
      it.v = vx[t].ref();
      it.zskip = scale ? 1 : 0;
      it.tol = tol * std::pow(level_decay, (double)lev);
      it.cap = max_rank < 0 ? -1 : std::max(0, max_rank - k1);
      const long long kcap = std::min<long long>(m, k1 + N);
      qbuf[li] = Mat{out.alloc((size_t)m * kcap), m, (int)kcap};
      bcbuf[li] = Mat{out.alloc((size_t)kcap * kx), (int)kcap, kx};
      it.q_out = qbuf[li].p;
      it.bc_out = bcbuf[li].p;
      sv.items.push_back(it);
    }
    g3.run(C);
    std::vector<int> rk = sv.run(C, lvl);

    GBatch g4;
    for (size_t li = 0; li < L.size(); ++li) {
      const int t = L[li];
      const int k = rk[li];
      const int m = vx[t].r, kx = vx[t].c;
      q.rank[t] = k;
      Mat Q{qbuf[li].p, m, k};
      R.bc[t] = Mat{bcbuf[li].p, k, kx};
      if (tr.leaf(t)) {
        q.leaf[t] = Q.p;
      } else {
        int off = 0;
        for (int i = 0; i < tr.nkids(t); ++i) {  // transfers = row split of Q_t (induced.py:143-146)
          const int c = tr.kid(t, i);
          q.xfer[c] = Q.p + (long long)off * k;
          off += q.rank[c];
        }
      }
      for (int b : mids[t]) {  // A_ts = Q_t^T blk for every middle (induced.py:138-139)
        const int s = x.col(b);
        Mat pm{out.alloc((size_t)k * VY.rank[s]), k, VY.rank[s]};
        g4.out(pm, false);
        g4.t2(Q.tref(), blk[b].ref(), m);
        R.proj[b] = pm;
      }
    }
    g4.run(C);
    for (int t : L)  // blk / rf entries of this level point into lvl
      if (!tr.leaf(t))
        for (int b : mids[t]) {
          blk[b] = Mat{};
          for (int i = 0; i < B.nkids(b); ++i) rfb[B.kid(b, i)] = Mat{};
        }
    mem_mark(("p1 L" + std::to_string(lev) + " ch" + std::to_string(C.channel)).c_str());
    if (part.on() && lev == part.level) {
      C.gate_enter();
      exchange_induced(C, out, part, x, y, mids, R, !x.T);  // row pass: x is X itself (not transposed)
      C.gate_leave();
    }
  }
  return R;
}

static void emit_push(GBatch& g, const Mat* E, const Mat& S, const Mat* F) {
  if (E && F) g.t3(E->ref(), S.ref(), F->tref(), E->c, S.c);
  else if (E) g.t2(E->ref(), S.ref(), E->c);
  else if (F) g.t2(S.ref(), F->tref(), S.c);
  else g.t1(S.ref());
}

// Dense targets of the product (inadmissible T^XY leaves) take only input factors -- kind a:
// (X|ts V_Y,s) S_Y W_Y,r^T, kind b: V_X,t S_X (Y|sr^T W_X,s)^T, kind c: N_X N_Y (induced.py:
// 286-307) -- so they are assembled as soon as T^XY exists, on the low-priority auxiliary stream,
// while the induced bases (the level-serial critical path) run.  assemble() then adds the push-down.
void assemble_dense_early(Ctx& A, HView x, HView y, PRef P, PTree& pt, cudaEvent_t inputs_ready, const Comm& comm) {
  const Blocks& B = *pt.bt;
  const Tree& rows = *B.rows;
  const Tree& cols = *B.cols;
  const Part part = make_part(rows, comm);
  PTree::Early& E = pt.early;
  E.near = std::make_shared<Arena>(A.st);
  E.near->cross_stream = true;  // read and written by the main stream later
  E.scratch = std::make_shared<Arena>(A.st);
  E.blk.assign(B.nb, nullptr);
  for (int b = 0; b < B.nb; ++b)
    if (B.near_leaf(b) && part.mine(B.row[b]))
      E.blk[b] = E.near->alloc((size_t)rows.size(B.row[b]) * cols.size(B.col[b]));
  if (inputs_ready) cuda_check(cudaStreamWaitEvent(A.st, inputs_ready, 0), "wait inputs");
  wait_near(A, *x.h);
  wait_near(A, *y.h);
  if (pt.dev.ready) cuda_check(cudaStreamWaitEvent(A.st, pt.dev.ready, 0), "wait upload");
  // memoised leaf products of the dense targets (induced.py:245-258)
  std::vector<Mat> xv, wy;
  HView yT{y.h, !y.T}, xT{x.h, !x.T};
  {
    std::vector<int> want;
    for (int b : pt.need_xv)
      if (part.mine(x.row(b))) want.push_back(b);
    xv_compute(A, *E.scratch, x, y, P, want, xv);
  }
  xv_compute(A, *E.scratch, yT, xT, PRef{P.P, !P.T}, pt.need_wy, wy);
  const Blocks& BX = *x.h->bt;
  const Blocks& BY = *y.h->bt;
  const Tree& mid = x.cols();
  const int ntrip = (int)pt.ts.size();
  std::vector<unsigned char> ndense(B.nb), xadm(BX.nb);
  for (int b = 0; b < B.nb; ++b) ndense[b] = B.near_leaf(b) ? 1 : 0;
  const MatRef z{nullptr, 0, 0};
  std::vector<MatRef> xcoup(BX.nb, z), xnear(BX.nb, z), xvr(BX.nb, z);
  for (int b = 0; b < BX.nb; ++b) {
    xadm[b] = BX.adm_leaf(b) ? 1 : 0;
    if (BX.adm_leaf(b)) xcoup[b] = x.coup(b);
    if (BX.near_leaf(b)) xnear[b] = x.near(b);
    if (b < (int)xv.size()) xvr[b] = xv[b].ref();
  }
  std::vector<MatRef> ycoup(BY.nb, z), ynear(BY.nb, z), wyl(BY.nb, z);
  for (int b = 0; b < BY.nb; ++b) {
    if (BY.adm_leaf(b)) ycoup[b] = y.coup(b);
    if (BY.near_leaf(b)) ynear[b] = y.near(b);
    if (b < (int)wy.size()) wyl[b] = wy[b].ref();
  }
  std::vector<MatRef> vxleaf(rows.n, z), wyleaf(cols.n, z);
  for (int t = 0; t < rows.n; ++t)
    if (rows.leaf(t)) vxleaf[t] = x.rb().leafm(t).ref();
  for (int r = 0; r < cols.n; ++r)
    if (cols.leaf(r)) wyleaf[r] = y.cb().leafm(r).ref();
  std::vector<int> size_mid(mid.n);
  for (int s = 0; s < mid.n; ++s) size_mid[s] = mid.size(s);
  AsmTables T{};
  T.tnode = pt.dev.tnode;
  T.ts = pt.dev.ts;
  T.tk = pt.dev.tk;
  T.tbx = pt.dev.tbx;
  T.tby = pt.dev.tby;
  T.node_row = A.push(B.row);
  T.node_col = A.push(B.col);
  T.node_dense = A.push(ndense);
  T.xcoup = A.push(xcoup);
  T.xnear = A.push(xnear);
  T.xadm = A.push(xadm);
  T.xv = A.push(xvr);
  T.ycoup = A.push(ycoup);
  T.ynear = A.push(ynear);
  T.wyl = A.push(wyl);
  T.vxleaf = A.push(vxleaf);
  T.wyleaf = A.push(wyleaf);
  T.kx_row = A.push(x.rb().rank);
  T.kwx_mid = A.push(x.cb().rank);
  T.ky_mid = A.push(y.rb().rank);
  T.kwy_col = A.push(y.cb().rank);
  T.size_mid = A.push(size_mid);
  T.grouped = 1;
  T.only = 1;  // coupling targets need the induced bases: assemble() does them
  GTerm* d_terms = (GTerm*)E.scratch->alloc_bytes(sizeof(GTerm) * std::max(1, ntrip));
  A.flush();
  cuda_check(launch_asm_expand(T, ntrip, d_terms, A.st), "asm_expand(dense)");
  ++A.launches;
  GBatch g;
  int k2max = 0;
  for (int k : y.cb().rank) k2max = std::max(k2max, k);
  for (int k : x.cb().rank) k2max = std::max(k2max, k);
  if (k2max > 256) throw StructureErr("gsum: 3-factor middle dimension above 256");
  g.k2max = std::max(k2max, 64);
  double fl = 0.0;
  for (int b = 0; b < B.nb; ++b) {
    if (!E.blk[b]) continue;
    const int t = B.row[b], r = B.col[b];
    const Mat tgt{E.blk[b], rows.size(t), cols.size(r)};
    GOut o{tgt.p, tgt.c, tgt.r, tgt.c, 0, pt.tptr[b], pt.tptr[b + 1]};
    const int ka = y.cb().rank[r], kb = x.rb().rank[t];
    if (ka <= 64) {
      o.ka = ka;
      o.da = y.cb().leafm(r).tref();
    }
    if (kb <= 64) {
      o.kb = kb;
      o.ab = x.rb().leafm(t).ref();
    }
    g.outs.push_back(o);
    if (A.prof)
      for (int i = pt.tptr[b]; i < pt.tptr[b + 1]; ++i) {
        const int s = pt.ts[i];
        const double m = tgt.r, n = tgt.c;
        if (pt.tk[i] == 'c') fl += 2 * m * n * mid.size(s);
        else if (pt.tk[i] == 'a') fl += 2 * m * y.rb().rank[s] * ka + 2 * m * ka * n;
        else fl += 2 * m * kb * x.cb().rank[s] + 2 * m * x.cb().rank[s] * n;
      }
  }
  {
    StageTag tag(A, "p1.dense");
    g.tag = 1;  // gsum_mma_kernel<1>: the dense-target launch, selectable by name in ncu
    g.run_device_terms(A, d_terms, fl);
  }
  cuda_check(cudaEventCreateWithFlags(&E.done, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(E.done, A.st), "event");
  A.flush();
  E.on = true;
}

// Row factors of the admissible X blocks of kind-a triples: bc_t S_X P_s (induced.py:260-265).
// They need only the row basis, so multiply() issues them as soon as the row pass is done, in the
// shadow of the column pass.
std::vector<Mat> row_factors(Ctx& C, Arena& sc, HView x, HView y, const Induced& qr, PRef P, const PTree& pt) {
  HostTimer hx(C, "asm_rf");
  const Basis& Q = *qr.q;
  const Part part = make_part(*pt.bt->rows, C.comm);
  std::vector<Mat> rf(x.h->bt->nb);
  GBatch g;
  for (int bts : pt.rf_blocks) {  // (planner thread: distinct X blocks of kind-a triples)
    const int t = x.row(bts), s = x.col(bts);
    if (!part.mine(t)) continue;
    Mat m{sc.alloc((size_t)Q.rank[t] * y.rb().rank[s]), Q.rank[t], y.rb().rank[s]};
    g.out(m, false);
    g.t3(qr.bc[t].ref(), x.coup(bts), P.at(s), qr.bc[t].c, P.rows(s));
    rf[bts] = m;
  }
  g.run(C);
  return rf;
}

// Product over T^XY in the induced bases + push-down (reference induced.py:220-355).
std::shared_ptr<H2> assemble(Ctx& C, HView x, HView y, Induced& qr, Induced& qc, PRef P, PTree& pt,
                             const std::vector<Mat>* rf_pre) {
  HostTimer ht(C, "assemble_total");
  HostTimer htpro(C, "asm_prologue");
  auto G = std::make_shared<H2>();
  G->bt = pt.bt;
  G->rb = qr.q;
  G->cb = qc.q;
  auto ar = std::make_shared<Arena>(C.st);
  G->owned.push_back(ar);
  G->near_owner = ar;
  const bool early = pt.early.on;  // dense targets already queued on the auxiliary stream
  if (early) {
    G->owned.push_back(pt.early.near);
    G->near_owner = pt.early.near;
  }
  Arena sc(C.st);
  const Blocks& B = *pt.bt;
  const Tree& rows = *B.rows;
  const Tree& cols = *B.cols;
  const BView bx = x.bv(), by = y.bv();
  const Basis& Q = *qr.q;
  const Basis& W = *qc.q;
  G->coup.assign(B.nb, nullptr);
  G->near.assign(B.nb, nullptr);
  // multi-GPU: this rank assembles the product blocks of its row subtrees (and the replicated top)
  const Part part = make_part(rows, C.comm);
  std::vector<Mat> cp(B.nb);
  for (int b = 0; b < B.nb; ++b) {
    const int t = B.row[b], r = B.col[b];
    if (!part.mine(t)) continue;
    if (B.near_leaf(b)) {
      G->near[b] = early ? pt.early.blk[b] : ar->alloc((size_t)rows.size(t) * cols.size(r));
    } else {
      Arena& a = B.adm_leaf(b) ? *ar : sc;
      cp[b] = Mat{a.alloc((size_t)Q.rank[t] * W.rank[r]), Q.rank[t], W.rank[r]};
      if (B.adm_leaf(b)) G->coup[b] = cp[b].p;
    }
  }
  htpro.stop();
  // the grouped launch's output list (one GOut per product block, its 64x64 tiles) is pure
  // structure: built on a helper thread while this one issues the xv / row-factor work and tables
  const bool prof = C.prof;
  auto outs_fut = std::async(std::launch::async, [&, prof] {
    GBatch g;
    int k2max = 0;
    for (int k : y.cb().rank) k2max = std::max(k2max, k);
    for (int k : x.cb().rank) k2max = std::max(k2max, k);
    if (k2max > 256) throw StructureErr("gsum: 3-factor middle dimension above 256");
    g.k2max = std::max(k2max, 64);  // group sums T (64 x ka) / U (kb x 64) share the Ts buffer
    g.outs.reserve(B.nb);
    double fl = 0.0;
    const Tree& mid = x.cols();
    for (int b = 0; b < B.nb; ++b) {
      const int t = B.row[b], r = B.col[b];
      if (!part.mine(t)) continue;
      const bool dense = B.near_leaf(b);
      if (dense && early) continue;
      const Mat tgt = dense ? Mat{G->near[b], rows.size(t), cols.size(r)} : cp[b];
      GOut o{tgt.p, tgt.c, tgt.r, tgt.c, 0, pt.tptr[b], pt.tptr[b + 1]};
      // grouped kind-a / kind-b terms (asm_expand_kernel emits nf = 4 / 5 under the same rule)
      const int ka = y.cb().rank[r], kb = x.rb().rank[t];
      if (ka <= 64) {
        o.ka = ka;
        o.da = dense ? y.cb().leafm(r).tref() : qc.bc[r].tref();
      }
      if (kb <= 64) {
        o.kb = kb;
        o.ab = dense ? x.rb().leafm(t).ref() : qr.bc[t].ref();
      }
      g.outs.push_back(o);
      if (prof)
        for (int i = pt.tptr[b]; i < pt.tptr[b + 1]; ++i) {
          const int s = pt.ts[i];
          const double m = tgt.r, n = tgt.c;
          if (pt.tk[i] == 'c') fl += 2 * m * n * mid.size(s);
          else if (pt.tk[i] == 'a') {
            const double k = y.rb().rank[s], k2 = y.cb().rank[r];
            fl += 2 * m * k * k2 + 2 * m * k2 * n;
          } else {
            const double k = x.rb().rank[t], k2 = x.cb().rank[s];
            fl += 2 * m * k * k2 + 2 * m * k2 * n;
          }
        }
    }
    g.whole = true;  // one CTA per output up to 128 x 128, grouped intermediates cached across its tiles
    g.prepare_tiles();
    return std::make_pair(std::move(g), fl);
  });
  struct JoinOuts {  // never leave the helper running past an exception
    std::future<std::pair<GBatch, double>>& f;
    ~JoinOuts() { if (f.valid()) f.wait(); }
  } join_outs{outs_fut};
  // memoised leaf products needed by dense targets, and row factors of admissible X blocks
  HostTimer ht1(C, "assemble_xv_rf");
  HView yT{y.h, !y.T}, xT{x.h, !x.T};
  if (!early) {
    HostTimer hx(C, "asm_xv1");
    if (part.on()) {
      std::vector<int> want;
      for (int b : pt.need_xv)
        if (part.mine(x.row(b))) want.push_back(b);
      xv_compute(C, sc, x, y, P, want, qr.xv);
    } else {
      xv_compute(C, sc, x, y, P, pt.need_xv, qr.xv);
    }
  }
  if (!early) {
    HostTimer hx(C, "asm_xv2");
    xv_compute(C, sc, yT, xT, PRef{P.P, !P.T}, pt.need_wy, qc.xv);
  }
  std::vector<Mat> rf_local;
  if (!rf_pre) rf_local = row_factors(C, sc, x, y, qr, P, pt);
  const std::vector<Mat>& rf = rf_pre ? *rf_pre : rf_local;
  // all terminal triples (induced.py:286-307), one output per product block; the terms are
  // expanded on the GPU from the triple list and per-block operand tables (asm_expand_kernel)
  {
    HostTimer ht2(C, "assemble_triples");
    const int ntrip = (int)pt.ts.size();
    const Blocks& BX = *x.h->bt;
    const Blocks& BY = *y.h->bt;
    const Tree& mid = x.cols();
    std::vector<unsigned char> ndense(B.nb), xadm(BX.nb);
    for (int b = 0; b < B.nb; ++b) ndense[b] = B.near_leaf(b) ? 1 : 0;
    const MatRef z{nullptr, 0, 0};
    std::vector<MatRef> xcoup(BX.nb, z), xnear(BX.nb, z), rfr(BX.nb, z), rproj(BX.nb, z), xvr(BX.nb, z);
    for (int b = 0; b < BX.nb; ++b) {
      xadm[b] = BX.adm_leaf(b) ? 1 : 0;
      if (BX.adm_leaf(b)) xcoup[b] = x.coup(b);
      if (BX.near_leaf(b)) xnear[b] = x.near(b);
      rfr[b] = rf[b].ref();
      if (b < (int)qr.proj.size()) rproj[b] = qr.proj[b].ref();
      if (b < (int)qr.xv.size()) xvr[b] = qr.xv[b].ref();
    }
    std::vector<MatRef> ycoup(BY.nb, z), ynear(BY.nb, z), cproj(BY.nb, z), wyl(BY.nb, z);
    for (int b = 0; b < BY.nb; ++b) {
      if (BY.adm_leaf(b)) ycoup[b] = y.coup(b);
      if (BY.near_leaf(b)) ynear[b] = y.near(b);
      if (b < (int)qc.proj.size()) cproj[b] = qc.proj[b].ref();
      if (b < (int)qc.xv.size()) wyl[b] = qc.xv[b].ref();
    }
    std::vector<MatRef> vxleaf(rows.n, z), bcr(rows.n, z), wyleaf(cols.n, z), bcc(cols.n, z);
    for (int t = 0; t < rows.n; ++t) {
      if (rows.leaf(t)) vxleaf[t] = x.rb().leafm(t).ref();
      bcr[t] = qr.bc[t].ref();
    }
    for (int r = 0; r < cols.n; ++r) {
      if (cols.leaf(r)) wyleaf[r] = y.cb().leafm(r).ref();
      bcc[r] = qc.bc[r].ref();
    }
    HostTimer htt(C, "asm_tables");
    std::vector<int> size_mid(mid.n);
    for (int s = 0; s < mid.n; ++s) size_mid[s] = mid.size(s);
    AsmTables T{};
    T.tnode = pt.dev.tnode;
    T.ts = pt.dev.ts;
    T.tk = pt.dev.tk;
    T.tbx = pt.dev.tbx;
    T.tby = pt.dev.tby;
    cudaEvent_t sw = C.sub_begin();
    if (pt.dev.ready) cuda_check(cudaStreamWaitEvent(C.st, pt.dev.ready, 0), "wait upload");
    T.node_row = C.push(B.row);
    T.node_col = C.push(B.col);
    T.node_dense = C.push(ndense);
    T.xcoup = C.push(xcoup);
    T.xnear = C.push(xnear);
    T.xadm = C.push(xadm);
    T.rf = C.push(rfr);
    T.rproj = C.push(rproj);
    T.xv = C.push(xvr);
    T.ycoup = C.push(ycoup);
    T.ynear = C.push(ynear);
    T.cproj = C.push(cproj);
    T.wyl = C.push(wyl);
    T.vxleaf = C.push(vxleaf);
    T.bcr = C.push(bcr);
    T.wyleaf = C.push(wyleaf);
    T.bcc = C.push(bcc);
    T.kx_row = C.push(x.rb().rank);
    T.kwx_mid = C.push(x.cb().rank);
    T.ky_mid = C.push(y.rb().rank);
    T.kwy_col = C.push(y.cb().rank);
    T.size_mid = C.push(size_mid);
    T.grouped = 1;
    T.only = early ? 2 : 0;
    GTerm* d_terms = (GTerm*)sc.alloc_bytes(sizeof(GTerm) * std::max(1, ntrip));
    C.flush();
    cuda_check(launch_asm_expand(T, ntrip, d_terms, C.st), "asm_expand");
    C.sub_end(S_MISC, sw);
    ++C.launches;
    htt.next("asm_outs");
    auto gf = outs_fut.get();
    GBatch& g = gf.first;
    const double fl = gf.second;
    static const bool dbg_asm = getenv("H2G_DEBUG_ASM") != nullptr;
    if (dbg_asm) {  // output-shape census of the assembly launch (algorithmic vs 64x64-tile work)
      auto up = [](double v, double q) { return std::ceil(v / q) * q; };
      double cnt[2] = {0, 0}, mn[2] = {0, 0}, nt[2] = {0, 0}, alg[2] = {0, 0}, pad[2] = {0, 0};
      for (int b = 0; b < B.nb; ++b) {
        const int t = B.row[b], r = B.col[b];
        const int d = B.near_leaf(b) ? 1 : 0;
        const double m = d ? rows.size(t) : Q.rank[t], n = d ? cols.size(r) : W.rank[r];
        if (m == 0 || n == 0) continue;
        cnt[d] += 1;
        mn[d] += m * n;
        nt[d] += pt.tptr[b + 1] - pt.tptr[b];
        const double tiles = up(m, 64) * up(n, 64) / 4096.0;
        for (int i = pt.tptr[b]; i < pt.tptr[b + 1]; ++i) {
          const int s = pt.ts[i];
          double k, k2 = 0;
          if (pt.tk[i] == 'c') k = mid.size(s);
          else if (pt.tk[i] == 'a') { k = y.rb().rank[s]; k2 = y.cb().rank[r]; }
          else { k = x.rb().rank[t]; k2 = x.cb().rank[s]; }
          if (k2 == 0) {
            alg[d] += 2 * m * n * k;
            pad[d] += tiles * 2 * 4096 * up(k, 16);
          } else {
            alg[d] += 2 * m * k * k2 + 2 * m * k2 * n;
            pad[d] += tiles * (2 * 64 * up(k2, 64) * up(k, 16) + 2 * 4096 * up(k2, 16));
          }
        }
      }
      for (int d = 0; d < 2; ++d)
        fprintf(stderr, "asm %s: %.0f outputs, mean m*n %.0f, mean terms %.1f, alg %.2f GF, tile work %.2f GF\n",
                d ? "dense" : "coupling", cnt[d], mn[d] / std::max(1.0, cnt[d]), nt[d] / std::max(1.0, cnt[d]),
                alg[d] * 1e-9, pad[d] * 1e-9);
    }
    g.run_device_terms(C, d_terms, fl);
  }
  // the dense targets (queued ahead) receive the push-down's expansions: the main stream waits for
  // them just before the first expansion launch (the coupling pushes of the upper levels do not
  // touch them); the triple arrays are consumed by both expansions, release them in stream order
  bool dense_wait = early;
  auto wait_dense = [&] {
    if (!dense_wait) return;
    cuda_check(cudaStreamWaitEvent(C.st, pt.early.done, 0), "wait dense targets");
    cudaEventDestroy(pt.early.done);
    pt.early.done = nullptr;
    dense_wait = false;
  };
  if (pt.dev.ready) {
    cudaEventDestroy(pt.dev.ready);
    pt.dev.ready = nullptr;
  }
  // push-down of couplings on subdivided blocks, parents first (induced.py:328-344)
  mem_mark("p1 before push-down");
  HostTimer ht3(C, "assemble_pushdown");
  StageTag tagp(C, "p1.push");
  struct Expansion {
    int ch;
    Mat part;
  };
  static const bool exp3 = getenv("H2G_EXPAND_3F") != nullptr;  // previous one-launch form (A/B)
  static const bool push3 = getenv("H2G_PUSH_3F") != nullptr;  // previous 3-factor pushes (A/B)
  constexpr size_t kPushBudget = size_t(1) << 27;  // doubles (1 GiB) of E_t2 S intermediates per chunk
  // The expansions into the dense targets write nothing a later push-down level reads: they run on
  // the normal-priority auxiliary stream, overlapping the next levels' coupling pushes and phase 2's
  // coupling norms and Z levels (which read couplings only).  Phase 2's nearfield readers follow
  // them on that stream (nearfield norms) or wait for G->near_ready.  Partitioned products exchange
  // G's blocks right after the push-down and keep them on the main stream.
  static const bool sync_exp = getenv("H2G_SYNC_EXPAND") != nullptr;  // A/B: expansions on the main stream
  Ctx* Ep = (!serial_passes() && !part.on() && !exp3 && !sync_exp) ? &C.aux(true) : nullptr;
  std::shared_ptr<Arena> pa;  // the expansions' k~ x k~ parts (read on Ep, freed after it)
  if (Ep) {
    Ep->sync();  // recycle its staging (a product without coarsen never joins it)
    pa = std::make_shared<Arena>(C.st);
    Ep->tag = "p1.expand";
  }
  bool dense_wait_ep = early;
  for (int lev = 0; lev < B.depth; ++lev) {
    GBatch g1, g2;
    std::vector<Expansion> exps;
    // children (t2, r2) of a subdivided block b receive E_t2 S F_r2^T (induced.py:328-344): E_t2 S is
    // shared by the children of one row child t2, so it is formed once per (b, t2) into scratch and the
    // children take one 2-factor term each -- no 3-factor term recomputing it for every output tile
    // and sibling.  Chunked over the parents to bound the scratch.
    const std::vector<int>& lvl = B.by_level[lev];
    for (size_t p0 = 0; p0 < lvl.size();) {
      size_t need = 0, p1 = p0;
      for (; p1 < lvl.size(); ++p1) {
        const int b = lvl[p1];
        if (B.leaf(b) || push3) continue;
        size_t sz = 0;
        for (int i = 0; i < B.nkids(b); ++i) {
          const int ch = B.kid(b, i);
          if (B.row[ch] != B.row[b]) sz += (size_t)Q.rank[B.row[ch]] * W.rank[B.col[b]];
        }
        if (p1 > p0 && need + sz > kPushBudget) break;
        need += sz;
      }
      if (push3) p1 = lvl.size();
      Arena ta(C.st);
      GBatch ge;
      for (size_t pi = p0; pi < p1; ++pi) {
        const int b = lvl[pi];
        if (B.leaf(b)) continue;
        const int t = B.row[b], r = B.col[b];
        const Mat& S = cp[b];
        std::vector<std::pair<int, Mat>> es;  // (t2, E_t2 S) of this parent
        for (int i = 0; i < B.nkids(b); ++i) {
          const int ch = B.kid(b, i);
          const int t2 = B.row[ch], r2 = B.col[ch];
          if (!part.mine(t2)) continue;
          Mat E, F;
          if (t2 != t) E = Q.xferm(t2);
          if (r2 != r) F = W.xferm(r2);
          Mat src = S;  // E_t2 S, or S itself when the row cluster does not change
          if (!push3 && t2 != t) {
            auto it = std::find_if(es.begin(), es.end(), [t2](const std::pair<int, Mat>& e) { return e.first == t2; });
            if (it == es.end()) {
              Mat m2{ta.alloc((size_t)Q.rank[t2] * S.c), Q.rank[t2], S.c};
              ge.out(m2, false);
              ge.t2(E.ref(), S.ref(), E.c);
              es.emplace_back(t2, m2);
              it = es.end() - 1;
            }
            src = it->second;
          }
          const bool push_e = push3 && t2 != t;
          if (B.near_leaf(ch)) {
            Mat part{(Ep ? *pa : sc).alloc((size_t)Q.rank[t2] * W.rank[r2]), Q.rank[t2], W.rank[r2]};
            g1.out(part, false);
            emit_push(g1, push_e ? &E : nullptr, src, r2 != r ? &F : nullptr);
            if (exp3) {
              g2.out(Mat{G->near[ch], rows.size(t2), cols.size(r2)}, true);
              g2.t3(Q.leafm(t2).ref(), part.ref(), W.leafm(r2).tref(), Q.rank[t2], W.rank[r2]);
            } else {
              exps.push_back(Expansion{ch, part});
            }
          } else {
            g1.out(cp[ch], true);
            emit_push(g1, push_e ? &E : nullptr, src, r2 != r ? &F : nullptr);
          }
        }
      }
      ge.run(C);
      g1.run(C);
      p0 = p1;
    }
    if (!g2.outs.empty() || (!exps.empty() && !Ep)) wait_dense();
    g2.run(C);
    Ctx& XC = Ep ? *Ep : C;  // stream of this level's expansions
    if (Ep && !exps.empty()) {
      if (dense_wait_ep) {  // the dense targets first
        cuda_check(cudaStreamWaitEvent(Ep->st, pt.early.done, 0), "wait dense targets");
        dense_wait_ep = false;
      }
      cudaEvent_t e;  // this level's parts are written on the main stream
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      cuda_check(cudaEventRecord(e, C.st), "event");
      cuda_check(cudaStreamWaitEvent(Ep->st, e, 0), "wait parts");
      cudaEventDestroy(e);
    }
    // expansion into the inadmissible children, N += Q_leaf(t2) (part W_leaf(r2)^T) as two
    // 2-factor launches: T = Q_leaf part once per target (a 3-factor term recomputes it for every
    // 64-column tile of the target and pads its middle dimension to 64), then N += T W_leaf^T.
    // Chunked so the intermediates stay within a bounded scratch (freed stream-ordered per chunk).
    constexpr size_t kExpBudget = size_t(1) << 27;  // doubles (1 GiB) of intermediates per chunk
    for (size_t e0 = 0; e0 < exps.size();) {
      size_t need = 0, e1 = e0;
      for (; e1 < exps.size(); ++e1) {
        const int ch = exps[e1].ch;
        const size_t sz = (size_t)rows.size(B.row[ch]) * W.rank[B.col[ch]];
        if (e1 > e0 && need + sz > kExpBudget) break;
        need += sz;
      }
      Arena ta(XC.st);
      GBatch ga, gb;
      for (size_t e = e0; e < e1; ++e) {
        const int ch = exps[e].ch;
        const int t2 = B.row[ch], r2 = B.col[ch];
        const Mat Tm{ta.alloc((size_t)rows.size(t2) * W.rank[r2]), rows.size(t2), W.rank[r2]};
        ga.out(Tm, false);
        ga.t2(Q.leafm(t2).ref(), exps[e].part.ref(), Q.rank[t2]);
        gb.out(Mat{G->near[ch], rows.size(t2), cols.size(r2)}, true);
        gb.t2(Tm.ref(), W.leafm(r2).tref(), W.rank[r2]);
      }
      ga.run(XC);
      gb.run(XC);
      e0 = e1;
    }
  }
  if (Ep && dense_wait_ep) {  // no expansion at all: the event below must still cover the dense targets
    cuda_check(cudaStreamWaitEvent(Ep->st, pt.early.done, 0), "wait dense targets");
    dense_wait_ep = false;
  }
  if (!Ep) wait_dense();
  if (Ep) {
    Ep->tag.clear();
    // the parts are freed on the expansion stream once it has consumed them
    pa->cross_stream = true;
    pa->free_st = Ep->st;
    pa->after = {C.st};
    pa.reset();
    // G's nearfield is complete at this event (dense targets and expansions): readers wait for it
    cuda_check(cudaEventCreateWithFlags(&G->near_ready, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(G->near_ready, Ep->st), "event");
  }
  if (pt.dev.block) {  // after the stream that frees them has waited for the dense targets' expansion
    cudaFreeAsync(pt.dev.block, Ep ? Ep->st : C.st);
    pt.dev.block = nullptr;
  }
  if (Ep && pt.early.done) {  // Ep waited for it above
    cudaEventDestroy(pt.early.done);
    pt.early.done = nullptr;
  }
  if (part.on()) {
    // G stays distributed by block rows: each rank keeps the blocks of its own rows (and the
    // replicated top rows).  Phase 2's column pass of cluster r reads the blocks (t, r) of column r:
    // each leaf block goes to its column's owner when that rank differs (the transpose halo, one
    // all-to-all); blocks of replicated top columns below partitioned rows (none on the balanced
    // BASELINE trees) are all-gathered.
    StageTag tagx(C, "p1.exchange");
    const Part pcol = make_part(cols, C.comm);
    std::vector<PItem> p2p;
    std::vector<XItem> ag;
    for (int b = 0; b < B.nb; ++b) {
      if (!B.leaf(b)) continue;
      const int t = B.row[b], r = B.col[b];
      if (part.top(t)) continue;
      const long long len = B.adm[b] ? (long long)Q.rank[t] * W.rank[r] : (long long)rows.size(t) * cols.size(r);
      double** dst = B.adm[b] ? &G->coup[b] : &G->near[b];
      const int src = part.owner[t];
      if (pcol.top(r)) ag.push_back(XItem{src, len, dst});
      else if (pcol.owner[r] != src) p2p.push_back(PItem{src, pcol.owner[r], len, dst});
    }
    exchange_p2p(C, *ar, p2p);
    exchange(C, *ar, ag);
    G->dist_rows = true;
    G->dist_halo = true;
  }
  // phase 2's block-norm batches are pure structure of G: build them on a host thread now, while
  // the assembly and push-down run on the GPU (coarsen picks them up)
  {
    const H2* gp = G.get();
    const Comm comm = C.comm;
    G->norm_prep = std::async(std::launch::async, [gp, comm] { return build_norm_prep(*gp, comm); }).share();
  }
  return G;  // scratch is released stream-ordered (cudaFreeAsync) after the queued work

}

static void record(Ctx& C, cudaEvent_t& e) {
  if (!C.timing) return;
  e = C.event();
  cudaEventRecord(e, C.st);
}

static float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (a && b) cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Phase-1 driver (reference induced.py:358-372).
std::shared_ptr<H2> multiply(Ctx& C, const H2& x, const H2& y, double tol, int max_rank, bool scaling) {
  x.start_near(C);  // deferred nearfield uploads: both operands' small arrays are queued by now
  y.start_near(C);
  if (!x.bt->cols->same(*y.bt->rows)) throw InvalidInput("x and y do not share the middle cluster tree");
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr, e4 = nullptr;
  record(C, e0);
  // T^XY is pure structure: build it on a host thread while the GPU computes weights and bases
  auto keep = std::make_shared<Arena>(C.st);
  Arena sc(C.st);
  HView X{&x, false}, Y{&y, false}, XT{&x, true}, YT{&y, true};
  StageTag tag0(C, "p1.weights");
  MatStore P = basis_product(C, sc, *x.cb, *y.rb);
  // T^XY is pure structure: build it on a host thread while the GPU computes weights and bases;
  // the same thread then queues the dense targets (inputs only) on the low-priority stream
  const bool ahead = !serial_passes();
  cudaEvent_t p_ready = nullptr;
  Ctx* A = nullptr;
  if (ahead) {
    A = &C.aux();
    // recycle its staging buffer (and free any retired one): the previous product's dense launch is
    // long finished (its coarsen joined the expansion stream, which waited for it), so this does not
    // wait in practice -- without it the buffer's offset only grew and every few products an
    // overflow reallocated it (pinned cudaMallocHost + cudaMalloc: +100-300 ms steps)
    A->sync();
    cuda_check(cudaEventCreateWithFlags(&p_ready, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(p_ready, C.st), "event");
  }
  static const bool dbg_plan = getenv("H2G_DEBUG_PLANNER") != nullptr;
  const auto t_mul0 = std::chrono::steady_clock::now();
  auto ms_since = [t_mul0] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_mul0).count();
  };
  auto pt_future = std::async(std::launch::async, [&x, &y, &C, &P, A, p_ready, X, Y, ms_since] {
    PTree pt = product_tree(BView{x.bt.get(), false}, BView{y.bt.get(), false});
    const double t1 = ms_since();
    ptree_prepare(pt, C, *x.bt, y.bt->nb);
    const double t2 = ms_since();
    if (A) assemble_dense_early(*A, X, Y, PRef{&P, false}, pt, p_ready, C.comm);
    if (dbg_plan)
      fprintf(stderr, "planner: product tree %.2f ms, prepared %.2f ms, dense targets queued %.2f ms\n", t1, t2,
              ms_since());
    return pt;
  });
  struct PtJoin {  // never leave the planner running past an exception
    std::future<PTree>& f;
    cudaEvent_t e;
    ~PtJoin() {
      if (f.valid()) f.wait();
      if (e) cudaEventDestroy(e);
    }
  } pt_join{pt_future, p_ready};
  record(C, e1);
  // the row and column bases are independent until the assembly: run them concurrently, the
  // column pass on a side stream driven by a second host thread
  auto keep2 = std::make_shared<Arena>(C.st);
  Induced qr, qc;
  PTree pt;
  std::vector<Mat> rf;
  bool have_rf = false;
  // each pass first forms its own total weights (weights.py:60-101): Z_Y for the rows, Z_X^T for
  // the columns
  cudaEvent_t ev_r[3] = {}, ev_c[3] = {};  // begin / weights done / end of each pass (timing mode)
  auto row_pass = [&](Ctx& c, Arena& out, Arena& scr) {
    ev_r[0] = mark_event(c);
    MatStore rwy = basis_weights(c, scr, *y.cb);
    MatStore zy = total_weights(c, scr, Y, rwy, scaling, tol < kFloorFreeTol);
    ev_r[1] = mark_event(c);
    Induced r = induced_rows(c, out, X, Y, zy, PRef{&P, false}, tol, max_rank, scaling, 1.0);
    ev_r[2] = mark_event(c);
    return r;
  };
  auto col_pass = [&](Ctx& c, Arena& out, Arena& scr) {
    ev_c[0] = mark_event(c);
    MatStore rwx = basis_weights(c, scr, *x.rb);
    MatStore zxt = total_weights(c, scr, XT, rwx, scaling, tol < kFloorFreeTol);
    ev_c[1] = mark_event(c);
    Induced r = induced_rows(c, out, YT, XT, zxt, PRef{&P, true}, tol, max_rank, scaling, 1.0);
    ev_c[2] = mark_event(c);
    return r;
  };
  if (serial_passes()) {  // profiling aid: deterministic single-stream launch order
    qr = row_pass(C, *keep, sc);
    qc = col_pass(C, *keep2, sc);
  } else {
    Ctx& S = C.side();
    keep2->st = S.st;
    C.order_free(*keep2);
    PassGate gate;  // partitioned products: the column pass's collectives follow the row pass's
    C.gate = &gate;
    S.gate = &gate;
    struct GateReset {
      Ctx &a, &b;
      ~GateReset() {
        a.gate_leave();  // never leave the column pass waiting (row pass done or failed)
        a.gate = b.gate = nullptr;
      }
    };
    std::exception_ptr err;
    std::thread th([&] {
      try {
        StageTag tg(S, "p1.weights");
        Arena sc2(S.st);
        qc = col_pass(S, *keep2, sc2);
        S.sync();
      } catch (...) {
        err = std::current_exception();
      }
    });
    GateReset gate_reset{C, S};
    try {
      qr = row_pass(C, *keep, sc);
      C.gate_leave();
      // the row factors need only the row basis: issue them while the column pass finishes
      // (only when the planner thread is done already -- it also queues the dense targets)
      static const bool early_rf = getenv("H2G_NO_EARLY_RF") == nullptr;
      if (early_rf && pt_future.wait_for(std::chrono::seconds(0)) == std::future_status::ready) {
        pt = pt_future.get();
        rf = row_factors(C, sc, X, Y, qr, PRef{&P, false}, pt);
        have_rf = true;
      }
    } catch (...) {
      C.gate_leave();
      th.join();
      throw;
    }
    HostTimer hj(C, "p1_join");
    th.join();
    if (err) std::rethrow_exception(err);
    C.join_side(S);
  }
  record(C, e2);
  e3 = e2;
  if (dbg_plan) fprintf(stderr, "main: induced passes issued and joined %.2f ms\n", ms_since());
  if (!have_rf) {
    HostTimer ht(C, "product_tree_wait");
    pt = pt_future.get();
  }
  if (pt.early.near) C.order_free(*pt.early.near);
  mem_mark("p1 induced bases");
  StageTag taga(C, "p1.asm");
  auto G = assemble(C, X, Y, qr, qc, PRef{&P, false}, pt, have_rf ? &rf : nullptr);
  mem_mark("p1 assembled");
  if (A) {
    if (G->near_ready && !C.prof) {
      // the push-down expansions (normal-priority auxiliary stream) waited for the dense targets
      // and G->near_ready completes both: the main stream goes on with phase 2 instead of waiting
      // here for the low-priority stream; its arena is freed after that stream's queued work
      C.launches += A->launches;
      A->launches = 0;
      if (pt.early.near) pt.early.near->after.push_back(A->st);
    } else {
      C.join_side(*A);  // counters / profile of the auxiliary stream's work
    }
  }
  record(C, e4);
  G->owned.push_back(keep);
  G->owned.push_back(keep2);
  G->own_rows = x.own_rows;
  G->own_cols = y.own_cols;
  if (C.timing) {
    C.sync();
    C.times.setup = elapsed(e0, e1) + elapsed(ev_r[0], ev_r[1]);
    C.times.setup_col = elapsed(ev_c[0], ev_c[1]);
    C.times.t1_row = elapsed(ev_r[1], ev_r[2]);
    C.times.t1_col = elapsed(ev_c[1], ev_c[2]);
    C.times.t1_span = elapsed(e1, e2);
    C.times.t1_mat = elapsed(e3, e4);
  }
  return G;
}

// ------------------------------------------------------------------ stage-level entry points
// compress_induced_row_basis (induced.py:76-184) with z = Z_Y and P = P_XY, or
// compress_induced_col_basis (induced.py:187-200: the row algorithm on Y^T X^T) with z = Z_X^T.
std::shared_ptr<InducedStage> induced_stage(Ctx& C, const H2& x, const H2& y, const MatStore& z, const MatStore& P,
                                            bool col, double tol, int max_rank, bool scale, double level_decay) {
  if (!x.bt->cols->same(*y.bt->rows)) throw InvalidInput("x and y do not share the middle cluster tree");
  if (tol < 0) throw InvalidInput("tolerance must be >= 0");
  wait_near(C, x);
  wait_near(C, y);
  auto out = std::make_shared<InducedStage>();
  out->ar = std::make_shared<Arena>(C.st);
  out->T = col;
  if ((int)z.size() != x.bt->cols->n) throw InvalidInput("total weights do not match the middle cluster tree");
  if ((int)P.size() != x.bt->cols->n) throw InvalidInput("basis product does not match the middle cluster tree");
  if (!col)
    out->ind = induced_rows(C, *out->ar, HView{&x, false}, HView{&y, false}, z, PRef{&P, false}, tol, max_rank, scale,
                            level_decay);
  else
    out->ind = induced_rows(C, *out->ar, HView{&y, true}, HView{&x, true}, z, PRef{&P, true}, tol, max_rank, scale,
                            level_decay);
  C.sync();
  return out;
}

// assemble_product (induced.py:220-355): T^XY built here (trees.py:314-359), every term on the GPU.
std::shared_ptr<H2> assemble_stage(Ctx& C, const H2& x, const H2& y, const InducedStage& qr, const InducedStage& qc,
                                   const MatStore& P, std::vector<ArenaPtr> keep) {
  if (!x.bt->cols->same(*y.bt->rows)) throw InvalidInput("x and y do not share the middle cluster tree");
  if (qr.T || !qc.T) throw InvalidInput("assemble_product needs an induced row basis and an induced column basis");
  if (qr.ind.q->tree != x.bt->rows || qc.ind.q->tree != y.bt->cols)
    throw InvalidInput("induced bases live on other cluster trees");
  wait_near(C, x);
  wait_near(C, y);
  PTree pt = product_tree(BView{x.bt.get(), false}, BView{y.bt.get(), false});
  ptree_prepare(pt, C, *x.bt, y.bt->nb);
  // assemble() memoises the leaf products it needs in the Induced it is given (scratch memory):
  // work on copies so the stage results stay reusable
  Induced r = qr.ind, c = qc.ind;
  auto G = assemble(C, HView{&x, false}, HView{&y, false}, r, c, PRef{&P, false}, pt, nullptr);
  G->owned.push_back(qr.ar);
  G->owned.push_back(qc.ar);
  for (auto& a : qr.keep) G->owned.push_back(a);
  for (auto& a : qc.keep) G->owned.push_back(a);
  for (auto& a : keep) G->owned.push_back(a);
  G->own_rows = x.own_rows;
  G->own_cols = y.own_cols;
  C.sync();
  return G;
}

}  // namespace h2g
