// extern "C" stage-level entry points (include/h2g.h, "Stage-level entry points"): the reference's
// stage functions (h2mul/__init__.py:11-32) one call at a time, with opaque result handles.
#include <cstring>

#include "capi_handles.h"

namespace {

h2g_mats* new_mats(const MatStore& m, std::vector<ArenaPtr> keep, std::shared_ptr<H2> owner = {}) {
  return new h2g_mats{m, std::move(keep), std::move(owner)};
}

void need(const void* p, const char* what) {
  if (!p) throw InvalidInput(std::string("null handle: ") + what);
}

}  // namespace

extern "C" {

int h2g_h2_basis(h2g_h2* g, int which, h2g_basis** out) {
  return guarded([&] {
    need(g, "g");
    auto b = new h2g_basis;
    b->b = which ? g->h->cb : g->h->rb;
    b->owner = g->h;
    *out = b;
  });
}

int h2g_basis_upload(h2g_ctx* ctx, h2g_tree* tree, const long long* rank, const long long* loff,
                     const long long* xoff, const double* data, long long len, h2g_basis** out) {
  return guarded([&] {
    need(tree, "tree");
    Ctx& C = ctx->c;
    auto ar = std::make_shared<Arena>(C.st);
    auto b = new h2g_basis;
    b->b = upload_basis(C, *ar, tree->t.get(), rank, loff, xoff, data, len);
    b->keep.push_back(ar);
    b->tree = tree->t;
    C.sync();
    *out = b;
  });
}

int h2g_basis_sizes(h2g_basis* b, long long* o) {
  return guarded([&] {
    const Basis& B = *b->b;
    const Tree& tr = *B.tree;
    long long len = 0;
    for (int t = 0; t < tr.n; ++t) {
      if (tr.leaf(t)) len += (long long)tr.size(t) * B.rank[t];
      if (tr.parent[t] >= 0) len += (long long)B.rank[t] * B.rank[tr.parent[t]];
    }
    o[0] = tr.n;
    o[1] = len;
  });
}

int h2g_basis_download(h2g_ctx* ctx, h2g_basis* b, long long* rank, long long* loff, long long* xoff, double* data) {
  return guarded([&] {
    Ctx& C = ctx->c;
    Arena ar(C.st);
    Gather g;
    pack_basis(*b->b, rank, loff, xoff, g);
    g.run(C, ar, data);
    C.sync();
  });
}

void h2g_basis_destroy(h2g_basis* b) { delete b; }

int h2g_mats_upload(h2g_ctx* ctx, int n, const long long* rows, const long long* cols, const long long* off,
                    const double* data, long long len, h2g_mats** out) {
  return guarded([&] {
    if (n < 0) throw InvalidInput("negative count");
    Ctx& C = ctx->c;
    auto ar = std::make_shared<Arena>(C.st);
    double* d = ar->alloc(len > 0 ? len : 1);
    if (len > 0) cuda_check(cudaMemcpyAsync(d, data, len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
    MatStore m(n);
    for (int i = 0; i < n; ++i) {
      if (off[i] < 0 || rows[i] <= 0 || cols[i] <= 0) {
        m[i] = Mat{nullptr, (int)std::max(0LL, rows[i]), (int)std::max(0LL, cols[i])};
        if (off[i] >= 0) m[i].p = d + off[i];
        continue;
      }
      if (off[i] + rows[i] * cols[i] > len) throw InvalidInput("matrix out of range");
      m[i] = Mat{d + off[i], (int)rows[i], (int)cols[i]};
    }
    C.sync();
    *out = new_mats(m, {ar});
  });
}

int h2g_mats_shapes(h2g_mats* m, int* n, long long* rows, long long* cols) {
  return guarded([&] {
    *n = (int)m->m.size();
    for (size_t i = 0; i < m->m.size(); ++i) {
      const Mat& a = m->m[i];
      const bool has = a.p != nullptr || (a.r == 0 || a.c == 0);
      if (rows) rows[i] = has ? a.r : 0;
      if (cols) cols[i] = has ? a.c : 0;
    }
  });
}

int h2g_mats_download(h2g_ctx* ctx, h2g_mats* m, long long* off, double* data) {
  return guarded([&] {
    Ctx& C = ctx->c;
    Arena ar(C.st);
    Gather g;
    for (size_t i = 0; i < m->m.size(); ++i) {
      const Mat& a = m->m[i];
      if (!a.p && a.r > 0 && a.c > 0) {
        off[i] = -1;
        continue;
      }
      off[i] = g.total;
      g.add(a.p, (long long)a.r * a.c);
    }
    g.run(C, ar, data);
    C.sync();
  });
}

void h2g_mats_destroy(h2g_mats* m) { delete m; }

int h2g_cluster_basis_product(h2g_ctx* ctx, h2g_basis* wx, h2g_basis* vy, h2g_mats** out) {
  return guarded([&] {
    need(wx, "wx");
    need(vy, "vy");
    Ctx& C = ctx->c;
    auto ar = std::make_shared<Arena>(C.st);
    MatStore P = basis_product(C, *ar, *wx->b, *vy->b);
    C.sync();
    std::vector<ArenaPtr> keep{ar};
    *out = new_mats(P, keep);
  });
}

int h2g_basis_weights(h2g_ctx* ctx, h2g_basis* w, h2g_mats** out) {
  return guarded([&] {
    need(w, "w");
    Ctx& C = ctx->c;
    auto ar = std::make_shared<Arena>(C.st);
    MatStore R = basis_weights(C, *ar, *w->b);
    C.sync();
    *out = new_mats(R, {ar});
  });
}

int h2g_total_weights(h2g_ctx* ctx, h2g_h2* y, int transposed, h2g_mats* rw, int scaling, h2g_mats** out) {
  return guarded([&] {
    need(y, "y");
    need(rw, "rw");
    Ctx& C = ctx->c;
    need_whole(C, *y->h);
    const H2& h = *y->h;
    const HView v{&h, transposed != 0};
    if ((int)rw->m.size() != v.cols().n) throw InvalidInput("basis weights do not match the column cluster tree");
    wait_near(C, h);
    auto ar = std::make_shared<Arena>(C.st);
    MatStore Z = total_weights(C, *ar, v, rw->m, scaling != 0);
    C.sync();
    *out = new_mats(Z, {ar});
  });
}

static int induced_impl(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_mats* z, h2g_mats* pxy, double tol, int max_rank,
                        int scale, double level_decay, bool col, h2g_induced** out) {
  return guarded([&] {
    need(x, "x");
    need(y, "y");
    need(z, "total weights");
    need(pxy, "pxy");
    need_whole(ctx->c, *x->h);
    need_whole(ctx->c, *y->h);
    auto s = induced_stage(ctx->c, *x->h, *y->h, z->m, pxy->m, col, tol, max_rank, scale != 0, level_decay);
    s->keep.insert(s->keep.end(), z->keep.begin(), z->keep.end());
    s->keep.insert(s->keep.end(), pxy->keep.begin(), pxy->keep.end());
    *out = new h2g_induced{s};
  });
}

int h2g_compress_induced_row_basis(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_mats* zy, h2g_mats* pxy, double tol,
                                   int max_rank, int scale_blocks, double level_decay, h2g_induced** out) {
  return induced_impl(ctx, x, y, zy, pxy, tol, max_rank, scale_blocks, level_decay, false, out);
}

int h2g_compress_induced_col_basis(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_mats* zxt, h2g_mats* pxy, double tol,
                                   int max_rank, int scale_blocks, double level_decay, h2g_induced** out) {
  return induced_impl(ctx, x, y, zxt, pxy, tol, max_rank, scale_blocks, level_decay, true, out);
}

int h2g_induced_parts(h2g_induced* r, h2g_basis** q, h2g_mats** bc, h2g_mats** proj) {
  return guarded([&] {
    need(r, "induced");
    const InducedStage& s = *r->s;
    std::vector<ArenaPtr> keep = s.keep;
    keep.push_back(s.ar);
    if (q) {
      auto b = new h2g_basis;
      b->b = s.ind.q;
      b->keep = keep;
      *q = b;
    }
    if (bc) *bc = new_mats(s.ind.bc, keep);
    if (proj) *proj = new_mats(s.ind.proj, keep);
  });
}

int h2g_induced_create(h2g_ctx* ctx, h2g_basis* q, h2g_mats* bc, h2g_mats* proj, int col, h2g_induced** out) {
  return guarded([&] {
    (void)ctx;
    need(q, "q");
    need(bc, "basis_change");
    need(proj, "block_projections");
    if ((int)bc->m.size() != q->b->tree->n) throw InvalidInput("basis_change does not match the basis's tree");
    auto s = std::make_shared<InducedStage>();
    s->ind.q = q->b;
    s->ind.bc = bc->m;
    s->ind.proj = proj->m;
    s->T = col != 0;
    s->keep = q->keep;
    s->keep.insert(s->keep.end(), bc->keep.begin(), bc->keep.end());
    s->keep.insert(s->keep.end(), proj->keep.begin(), proj->keep.end());
    *out = new h2g_induced{s};
  });
}

void h2g_induced_destroy(h2g_induced* r) { delete r; }

int h2g_assemble_product(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, h2g_induced* qrow, h2g_induced* qcol, h2g_mats* pxy,
                         h2g_h2** out) {
  return guarded([&] {
    need(x, "x");
    need(y, "y");
    need(qrow, "qrow");
    need(qcol, "qcol");
    need(pxy, "pxy");
    if ((int)pxy->m.size() != x->h->bt->cols->n) throw InvalidInput("pxy does not match the middle cluster tree");
    need_whole(ctx->c, *x->h);
    need_whole(ctx->c, *y->h);
    auto G = assemble_stage(ctx->c, *x->h, *y->h, *qrow->s, *qcol->s, pxy->m, pxy->keep);
    *out = new h2g_h2{G};
  });
}

int h2g_block_norms(h2g_ctx* ctx, h2g_h2* g, double* cn, double* nn) {
  return guarded([&] {
    need(g, "g");
    if (!cn || !nn) throw InvalidInput("norm arrays are required");
    need_rows_halo(ctx->c, *g->h);
    block_norms_stage(ctx->c, *g->h, cn, nn);
  });
}

static int coarse_impl(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank, int scale,
                       const double* cn, const double* nn, bool col, h2g_cstate** out) {
  return guarded([&] {
    need(g, "g");
    need(coarse, "coarse");
    need_rows_halo(ctx->c, *g->h);
    auto s = coarse_basis_stage(ctx->c, *g->h, coarse->b, col, tol, max_rank, scale != 0, cn, nn);
    *out = new h2g_cstate{s, g->h};
  });
}

int h2g_build_coarse_row_basis(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank,
                               int scale_blocks, const double* cn, const double* nn, h2g_cstate** out) {
  return coarse_impl(ctx, g, coarse, tol, max_rank, scale_blocks, cn, nn, false, out);
}

int h2g_build_coarse_col_basis(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank,
                               int scale_blocks, const double* cn, const double* nn, h2g_cstate** out) {
  return coarse_impl(ctx, g, coarse, tol, max_rank, scale_blocks, cn, nn, true, out);
}

int h2g_cstate_parts(h2g_cstate* s, h2g_basis** q, h2g_mats** r, h2g_mats** z, long long* nreps) {
  return guarded([&] {
    need(s, "state");
    MatStore rr, zz;
    ArenaPtr ar;
    int nrep = 0;
    std::shared_ptr<Basis> b = coarse_stage_basis(*s->s, &rr, &zz, &ar, &nrep);
    std::vector<ArenaPtr> keep{ar};
    if (q) {
      auto hb = new h2g_basis;
      hb->b = b;
      hb->keep = keep;
      hb->owner = s->g;
      *q = hb;
    }
    if (r) *r = new_mats(rr, keep, s->g);
    if (z) *z = new_mats(zz, keep, s->g);
    if (nreps) *nreps = nrep;
  });
}

void h2g_cstate_destroy(h2g_cstate* s) { delete s; }

int h2g_project_final(h2g_ctx* ctx, h2g_h2* g, h2g_cstate* rs, h2g_cstate* cs, h2g_blocks* coarse, h2g_h2** out) {
  return guarded([&] {
    need(g, "g");
    need(rs, "rowstate");
    need(cs, "colstate");
    need(coarse, "coarse");
    auto Z = project_final_stage(ctx->c, *g->h, *rs->s, *cs->s, coarse->b);
    *out = new h2g_h2{Z};
  });
}

}  // extern "C"
