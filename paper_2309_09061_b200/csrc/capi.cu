// extern "C" boundary (include/h2g.h): handles, upload / download in the packed layout, status codes.
#include <malloc.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "../../include/h2g.h"
#include "engine.h"

using namespace h2g;

#include "capi_handles.h"

thread_local std::string g_err;

extern "C" {

const char* h2g_last_error(void) { return g_err.c_str(); }

int h2g_ctx_create(int device, void* stream, h2g_ctx** out) {
  return guarded([&] {
    // The planner and batch builders allocate and free large host vectors every product; keep them on
    // the heap (no per-product mmap / munmap and page-fault storms once glibc's thresholds adapt)
    static std::once_flag malloc_once;
    std::call_once(malloc_once, [] {
      mallopt(M_MMAP_THRESHOLD, 512 << 20);
      mallopt(M_TRIM_THRESHOLD, 1 << 30);
    });
    *out = new h2g_ctx(device, (cudaStream_t)stream);
  });
}

int h2g_ctx_destroy(h2g_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int h2g_ctx_set_timing(h2g_ctx* ctx, int on) {
  ctx->c.timing = on != 0;
  return 0;
}

int h2g_ctx_set_comm(h2g_ctx* ctx, int rank, int size, h2g_allgather_fn fn, void* user) {
  return guarded([&] {
    if (size < 1 || rank < 0 || rank >= size) throw InvalidInput("rank outside [0, size)");
    if (size > 1 && !fn) throw InvalidInput("a partitioned product needs an all-gather function");
    const Comm prev = ctx->c.comm;
    ctx->c.comm = Comm{rank, size, (AllgatherFn)fn, user, prev.a2a, prev.a2a_user};
    if (ctx->c.side_) {
      ctx->c.side_->comm = ctx->c.comm;
      ctx->c.side_->channel = 1;
    }
  });
}

int h2g_ctx_set_alltoall(h2g_ctx* ctx, h2g_alltoall_fn fn, void* user) {
  return guarded([&] {
    ctx->c.comm.a2a = (AlltoallFn)fn;
    ctx->c.comm.a2a_user = user;
    if (ctx->c.side_) ctx->c.side_->comm = ctx->c.comm;
  });
}

int h2g_ctx_stage_times(h2g_ctx* ctx, double* o) {
  const StageTimes& t = ctx->c.times;
  o[0] = t.setup; o[1] = t.t1_row; o[2] = t.t1_col; o[3] = t.t1_mat;
  o[4] = t.t2_row; o[5] = t.t2_col; o[6] = t.t2_mat;
  return 0;
}

int h2g_ctx_stage_times_ext(h2g_ctx* ctx, double* o, int n) {
  const StageTimes& t = ctx->c.times;
  const double v[11] = {t.setup, t.t1_row, t.t1_col, t.t1_mat, t.t2_row, t.t2_col, t.t2_mat,
                        t.setup_col, t.t1_span, t.t2_span, t.t2_norms};
  for (int i = 0; i < n && i < 11; ++i) o[i] = v[i];
  return 0;
}

int h2g_ctx_mem(h2g_ctx* ctx, long long* o, int reset) {
  return guarded([&] {
    cudaMemPool_t pool;
    cuda_check(cudaDeviceGetDefaultMemPool(&pool, ctx->c.device), "default pool");
    unsigned long long v[4] = {0, 0, 0, 0};
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &v[0]);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &v[1]);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &v[2]);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v[3]);
    for (int i = 0; i < 4; ++i) o[i] = (long long)v[i];
    o[4] = g_arena_payload_high.load();
    o[5] = g_arena_payload.load();
    if (reset) {
      unsigned long long z = 0;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &z);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReservedMemHigh, &z);
      g_arena_payload_high = g_arena_payload.load();
    }
  });
}

int h2g_ctx_counters(h2g_ctx* ctx, long long* o, int reset) {
  o[0] = ctx->c.launches;
  o[1] = ctx->c.syncs;
  if (reset) ctx->c.launches = ctx->c.syncs = 0;
  return 0;
}

int h2g_ctx_set_profile(h2g_ctx* ctx, int on) {
  ctx->c.prof = on != 0;
  return 0;
}

int h2g_set_serial(int on) {
  g_serial.store(on != 0);
  return 0;
}

int h2g_ctx_kernel_stats(h2g_ctx* ctx, double* o, int reset) {
  return guarded([&] {
    ctx->c.sync();
    for (int k = 0; k < K_NCLASS; ++k) {
      KStat& s = ctx->c.kstat[k];
      o[4 * k + 0] = (double)s.launches;
      o[4 * k + 1] = s.ms;
      o[4 * k + 2] = s.flops;
      o[4 * k + 3] = s.bytes;
      if (reset) s = KStat{};
    }
  });
}

int h2g_ctx_host_times(h2g_ctx* ctx, char* buf, int len, int reset) {
  std::string out;
  for (auto& kv : ctx->c.htime) out += kv.first + "=" + std::to_string(kv.second) + ";";
  if (reset) ctx->c.htime.clear();
  if (buf && len > 0) {
    strncpy(buf, out.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)out.size();
}

int h2g_ctx_trace_begin(h2g_ctx* ctx) {
  return guarded([&] {
    Ctx& C = ctx->c;
    C.sync();
    C.prof = true;
    C.trace = true;
    C.trace_recs.clear();
    C.trace_out = &C.trace_recs;
    if (!C.trace_base) cuda_check(cudaEventCreate(&C.trace_base), "event");
    cudaEventRecord(C.trace_base, C.st);
    cudaEventSynchronize(C.trace_base);
    C.trace_host0 = std::chrono::steady_clock::now();
  });
}

int h2g_ctx_trace_dump(h2g_ctx* ctx, const char* path) {
  return guarded([&] {
    Ctx& C = ctx->c;
    C.sync();
    static const char* names[] = {"gsum", "qr_r", "svd", "norm", "gather", "mv", "svd.tsqr", "merge", "svd.finish", "qr.chunk", "misc"};
    FILE* f = fopen(path, "w");
    if (!f) throw InvalidInput("cannot open trace file");
    fprintf(f, "{\"traceEvents\":[\n");
    bool first = true;
    for (auto& r : C.trace_recs) {
      const bool host = r.cls < 0;
      fprintf(f,
              "%s{\"name\":\"%s\",\"ph\":\"X\",\"ts\":%.3f,\"dur\":%.3f,\"pid\":%d,\"tid\":%d,"
              "\"args\":{\"tag\":\"%s\",\"gflop\":%.4f}}",
              first ? "" : ",\n", host ? "host_sync_wait" : names[r.cls], r.t0_us, r.dur_us, host ? 1 : 0, r.tid,
              r.tag.c_str(), r.flops * 1e-9);
      first = false;
    }
    fprintf(f, "\n]}\n");
    fclose(f);
    C.trace = false;
    C.prof = false;
    C.trace_out = nullptr;
  });
}

int h2g_ctx_synchronize(h2g_ctx* ctx) {
  return guarded([&] {
    // asynchronous uploads: the caller may release near_data after this call, so deferred nearfield
    // copies start now and the copy stream is drained too
    Ctx& C = ctx->c;
    for (auto& w : C.deferred_near)
      if (auto h = w.lock()) h->start_near(C);
    C.deferred_near.clear();
    if (C.up_stream) cuda_check(cudaStreamSynchronize(C.up_stream), "cudaStreamSynchronize");
    C.sync();
  });
}

int h2g_tree_create(h2g_ctx*, int n, const long long* start, const long long* stop, const long long* cptr,
                    const long long* cidx, h2g_tree** out) {
  return guarded([&] {
    if (n <= 0) throw InvalidInput("cluster tree must be non-empty");
    *out = new h2g_tree{make_tree(n, start, stop, cptr, cidx)};
  });
}

void h2g_tree_destroy(h2g_tree* t) { delete t; }

int h2g_tree_partition(h2g_tree* t, int nparts, long long* owner, int* level) {
  return guarded([&] {
    if (nparts < 1) throw InvalidInput("number of parts must be >= 1");
    const Part p = make_part(*t->t, nparts, 0);
    *level = p.level;
    for (int i = 0; i < t->t->n; ++i) owner[i] = p.on() ? p.owner[i] : -1;
  });
}

int h2g_blocks_create(h2g_ctx*, h2g_tree* rows, h2g_tree* cols, int nb, const long long* row,
                      const long long* col, const long long* cptr, const long long* cidx,
                      const unsigned char* adm, h2g_blocks** out) {
  return guarded([&] {
    if (nb <= 0) throw InvalidInput("block tree must be non-empty");
    for (int b = 0; b < nb; ++b)
      if (row[b] < 0 || row[b] >= rows->t->n || col[b] < 0 || col[b] >= cols->t->n)
        throw InvalidInput("block references a cluster outside its tree");
    auto bl = make_blocks(rows->t.get(), cols->t.get(), nb, row, col, cptr, cidx, adm);
    *out = new h2g_blocks{bl, rows->t, cols->t};
  });
}

void h2g_blocks_destroy(h2g_blocks* b) { delete b; }

}  // extern "C"

std::shared_ptr<Basis> upload_basis(Ctx& C, Arena& ar, const Tree* tree, const long long* rank,
                                           const long long* loff, const long long* xoff, const double* data,
                                           long long len) {
  auto B = std::make_shared<Basis>();
  B->tree = tree;
  B->rank.assign(rank, rank + tree->n);
  B->leaf.assign(tree->n, nullptr);
  B->xfer.assign(tree->n, nullptr);
  double* d = ar.alloc(len > 0 ? len : 1);
  if (len > 0) cuda_check(cudaMemcpyAsync(d, data, len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  for (int t = 0; t < tree->n; ++t) {
    if (B->rank[t] < 0) throw InvalidInput("negative rank");
    if (tree->leaf(t)) {
      if (loff[t] < 0 || loff[t] + (long long)tree->size(t) * B->rank[t] > len) throw InvalidInput("leaf matrix out of range");
      B->leaf[t] = d + loff[t];
    }
    if (tree->parent[t] >= 0) {
      if (xoff[t] < 0 || xoff[t] + (long long)B->rank[t] * rank[tree->parent[t]] > len)
        throw InvalidInput("transfer matrix out of range");
      B->xfer[t] = d + xoff[t];
    }
  }
  return B;
}

extern "C" {

static int upload_impl(h2g_ctx* ctx, h2g_blocks* bt, const long long* rb_rank, const long long* rb_loff,
                       const long long* rb_xoff, const double* rb_data, long long rb_len, const long long* cb_rank,
                       const long long* cb_loff, const long long* cb_xoff, const double* cb_data, long long cb_len,
                       int share, const long long* coup_off, const double* coup_data, long long coup_len,
                       const long long* near_off, const double* near_data, long long near_len, h2g_h2** out,
                       bool async_near) {
  return guarded([&] {
    Ctx& C = ctx->c;
    auto h = std::make_shared<H2>();
    auto ar = std::make_shared<Arena>(C.st);
    h->owned.push_back(ar);
    h->bt = bt->b;
    h->own_rows = bt->rows;
    h->own_cols = bt->cols;
    const Blocks& B = *bt->b;
    h->rb = upload_basis(C, *ar, B.rows, rb_rank, rb_loff, rb_xoff, rb_data, rb_len);
    if (share) {
      if (!B.rows->same(*B.cols)) throw InvalidInput("shared bases need identical row and column trees");
      h->cb = h->rb;
    } else {
      h->cb = upload_basis(C, *ar, B.cols, cb_rank, cb_loff, cb_xoff, cb_data, cb_len);
    }
    double* dc = ar->alloc(coup_len > 0 ? coup_len : 1);
    double* dn = ar->alloc(near_len > 0 ? near_len : 1);
    if (coup_len > 0)
      cuda_check(cudaMemcpyAsync(dc, coup_data, coup_len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
    if (near_len > 0) {
      if (async_near) {  // the nearfield streams in on the copy stream while the product starts;
                         // the copy is issued at the matrix's first use (H2::start_near)
        cuda_check(cudaEventCreateWithFlags(&h->near_alloc, cudaEventDisableTiming), "event");
        cuda_check(cudaEventRecord(h->near_alloc, C.st), "event");
        h->near_src = near_data;
        h->near_dst = dn;
        h->near_bytes = (size_t)near_len * sizeof(double);
        if (C.deferred_near.size() >= 64)  // drop matrices already destroyed or started
          C.deferred_near.erase(std::remove_if(C.deferred_near.begin(), C.deferred_near.end(),
                                               [](const std::weak_ptr<H2>& w) {
                                                 auto p = w.lock();
                                                 return !p || !p->near_src;
                                               }),
                                C.deferred_near.end());
        C.deferred_near.push_back(h);
      } else {
        cuda_check(cudaMemcpyAsync(dn, near_data, near_len * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
      }
    }
    h->coup.assign(B.nb, nullptr);
    h->near.assign(B.nb, nullptr);
    for (int b = 0; b < B.nb; ++b) {
      if (!B.leaf(b)) continue;
      const int t = B.row[b], s = B.col[b];
      if (B.adm[b]) {
        const long long n = (long long)h->rb->rank[t] * h->cb->rank[s];
        if (coup_off[b] < 0 || coup_off[b] + n > coup_len) throw InvalidInput("coupling out of range");
        h->coup[b] = dc + coup_off[b];
      } else {
        const long long n = (long long)B.rows->size(t) * B.cols->size(s);
        if (near_off[b] < 0 || near_off[b] + n > near_len) throw InvalidInput("nearfield out of range");
        h->near[b] = dn + near_off[b];
      }
    }
    if (!async_near) C.sync();  // host arrays may be released by the caller after return
    *out = new h2g_h2{h};
  });
}

int h2g_h2_upload(h2g_ctx* ctx, h2g_blocks* bt, const long long* rb_rank, const long long* rb_loff,
                  const long long* rb_xoff, const double* rb_data, long long rb_len, const long long* cb_rank,
                  const long long* cb_loff, const long long* cb_xoff, const double* cb_data, long long cb_len,
                  int share, const long long* coup_off, const double* coup_data, long long coup_len,
                  const long long* near_off, const double* near_data, long long near_len, h2g_h2** out) {
  return upload_impl(ctx, bt, rb_rank, rb_loff, rb_xoff, rb_data, rb_len, cb_rank, cb_loff, cb_xoff, cb_data, cb_len,
                     share, coup_off, coup_data, coup_len, near_off, near_data, near_len, out, false);
}

int h2g_h2_upload_async(h2g_ctx* ctx, h2g_blocks* bt, const long long* rb_rank, const long long* rb_loff,
                        const long long* rb_xoff, const double* rb_data, long long rb_len, const long long* cb_rank,
                        const long long* cb_loff, const long long* cb_xoff, const double* cb_data, long long cb_len,
                        int share, const long long* coup_off, const double* coup_data, long long coup_len,
                        const long long* near_off, const double* near_data, long long near_len, h2g_h2** out) {
  return upload_impl(ctx, bt, rb_rank, rb_loff, rb_xoff, rb_data, rb_len, cb_rank, cb_loff, cb_xoff, cb_data, cb_len,
                     share, coup_off, coup_data, coup_len, near_off, near_data, near_len, out, true);
}

void h2g_h2_destroy(h2g_h2* h) { delete h; }

static long long basis_len(const Basis& B) {
  const Tree& tr = *B.tree;
  long long n = 0;
  for (int t = 0; t < tr.n; ++t) {
    if (tr.leaf(t)) n += (long long)tr.size(t) * B.rank[t];
    if (tr.parent[t] >= 0) n += (long long)B.rank[t] * B.rank[tr.parent[t]];
  }
  return n;
}

int h2g_h2_sizes(h2g_h2* hh, long long* o) {
  return guarded([&] {
    const H2& h = *hh->h;
    const Blocks& B = *h.bt;
    long long cl = 0, nl = 0;
    for (int b = 0; b < B.nb; ++b) {
      if (!B.leaf(b)) continue;
      const int t = B.row[b], s = B.col[b];
      if (B.adm[b]) cl += (long long)h.rb->rank[t] * h.cb->rank[s];
      else nl += (long long)B.rows->size(t) * B.cols->size(s);
    }
    o[0] = B.nb;
    o[1] = B.rows->n;
    o[2] = B.cols->n;
    o[3] = basis_len(*h.rb);
    o[4] = basis_len(*h.cb);
    o[5] = cl;
    o[6] = nl;
    o[7] = (long long)B.cidx.size();
  });
}

int h2g_h2_ranks(h2g_h2* hh, long long* rr, long long* cr) {
  return guarded([&] {
    const H2& h = *hh->h;
    for (size_t i = 0; i < h.rb->rank.size(); ++i) rr[i] = h.rb->rank[i];
    for (size_t i = 0; i < h.cb->rank.size(); ++i) cr[i] = h.cb->rank[i];
  });
}

int h2g_h2_structure(h2g_h2* hh, long long* row, long long* col, long long* cptr, long long* cidx,
                     unsigned char* adm) {
  return guarded([&] {
    const Blocks& B = *hh->h->bt;
    for (int b = 0; b < B.nb; ++b) {
      row[b] = B.row[b];
      col[b] = B.col[b];
      adm[b] = B.adm[b];
      cptr[b] = B.cptr[b];
    }
    cptr[B.nb] = B.cptr[B.nb];
    for (size_t i = 0; i < B.cidx.size(); ++i) cidx[i] = B.cidx[i];
  });
}

}  // extern "C"

void pack_basis(const Basis& B, long long* rank, long long* loff, long long* xoff, Gather& g) {
  const Tree& tr = *B.tree;
  for (int t = 0; t < tr.n; ++t) {
    rank[t] = B.rank[t];
    loff[t] = -1;
    xoff[t] = -1;
  }
  for (int t = 0; t < tr.n; ++t)
    if (tr.leaf(t)) {
      loff[t] = g.total;
      g.add(B.leaf[t], (long long)tr.size(t) * B.rank[t]);
    }
  for (int t = 0; t < tr.n; ++t)
    if (tr.parent[t] >= 0) {
      xoff[t] = g.total;
      g.add(B.xfer[t], (long long)B.rank[t] * B.rank[tr.parent[t]]);
    }
}

extern "C" {

int h2g_h2_download(h2g_ctx* ctx, h2g_h2* hh, long long* rb_rank, long long* rb_loff, long long* rb_xoff,
                    double* rb_data, long long* cb_rank, long long* cb_loff, long long* cb_xoff, double* cb_data,
                    long long* coup_off, double* coup_data, long long* near_off, double* near_data) {
  return guarded([&] {
    Ctx& C = ctx->c;
    gather_rows(C, *hh->h);  // a partitioned product: complete it first
    const H2& h = *hh->h;
    const Blocks& B = *h.bt;
    wait_near(C, h);
    Arena ar(C.st);
    Gather gr, gc, gcp, gn;
    pack_basis(*h.rb, rb_rank, rb_loff, rb_xoff, gr);
    pack_basis(*h.cb, cb_rank, cb_loff, cb_xoff, gc);
    // blocks prefetched into this very host buffer during coarsen are skipped (their bytes are there)
    const bool pre = h.near_host && h.near_host == near_data && h.near_host_ready;
    std::vector<std::pair<long long, long long>> runs;  // non-prefetched dense ranges [lo, hi)
    for (int b = 0; b < B.nb; ++b) {
      coup_off[b] = -1;
      near_off[b] = -1;
      if (!B.leaf(b)) continue;
      const int t = B.row[b], s = B.col[b];
      if (B.adm[b]) {
        coup_off[b] = gcp.total;
        gcp.add(h.coup[b], (long long)h.rb->rank[t] * h.cb->rank[s]);
      } else {
        const long long sz = (long long)B.rows->size(t) * B.cols->size(s);
        near_off[b] = gn.total;
        if (pre && h.near_on_host[b]) {
          gn.total += sz;  // already on the host
        } else {
          if (pre) {
            if (!runs.empty() && runs.back().second == gn.total) runs.back().second += sz;
            else runs.emplace_back(gn.total, gn.total + sz);
          }
          gn.add(h.near[b], sz);
        }
      }
    }
    gr.run(C, ar, rb_data);
    gc.run(C, ar, cb_data);
    gcp.run(C, ar, coup_data);
    if (pre) {
      gn.run_runs(C, ar, near_data, runs);
      cuda_check(cudaStreamWaitEvent(C.st, h.near_host_ready, 0), "wait prefetch");
    } else {
      gn.run(C, ar, near_data);
    }
    C.sync();
  });
}

int h2g_product_tree(h2g_blocks* bx, h2g_blocks* by, h2g_blocks** out, long long* ntriples) {
  return guarded([&] {
    PTree pt = product_tree(BView{bx->b.get(), false}, BView{by->b.get(), false});
    *out = new h2g_blocks{pt.bt, bx->rows, by->cols};
    if (ntriples) {
      long long na = 0, nb = 0, nc = 0;
      for (char k : pt.tk) { na += k == 'a'; nb += k == 'b'; nc += k == 'c'; }
      ntriples[0] = na; ntriples[1] = nb; ntriples[2] = nc;
    }
  });
}

int h2g_blocks_structure(h2g_blocks* bb, long long* sizes2, long long* row, long long* col, long long* cptr,
                         long long* cidx, unsigned char* adm) {
  return guarded([&] {
    const Blocks& B = *bb->b;
    sizes2[0] = B.nb;
    sizes2[1] = (long long)B.cidx.size();
    if (!row) return;
    for (int b = 0; b < B.nb; ++b) {
      row[b] = B.row[b];
      col[b] = B.col[b];
      adm[b] = B.adm[b];
      cptr[b] = B.cptr[b];
    }
    cptr[B.nb] = B.cptr[B.nb];
    for (size_t i = 0; i < B.cidx.size(); ++i) cidx[i] = B.cidx[i];
  });
}

int h2g_h2_build_kernel(h2g_ctx* ctx, h2g_blocks* bt, int kernel, int dim, const double* points,
                        const double* weights, const long long* rank, const long long* loff, const long long* xoff,
                        const double* basis, long long basis_len, const long long* node_off, const double* nodes,
                        long long nodes_len, h2g_h2** out) {
  return guarded([&] {
    auto h = build_kernel_h2(ctx->c, bt->b, kernel, dim, points, weights, rank, loff, xoff, basis, basis_len,
                             node_off, nodes, nodes_len);
    h->own_rows = bt->rows;
    h->own_cols = bt->cols;
    *out = new h2g_h2{h};
  });
}

int h2g_matvec(h2g_ctx* ctx, h2g_h2* g, int trans, const double* x, double* y, double alpha, int accumulate) {
  return guarded([&] {
    if (!x || !y) throw InvalidInput("matvec: null vector");
    gather_rows(ctx->c, *g->h);  // a partitioned product: complete it first
    h2_matvec(ctx->c, HView{g->h.get(), trans != 0}, x, y, alpha, accumulate != 0);
  });
}

int h2g_multiply(h2g_ctx* ctx, h2g_h2* x, h2g_h2* y, double tol, int max_rank, int scaling, h2g_h2** g) {
  return guarded([&] {
    x->h->start_near(ctx->c);
    y->h->start_near(ctx->c);
    need_whole(ctx->c, *x->h);
    need_whole(ctx->c, *y->h);
    auto G = multiply(ctx->c, *x->h, *y->h, tol, max_rank, scaling != 0);
    G->keep.push_back(x->h->bt);
    G->keep.push_back(y->h->bt);
    G->keep.push_back(x->h->own_rows);
    G->keep.push_back(y->h->own_cols);
    *g = new h2g_h2{G};
  });
}

int h2g_coarsen(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank, int scale_blocks,
                h2g_h2** z) {
  return h2g_coarsen_prefetch(ctx, g, coarse, tol, max_rank, scale_blocks, nullptr, 0, z);
}

int h2g_coarsen_prefetch(h2g_ctx* ctx, h2g_h2* g, h2g_blocks* coarse, double tol, int max_rank, int scale_blocks,
                         double* near_host, long long near_len, h2g_h2** z) {
  return guarded([&] {
    need_rows_halo(ctx->c, *g->h);
    auto Z = coarsen(ctx->c, *g->h, coarse->b, tol, max_rank, scale_blocks != 0, near_host, near_len);
    Z->keep.push_back(coarse->rows);
    Z->keep.push_back(coarse->cols);
    Z->keep.push_back(g->h->bt);
    Z->keep.push_back(g->h->own_rows);
    Z->keep.push_back(g->h->own_cols);
    for (auto& k : g->h->keep) Z->keep.push_back(k);
    *z = new h2g_h2{Z};
  });
}

int h2g_recompress(h2g_ctx* ctx, h2g_h2* x, double tol, int max_rank, h2g_h2** z) {
  return guarded([&] {
    if (tol < 0) throw InvalidInput("tolerance must be >= 0");
    need_whole(ctx->c, *x->h);
    auto Z = recompress(ctx->c, *x->h, tol, max_rank);
    Z->keep.push_back(x->h->bt);
    Z->keep.push_back(x->h->own_rows);
    Z->keep.push_back(x->h->own_cols);
    *z = new h2g_h2{Z};
  });
}

}  // extern "C"
