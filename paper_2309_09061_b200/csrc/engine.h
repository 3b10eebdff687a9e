// Host-side engine of the B200 H^2 product: structure, device arenas, batch planning.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <future>
#include <mutex>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "h2g_types.h"

namespace h2g {

// ------------------------------------------------------------------ errors (C-ABI status codes)
struct InvalidInput : std::runtime_error { using std::runtime_error::runtime_error; };   // 1
struct StructureErr : std::runtime_error { using std::runtime_error::runtime_error; };   // 2
struct CudaFailure : std::runtime_error { using std::runtime_error::runtime_error; };    // 3

void cuda_check(cudaError_t e, const char* what);

// ------------------------------------------------------------------ kernels (kernels.cu)
cudaError_t launch_gsum(const GOut*, const GTerm*, const GTile*, int ntiles, int k2max, cudaStream_t, int tag = 0);
cudaError_t launch_gsum_lean(const GOut*, const GTerm*, const GLTile*, int ntiles, bool wide, cudaStream_t);
cudaError_t launch_gsum_sum(const GOut*, const GTerm*, const GLTile*, int ntiles, cudaStream_t);
int gsum_sum_chunk();
cudaError_t launch_gsum_whole(const GOut*, const GTerm*, const GTile*, int ntiles, int k2max, cudaStream_t);
cudaError_t launch_qr_chunks(const QrItem*, const Seg*, const SvdWork*, int nwork, size_t smem, bool rsmem,
                             cudaStream_t);
cudaError_t launch_tsqr_merge(const MergeWork*, int nwork, size_t smem, bool rsmem, cudaStream_t);
cudaError_t launch_qr_out(const QrItem*, int nitems, cudaStream_t);
cudaError_t launch_svd_tsqr(const SvdItem*, const Seg*, const SvdWork*, int nwork, size_t smem, bool rsmem,
                            cudaStream_t);
cudaError_t launch_gram(const GramItem* items, const Seg* segs, const GramWork* work, int nwork, int nflat,
                        int nitems, int mmax, cudaStream_t st);
size_t gram_chol_smem(int m);
cudaError_t launch_svd_finish(const SvdItem*, const Seg*, int nitems, size_t smem, bool rsmem, bool vsmem, int nmax,
                              cudaStream_t, bool tight = false);
cudaError_t launch_norm(const NormItem*, const Seg*, int nitems, size_t smem, cudaStream_t);
cudaError_t launch_gather(const long long* items, int nitems, cudaStream_t);
cudaError_t launch_norm_warp(const NormItem* items, const Seg* segs, int nitems, cudaStream_t);
cudaError_t launch_norm_cta(const NormItem* items, const Seg* segs, int nitems, size_t smem, cudaStream_t);
cudaError_t launch_norm_lz(const NormItem* items, const Seg* segs, int nitems, int mmax, int nmax, cudaStream_t);
size_t norm_cta_smem(int m, int N);
cudaError_t launch_asm_expand(const AsmTables& T, int ntrip, GTerm* terms, cudaStream_t);
cudaError_t launch_tile_absorb(const TileItem*, const Seg*, const TileWork*, int nwork, int nmax, cudaStream_t);
cudaError_t launch_svd_prep(const SvdItem*, const int* ids, int nids, size_t smem, cudaStream_t);
size_t tile_absorb_smem(int n);
size_t svd_prep_smem(int m, int kx, bool with_q = true);
size_t qr_smem(int n, bool rsmem);
size_t svd_tsqr_smem(int m, int kx, bool rsmem);
size_t merge_smem(int n, bool rsmem);
size_t svd_finish_smem(int m, int kx, bool rsmem, bool vsmem = true, bool tight = false);
size_t norm_smem(int m, long long N, bool gram_in_smem = true);

// ------------------------------------------------------------------ structure
struct Tree {
  int n = 0, depth = 0;
  std::vector<long long> start, stop;
  std::vector<int> parent, level, cptr, cidx;
  std::vector<std::vector<int>> by_level;
  bool leaf(int t) const { return cptr[t + 1] == cptr[t]; }
  int size(int t) const { return (int)(stop[t] - start[t]); }
  int nkids(int t) const { return cptr[t + 1] - cptr[t]; }
  int kid(int t, int i) const { return cidx[cptr[t] + i]; }
  bool same(const Tree& o) const;
  void finalize();
};

struct Blocks {
  const Tree* rows = nullptr;
  const Tree* cols = nullptr;
  int nb = 0, depth = 0;
  std::vector<int> row, col, cptr, cidx, parent, level;
  std::vector<unsigned char> adm;
  std::vector<int> rptr, rcol, rblk;  // per row cluster: blocks sorted by column (lookup table)
  std::vector<std::vector<int>> by_level;
  bool leaf(int b) const { return cptr[b + 1] == cptr[b]; }
  bool adm_leaf(int b) const { return leaf(b) && adm[b]; }
  bool near_leaf(int b) const { return leaf(b) && !adm[b]; }
  int nkids(int b) const { return cptr[b + 1] - cptr[b]; }
  int kid(int b, int i) const { return cidx[cptr[b] + i]; }
  int find(int t, int s) const {  // binary search in row t's blocks (replaces the reference's dict)
    int lo = rptr[t], hi = rptr[t + 1];
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (rcol[mid] < s) lo = mid + 1; else hi = mid;
    }
    return (lo < rptr[t + 1] && rcol[lo] == s) ? rblk[lo] : -1;
  }
  void finalize();
};

// Row/column-swapped view of a block tree (reference BlockTree.transposed, trees.py:211-214).
struct BView {
  const Blocks* b;
  bool T;
  const Tree& rows() const { return T ? *b->cols : *b->rows; }
  const Tree& cols() const { return T ? *b->rows : *b->cols; }
  int row(int i) const { return T ? b->col[i] : b->row[i]; }
  int col(int i) const { return T ? b->row[i] : b->col[i]; }
  int find(int t, int s) const { return T ? b->find(s, t) : b->find(t, s); }
  int nb() const { return b->nb; }
};

// ------------------------------------------------------------------ device memory
struct Arena {  // bump allocator over cudaMalloc'd chunks, freed together
  cudaStream_t st = nullptr;
  bool cross_stream = false;  // used by other streams too: free after a device-wide sync
  // cross-stream arenas with a free stream: freed stream-ordered on free_st after everything queued
  // so far on the `after` streams (no device-wide synchronisation; see Ctx::order_free)
  cudaStream_t free_st = nullptr;
  std::vector<cudaStream_t> after;
  std::vector<void*> chunks;
  char* cur = nullptr;
  size_t left = 0;
  size_t bytes = 0;
  explicit Arena(cudaStream_t s) : st(s) {}
  ~Arena();
  double* alloc(size_t ndoubles);
  void* alloc_bytes(size_t nbytes);
};
using ArenaPtr = std::shared_ptr<Arena>;
extern std::atomic<long long> g_arena_payload, g_arena_payload_high;
// H2G_DEBUG_MEM=1: arena payload (now / high-water, MB) at the stage boundaries of a product
void mem_mark(const char* where);

struct Mat {
  double* p = nullptr;
  int r = 0, c = 0;
  MatRef ref() const { return MatRef{p, c, 1}; }
  MatRef tref() const { return MatRef{p, 1, c}; }
  Mat band(int r0, int nr) const { return Mat{p + (long long)r0 * c, nr, c}; }
};
inline MatRef trn(MatRef m) { return MatRef{m.p, m.cs, m.rs}; }

struct Basis {  // leaf (size x k, ld k); xfer (k_c x k_parent, ld k_parent)
  const Tree* tree = nullptr;
  std::vector<int> rank;
  std::vector<double*> leaf, xfer;
  Mat leafm(int t) const { return Mat{leaf[t], tree->size(t), rank[t]}; }
  Mat xferm(int c) const { return Mat{xfer[c], rank[c], rank[tree->parent[c]]}; }
};

struct Ctx;

struct H2 {
  std::shared_ptr<const Blocks> bt;
  // partitioned product (multi-GPU): this rank holds the leaf blocks of its own block rows (plus the
  // replicated top rows and, for G, the halo its column passes read); gather_rows() completes it
  bool dist_rows = false;
  bool dist_halo = false;  // a partitioned product G: also holds the blocks its column passes read
  std::shared_ptr<Basis> rb, cb;
  std::vector<double*> coup, near;
  std::vector<ArenaPtr> owned;
  ArenaPtr near_owner;  // arena holding the nearfield blocks (shared by a coarsened result)
  // asynchronous upload: the nearfield copy completes at this event.  The copy itself is deferred
  // (start_near) until the matrix is first used, so that the small arrays (bases, couplings) of a
  // second operand uploaded right after do not queue behind 3 GB of nearfield on the copy engine:
  // multiply starts both operands' copies after all the small ones.
  mutable cudaEvent_t near_ready = nullptr;
  mutable const double* near_src = nullptr;  // pending host source (pinned or pageable), null once started
  mutable double* near_dst = nullptr;
  mutable size_t near_bytes = 0;
  mutable cudaEvent_t near_alloc = nullptr;  // the device allocation is stream-ordered: the copy follows it
  void start_near(Ctx& C) const;
  // nearfield prefetch to the host (coarsen with a host buffer): blocks already copied, the target
  // buffer and the event that completes the copy
  std::vector<char> near_on_host;
  double* near_host = nullptr;
  cudaEvent_t near_host_ready = nullptr;
  ~H2() {
    if (near_ready) cudaEventDestroy(near_ready);
    if (near_alloc) cudaEventDestroy(near_alloc);
    if (near_host_ready) cudaEventDestroy(near_host_ready);
  }
  std::shared_ptr<Tree> own_rows, own_cols;  // trees owned by this matrix (when built here)
  std::vector<std::shared_ptr<const void>> keep;  // other structure this matrix points into
  mutable std::shared_ptr<struct MvPlan> mv_plan[2];  // cached matvec launch plans (plain, transposed)
  // phase-2 block-norm batches of this matrix (product output): built on a host thread while the
  // assembly runs on the GPU, consumed by coarsen (declared last: joined before the rest goes)
  std::shared_future<std::shared_ptr<struct NormPrep>> norm_prep;
};

// Transposable view of an H^2 matrix (reference H2Matrix.transposed, h2.py:169-173).
struct HView {
  const H2* h;
  bool T;
  BView bv() const { return BView{h->bt.get(), T}; }
  const Tree& rows() const { return T ? *h->bt->cols : *h->bt->rows; }
  const Tree& cols() const { return T ? *h->bt->rows : *h->bt->cols; }
  const Basis& rb() const { return T ? *h->cb : *h->rb; }
  const Basis& cb() const { return T ? *h->rb : *h->cb; }
  int row(int b) const { return T ? h->bt->col[b] : h->bt->row[b]; }
  int col(int b) const { return T ? h->bt->row[b] : h->bt->col[b]; }
  int find(int t, int s) const { return T ? h->bt->find(s, t) : h->bt->find(t, s); }
  MatRef coup(int b) const {
    const int ld = h->cb->rank[h->bt->col[b]];
    return T ? MatRef{h->coup[b], 1, ld} : MatRef{h->coup[b], ld, 1};
  }
  MatRef near(int b) const {
    const int ld = h->bt->cols->size(h->bt->col[b]);
    return T ? MatRef{h->near[b], 1, ld} : MatRef{h->near[b], ld, 1};
  }
};

// ------------------------------------------------------------------ multi-GPU
// In-place variable all-gather over the ranks of one product: dbuf holds nseg = P segments
// [off[i], off[i+1]) bytes; on entry segment `rank` is valid, on return every segment is.  Issued on
// `stream` (the device buffer is stream-ordered); returns 0 on success.  Supplied by the host
// (torch.distributed over NCCL in production, gloo with host staging in tests); `channel` 0 / 1 keeps
// the concurrent row / column passes on separate communicators.
typedef int (*AllgatherFn)(void* user, int channel, void* dbuf, const long long* off, int nseg, void* stream);
// Variable all-to-all: rank i sends bytes [soff[j], soff[j+1]) of sbuf to rank j and receives rank j's
// bytes into [roff[j], roff[j+1]) of rbuf (device buffers, stream-ordered).  Optional: without it the
// engine falls back to all-gathers (every rank then receives every exchanged block).
typedef int (*AlltoallFn)(void* user, int channel, const void* sbuf, const long long* soff, void* rbuf,
                          const long long* roff, int nseg, void* stream);
struct Comm {
  int rank = 0, size = 1;
  AllgatherFn fn = nullptr;
  void* user = nullptr;
  AlltoallFn a2a = nullptr;
  void* a2a_user = nullptr;
  bool on() const { return size > 1 && fn != nullptr; }
};

// Orders the collectives of the two concurrent passes of a partitioned product (row pass: channel 0,
// column pass: channel 1, each on its own host thread, stream and communicator): channel 1 issues its
// exchanges only after channel 0 has issued all of its own, and its stream waits for them, so every
// rank issues -- and every GPU runs -- the collectives of the two communicators in the same order (no
// cross-communicator circular wait).  Channel 0 never waits.
struct PassGate {
  std::mutex m;
  std::condition_variable cv;
  bool ch0_done = false;
  cudaEvent_t ev0 = nullptr;  // channel 0's stream after its exchanges
  ~PassGate() {
    if (ev0) cudaEventDestroy(ev0);
  }
};

// ------------------------------------------------------------------ context: stream + staging
// Device times (ms) in the reference harness's stage split (bench.py:195-237).  The row and column
// passes of each phase run concurrently on two streams: t1_row / t1_col (t2_row / t2_col) are each
// pass's own span on its stream, the *_span fields the joint span; setup = basis product + the row
// pass's total weights, setup_col = the column pass's weights (concurrent with setup's weights);
// t2_norms = the block norms (part of t2_row, as in the reference).
struct StageTimes {
  float setup = 0, t1_row = 0, t1_col = 0, t1_mat = 0, t2_row = 0, t2_col = 0, t2_mat = 0;
  float setup_col = 0, t1_span = 0, t2_span = 0, t2_norms = 0;
};
// event on the context's stream when timing (null otherwise)
inline cudaEvent_t mark_event(struct Ctx& c);

// Per-kernel-class accounting for the roofline (profile mode only; never inside a timed step).
enum KClass { K_GSUM = 0, K_QR = 1, K_SVD = 2, K_NORM = 3, K_GATHER = 4, K_MV = 5, K_NCLASS = 6 };
// trace-only sub-intervals (not counted in the kernel-class statistics)
enum KSub { S_SVD_TSQR = 6, S_MERGE = 7, S_SVD_FIN = 8, S_QR_CHUNK = 9, S_MISC = 10, S_NSUB = 11 };
struct KStat {
  long long launches = 0;
  double ms = 0, flops = 0, bytes = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  // pinned host staging and device staging for descriptors (reset at every host sync)
  char* hstage = nullptr;
  char* dstage = nullptr;
  std::vector<std::pair<char*, char*>> retired;  // full staging buffers awaiting the next sync
  size_t stage_cap = 0, stage_off = 0, stage_flushed = 0;
  char* hread = nullptr;  // pinned read-back area
  size_t read_cap = 0;
  long long launches = 0;  // kernels launched since the last reset
  long long syncs = 0;
  StageTimes times;
  bool timing = false;
  std::vector<cudaEvent_t> evpool;
  bool prof = false;
  KStat kstat[K_NCLASS];
  struct Pending {
    int cls;
    cudaEvent_t a, b;
    double flops, bytes;
    std::string tag;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> free_ev;
  std::map<std::string, double> htime;  // host-side ms per named section (timing mode)
  // timeline tracing (profile mode + trace): device intervals per launch, host sync waits
  struct TraceRec {
    int cls, tid;
    double t0_us, dur_us;
    double flops;
    std::string tag;
  };
  std::string tag;  // current stage label (profile/trace mode), set by StageTag
  bool trace = false;
  int trace_tid = 0;
  cudaEvent_t trace_base = nullptr;
  std::chrono::steady_clock::time_point trace_host0;
  std::vector<TraceRec>* trace_out = nullptr;  // shared with the side context
  std::vector<TraceRec> trace_recs;
  cudaEvent_t prof_begin();
  void prof_end(int cls, cudaEvent_t a, double flops, double bytes);
  cudaEvent_t sub_begin() { return trace ? prof_begin() : nullptr; }
  void sub_end(int cls, cudaEvent_t a) { if (trace) prof_end(cls, a, 0.0, 0.0); }
  void drain_prof();

  Comm comm;        // ranks sharing this product (size 1: single GPU)
  PassGate* gate = nullptr;  // set while two passes run concurrently (partitioned products)
  void gate_enter();         // before this pass's partition-level exchanges
  void gate_leave();         // after them (channel 0: releases channel 1; idempotent)
  int channel = 0;  // communicator of this context's host thread (side context: 1)
  std::unique_ptr<Ctx> side_;  // second stream + staging for the concurrent column passes
  cudaStream_t up_stream = nullptr;  // structure uploads from the planner thread
  std::vector<std::weak_ptr<H2>> deferred_near;  // asynchronous uploads whose nearfield copy has not started
  char* up_host = nullptr;
  size_t up_cap = 0;
  std::unique_ptr<Ctx> aux_;   // low-priority stream: work ahead of the critical path (dense targets)
  std::unique_ptr<Ctx> aux_hi_;  // normal-priority auxiliary stream (phase-2 nearfield norms)
  cudaStream_t mv_st = nullptr;  // matvec nearfield stream (concurrent with the transform chain)
  cudaStream_t mv_stream();
  Ctx(int dev, cudaStream_t s, int priority = 0);
  ~Ctx();
  Ctx& side();
  Ctx& aux(bool urgent = false);  // urgent: main-stream priority instead of the lowest
  void join_side(Ctx& S);  // main stream waits for the side stream's queued work
  void* stage(const void* src, size_t bytes);  // returns device pointer (copied at the next flush())
  void flush();  // enqueue the host->device copy of everything staged since the last flush
  template <class T> T* push(const std::vector<T>& v) {
    return v.empty() ? nullptr : (T*)stage(v.data(), v.size() * sizeof(T));
  }
  void sync();
  template <class T> std::vector<T> read(const T* dptr, size_t n) {
    std::vector<T> out(n);
    if (n == 0) return out;
    ensure_read(n * sizeof(T));
    cuda_check(cudaMemcpyAsync(hread, dptr, n * sizeof(T), cudaMemcpyDeviceToHost, st), "read");
    sync();
    memcpy(out.data(), hread, n * sizeof(T));
    return out;
  }
  void ensure_read(size_t bytes);
  cudaEvent_t event();
  // a cross-stream arena of this context's product: free it on the main stream after the work
  // queued on every stream of the context (main, side, auxiliary, uploads) at destruction time
  void order_free(Arena& a);
};

inline cudaEvent_t mark_event(Ctx& c) {
  if (!c.timing) return nullptr;
  cudaEvent_t e = c.event();
  cudaEventRecord(e, c.st);
  return e;
}
inline float event_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  if (a && b) cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Scoped host timer, active when the context is in timing mode.
struct HostTimer {
  Ctx& C;
  const char* name;
  std::chrono::steady_clock::time_point t0;
  HostTimer(Ctx& c, const char* n) : C(c), name(n), t0(std::chrono::steady_clock::now()) {}
  ~HostTimer() { stop(); }
  void stop() {  // book the running section (no-op once stopped)
    if (name && C.timing)
      C.htime[name] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    name = nullptr;
  }
  void next(const char* n) {  // book the running section and start the next one
    stop();
    name = n;
    t0 = std::chrono::steady_clock::now();
  }
};

// H2G_SERIAL=1 (or h2g_set_serial): run the row and column passes one after the other on the main
// stream (profiling).  Read at the start of each pass structure decision; toggle between products only.
extern std::atomic<bool> g_serial;
inline bool serial_passes() {
  static const bool env = getenv("H2G_SERIAL") != nullptr;
  return env || g_serial.load();
}

// Labels the launches issued in its scope (trace mode only).
struct StageTag {
  Ctx& C;
  std::string prev;
  StageTag(Ctx& c, const std::string& t) : C(c) {
    if (C.trace) {
      prev = C.tag;
      C.tag = t;
    }
  }
  ~StageTag() {
    if (C.trace) C.tag = prev;
  }
};

// ------------------------------------------------------------------ batches
struct GBatch {
  std::vector<GOut> outs;
  std::vector<GTerm> terms;
  int k2max = 0;
  void out(Mat c, bool beta) { outs.push_back(GOut{c.p, c.c, c.r, c.c, beta ? 1 : 0, (int)terms.size(), (int)terms.size()}); }
  void t1(MatRef a, double al = 1.0);
  void t2(MatRef a, MatRef b, int k, double al = 1.0);
  void t3(MatRef a, MatRef b, MatRef d, int k, int k2, double al = 1.0);
  void run(Ctx& C);
  // launch with a device-resident term array (terms generated on the GPU); `outs` index into it
  void run_device_terms(Ctx& C, const GTerm* d_terms, double flops_hint);
  int tag = 0;               // kernel symbol (1: dense-target assembly, selectable in profilers)
  bool whole = false;        // outputs up to 128 x 128 as one CTA each (gsum_whole_kernel: cached T / U)
  std::vector<GTile> tiles;  // prepare_tiles(): the 64x64 output tiles, built ahead (any thread)
  std::vector<GTile> whole_tiles;  // outputs handled whole (one CTA each), when `whole`
  bool tiles_ready = false;
  void prepare_tiles();
  bool empty() const { return outs.empty(); }
};

struct SegList {  // segments of the batch's items; begin() opens (and closes) an item
  std::vector<Seg> segs;
  long long cur = 0;
  int begin() {
    cur = 0;
    return (int)segs.size();
  }
  void add(MatRef a, int w, double scale = 1.0, const double* sdiv = nullptr) {
    if (w > 0) {
      segs.push_back(Seg{a, w, 0, scale, cur, sdiv});
      cur += w;
    }
  }
};

struct QrBatch {
  SegList sl;
  std::vector<QrItem> items;
  // returns Mat (min(M, n) x n) output allocated from `ar`
  void run(Ctx& C, Arena& scratch);
};

struct NormBatch {
  SegList sl;
  std::vector<NormItem> items;
  std::vector<double> run(Ctx& C, Arena& scratch);  // sync + values
  // no host synchronisation: each item writes sigma_1 to its preset `out` (caller zero-fills)
  void run_async(Ctx& C);
  Arena* scratch = nullptr;  // for Gram matrices of large items (else a local arena)
};

// Spectral-norm batches of every leaf block of an H^2 matrix (reference coarsening.py:342-351):
// nearfield norms (device-resident divisors) and coupling norms (read back), pure host structure.
struct NormPrep {
  NormBatch nbn, nbc;
  std::vector<int> ids;   // block of each coupling item
  std::vector<int> nids;  // block of each nearfield item (its output slot in the divisor array)
};
std::shared_ptr<NormPrep> build_norm_prep(const H2& g, const Comm& comm);

struct SvdBatch {
  SegList sl;
  std::vector<SvdItem> items;
  std::vector<int> run(Ctx& C, Arena& scratch);  // sync + ranks (k1 + k2)
};

// H^2 matvec launch plan (matvec.cu): descriptors built and uploaded once per matrix and orientation,
// replayed with the call's x, y, alpha and accumulate flag.
struct MvPlan;

using MatStore = std::vector<Mat>;
struct PRef {  // basis product view (transposed for the column pass)
  const MatStore* P;
  bool T;
  MatRef at(int s) const { return T ? (*P)[s].tref() : (*P)[s].ref(); }
  int rows(int s) const { return T ? (*P)[s].c : (*P)[s].r; }
  int cols(int s) const { return T ? (*P)[s].r : (*P)[s].c; }
};

struct PairMap {
  std::unordered_map<long long, Mat> m;
  static long long key(int a, int b) { return ((long long)a << 32) | (unsigned)b; }
  Mat* get(int a, int b) {
    auto it = m.find(key(a, b));
    return it == m.end() ? nullptr : &it->second;
  }
  void put(int a, int b, Mat v) { m[key(a, b)] = v; }
};

struct Induced {
  std::shared_ptr<Basis> q;
  MatStore bc;
  std::vector<Mat> proj;    // per block of X (view): Q_t^T X|ts V_Y,s for non-admissible-leaf blocks
  std::vector<Mat> xv;      // per block of X (view), leaf rows: X|ts V_Y,s (induced.py:59-73)
  std::vector<double> gap;  // min |sigma - thr| / thr per cluster (diagnostic)
};

struct PTree {  // product block tree with the classified triples per node
  std::shared_ptr<Blocks> bt;
  std::vector<int> tptr;  // per node: triples [tptr[b], tptr[b+1])
  std::vector<int> ts;    // middle cluster
  std::vector<char> tk;   // kind 'a' 'b' 'c'
  std::vector<int> tbx, tby;  // block ids of X|ts and Y|sr
  // filled by the asynchronous planner thread: distinct X / Y blocks feeding dense targets
  // (kinds a / b) and the triple arrays already copied to the device
  std::vector<int> need_xv, need_wy;
  std::vector<int> rf_blocks;  // distinct admissible-leaf X blocks of kind-a triples on non-dense targets
  // dense targets assembled ahead (assemble_dense_early): they depend on the inputs only, so they
  // run on the auxiliary stream while the induced bases are computed
  struct Early {
    bool on = false;
    ArenaPtr near;             // the dense target blocks (become G's nearfield)
    std::vector<double*> blk;  // per product block: its dense target (this rank's rows) or null
    ArenaPtr scratch;          // memoised leaf products and the expanded terms
    cudaEvent_t done = nullptr;
  } early;
  struct Dev {
    int *tnode = nullptr, *ts = nullptr, *tbx = nullptr, *tby = nullptr;
    char* tk = nullptr;
    void* block = nullptr;
    cudaEvent_t ready = nullptr;
  } dev;
};
void ptree_prepare(PTree& P, Ctx& C, const Blocks& BX, int nby);

// ------------------------------------------------------------------ row-subtree partition (shard.cu)
// Ownership of the clusters of one tree among P ranks: the subtrees rooted at the first level with
// at least P clusters (level log2 P on the balanced BASELINE trees) are dealt out in contiguous runs;
// clusters above that level are replicated (owner -1) and computed by every rank.
struct Part {
  int P = 1, me = 0, level = -1;
  std::vector<int> owner;
  bool on() const { return level >= 0; }
  bool mine(int t) const { return !on() || owner[t] < 0 || owner[t] == me; }
  bool top(int t) const { return !on() || owner[t] < 0; }
  std::vector<int> filter(const std::vector<int>& L) const;  // the clusters of L this rank computes
};
Part make_part(const Tree& tr, int P, int me);
inline Part make_part(const Tree& tr, const Comm& c) {
  return c.on() ? make_part(tr, c.size, c.rank) : Part{};
}
// One exchanged array: `len` doubles produced by rank `owner`; on the owner *dst is the source, on
// every other rank *dst is set to the received copy (allocated from the arena passed to exchange()).
struct XItem {
  int owner;
  long long len;
  double** dst;
};
void exchange(Ctx& C, Arena& ar, const std::vector<XItem>& items);
// Point-to-point exchange: `len` doubles produced by rank `src` are needed by rank `dst` (src != dst);
// every rank lists the same items in the same order.  On dst, *ptr is set to the received copy
// (allocated from `ar`); on src, *ptr is the source.  One all-to-all (Comm::a2a), or an all-gather
// when the host supplied none.
struct PItem {
  int src, dst;
  long long len;
  double** ptr;
};
void exchange_p2p(Ctx& C, Arena& ar, const std::vector<PItem>& items);
// Complete a row-distributed matrix (H2::dist_rows) on every rank: all-gather of the leaf blocks of
// the partitioned block rows (downloads and matvecs of a partitioned product call it).
void gather_rows(Ctx& C, H2& h);
// inputs of the partitioned stages: a product's factors must be whole (gathered if distributed);
// coarsen reads its own rows plus the column halo (a partitioned product G has it, anything else
// distributed is gathered)
void need_whole(Ctx& C, H2& h);
void need_rows_halo(Ctx& C, H2& h);
// Integer per-cluster values (ranks): v[t] for the listed clusters is taken from owner[t].
void exchange_ints(Ctx& C, const Part& part, const std::vector<int>& ids, std::vector<int>& v);

// ------------------------------------------------------------------ stages
std::shared_ptr<Tree> make_tree(int n, const long long* start, const long long* stop, const long long* cptr,
                                const long long* cidx);
std::shared_ptr<Blocks> make_blocks(const Tree* rows, const Tree* cols, int nb, const long long* row,
                                    const long long* col, const long long* cptr, const long long* cidx,
                                    const unsigned char* adm);

void xv_compute(Ctx& C, Arena& ar, HView x, HView y, PRef P, const std::vector<int>& want,
                std::vector<Mat>& memo);
MatStore basis_product(Ctx& C, Arena& ar, const Basis& W, const Basis& V);
MatStore basis_weights(Ctx& C, Arena& ar, const Basis& W);
// exact_rows: leave exactly-zero blocks out of the stacks' row counts (one norm read-back); callers
// whose truncation tolerance makes the eps * max(rows, cols) floor irrelevant (floor_free_tol) skip it
MatStore total_weights(Ctx& C, Arena& ar, HView h, const MatStore& rw, bool scaling, bool exact_rows = true);
// Above this tolerance the SVD floor max(rows, cols) eps sigma_1 (rows, cols <= 1e5, sigma_1 of block-
// normalised stacks <= 1e2) stays below tol, so the exact row counts of zero-block stacks cannot matter
constexpr double kFloorFreeTol = 1e-8;
Induced induced_rows(Ctx& C, Arena& out, HView x, HView y, const MatStore& zy, PRef P, double tol,
                     int max_rank, bool scale, double level_decay);
PTree product_tree(BView bx, BView by);
std::vector<Mat> row_factors(Ctx& C, Arena& sc, HView x, HView y, const Induced& qr, PRef P, const PTree& pt);
std::shared_ptr<H2> assemble(Ctx& C, HView x, HView y, Induced& qr, Induced& qc, PRef P, PTree& pt,
                             const std::vector<Mat>* rf_pre = nullptr);
void assemble_dense_early(Ctx& A, HView x, HView y, PRef P, PTree& pt, cudaEvent_t inputs_ready, const Comm& comm);
std::shared_ptr<H2> multiply(Ctx& C, const H2& x, const H2& y, double tol, int max_rank, bool scaling);
std::shared_ptr<H2> coarsen(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, double tol, int max_rank,
                            bool scale, double* near_host, long long near_cap);
std::shared_ptr<H2> coarsen(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, double tol, int max_rank,
                            bool scale);
void h2_matvec(Ctx& C, HView g, const double* x, double* y, double alpha, bool accumulate);
// make the context's stream wait for an asynchronously uploaded nearfield (no-op otherwise)
inline void wait_near(Ctx& C, const H2& h) {
  h.start_near(C);
  if (h.near_ready) cuda_check(cudaStreamWaitEvent(C.st, h.near_ready, 0), "wait nearfield upload");
}
std::shared_ptr<H2> build_kernel_h2(Ctx& C, std::shared_ptr<const Blocks> bt, int kind, int dim,
                                    const double* points, const double* weights, const long long* rank,
                                    const long long* loff, const long long* xoff, const double* basis,
                                    long long basis_len, const long long* node_off, const double* nodes,
                                    long long nodes_len);
std::shared_ptr<H2> recompress(Ctx& C, const H2& g, double tol, int max_rank);

// ------------------------------------------------------------------ stage-level entry points
// The reference's stage functions one call at a time (bench.py:195-237 times them individually):
// results own their device arenas and can be inspected or fed to the next stage.
struct InducedStage {  // InducedBasisResult (induced.py:33-46) of a row (T = false) or column pass
  Induced ind;
  ArenaPtr ar;
  std::vector<ArenaPtr> keep;
  bool T = false;
};
std::shared_ptr<InducedStage> induced_stage(Ctx& C, const H2& x, const H2& y, const MatStore& z, const MatStore& P,
                                            bool col, double tol, int max_rank, bool scale, double level_decay);
std::shared_ptr<H2> assemble_stage(Ctx& C, const H2& x, const H2& y, const InducedStage& qr, const InducedStage& qc,
                                   const MatStore& P, std::vector<ArenaPtr> keep);
struct CoarseStage;  // CoarsenState (coarsening.py:36-50), phase2.cu
std::shared_ptr<CoarseStage> coarse_basis_stage(Ctx& C, const H2& g, std::shared_ptr<const Blocks> coarse, bool col,
                                                double tol, int max_rank, bool scale, const double* d_cn,
                                                const double* d_nn);
void block_norms_stage(Ctx& C, const H2& g, double* d_cn, double* d_nn);
std::shared_ptr<H2> project_final_stage(Ctx& C, const H2& g, const CoarseStage& rs, const CoarseStage& cs,
                                        std::shared_ptr<const Blocks> coarse);
std::shared_ptr<Basis> coarse_stage_basis(const CoarseStage& s, MatStore* r, MatStore* z, ArenaPtr* ar, int* nreps);

}  // namespace h2g
