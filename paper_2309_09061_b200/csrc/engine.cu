// Host engine: structure, staging, batch planning and the stage drivers of the adaptive H^2 product.
//
// Every stage walks the reference recursion (h2mul induced.py / coarsening.py / weights.py) level by
// level over the cluster tree and emits one batched launch per dependency level; the only host
// round trips are the ones the algorithm forces (exact zero-norm skips and the data-dependent ranks
// that size the next level).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <functional>
#include <memory>
#include <thread>
#include <mutex>

#include "engine.h"

namespace h2g {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

// ============================================================================ infrastructure

std::atomic<bool> g_serial{false};  // h2g_set_serial (engine.h serial_passes)

// Process-wide payload of the arenas (bytes handed out, not the chunks behind them): the memory a
// product actually needs, independent of the 64 MB chunk granularity (h2g_ctx_mem).
std::atomic<long long> g_arena_payload{0}, g_arena_payload_high{0};

// Destructors cannot throw: failed CUDA calls there are reported (and cleared, so that they do not
// surface later as the "last error" of an unrelated launch) when H2G_DEBUG_API is set.
static void dtor_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  static const bool dbg = getenv("H2G_DEBUG_API") != nullptr;
  if (dbg) fprintf(stderr, "h2g: %s failed in a destructor: %s\n", what, cudaGetErrorString(e));
  cudaGetLastError();
}

void mem_mark(const char* where) {
  static const bool on = getenv("H2G_DEBUG_MEM") != nullptr;
  if (on)
    fprintf(stderr, "mem %-24s payload %9.1f MB  high %9.1f MB\n", where, g_arena_payload.load() / 1e6,
            g_arena_payload_high.load() / 1e6);
}

Arena::~Arena() {
  g_arena_payload -= (long long)bytes;
  if (cross_stream && free_st) {
    for (cudaStream_t s : after) {
      if (!s || s == free_st) continue;
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) continue;
      dtor_check(cudaEventRecord(e, s), "arena: event record on a user stream");
      dtor_check(cudaStreamWaitEvent(free_st, e, 0), "arena: free stream wait");
      cudaEventDestroy(e);
    }
    for (void* p : chunks) dtor_check(cudaFreeAsync(p, free_st), "arena: cudaFreeAsync (cross-stream)");
    return;
  }
  if (cross_stream) {
    cudaDeviceSynchronize();
    for (void* p : chunks) cudaFree(p);
    return;
  }
  for (void* p : chunks) dtor_check(cudaFreeAsync(p, st), "arena: cudaFreeAsync");
}

void* Arena::alloc_bytes(size_t nb) {
  nb = (nb + 255) & ~size_t(255);
  if (nb == 0) return nullptr;
  if (nb > left) {
    size_t chunk = std::max(nb, size_t(64) << 20);
    void* p = nullptr;
    static const bool dbg = getenv("H2G_DEBUG_ALLOC") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cuda_check(cudaMallocAsync(&p, chunk, st), "cudaMallocAsync");
    if (dbg) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 5.0) fprintf(stderr, "h2g: cudaMallocAsync(%.0f MB) took %.1f ms\n", chunk / 1e6, ms);
    }
    chunks.push_back(p);
    cur = (char*)p;
    left = chunk;
  }
  {
    const long long now = (g_arena_payload += (long long)nb);
    long long hw = g_arena_payload_high.load();
    while (now > hw && !g_arena_payload_high.compare_exchange_weak(hw, now)) {
    }
  }
  void* r = cur;
  cur += nb;
  left -= nb;
  bytes += nb;
  return r;
}

double* Arena::alloc(size_t n) { return (double*)alloc_bytes(n * sizeof(double)); }

Ctx::Ctx(int dev, cudaStream_t s, int priority) : device(dev), st(s) {
  cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  if (!st) {
    cuda_check(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, priority), "stream");
    own_stream = true;
  }
  // keep freed stream-ordered allocations in the pool between products (the default threshold of 0
  // hands every arena back to the driver at each synchronisation)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // no hidden cross-stream waits: by default an allocation may reuse memory freed on another stream
    // by making its stream wait for that stream's pending work (a level batch on the side stream
    // stalling behind the main stream's queue); the pool grows instead (H2G_POOL_DEPS=1: default)
    if (!getenv("H2G_POOL_DEPS")) {
      int zero = 0;
      cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
    }
    // H2G_POOL_RESERVE_GB=n: map n GB into the pool once, up front (growing it later maps memory on
    // the host thread of whichever allocation needs it)
    if (const char* r = getenv("H2G_POOL_RESERVE_GB")) {
      const double gb = atof(r);
      unsigned long long cur = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &cur);
      if (gb > 0 && (double)cur < gb * 1e9) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, (size_t)(gb * 1e9), st) == cudaSuccess) {
          cudaFreeAsync(p, st);
          cudaStreamSynchronize(st);
        }
        cudaGetLastError();
      }
    }
  }
  stage_cap = size_t(64) << 20;
  cuda_check(cudaMallocHost(&hstage, stage_cap), "cudaMallocHost");
  cuda_check(cudaMalloc(&dstage, stage_cap), "cudaMalloc stage");
  ensure_read(1 << 20);
}

Ctx::~Ctx() {
  cudaStreamSynchronize(st);
  if (mv_st) {
    cudaStreamSynchronize(mv_st);
    cudaStreamDestroy(mv_st);
  }
  if (up_stream) {
    cudaStreamSynchronize(up_stream);
    cudaStreamDestroy(up_stream);
  }
  if (up_host) cudaFreeHost(up_host);
  for (auto e : evpool) cudaEventDestroy(e);
  cudaFreeHost(hstage);
  cudaFree(dstage);
  for (auto& r : retired) {
    cudaFreeHost(r.first);
    cudaFree(r.second);
  }
  if (hread) cudaFreeHost(hread);
  if (own_stream) cudaStreamDestroy(st);
}

void Ctx::ensure_read(size_t bytes) {
  if (bytes <= read_cap) return;
  if (hread) cudaFreeHost(hread);
  read_cap = std::max(bytes, read_cap * 2);
  cuda_check(cudaMallocHost(&hread, read_cap), "cudaMallocHost read");
}

static std::mutex g_trace_mu;  // the main and side contexts share one trace vector

void Ctx::sync() {
  flush();
  HostTimer ht(*this, "sync_wait");
  const auto h0 = std::chrono::steady_clock::now();
  cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (trace && trace_out) {
    const auto h1 = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> lk(g_trace_mu);
    trace_out->push_back(TraceRec{-1 - trace_tid, trace_tid,
                                  std::chrono::duration<double, std::micro>(h0 - trace_host0).count(),
                                  std::chrono::duration<double, std::micro>(h1 - h0).count(), 0.0, tag});
  }
  stage_off = 0;
  stage_flushed = 0;
  for (auto& r : retired) {  // staging buffers retired by an overflow: consumed now
    cudaFreeHost(r.first);
    cudaFree(r.second);
  }
  retired.clear();
  ++syncs;
  if (!pending.empty()) drain_prof();
}

cudaEvent_t Ctx::prof_begin() {
  if (!prof) return nullptr;
  cudaEvent_t e;
  if (free_ev.empty()) {
    cuda_check(cudaEventCreate(&e), "event");
  } else {
    e = free_ev.back();
    free_ev.pop_back();
  }
  cudaEventRecord(e, st);
  return e;
}

void Ctx::prof_end(int cls, cudaEvent_t a, double flops, double bytes) {
  if (!prof || !a) return;
  cudaEvent_t b;
  if (free_ev.empty()) {
    cuda_check(cudaEventCreate(&b), "event");
  } else {
    b = free_ev.back();
    free_ev.pop_back();
  }
  cudaEventRecord(b, st);
  pending.push_back(Pending{cls, a, b, flops, bytes, trace ? tag : std::string()});
}

void Ctx::drain_prof() {
  for (auto& p : pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p.a, p.b);
    if (trace && trace_out && trace_base) {
      float t0 = 0;
      cudaEventElapsedTime(&t0, trace_base, p.a);
      std::lock_guard<std::mutex> lk(g_trace_mu);
      trace_out->push_back(TraceRec{p.cls, trace_tid, 1e3 * t0, 1e3 * ms, p.flops, p.tag});
    }
    free_ev.push_back(p.a);
    free_ev.push_back(p.b);
    if (p.cls >= K_NCLASS) continue;
    KStat& k = kstat[p.cls];
    k.launches += 1;
    k.ms += ms;
    k.flops += p.flops;
    k.bytes += p.bytes;
  }
  pending.clear();
}

void* Ctx::stage(const void* src, size_t bytes) {
  const size_t need = (bytes + 255) & ~size_t(255);
  if (stage_off + need > stage_cap) {
    // The buffer is full, but earlier pushes of the launch being prepared may still sit in it
    // (their device pointers are already handed out): never recycle it here.  Flush it, retire it
    // (freed at the next host sync, once the stream has consumed it) and continue in a new one.
    flush();
    retired.emplace_back(hstage, dstage);
    stage_cap = std::max(need, stage_cap * 2);
    static const bool dbg = getenv("H2G_DEBUG_STAGE") != nullptr;
    if (dbg) fprintf(stderr, "h2g: staging overflow, new buffer %.0f MB\n", stage_cap / 1e6);
    cuda_check(cudaMallocHost(&hstage, stage_cap), "cudaMallocHost");
    cuda_check(cudaMalloc(&dstage, stage_cap), "cudaMalloc stage");
    stage_off = 0;
    stage_flushed = 0;
  }
  char* h = hstage + stage_off;
  char* d = dstage + stage_off;
  HostTimer ht(*this, "stage_memcpy");
  memcpy(h, src, bytes);
  stage_off += need;  // copied to the device by the next flush() (one transfer per launch)
  return d;
}

void Ctx::flush() {
  if (stage_off > stage_flushed) {
    cuda_check(cudaMemcpyAsync(dstage + stage_flushed, hstage + stage_flushed, stage_off - stage_flushed,
                               cudaMemcpyHostToDevice, st),
               "stage copy");
    stage_flushed = stage_off;
  }
}

Ctx& Ctx::aux(bool urgent) {
  std::unique_ptr<Ctx>& a = urgent ? aux_hi_ : aux_;
  if (!a) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    int prio = least;
    if (urgent) cudaStreamGetPriority(st, &prio);  // as urgent as the main stream
    a.reset(new Ctx(device, nullptr, prio));
  }
  a->timing = timing;
  a->prof = prof;
  a->trace = trace;
  a->trace_tid = urgent ? 3 : 2;
  a->trace_base = trace_base;
  a->trace_host0 = trace_host0;
  a->trace_out = trace_out;
  a->channel = 2;  // no collectives
  return *a;
}

cudaStream_t Ctx::mv_stream() {
  if (!mv_st) {
    int prio = 0;
    cudaStreamGetPriority(st, &prio);
    cuda_check(cudaStreamCreateWithPriority(&mv_st, cudaStreamNonBlocking, prio), "matvec stream");
  }
  return mv_st;
}

Ctx& Ctx::side() {
  if (!side_) {
    int prio = 0;
    cudaStreamGetPriority(st, &prio);  // as urgent as the main stream
    side_.reset(new Ctx(device, nullptr, prio));
  }
  side_->timing = timing;
  side_->prof = prof;
  side_->trace = trace;
  side_->trace_tid = 1;
  side_->trace_base = trace_base;
  side_->trace_host0 = trace_host0;
  side_->trace_out = trace_out;
  side_->comm = comm;
  side_->channel = 1;
  // the side stream starts after everything queued so far on the main stream
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cudaEventRecord(e, st);
  cudaStreamWaitEvent(side_->st, e, 0);
  cudaEventDestroy(e);
  return *side_;
}

void Ctx::join_side(Ctx& S) {
  cudaEvent_t e;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cudaEventRecord(e, S.st);
  cudaStreamWaitEvent(st, e, 0);
  cudaEventDestroy(e);
  launches += S.launches;
  syncs += S.syncs;
  S.launches = S.syncs = 0;
  S.sync();  // drains the side's profile events (already complete once the join is waited on)
  for (int k = 0; k < K_NCLASS; ++k) {
    kstat[k].launches += S.kstat[k].launches;
    kstat[k].ms += S.kstat[k].ms;
    kstat[k].flops += S.kstat[k].flops;
    kstat[k].bytes += S.kstat[k].bytes;
    S.kstat[k] = KStat{};
  }
  for (auto& kv : S.htime) htime["side." + kv.first] += kv.second;
  S.htime.clear();
}

void Ctx::gate_enter() {
  if (!gate || !comm.on() || channel != 1) return;
  std::unique_lock<std::mutex> lk(gate->m);
  gate->cv.wait(lk, [this] { return gate->ch0_done; });
  if (gate->ev0) cuda_check(cudaStreamWaitEvent(st, gate->ev0, 0), "gate wait");
}

void Ctx::gate_leave() {
  if (!gate || channel != 0) return;
  std::lock_guard<std::mutex> lk(gate->m);
  if (gate->ch0_done) return;
  if (comm.on()) {
    cuda_check(cudaEventCreateWithFlags(&gate->ev0, cudaEventDisableTiming), "event");
    cuda_check(cudaEventRecord(gate->ev0, st), "event");
  }
  gate->ch0_done = true;
  gate->cv.notify_all();
}

// Every use of a product's memory on the side, auxiliary or copy streams is joined into the main
// stream before multiply / coarsen return (join_side, wait_near, the prefetch gather's event), so a
// cross-stream arena is freed stream-ordered on the main stream alone -- no device-wide sync, and no
// event on a stream that may be gone by then (the side / aux / copy streams die with their context;
// the main stream is the caller's).
void Ctx::order_free(Arena& a) {
  a.cross_stream = true;
  a.free_st = st;
  a.after.clear();
}

cudaEvent_t Ctx::event() {
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "event");
  evpool.push_back(e);
  return e;
}

void H2::start_near(Ctx& C) const {
  if (!near_src) return;
  if (!C.up_stream) cuda_check(cudaStreamCreateWithFlags(&C.up_stream, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamWaitEvent(C.up_stream, near_alloc, 0), "wait");
  cuda_check(cudaMemcpyAsync(near_dst, near_src, near_bytes, cudaMemcpyHostToDevice, C.up_stream), "upload");
  cuda_check(cudaEventCreateWithFlags(&near_ready, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(near_ready, C.up_stream), "event");
  near_src = nullptr;
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


// H2G_DEBUG_GSUM=1: per launch, how full its 64 x 64 tiles are (live 16 x 32 warp quadrants of 8)
static void gsum_tile_stats(const char* tag, const std::vector<GOut>& outs, const std::vector<GTile>& tiles,
                            const std::vector<GTerm>* terms) {
  static const bool dbg = getenv("H2G_DEBUG_GSUM") != nullptr;
  if (!dbg || tiles.size() < 500) return;
  double live = 0, full = 0, cells = 0, ksum = 0, kcnt = 0;
  long long hist[9] = {0};
  for (const GTile& t : tiles) {
    const GOut& o = outs[t.out];
    const int i0 = (t.tij & 0xffff) * 64, j0 = (t.tij >> 16) * 64;
    const int mt = std::min(64, o.m - i0), nt = std::min(64, o.n - j0);
    const int lw = ((mt + 15) / 16) * ((nt + 31) / 32);
    live += lw;
    ++hist[lw];
    full += (mt == 64 && nt == 64);
    cells += (double)mt * nt;
    if (terms)
      for (int i = o.t0; i < o.t1; ++i) {
        const GTerm& u = (*terms)[i];
        if (u.nf >= 2) { ksum += u.k; ++kcnt; }
      }
  }
  const double n = (double)tiles.size();
  fprintf(stderr, "gsum[%s] tiles %zu outs %zu: full %.2f, live warps %.2f/8, cell fill %.2f, mean k %.1f (%.1f terms/tile), live hist",
          tag ? tag : "", tiles.size(), outs.size(), full / n, live / n, cells / (4096.0 * n), ksum / std::max(1.0, kcnt), kcnt / n);
  for (int i = 1; i <= 8; ++i) fprintf(stderr, " %lld", hist[i]);
  fprintf(stderr, "\n");
}

void GBatch::run(Ctx& C) {
  HostTimer ht(C, "gbatch_run");
  std::vector<GTile> tiles;
  // outputs whose terms are plain sums and 2-factor products (no grouped / 3-factor terms) take the lean kernel:
  // 4-warp CTAs in the arrangement (32 x 64, 64 x 32, 16 x 128) that covers each output with the
  // fewest CTAs (H2G_GSUM_NO_LEAN=1: 64 x 64 tiles, for A/B)
  static const bool no_lean = getenv("H2G_GSUM_NO_LEAN") != nullptr;
  const bool lean_ok = !no_lean && tag == 0;  // decided per output: a batch may mix both kinds
  std::vector<GLTile> ltiles, stiles;
  bool wide = false;
  static const bool no_sum = getenv("H2G_GSUM_NO_SUM") != nullptr;  // A/B: sums through the GEMM kernels
  const int sum_chunk = gsum_sum_chunk();
  for (int i = 0; i < (int)outs.size(); ++i) {
    const GOut& o = outs[i];
    if (o.m <= 0 || o.n <= 0) continue;
    if (!no_sum && !o.ka && !o.kb) {  // plain sums / copies: the elementwise kernel
      bool sum_only = true;
      for (int t = o.t0; t < o.t1 && sum_only; ++t) sum_only = terms[t].nf <= 1;
      if (sum_only) {
        const long long tot = (long long)o.m * o.n;
        for (long long a = 0; a * sum_chunk < tot; ++a) stiles.push_back(GLTile{i, (int)a, 0, 0});
        continue;
      }
    }
    bool lean = lean_ok && !o.ka && !o.kb;
    for (int t = o.t0; t < o.t1 && lean; ++t) lean = terms[t].nf <= 2;
    if (lean) {
      auto cd = [](int a, int b) { return (a + b - 1) / b; };
      const int n0 = cd(o.m, 32) * cd(o.n, 64), n1 = cd(o.m, 64) * cd(o.n, 32), n2 = cd(o.m, 16) * cd(o.n, 128);
      // the 16 x 128 arrangement needs the larger stage (3 CTAs per SM instead of 4 for the whole
      // launch): only where it halves the CTA count
      const int lay = (2 * n2 <= n0 && 2 * n2 <= n1) ? 2 : (n1 < n0 ? 1 : 0);
      const int TM = lay == 0 ? 32 : (lay == 1 ? 64 : 16), TN = lay == 0 ? 64 : (lay == 1 ? 32 : 128);
      wide |= lay == 2;
      for (int a = 0; a < o.m; a += TM)
        for (int b = 0; b < o.n; b += TN) ltiles.push_back(GLTile{i, a, b, lay});
      continue;
    }
    const int tm = (o.m + 63) / 64, tn = (o.n + 63) / 64;
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) tiles.push_back(GTile{i, a | (b << 16)});
  }
  if (tiles.empty() && ltiles.empty() && stiles.empty()) return;
  {
    static const bool dbg = getenv("H2G_DEBUG_GSUM") != nullptr;
    if (dbg && ltiles.size() >= 500) {
      long long n1 = 0, n2 = 0, no = 0, k2 = 0, cells = 0;
      std::vector<char> seen(outs.size(), 0);
      for (const GLTile& t : ltiles) {
        if (seen[t.out]) continue;
        seen[t.out] = 1;
        const GOut& o = outs[t.out];
        ++no;
        cells += (long long)o.m * o.n;
        for (int i = o.t0; i < o.t1; ++i) {
          if (terms[i].nf == 1) ++n1;
          else if (terms[i].nf == 2) { ++n2; k2 += terms[i].k; }
        }
      }
      fprintf(stderr, "gsum-lean[%s] tiles %zu (sum tiles %zu) outs %lld: mean m*n %.0f, nf1 terms/out %.2f, nf2 terms/out %.2f, mean k %.1f, wide %d\n",
              C.tag.c_str(), ltiles.size(), stiles.size(), no, (double)cells / std::max(1LL, no), (double)n1 / std::max(1LL, no),
              (double)n2 / std::max(1LL, no), (double)k2 / std::max(1LL, n2), (int)wide);
    }
  }
  gsum_tile_stats(C.tag.c_str(), outs, tiles, &terms);
  GOut* d_o = C.push(outs);
  GTerm* d_t = C.push(terms);
  GTile* d_l = C.push(tiles);
  GLTile* d_ll = C.push(ltiles);
  GLTile* d_sl = C.push(stiles);
  double fl = 0, by = 0;
  if (C.prof) {  // algorithmic work: each product once at its own shape
    for (const GOut& o : outs) {
      if (o.m <= 0 || o.n <= 0) continue;
      by += 8.0 * o.m * o.n * (1 + o.beta);
      for (int i = o.t0; i < o.t1; ++i) {
        const GTerm& t = terms[i];
        if (t.nf == 1) { fl += (double)o.m * o.n; by += 8.0 * o.m * o.n; }
        else if (t.nf == 2) { fl += 2.0 * o.m * o.n * t.k; by += 8.0 * ((double)o.m * t.k + (double)t.k * o.n); }
        else {
          fl += 2.0 * o.m * t.k * t.k2 + 2.0 * o.m * t.k2 * o.n;
          by += 8.0 * ((double)o.m * t.k + (double)t.k * t.k2 + (double)t.k2 * o.n);
        }
      }
    }
  }
  cudaEvent_t ev = C.prof_begin();
  C.flush();
  if (!stiles.empty()) {
    cuda_check(launch_gsum_sum(d_o, d_t, d_sl, (int)stiles.size(), C.st), "gsum(sum)");
    ++C.launches;
  }
  if (!ltiles.empty()) {
    cuda_check(launch_gsum_lean(d_o, d_t, d_ll, (int)ltiles.size(), wide, C.st), "gsum(lean)");
    ++C.launches;
  }
  if (!tiles.empty()) {
    cuda_check(launch_gsum(d_o, d_t, d_l, (int)tiles.size(), k2max, C.st), "gsum");
    ++C.launches;
  }
  C.prof_end(K_GSUM, ev, fl, by);
  outs.clear();
  terms.clear();
  tiles.clear();
  tiles_ready = false;
  k2max = 0;
}

// H2G_GSUM_NO_WHOLE=1: every output through 64 x 64 tiles (A/B of the whole-output kernel)
static bool whole_ok() {
  static const bool off = getenv("H2G_GSUM_NO_WHOLE") != nullptr;
  return !off;
}

void GBatch::prepare_tiles() {
  tiles.clear();
  whole_tiles.clear();
  tiles.reserve(outs.size());
  const bool w = whole && whole_ok();
  for (int i = 0; i < (int)outs.size(); ++i) {
    const GOut& o = outs[i];
    if (o.m <= 0 || o.n <= 0) continue;
    const int tm = (o.m + 63) / 64, tn = (o.n + 63) / 64;
    if (w && tm <= 2 && tn <= 2 && (tm > 1 || tn > 1)) {
      whole_tiles.push_back(GTile{i, 0});
      continue;
    }
    for (int a = 0; a < tm; ++a)
      for (int b = 0; b < tn; ++b) tiles.push_back(GTile{i, a | (b << 16)});
  }
  tiles_ready = true;
}

void GBatch::run_device_terms(Ctx& C, const GTerm* d_terms, double flops_hint) {
  HostTimer ht(C, "gbatch_run");
  if (!tiles_ready) prepare_tiles();
  if (!tiles.empty() || !whole_tiles.empty()) {
    gsum_tile_stats(C.tag.c_str(), outs, tiles, nullptr);
    GOut* d_o = C.push(outs);
    GTile* d_l = C.push(tiles);
    GTile* d_w = C.push(whole_tiles);
    cudaEvent_t ev = C.prof_begin();
    C.flush();
    if (!whole_tiles.empty()) {
      cuda_check(launch_gsum_whole(d_o, d_terms, d_w, (int)whole_tiles.size(), std::max(k2max, 64), C.st),
                 "gsum(whole)");
      ++C.launches;
    }
    if (!tiles.empty()) {
      cuda_check(launch_gsum(d_o, d_terms, d_l, (int)tiles.size(), k2max, C.st, tag), "gsum");
      ++C.launches;
    }
    C.prof_end(K_GSUM, ev, flops_hint, 0.0);
  }
  outs.clear();
  terms.clear();
  k2max = 0;
}

static constexpr size_t kSmemLimit = 227 * 1024 - 1024;  // minus the kernels' static shared memory

// Pairwise tree of partial-R merges; `parts` = (rbuf, n, nchunk) per item.
static void run_merges(Ctx& C, const std::vector<std::tuple<double*, int, int>>& parts, bool rsmem, size_t smem) {
  int maxchunk = 1;
  for (auto& p : parts) maxchunk = std::max(maxchunk, std::get<2>(p));
  for (int stride = 1; stride < maxchunk; stride *= 2) {
    std::vector<MergeWork> lvl;
    for (auto& p : parts) {
      if (std::get<1>(p) == 0) continue;
      for (int a = 0; a + stride < std::get<2>(p); a += 2 * stride)
        lvl.push_back(MergeWork{std::get<0>(p), std::get<1>(p), a, a + stride, 0});
    }
    if (lvl.empty()) continue;
    cudaEvent_t sv = C.sub_begin();
    MergeWork* d_lvl = C.push(lvl);
    C.flush();
    cuda_check(launch_tsqr_merge(d_lvl, (int)lvl.size(), smem, rsmem, C.st), "tsqr_merge");
    C.sub_end(S_MERGE, sv);
    ++C.launches;
  }
}

// Register-tile TSQR (tileqr.cu) handles R factors up to 128 columns; H2G_NO_TILE=1 forces the
// panel kernels (A/B comparisons).
// Wide SVD inputs without a protected basis go through the double-double Gram (gram.cu) when the
// Gram fits the Cholesky CTA's shared memory (H2G_NO_GRAM=1: Householder TSQR, for A/B).
// columns per Gram CTA (H2G_GRAM_COLS overrides, for tuning)
static long long gram_cols() {
  static const long long v = getenv("H2G_GRAM_COLS") ? std::max(32LL, atoll(getenv("H2G_GRAM_COLS"))) : 512;
  return v;
}
static bool gram_path(int kx, int n, long long N) {
  static const bool off = getenv("H2G_NO_GRAM") != nullptr;
  return !off && kx == 0 && n > 0 && N > 0 && gram_chol_smem(n) <= (size_t)kSmemLimit;
}

// Items of one double-double Gram launch pair (gram.cu), shared by the SVD and QR batches.
struct GramBatch {
  std::vector<GramItem> items;
  std::vector<GramWork> work, wflat;  // tiled / flat (m <= kGramFlatMax) work units
  int mmax = 0;
  // lines of hstack(segs[s0:s1]) (hcols) or vstack (rows), m-dimensional; factor into rbuf, rows into *nr
  void add(Arena& scratch, int s0, int s1, int m, long long N, int hcols, double tol, double* rbuf, int* nr) {
    const int ncc = (int)std::max<long long>(1, (N + gram_cols() - 1) / gram_cols());
    GramItem g{};
    g.s0 = s0;
    g.s1 = s1;
    g.m = m;
    static const bool tiled = getenv("H2G_GRAM_TILED") != nullptr;  // A/B: 64 x 64 tiles for every m
    const bool flat = m > 64 && m <= kGramFlatMax && !tiled;
    g.nslice = flat ? ncc : ncc * gram_reps(m);  // partial slices summed by the Cholesky CTA
    g.N = N;
    g.hcols = hcols;
    g.tol = tol;
    g.gpart = scratch.alloc((size_t)g.nslice * 2 * m * m);
    g.rbuf = rbuf;
    g.nr = nr;
    const int gi = (int)items.size(), nt = (m + 63) / 64;
    if (flat) {
      // 64 < m <= 128: the upper triangle's 4 x 4 blocks dealt out evenly in contiguous runs, one
      // block per thread over all of a panel's lines (64 x 64 tiles left most of the second tile
      // row idle for m ~ 66-97: 20-40 % of the threads busy; splitting lines over replicas costs
      // more staging per product than it gains, measured)
      const int nb = (m + 3) / 4, nblk = nb * (nb + 1) / 2;
      const int best_r = 1;
      const int ncta = (nblk + kGramFlatThreads - 1) / kGramFlatThreads;
      const int bpc = (nblk + ncta - 1) / ncta;
      for (int c = 0; c < ncc; ++c)
        for (int b0 = 0; b0 < nblk; b0 += bpc)
          wflat.push_back(GramWork{gi, b0, std::min(bpc, nblk - b0) | (best_r << 16), c, (long long)c * gram_cols(),
                                   std::min<long long>(N, (long long)(c + 1) * gram_cols())});
    } else {
      for (int c = 0; c < ncc; ++c)
        for (int ti = 0; ti < nt; ++ti)
          for (int tj = ti; tj < nt; ++tj)
            work.push_back(GramWork{gi, ti, tj, c, (long long)c * gram_cols(), std::min<long long>(N, (long long)(c + 1) * gram_cols())});
    }
    items.push_back(g);
    mmax = std::max(mmax, m);
  }
  void launch(Ctx& C, const Seg* d_segs) {
    if (items.empty()) return;
    GramItem* d_it = C.push(items);
    const int nflat = (int)wflat.size();
    wflat.insert(wflat.end(), work.begin(), work.end());
    GramWork* d_w = C.push(wflat);
    C.flush();
    cuda_check(launch_gram(d_it, d_segs, d_w, (int)wflat.size(), nflat, (int)items.size(), mmax, C.st), "gram");
    C.launches += 1 + (nflat > 0 && nflat < (int)wflat.size() ? 2 : 1);
  }
};

// Protected-basis items (phase 1) through the Gram as well: opt-in (H2G_GRAM_PROT=1) -- measured
// neutral on c2 / c4 (the projection GEMM costs what the TSQR and QRCP saved).
static bool gram_prot_path(int n) {
  static const bool on = getenv("H2G_GRAM_PROT") != nullptr;
  return on && gram_path(0, n, 1);
}

static bool gram_qr_path(int n, long long M) {
  static const bool off = getenv("H2G_NO_GRAM_QR") != nullptr;
  return !off && gram_path(0, n, M);
}

// H2G_DEFER_OUT=1: the finish kernel writes U and Q_t = Q_V [[I, 0], [0, U]] is one batched GEMM
// (explicit Q_V from svd_prep_kernel for every protected item).  Measured slower at c4 (the explicit
// Q_V costs more than the in-kernel reflector application saves), so off by default.
static bool defer_out() {
  static const bool on = getenv("H2G_DEFER_OUT") != nullptr;
  return on;
}

static bool tile_path(int n) {
  static const bool off = getenv("H2G_NO_TILE") != nullptr;
  return !off && n <= 128;
}

// Tiles (128 lines) per chunk CTA.  Time model in units of one tile absorb, `slots` concurrent
// CTAs: chunk stage ceil(ctas / slots) x tpc, then each pairwise merge level ceil(merges / slots).
// Pick tpc in {1, 2, 4, 8} minimising it (few items: many short CTAs; many items: fewer merges).
static int tiles_per_cta(const std::vector<long long>& lines) {
  const long long slots = 148 * 2;
  int best = 1;
  double bcost = 1e300;
  for (int tpc = 1; tpc <= 8; tpc *= 2) {
    std::vector<long long> ch;
    long long ctas = 0;
    for (long long M : lines) {
      ch.push_back(std::max<long long>(1, (M + 128LL * tpc - 1) / (128LL * tpc)));
      ctas += ch.back();
    }
    double cost = std::ceil((double)ctas / slots) * tpc;
    for (;;) {  // merge levels: every item with c > 1 partial factors merges floor(c / 2) pairs
      long long merges = 0;
      for (long long& c : ch)
        if (c > 1) {
          merges += c / 2;
          c = (c + 1) / 2;
        }
      if (!merges) break;
      cost += std::ceil((double)merges / slots);
    }
    if (cost < bcost - 1e-9) { bcost = cost; best = tpc; }
  }
  return best;
}

static void run_tile_merges(Ctx& C, const std::vector<std::tuple<double*, int, int, int>>& parts,
                            const TileItem* d_items, int nmax) {
  int maxchunk = 1;
  for (auto& p : parts) maxchunk = std::max(maxchunk, std::get<2>(p));
  for (int stride = 1; stride < maxchunk; stride *= 2) {
    std::vector<TileWork> lvl;
    for (auto& p : parts) {
      const int n = std::get<1>(p);
      double* rb = std::get<0>(p);
      for (int a = 0; a + stride < std::get<2>(p); a += 2 * stride) {
        TileWork w{};
        w.item = std::get<3>(p);
        w.rinit = rb + (size_t)a * n * n;
        w.rsrc = rb + (size_t)(a + stride) * n * n;
        w.rout = rb + (size_t)a * n * n;
        lvl.push_back(w);
      }
    }
    if (lvl.empty()) continue;
    cudaEvent_t sv = C.sub_begin();
    TileWork* d_lvl = C.push(lvl);
    C.flush();
    cuda_check(launch_tile_absorb(d_items, nullptr, d_lvl, (int)lvl.size(), nmax, C.st), "tile_merge");
    C.sub_end(S_MERGE, sv);
    ++C.launches;
  }
}

void QrBatch::run(Ctx& C, Arena& scratch) {
  static constexpr long long kChunkRows = 256;  // rows per chunk CTA (8 panels of 32)
  std::vector<QrItem> live;
  bool rsmem = true;
  std::vector<long long> tile_lines;
  for (auto& it : items)
    if (it.n > 0 && it.M > 0 && tile_path(it.n) && !gram_qr_path(it.n, it.M)) tile_lines.push_back(it.M);
  const int tpc = tiles_per_cta(tile_lines);
  std::vector<TileItem> titems;
  std::vector<TileWork> twork;
  std::vector<std::tuple<double*, int, int, int>> tparts;
  int tnmax = 0;
  GramBatch gb;
  int* g_nr = nullptr;
  for (auto& it : items) {
    if (it.n == 0 || it.M == 0) continue;
    if (gram_qr_path(it.n, it.M)) {
      // R-only QR as the pivoted double-double Cholesky factor of the stack's Gram: every consumer
      // of these factors (weights.py:37-101, coarsening.py:231-245) uses only R^T R
      if (!g_nr) g_nr = (int*)scratch.alloc_bytes(items.size() * sizeof(int));
      it.rbuf = scratch.alloc((size_t)it.n * it.n);
      it.full = 1;
      gb.add(scratch, it.s0, it.s1, it.n, it.M, 0, 0.0, it.rbuf, g_nr + gb.items.size());
      live.push_back(it);
      continue;
    }
    if (tile_path(it.n)) {
      const long long per = 128LL * tpc;
      it.nchunk = (int)((it.M + per - 1) / per);
      it.rbuf = scratch.alloc((size_t)it.nchunk * it.n * it.n);
      const int ti = (int)titems.size();
      titems.push_back(TileItem{it.s0, it.s1, it.n, it.n, 0, 0, nullptr});  // no projection
      for (int c = 0; c < it.nchunk; ++c) {
        TileWork w{};
        w.item = ti;
        w.l0 = c * per;
        w.l1 = std::min(it.M, w.l0 + per);
        w.rout = it.rbuf + (size_t)c * it.n * it.n;
        twork.push_back(w);
      }
      tparts.emplace_back(it.rbuf, it.n, it.nchunk, ti);
      tnmax = std::max(tnmax, it.n);
      live.push_back(it);
      continue;
    }
    it.nchunk = (int)std::max<long long>(1, (it.M + kChunkRows - 1) / kChunkRows);
    it.rbuf = scratch.alloc((size_t)it.nchunk * it.n * it.n);
    if (qr_smem(it.n, true) > kSmemLimit || merge_smem(it.n, true) > kSmemLimit) rsmem = false;
    live.push_back(it);
  }
  if (live.empty()) { items.clear(); sl.segs.clear(); return; }
  static const bool dbg_qr = getenv("H2G_DEBUG_SWEEPS") != nullptr;
  if (dbg_qr) {
    double mn = 0, mM = 0, mc = 0;
    int mxn = 0, mxc = 0;
    for (auto& it : live) {
      mn += it.n; mM += (double)it.M; mc += it.nchunk;
      mxn = std::max(mxn, it.n); mxc = std::max(mxc, it.nchunk);
    }
    const double ni = (double)live.size();
    fprintf(stderr, "qr batch: %zu items, n mean %.1f max %d, M mean %.0f, chunks mean %.1f max %d, tiles/cta %d\n",
            live.size(), mn / ni, mxn, mM / ni, mc / ni, mxc, tpc);
  }
  size_t sm_chunk = 0, sm_merge = 0;
  std::vector<SvdWork> work;
  std::vector<std::tuple<double*, int, int>> parts;
  for (size_t i = 0; i < live.size(); ++i) {
    if (live[i].full || tile_path(live[i].n)) continue;
    sm_chunk = std::max(sm_chunk, qr_smem(live[i].n, rsmem));
    sm_merge = std::max(sm_merge, merge_smem(live[i].n, rsmem));
    for (int c = 0; c < live[i].nchunk; ++c) work.push_back(SvdWork{(int)i, c, 0, 0});
    parts.emplace_back(live[i].rbuf, live[i].n, live[i].nchunk);
  }
  double fl = 0, by = 0;
  if (C.prof)
    for (auto& it : live) {  // Householder R-only: 2 M n^2 - 2/3 n^3 (M >= n)
      const double M = (double)it.M, n = it.n;
      fl += M >= n ? 2 * M * n * n - 2.0 / 3 * n * n * n : 2 * n * M * M - 2.0 / 3 * M * M * M;
      by += 8 * (M * n + std::min(M, n) * n);
    }
  Seg* d_s = C.push(sl.segs);
  QrItem* d_items = C.push(live);
  SvdWork* d_work = C.push(work);
  cudaEvent_t ev = C.prof_begin();
  cudaEvent_t sv = C.sub_begin();
  gb.launch(C, d_s);
  if (!work.empty()) {
    C.flush();
    cuda_check(launch_qr_chunks(d_items, d_s, d_work, (int)work.size(), sm_chunk, rsmem, C.st), "qr_chunks");
    ++C.launches;
  }
  const TileItem* d_ti = nullptr;
  if (!twork.empty()) {
    d_ti = C.push(titems);
    TileWork* d_tw = C.push(twork);
    C.flush();
    cuda_check(launch_tile_absorb(d_ti, d_s, d_tw, (int)twork.size(), tnmax, C.st), "tile_absorb");
    ++C.launches;
  }
  C.sub_end(S_QR_CHUNK, sv);
  run_merges(C, parts, rsmem, sm_merge);
  if (!tparts.empty()) run_tile_merges(C, tparts, d_ti, tnmax);
  C.flush();
  cuda_check(launch_qr_out(d_items, (int)live.size(), C.st), "qr_out");
  ++C.launches;
  C.prof_end(K_QR, ev, fl, by);
  items.clear();
  sl.segs.clear();
}

void NormBatch::run_async(Ctx& C) {
  size_t smem = 0, smem_g = 0;
  // small: single segment, both sides <= 64 / 128 (warp Lanczos); big: CTA Gram in shared memory;
  // huge: CTA Gram in global scratch
  std::vector<NormItem> big, small, huge, mid, lz, lz64, lz96;  // mid / lz*: single segment up to 128 x 128
  size_t smem_mid = 0;
  std::unique_ptr<Arena> local;
  for (auto& it : items) {
    if (it.m == 0 || it.N == 0) continue;
    const long long mn = std::min<long long>(it.m, it.N), mx = std::max<long long>(it.m, it.N);
    if (it.s1 - it.s0 == 1 && mn <= 64 && mx <= 128 && it.m * (it.N | 1) <= 64 * 65) {
      small.push_back(it);
      continue;
    }
    if (it.s1 - it.s0 == 1 && it.m <= 128 && it.N <= 128) {
      // large ones (the 128 x 128 nearfield blocks) keep A in registers (norm_lz_kernel, one CTA per
      // SM: 1.9x on them); smaller ones run several shared-memory CTAs per SM (norm_cta_kernel)
      static const bool cta_all = getenv("H2G_NORM_CTA") != nullptr;  // A/B: shared-memory kernel only
      if (!cta_all) {
        (it.m <= 64 && it.N <= 64 ? lz64 : (it.m <= 96 && it.N <= 96 ? lz96 : lz)).push_back(it);
        continue;
      }
      smem_mid = std::max(smem_mid, norm_cta_smem(it.m, (int)it.N));
      mid.push_back(it);
      continue;
    }
    const bool rowside = it.m <= it.N;
    const long long g = rowside ? it.m : it.N;
    if (norm_smem(it.m, it.N, true) <= kSmemLimit) {
      smem = std::max(smem, norm_smem(it.m, it.N, true));
      big.push_back(it);
      continue;
    }
    if (norm_smem(it.m, it.N, false) > kSmemLimit) throw StructureErr("spectral norm: panel too wide for shared memory");
    if (!scratch) {
      local.reset(new Arena(C.st));
      scratch = local.get();
    }
    it.gbuf = scratch->alloc((size_t)g * g);
    smem_g = std::max(smem_g, norm_smem(it.m, it.N, false));
    huge.push_back(it);
  }
  if (!big.empty() || !small.empty() || !huge.empty() || !mid.empty() || !lz.empty() || !lz64.empty() || !lz96.empty()) {
    double fl = 0, by = 0;
    if (C.prof)
      for (auto* v : {&big, &small, &huge, &mid, &lz, &lz64, &lz96})
        for (auto& it : *v) {  // Gram on the short side + tridiagonalisation (reference's work)
          const double mn = std::min<double>(it.m, (double)it.N), mx = std::max<double>(it.m, (double)it.N);
          fl += 2 * mn * mn * mx + 4.0 / 3 * mn * mn * mn;
          by += 8 * mn * mx;
        }
    Seg* d_s = C.push(sl.segs);
    NormItem* d_big = C.push(big);
    NormItem* d_small = C.push(small);
    cudaEvent_t ev = C.prof_begin();
    if (!big.empty()) {
      C.flush();
      cuda_check(launch_norm(d_big, d_s, (int)big.size(), smem, C.st), "norm");
      ++C.launches;
    }
    if (!small.empty()) {
      C.flush();
      cuda_check(launch_norm_warp(d_small, d_s, (int)small.size(), C.st), "norm_warp");
      ++C.launches;
    }
    if (!huge.empty()) {
      NormItem* d_huge = C.push(huge);
      C.flush();
      cuda_check(launch_norm(d_huge, d_s, (int)huge.size(), smem_g, C.st), "norm(global gram)");
      ++C.launches;
    }
    if (!mid.empty()) {
      NormItem* d_mid = C.push(mid);
      C.flush();
      cuda_check(launch_norm_cta(d_mid, d_s, (int)mid.size(), smem_mid, C.st), "norm_cta");
      ++C.launches;
    }
    for (auto* v : {&lz64, &lz96, &lz}) {
      if (v->empty()) continue;
      NormItem* d_lz = C.push(*v);
      C.flush();
      const int cap = v == &lz64 ? 64 : (v == &lz96 ? 96 : 128);
      cuda_check(launch_norm_lz(d_lz, d_s, (int)v->size(), cap, cap, C.st), "norm_lz");
      ++C.launches;
    }
    C.prof_end(K_NORM, ev, fl, by);
  }
  items.clear();
  sl.segs.clear();
  if (local) scratch = nullptr;
}

std::vector<double> NormBatch::run(Ctx& C, Arena& scratch) {
  std::vector<double> res(items.size(), 0.0);
  if (items.empty()) return res;
  double* d_out = scratch.alloc(items.size());
  cuda_check(cudaMemsetAsync(d_out, 0, items.size() * sizeof(double), C.st), "memset");
  for (size_t i = 0; i < items.size(); ++i) items[i].out = d_out + i;
  const size_t n = items.size();
  run_async(C);
  return C.read(d_out, n);
}

std::vector<int> SvdBatch::run(Ctx& C, Arena& scratch) {
  std::vector<int> ranks(items.size(), 0);
  if (items.empty()) return ranks;
  int* d_rank = (int*)scratch.alloc_bytes(items.size() * sizeof(int));
  cuda_check(cudaMemsetAsync(d_rank, 0, items.size() * sizeof(int), C.st), "memset");
  static constexpr long long kChunkCols = 256;  // columns per stage-1 CTA (8 panels of 32)
  std::vector<SvdItem> live;
  bool rsmem = true, fin_rsmem = true;
  size_t sm_tsqr = 0, sm_merge = 0, sm_fin = 0, sm_prep = 0;
  std::vector<long long> tile_lines;
  for (auto& it : items) {
    const int n = it.m - std::min(it.m, it.kx);
    if (it.m > 0 && n > 0 && tile_path(n) && !gram_path(it.kx, n, it.N) && !(it.kx > 0 && it.N > 0 && gram_prot_path(n)))
      tile_lines.push_back(it.N);
  }
  const int tpc = tiles_per_cta(tile_lines);
  std::vector<TileItem> titems;
  std::vector<TileWork> twork;
  std::vector<std::tuple<double*, int, int, int>> tparts;
  std::vector<int> prep_ids;
  int tnmax = 0;
  GramBatch gb;
  GBatch gproj;  // projections of protected-basis items onto Q_V[:, k1:]
  int* g_nr = (int*)scratch.alloc_bytes(items.size() * sizeof(int));
  for (size_t i = 0; i < items.size(); ++i) {
    SvdItem& it = items[i];
    it.rank_out = d_rank + i;
    if (it.m == 0) continue;
    const int k1 = std::min(it.m, it.kx);
    const int n = it.m - k1;
    it.vws = it.kx > 0 ? scratch.alloc((size_t)it.m * (it.kx | 1) + it.kx) : nullptr;
    if (svd_finish_smem(it.m, it.kx, true, false) > kSmemLimit) fin_rsmem = false;
    if (it.kx > 0 && n > 0 && it.N > 0 && gram_prot_path(n)) {
      // protected basis: B = Q_V[:, k1:]^T A (double, as the reference forms Q_full^T hstack(w),
      // induced.py:127-137) per segment, then the same double-double Gram of B; svd_prep_kernel
      // supplies the explicit Q_V and the finish forms Q_t = Q_V [[I, 0], [0, U]]
      it.q2 = scratch.alloc((size_t)it.m * it.m);
      prep_ids.push_back((int)live.size());
      const size_t full = svd_prep_smem(it.m, it.kx, true);
      sm_prep = std::max(sm_prep, full <= kSmemLimit ? full : svd_prep_smem(it.m, it.kx, false));
      it.rbuf = scratch.alloc((size_t)n * n);
      it.pre_nr = g_nr + gb.items.size();
      const int s0n = (int)sl.segs.size();
      for (int q = it.s0; q < it.s1; ++q) {
        Seg sg = sl.segs[q];
        const Mat b{scratch.alloc((size_t)n * sg.w), n, sg.w};
        gproj.out(b, false);
        gproj.t2(MatRef{it.q2 + k1, 1, it.m}, sg.a, it.m);
        sg.a = b.ref();  // scale and device divisor apply to B's columns as to A's
        sl.segs.push_back(sg);
      }
      gb.add(scratch, s0n, (int)sl.segs.size(), n, it.N, 1, it.tol, it.rbuf, it.pre_nr);
      live.push_back(it);
      continue;
    }
    if (gram_path(it.kx, n, it.N)) {
      // double-double Gram + pivoted Cholesky (gram.cu) instead of the Householder TSQR
      it.rbuf = scratch.alloc((size_t)n * n);
      it.pre_nr = g_nr + gb.items.size();
      gb.add(scratch, it.s0, it.s1, n, it.N, 1, it.tol, it.rbuf, it.pre_nr);
      live.push_back(it);
      continue;
    }
    if (tile_path(n)) {
      const long long per = 128LL * tpc;
      it.nchunk = (int)std::max<long long>(1, (it.N + per - 1) / per);
      it.rbuf = n > 0 ? scratch.alloc((size_t)it.nchunk * n * n) : nullptr;
      it.q2 = it.kx > 0 ? scratch.alloc((size_t)it.m * it.m) : nullptr;
      if (it.q2 && n > 0 && defer_out()) it.u_out = scratch.alloc((size_t)n * n);
      if (it.kx > 0) {
        prep_ids.push_back((int)live.size());
        const size_t full = svd_prep_smem(it.m, it.kx, true);
        sm_prep = std::max(sm_prep, full <= kSmemLimit ? full : svd_prep_smem(it.m, it.kx, false));
      }
      if (n > 0) {
        const int ti = (int)titems.size();
        titems.push_back(TileItem{it.s0, it.s1, n, it.kx > 0 ? it.m : n, 1, it.m, it.q2 ? it.q2 + k1 : nullptr});
        for (int c = 0; c < it.nchunk; ++c) {
          TileWork w{};
          w.item = ti;
          w.l0 = c * per;
          w.l1 = std::min(it.N, w.l0 + per);
          w.rout = it.rbuf + (size_t)c * n * n;
          twork.push_back(w);
        }
        tparts.emplace_back(it.rbuf, n, it.nchunk, ti);
        tnmax = std::max(tnmax, n);
      }
      live.push_back(it);
      continue;
    }
    it.nchunk = (int)std::max<long long>(1, (it.N + kChunkCols - 1) / kChunkCols);
    it.rbuf = n > 0 ? scratch.alloc((size_t)it.nchunk * n * n) : nullptr;
    if (svd_tsqr_smem(it.m, it.kx, true) > kSmemLimit || merge_smem(n, true) > kSmemLimit) rsmem = false;
    if (it.kx > 0 && n > 0 && defer_out()) {
      // explicit Q_V (svd_prep_kernel) so that the output is one GEMM instead of k1 sequential
      // reflector applications per column inside the finish kernel
      it.q2 = scratch.alloc((size_t)it.m * it.m);
      it.u_out = scratch.alloc((size_t)n * n);
      prep_ids.push_back((int)live.size());
      const size_t full = svd_prep_smem(it.m, it.kx, true);
      sm_prep = std::max(sm_prep, full <= kSmemLimit ? full : svd_prep_smem(it.m, it.kx, false));
    }
    live.push_back(it);
  }
  if (live.empty()) return ranks;
  if (sm_prep > kSmemLimit) throw StructureErr("svd: protected basis too large for shared memory");
  std::vector<SvdWork> work;
  std::vector<std::tuple<double*, int, int>> parts;
  // the finish stage keeps R in shared memory when it fits (first choice), V beside it when that fits too;
  // else R alone at its unpadded stride ("tight": the top-level row clusters of c4, n up to ~168)
  bool fin_tight = false;
  if (!fin_rsmem) {
    fin_tight = true;
    for (const SvdItem& it : live)
      if (svd_finish_smem(it.m, it.kx, true, false, true) > kSmemLimit) fin_tight = false;
    if (fin_tight) fin_rsmem = true;
  }
  bool fin_vsmem = !fin_tight;
  for (const SvdItem& it : live)
    if (!fin_tight && svd_finish_smem(it.m, it.kx, fin_rsmem, true) > kSmemLimit) fin_vsmem = false;
  for (size_t i = 0; i < live.size(); ++i) {
    const SvdItem& it = live[i];
    const int n = it.m - std::min(it.m, it.kx);
    sm_fin = std::max(sm_fin, svd_finish_smem(it.m, it.kx, fin_rsmem, fin_vsmem, fin_tight));
    if (sm_fin > kSmemLimit) throw StructureErr("svd: item too large for shared memory");
    if (it.pre_nr || tile_path(n)) continue;
    sm_tsqr = std::max(sm_tsqr, svd_tsqr_smem(it.m, it.kx, rsmem));
    sm_merge = std::max(sm_merge, merge_smem(n, rsmem));
    if (sm_tsqr > kSmemLimit) throw StructureErr("svd: item too large for shared memory");
    for (int c = 0; c < it.nchunk; ++c) work.push_back(SvdWork{(int)i, c, 0, 0});
    if (n > 0) parts.emplace_back(it.rbuf, n, it.nchunk);
  }
  static const bool dbg_sweeps = getenv("H2G_DEBUG_SWEEPS") != nullptr;
  int* d_sw = nullptr;
  if (dbg_sweeps) {
    d_sw = (int*)scratch.alloc_bytes(live.size() * 8 * sizeof(int));
    cuda_check(cudaMemsetAsync(d_sw, 0, live.size() * 8 * sizeof(int), C.st), "memset");
    for (size_t i = 0; i < live.size(); ++i) live[i].sweeps_out = d_sw + 8 * i;
  }
  Seg* d_s = C.push(sl.segs);
  SvdItem* d_items = C.push(live);
  SvdWork* d_work = C.push(work);
  double fl = 0, by = 0;
  if (C.prof)
    for (auto& it : live) {  // reference ops: full QR of V, Q^T A, gesdd of the remainder
      const double m = it.m, kx = it.kx, N = (double)it.N, k1 = std::min(m, kx), r = m - k1;
      if (kx > 0) fl += 2 * m * kx * kx - 2.0 / 3 * kx * kx * kx + 4.0 / 3 * m * m * m + 2 * r * m * N;
      const double mn = std::min(r, N), mx = std::max(r, N);
      fl += 4 * mx * mn * mn + 8 * mn * mn * mn;
      by += 8 * (m * N + m * kx + m * m);
    }
  cudaEvent_t ev = C.prof_begin();
  cudaEvent_t sv = C.sub_begin();
  if (!prep_ids.empty()) {  // explicit Q_V first: the Gram projections and the tile path read it
    int* d_ids = C.push(prep_ids);
    C.flush();
    cuda_check(launch_svd_prep(d_items, d_ids, (int)prep_ids.size(), sm_prep, C.st), "svd_prep");
    ++C.launches;
  }
  if (!gproj.outs.empty()) gproj.run(C);
  gb.launch(C, d_s);
  if (!work.empty()) {
    C.flush();
    cuda_check(launch_svd_tsqr(d_items, d_s, d_work, (int)work.size(), sm_tsqr, rsmem, C.st), "svd_tsqr");
    ++C.launches;
  }
  const TileItem* d_ti = nullptr;
  if (!twork.empty()) {
    d_ti = C.push(titems);
    TileWork* d_tw = C.push(twork);
    C.flush();
    cuda_check(launch_tile_absorb(d_ti, d_s, d_tw, (int)twork.size(), tnmax, C.st), "tile_absorb");
    ++C.launches;
  }
  C.sub_end(S_SVD_TSQR, sv);
  run_merges(C, parts, rsmem, sm_merge);
  if (!tparts.empty()) run_tile_merges(C, tparts, d_ti, tnmax);
  cudaEvent_t sf = C.sub_begin();
  int fin_nmax = 0;
  for (auto& it : live) fin_nmax = std::max(fin_nmax, it.m - std::min(it.m, it.kx));
  C.flush();
  cuda_check(launch_svd_finish(d_items, d_s, (int)live.size(), sm_fin, fin_rsmem, fin_vsmem, fin_nmax, C.st, fin_tight),
             "svd_finish");
  C.sub_end(S_SVD_FIN, sf);
  ++C.launches;
  C.prof_end(K_SVD, ev, fl, by);
  ranks = C.read(d_rank, items.size());
  {  // deferred outputs: Q_t = [Q_V[:, :k1] | Q_V[:, k1:] U] (m x kt), one grouped GEMM
    GBatch qo;
    for (const SvdItem& it : live) {
      if (!it.u_out) continue;
      const int kt = ranks[it.rank_out - d_rank];
      const int k1 = std::min(it.m, it.kx), n = it.m - k1, k2 = kt - k1;
      if (k1 > 0) {
        qo.out(Mat{it.q_out, it.m, k1}, false);
        qo.outs.back().ldc = kt;
        qo.t1(MatRef{it.q2, it.m, 1});
      }
      if (k2 > 0) {
        qo.out(Mat{it.q_out + k1, it.m, k2}, false);
        qo.outs.back().ldc = kt;
        qo.t2(MatRef{it.q2 + k1, it.m, 1}, MatRef{it.u_out, n, 1}, n);
      }
    }
    if (!qo.empty()) qo.run(C);
  }
  if (dbg_sweeps) {
    std::vector<int> sw = C.read(d_sw, live.size() * 8);
    int mx = 0, mxn = 0;
    double mean = 0, mn = 0, mnr = 0, mk = 0, mN = 0, ph[4] = {0, 0, 0, 0};
    const size_t ni = live.size();
    for (size_t i = 0; i < ni; ++i) {
      const int* r = &sw[8 * i];
      mx = std::max(mx, r[0]);
      mean += r[0];
      mn += r[1];
      mnr += r[2];
      mk += r[3];
      for (int q = 0; q < 4; ++q) ph[q] = std::max(ph[q], (double)r[4 + q]);
      mN += (double)live[i].N;
      mxn = std::max(mxn, r[1]);
    }
    fprintf(stderr,
            "svd batch: %zu items, n<=%d, mean n %.1f live %.1f k2 %.1f N %.0f, sweeps max %d mean %.1f | max kcyc "
            "load %.0f qrcp %.0f jacobi %.0f out %.0f\n",
            ni, mxn, mn / ni, mnr / ni, mk / ni, mN / ni, mx, mean / ni, ph[0], ph[1], ph[2], ph[3]);
  }
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
  rptr.assign(rows->n + 1, 0);
  for (int b = 0; b < nb; ++b) {
    if (row[b] < 0 || row[b] >= rows->n || col[b] < 0 || col[b] >= cols->n)
      throw InvalidInput("block references a cluster outside its tree");
    ++rptr[row[b] + 1];
  }
  for (int t = 0; t < rows->n; ++t) rptr[t + 1] += rptr[t];
  rcol.assign(nb, 0);
  rblk.assign(nb, 0);
  {
    std::vector<int> fill(rptr.begin(), rptr.end() - 1);
    for (int b = 0; b < nb; ++b) {
      rcol[fill[row[b]]] = col[b];
      rblk[fill[row[b]]++] = b;
    }
    for (int t = 0; t < rows->n; ++t) {
      std::vector<std::pair<int, int>> v;
      for (int i = rptr[t]; i < rptr[t + 1]; ++i) v.emplace_back(rcol[i], rblk[i]);
      std::sort(v.begin(), v.end());
      for (int i = rptr[t]; i < rptr[t + 1]; ++i) {
        rcol[i] = v[i - rptr[t]].first;
        rblk[i] = v[i - rptr[t]].second;
      }
    }
  }
  for (int b = 0; b < nb; ++b) {
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

// Locate block (row, col) of a block tree starting from a hint block: the hint itself, one of its
// children, or (fallback) a binary search.  The product recursion always has the parent blocks of
// X|ts and Y|sr at hand, so this replaces the reference's dict lookups (trees.py:187, :289-290).
static inline int locate(BView v, int hint, int row, int col) {
  if (hint >= 0) {
    if (v.row(hint) == row && v.col(hint) == col) return hint;
    const Blocks& B = *v.b;
    for (int i = B.cptr[hint]; i < B.cptr[hint + 1]; ++i) {
      const int c = B.cidx[i];
      if (v.row(c) == row && v.col(c) == col) return c;
    }
  }
  return v.find(row, col);
}

// Triple kind (reference trees.py:288-300): 'a' > 'b' > 'c' > 'n'.
static inline char classify(BView bx, BView by, int bts, int bsr) {
  if (bts < 0 || bsr < 0) throw StructureErr("triple not covered by the factor block trees");
  if (by.b->adm_leaf(bsr)) return 'a';
  if (bx.b->adm_leaf(bts)) return 'b';
  if (by.b->leaf(bsr) && bx.b->leaf(bts)) return 'c';
  return 'n';
}

// Product block tree T^XY with the per-node terminal triples (trees.py:314-359, induced.py:280-326).
//
// The recursion `rec(t, r, middles)` is a depth-first preorder walk.  It is built in parallel: a
// breadth-first prefix expands the top frames until there are enough independent subtrees, each
// subtree is built by its own host thread with the same per-node logic, and the pieces are
// stitched back in exact preorder (prefix node, then its children's subtrees in slot order), so
// block ids, children and triple order are identical to the sequential walk.
namespace {

struct PtMid {
  int s, hx, hy;  // middle cluster and hint blocks (parents of X|ts, Y|sr)
};
struct PtFrame {
  int t, r, parent, slot, m0, m1;  // middles in `pool[m0:m1]`
};

struct PtBuilder {
  BView bx, by;
  const Tree *rows, *mid, *cols;
  std::vector<PtMid> pool;
  std::vector<int> row, col;
  std::vector<unsigned char> adm;
  std::vector<std::vector<int>> kids;
  std::vector<int> tptr, ts, tbx, tby;
  std::vector<char> tk;
  struct Live {
    int s, bts, bsr;
  };
  std::vector<Live> pend, open;

  PtBuilder(BView x, BView y) : bx(x), by(y), rows(&x.rows()), mid(&x.cols()), cols(&y.cols()) {}

  // creates node for frame f (linking it to its parent slot) and appends its child frames
  int node(const PtFrame& f, std::vector<PtFrame>& out) {
    const int b = (int)row.size();
    if (f.parent >= 0) kids[f.parent][f.slot] = b;
    row.push_back(f.t);
    col.push_back(f.r);
    adm.push_back(1);
    kids.emplace_back();
    tptr.push_back((int)ts.size());
    const bool both_leaf = rows->leaf(f.t) && cols->leaf(f.r);
    pend.clear();
    for (int i = f.m0; i < f.m1; ++i) {
      const PtMid& m = pool[i];
      pend.push_back(Live{m.s, locate(bx, m.hx, f.t, m.s), locate(by, m.hy, m.s, f.r)});
    }
    open.clear();
    bool dense = false;
    while (!pend.empty()) {
      const Live l = pend.back();
      pend.pop_back();
      const char k = classify(bx, by, l.bts, l.bsr);
      if (k == 'n') {
        if (both_leaf) {  // both clusters exhausted: chase the middle only (trees.py:343-345)
          for (int i = 0; i < mid->nkids(l.s); ++i) {
            const int s2 = mid->kid(l.s, i);
            pend.push_back(Live{s2, locate(bx, l.bts, f.t, s2), locate(by, l.bsr, s2, f.r)});
          }
        } else {
          open.push_back(l);
        }
        continue;
      }
      if (k == 'c') dense = true;
      ts.push_back(l.s);
      tk.push_back(k);
      tbx.push_back(l.bts);
      tby.push_back(l.bsr);
    }
    if (!open.empty()) {
      const int m0 = (int)pool.size();
      for (const Live& l : open) {  // _sub_middles (trees.py:303-311)
        if (!bx.b->leaf(l.bts) && !by.b->leaf(l.bsr) && mid->nkids(l.s) > 0) {
          for (int i = 0; i < mid->nkids(l.s); ++i) pool.push_back(PtMid{mid->kid(l.s, i), l.bts, l.bsr});
        } else {
          pool.push_back(PtMid{l.s, l.bts, l.bsr});
        }
      }
      const int m1 = (int)pool.size();
      const int nt = std::max(1, rows->nkids(f.t)), nr = std::max(1, cols->nkids(f.r));
      kids[b].assign(nt * nr, -1);
      for (int i = 0; i < nt * nr; ++i) {
        const int t2 = rows->nkids(f.t) ? rows->kid(f.t, i / nr) : f.t;
        const int r2 = cols->nkids(f.r) ? cols->kid(f.r, i % nr) : f.r;
        out.push_back(PtFrame{t2, r2, b, i, m0, m1});
      }
    } else if (dense) {
      adm[b] = 0;
    }
    return b;
  }

  // sequential preorder walk from `root` (its middles already in pool[root.m0:root.m1])
  void dfs(const PtFrame& root) {
    std::vector<PtFrame> stack{root}, tmp;
    while (!stack.empty()) {
      const PtFrame f = stack.back();
      stack.pop_back();
      tmp.clear();
      node(f, tmp);
      for (int i = (int)tmp.size() - 1; i >= 0; --i) stack.push_back(tmp[i]);  // slot 0 first
    }
    tptr.push_back((int)ts.size());
  }
};

}  // namespace

PTree product_tree(BView bx, BView by) {
  const Tree& rows = bx.rows();
  const Tree& cols = by.cols();
  if (!bx.cols().same(by.rows())) throw InvalidInput("factors do not share the middle cluster tree");
  // breadth-first prefix until there are enough subtrees for the worker threads
  PtBuilder pre(bx, by);
  pre.pool.push_back(PtMid{0, 0, 0});
  std::vector<PtFrame> level{PtFrame{0, 0, -1, 0, 0, 1}}, next;
  // prefix children: >= 0 prefix node, < 0: -(1 + fragment index)
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t want = std::max<size_t>(1, 8 * (size_t)std::min(hw, 16u));
  std::vector<PtFrame> frags;
  while (!level.empty()) {
    if (level.size() >= want) {
      for (const PtFrame& f : level) {
        pre.kids[f.parent][f.slot] = -1 - (int)frags.size();
        frags.push_back(f);
      }
      break;
    }
    next.clear();
    for (const PtFrame& f : level) pre.node(f, next);
    level.swap(next);
  }
  pre.tptr.push_back((int)pre.ts.size());
  // subtrees in parallel
  std::vector<std::unique_ptr<PtBuilder>> fb(frags.size());
  {
    std::atomic<size_t> nextf{0};
    std::exception_ptr err;
    std::mutex emu;
    auto work = [&] {
      try {
        for (size_t i; (i = nextf.fetch_add(1)) < frags.size();) {
          auto B = std::make_unique<PtBuilder>(bx, by);
          const PtFrame& f = frags[i];
          B->pool.assign(pre.pool.begin() + f.m0, pre.pool.begin() + f.m1);
          B->dfs(PtFrame{f.t, f.r, -1, 0, 0, f.m1 - f.m0});
          fb[i] = std::move(B);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(emu);
        if (!err) err = std::current_exception();
      }
    };
    const int nth = (int)std::min<size_t>(frags.size(), std::min(hw, 16u));
    std::vector<std::thread> th;
    for (int k = 1; k < nth; ++k) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    if (err) std::rethrow_exception(err);
  }
  // stitch in preorder
  PTree P;
  auto bt = std::make_shared<Blocks>();
  bt->rows = &rows;
  bt->cols = &cols;
  size_t nnodes = pre.row.size(), ntrip = pre.ts.size();
  for (auto& B : fb) {
    nnodes += B->row.size();
    ntrip += B->ts.size();
  }
  bt->row.reserve(nnodes);
  bt->col.reserve(nnodes);
  bt->adm.reserve(nnodes);
  P.tptr.reserve(nnodes + 1);
  P.ts.reserve(ntrip);
  P.tk.reserve(ntrip);
  P.tbx.reserve(ntrip);
  P.tby.reserve(ntrip);
  std::vector<std::vector<int>> kids;
  kids.reserve(nnodes);
  auto append = [&](const PtBuilder& B, int b, int base) {
    bt->row.push_back(B.row[b]);
    bt->col.push_back(B.col[b]);
    bt->adm.push_back(B.adm[b]);
    P.tptr.push_back((int)P.ts.size());
    for (int i = B.tptr[b]; i < B.tptr[b + 1]; ++i) {
      P.ts.push_back(B.ts[i]);
      P.tk.push_back(B.tk[i]);
      P.tbx.push_back(B.tbx[i]);
      P.tby.push_back(B.tby[i]);
    }
    kids.emplace_back(B.kids[b]);
    if (base)
      for (int& c : kids.back()) c += base;
  };
  std::function<int(int)> emit = [&](int p) -> int {
    const int g = (int)bt->row.size();
    append(pre, p, 0);
    const std::vector<int> ch = pre.kids[p];
    for (size_t i = 0; i < ch.size(); ++i) {
      int gid;
      if (ch[i] >= 0) {
        gid = emit(ch[i]);
      } else {
        const PtBuilder& B = *fb[-1 - ch[i]];
        gid = (int)bt->row.size();
        for (int b = 0; b < (int)B.row.size(); ++b) append(B, b, gid);
      }
      kids[g][i] = gid;
    }
    return g;
  };
  if (pre.row.empty()) {  // the root itself was a fragment (cannot happen: want >= 1 frame > 0)
    throw StructureErr("product tree: empty prefix");
  }
  emit(0);
  P.tptr.push_back((int)P.ts.size());
  bt->nb = (int)bt->row.size();
  bt->cptr.assign(bt->nb + 1, 0);
  for (int b = 0; b < bt->nb; ++b) bt->cptr[b + 1] = bt->cptr[b] + (int)kids[b].size();
  bt->cidx.reserve(bt->cptr[bt->nb]);
  for (int b = 0; b < bt->nb; ++b)
    for (int c : kids[b]) bt->cidx.push_back(c);
  bt->finalize();
  P.bt = bt;
  return P;
}

// Planner-thread epilogue: distinct dense-target operand blocks, and the triple arrays copied to the
// device on a private stream (overlapping the GPU's basis construction).
void ptree_prepare(PTree& P, Ctx& C, const Blocks& BX, int nby) {
  static const bool dbg = getenv("H2G_DEBUG_PLANNER") != nullptr;
  const auto tp0 = std::chrono::steady_clock::now();
  auto tms = [tp0] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count(); };
  const Blocks& B = *P.bt;
  const int nt = (int)P.ts.size();
  // order each node's triples c, a, b (stable): the assembly sums kind-a terms into one T and
  // kind-b terms into one U before applying their shared factor (GOut ka / kb).  Nodes are
  // independent: block ranges of about equal triple counts go to host threads.
  const int nthr = (int)std::min<long long>(8, std::max<long long>(1, nt / 65536));
  std::vector<int> cut(nthr + 1, B.nb);
  cut[0] = 0;
  for (int k = 1, b = 0; k < nthr; ++k) {
    const long long target = (long long)nt * k / nthr;
    while (b < B.nb && P.tptr[b] < target) ++b;
    cut[k] = b;
  }
  auto par = [&](auto&& fn) {  // fn(b0, b1) over the block ranges
    std::vector<std::thread> th;
    for (int k = 1; k < nthr; ++k) th.emplace_back(fn, cut[k], cut[k + 1]);
    fn(cut[0], cut[1]);
    for (auto& t : th) t.join();
  };
  {
    std::atomic<int> bad{0};
    par([&](int b0, int b1) {  // in place, one node at a time through a small local buffer
      std::vector<int> ts2, tbx2, tby2;
      std::vector<char> tk2;
      for (int b = b0; b < b1; ++b) {
        const int i0 = P.tptr[b], i1 = P.tptr[b + 1], cnt = i1 - i0;
        ts2.resize(cnt); tbx2.resize(cnt); tby2.resize(cnt); tk2.resize(cnt);
        int o = 0;
        for (const char kind : {'c', 'a', 'b'})
          for (int i = i0; i < i1; ++i)
            if (P.tk[i] == kind) {
              ts2[o] = P.ts[i];
              tbx2[o] = P.tbx[i];
              tby2[o] = P.tby[i];
              tk2[o] = kind;
              ++o;
            }
        if (o != cnt) { bad = 1; continue; }
        std::copy(ts2.begin(), ts2.end(), P.ts.begin() + i0);
        std::copy(tbx2.begin(), tbx2.end(), P.tbx.begin() + i0);
        std::copy(tby2.begin(), tby2.end(), P.tby.begin() + i0);
        std::copy(tk2.begin(), tk2.end(), P.tk.begin() + i0);
      }
    });
    if (bad) throw StructureErr("product tree: unknown triple kind");
  }
  const double t_re = tms();
  const int nbx = BX.nb;
  const Part part = make_part(*B.rows, C.comm);  // multi-GPU: only this rank's product rows
  // per range: first appearances within the range; merged in range order (= global first
  // appearance, the serial order)
  std::vector<std::vector<int>> lx(nthr), ly(nthr), lf(nthr);
  {
    std::vector<std::thread> th;
    auto run = [&](int k) {
      std::vector<char> sx(nbx, 0), sy(nby, 0), sf(nbx, 0);
      for (int b = cut[k]; b < cut[k + 1]; ++b) {
        if (!part.mine(B.row[b])) continue;
        if (!B.near_leaf(b)) {
          for (int i = P.tptr[b]; i < P.tptr[b + 1]; ++i) {
            const int bts = P.tbx[i];
            if (P.tk[i] == 'a' && BX.adm_leaf(bts) && !sf[bts]) { sf[bts] = 1; lf[k].push_back(bts); }
          }
          continue;
        }
        for (int i = P.tptr[b]; i < P.tptr[b + 1]; ++i) {
          if (P.tk[i] == 'a' && !sx[P.tbx[i]]) { sx[P.tbx[i]] = 1; lx[k].push_back(P.tbx[i]); }
          if (P.tk[i] == 'b' && !sy[P.tby[i]]) { sy[P.tby[i]] = 1; ly[k].push_back(P.tby[i]); }
        }
      }
    };
    for (int k = 1; k < nthr; ++k) th.emplace_back(run, k);
    run(0);
    for (auto& t : th) t.join();
  }
  {
    std::vector<char> seenx(nbx, 0), seeny(nby, 0), seenf(nbx, 0);
    for (int k = 0; k < nthr; ++k) {
      for (int v : lf[k]) if (!seenf[v]) { seenf[v] = 1; P.rf_blocks.push_back(v); }
      for (int v : lx[k]) if (!seenx[v]) { seenx[v] = 1; P.need_xv.push_back(v); }
      for (int v : ly[k]) if (!seeny[v]) { seeny[v] = 1; P.need_wy.push_back(v); }
    }
  }
  const double t_dd = tms();
  if (nt == 0) return;
  const size_t n4 = (size_t)nt * 4, pad = 256;
  const size_t bytes = 4 * ((n4 + pad - 1) / pad * pad) + nt + pad;
  if (!C.up_stream) cuda_check(cudaStreamCreateWithFlags(&C.up_stream, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamSynchronize(C.up_stream), "up sync");
  if (bytes > C.up_cap) {
    if (C.up_host) cudaFreeHost(C.up_host);
    C.up_cap = bytes * 2;
    cuda_check(cudaMallocHost(&C.up_host, C.up_cap), "cudaMallocHost");
  }
  const double t_sy = tms();
  const size_t stride = (n4 + pad - 1) / pad * pad;
  char* h = C.up_host;
  int* htnode = (int*)h;
  par([&](int b0, int b1) {  // staging into the pinned buffer, by block ranges
    if (b0 >= b1) return;
    const int i0 = P.tptr[b0], i1 = P.tptr[b1];
    for (int b = b0; b < b1; ++b)
      for (int i = P.tptr[b]; i < P.tptr[b + 1]; ++i) htnode[i] = b;
    memcpy(h + stride + 4 * (size_t)i0, P.ts.data() + i0, 4 * (size_t)(i1 - i0));
    memcpy(h + 2 * stride + 4 * (size_t)i0, P.tbx.data() + i0, 4 * (size_t)(i1 - i0));
    memcpy(h + 3 * stride + 4 * (size_t)i0, P.tby.data() + i0, 4 * (size_t)(i1 - i0));
    memcpy(h + 4 * stride + i0, P.tk.data() + i0, (size_t)(i1 - i0));
  });
  cuda_check(cudaMallocAsync(&P.dev.block, bytes, C.up_stream), "cudaMallocAsync");
  cuda_check(cudaMemcpyAsync(P.dev.block, h, bytes, cudaMemcpyHostToDevice, C.up_stream), "upload");
  char* d = (char*)P.dev.block;
  P.dev.tnode = (int*)d;
  P.dev.ts = (int*)(d + stride);
  P.dev.tbx = (int*)(d + 2 * stride);
  P.dev.tby = (int*)(d + 3 * stride);
  P.dev.tk = d + 4 * stride;
  cuda_check(cudaEventCreateWithFlags(&P.dev.ready, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(P.dev.ready, C.up_stream), "event");
  if (dbg)
    fprintf(stderr, "ptree_prepare: %d triples, reorder %.2f, dedupe %.2f, sync/alloc %.2f, staged+queued %.2f ms\n", nt,
            t_re, t_dd, t_sy, tms());
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
MatStore total_weights(Ctx& C, Arena& ar, HView h, const MatStore& rw, bool scaling, bool exact_rows) {
  const Tree& tr = h.rows();
  const int nb = h.h->bt->nb;
  std::vector<std::vector<int>> adm_of(tr.n);
  for (int b = 0; b < nb; ++b)
    if (h.h->bt->adm_leaf(b)) adm_of[h.row(b)].push_back(b);
  // T_b = R_{col b} S_b^T and their norms
  std::vector<Mat> Tb(nb);
  GBatch g;
  NormBatch nbatch;
  // sigma_1 of every T_b stays on the device as its segment's divisor (no host round trip); an
  // exactly-zero T_b (sigma_1 = 0, skipped by the reference, weights.py:86-89) contributes zero rows,
  // which leave the stack's Gram -- all its factor's consumers see -- unchanged
  double* d_nrm = scaling ? ar.alloc(std::max(1, nb)) : nullptr;
  if (scaling) cuda_check(cudaMemsetAsync(d_nrm, 0, sizeof(double) * std::max(1, nb), C.st), "memset");
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
        it.out = d_nrm + b;
        nbatch.items.push_back(it);
      }
    }
  g.run(C);
  std::vector<double> nrm;
  if (scaling) {
    nbatch.scratch = &ar;
    nbatch.run_async(C);
    // exactly-zero blocks are not rows of the reference's stack (weights.py:86-89): the factor's
    // row count min(M, k) -- which sets the column counts (and so the eps * max(rows, cols) floor)
    // of the SVD inputs built from these weights -- counts the nonzero blocks only
    if (exact_rows) nrm = C.read(d_nrm, (size_t)std::max(1, nb));
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
        if (scaling && exact_rows && nrm[b] == 0.0) continue;
        q.sl.add(Tb[b].ref(), Tb[b].r, 1.0, scaling ? d_nrm + b : nullptr);
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
