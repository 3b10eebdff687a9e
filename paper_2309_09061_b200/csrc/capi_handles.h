// Opaque handle types of the C ABI (include/h2g.h) and the status-code guard, shared by the
// translation units that implement it (capi.cu, capi_stages.cu).
#pragma once
#include <string>

#include "../../include/h2g.h"
#include "engine.h"

using namespace h2g;

struct h2g_ctx {
  Ctx c;
  h2g_ctx(int dev, cudaStream_t s) : c(dev, s) {}
};
struct h2g_tree {
  std::shared_ptr<Tree> t;
};
struct h2g_blocks {
  std::shared_ptr<Blocks> b;
  std::shared_ptr<Tree> rows, cols;
};
struct h2g_h2 {
  std::shared_ptr<H2> h;
};

// stage-level results (capi_stages.cu)
struct h2g_basis {
  std::shared_ptr<Basis> b;
  std::vector<ArenaPtr> keep;
  std::shared_ptr<H2> owner;  // matrix the basis belongs to (views)
  std::shared_ptr<Tree> tree;  // tree kept alive for uploaded bases
};
struct h2g_mats {
  MatStore m;
  std::vector<ArenaPtr> keep;
  std::shared_ptr<H2> owner;
};
struct h2g_induced {
  std::shared_ptr<InducedStage> s;
};
struct h2g_cstate {
  std::shared_ptr<CoarseStage> s;
  std::shared_ptr<H2> g;  // the product the state was built from
};

extern thread_local std::string g_err;

struct Gather {
  std::vector<long long> items;  // src, n, dst-offset (patched to absolute)
  long long total = 0;
  void add(const double* src, long long n) {
    if (n <= 0) return;
    items.push_back((long long)src);
    items.push_back(n);
    items.push_back(total);
    total += n;
  }
  // as run(), but only the ranges `runs` of the packed layout are copied to the host
  void run_runs(Ctx& C, Arena& ar, double* host, const std::vector<std::pair<long long, long long>>& runs) {
    if (total == 0 || items.empty()) return;
    double* d = ar.alloc(total);
    for (size_t i = 2; i < items.size(); i += 3) items[i] = (long long)(d + items[i]);
    long long* di = C.push(items);
    C.flush();
    cuda_check(launch_gather(di, (int)(items.size() / 3), C.st), "gather");
    for (auto& r : runs)
      cuda_check(cudaMemcpyAsync(host + r.first, d + r.first, (r.second - r.first) * sizeof(double),
                                 cudaMemcpyDeviceToHost, C.st),
                 "download");
  }
  void run(Ctx& C, Arena& ar, double* host) {
    if (total == 0) return;
    double* d = ar.alloc(total);
    for (size_t i = 2; i < items.size(); i += 3) items[i] = (long long)(d + items[i]);
    long long* di = C.push(items);
    C.flush();
    cuda_check(launch_gather(di, (int)(items.size() / 3), C.st), "gather");
    cuda_check(cudaMemcpyAsync(host, d, total * sizeof(double), cudaMemcpyDeviceToHost, C.st), "download");
  }
};

std::shared_ptr<Basis> upload_basis(Ctx& C, Arena& ar, const Tree* tree, const long long* rank,
                                    const long long* loff, const long long* xoff, const double* data,
                                    long long len);
void pack_basis(const Basis& B, long long* rank, long long* loff, long long* xoff, Gather& g);


template <class F>
inline int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidInput& e) {
    g_err = e.what();
    return 1;
  } catch (const StructureErr& e) {
    g_err = e.what();
    return 2;
  } catch (const CudaFailure& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

