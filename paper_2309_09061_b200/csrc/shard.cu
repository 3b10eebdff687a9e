// Multi-GPU partition of one product: the row cluster tree (and, for the column
// passes, the column tree) is split into subtrees at the first level with >= P clusters; each rank
// computes the clusters and product blocks of its subtrees, every rank computes the few replicated
// top levels, and the per-cluster results (ranks, bases, transfers, projections, couplings,
// nearfield) are all-gathered in place so that each rank continues with the full state.
//
// The collective itself is the host's (Comm::fn): torch.distributed over NCCL on the context's
// stream in production, gloo with host staging in the tests.  The engine only lays out the
// segments: one contiguous device buffer, segment i holding rank i's arrays in a canonical order
// that every rank derives from the same structure.
#include <algorithm>

#include "engine.h"

namespace h2g {

Part make_part(const Tree& tr, int P, int me) {
  Part p;
  p.P = P;
  p.me = me;
  if (P <= 1) return p;
  int lev = -1;
  for (int l = 0; l <= tr.depth; ++l)
    if ((int)tr.by_level[l].size() >= P) {
      lev = l;
      break;
    }
  if (lev < 0) return p;  // fewer clusters than ranks at every level: fully replicated
  p.level = lev;
  p.owner.assign(tr.n, -1);
  const std::vector<int>& L = tr.by_level[lev];  // preorder ids ascending = left to right
  const long long m = (long long)L.size();
  for (long long i = 0; i < m; ++i) p.owner[L[i]] = (int)(i * P / m);
  for (int l = lev + 1; l <= tr.depth; ++l)
    for (int t : tr.by_level[l]) p.owner[t] = p.owner[tr.parent[t]];
  return p;
}

std::vector<int> Part::filter(const std::vector<int>& L) const {
  std::vector<int> out;
  out.reserve(L.size());
  for (int t : L)
    if (mine(t)) out.push_back(t);
  return out;
}

void exchange(Ctx& C, Arena& ar, const std::vector<XItem>& items) {
  if (!C.comm.on() || items.empty()) return;
  const int P = C.comm.size, me = C.comm.rank;
  std::vector<long long> off(P + 1, 0);
  for (const XItem& it : items) {
    if (it.owner < 0 || it.owner >= P) throw StructureErr("exchange: item without an owning rank");
    off[it.owner + 1] += it.len;
  }
  for (int i = 0; i < P; ++i) off[i + 1] += off[i];
  const long long total = off[P];
  if (total == 0) return;
  double* buf = ar.alloc(total);
  std::vector<long long> run(off.begin(), off.end() - 1), g;
  std::vector<double*> pos(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    const XItem& it = items[i];
    pos[i] = buf + run[it.owner];
    run[it.owner] += it.len;
    if (it.owner == me && it.len > 0) {
      if (!*it.dst) throw StructureErr("exchange: owned item was not computed");
      g.push_back((long long)*it.dst);
      g.push_back(it.len);
      g.push_back((long long)pos[i]);
    }
  }
  if (!g.empty()) {  // pack this rank's arrays into its segment
    long long* di = C.push(g);
    C.flush();
    cuda_check(launch_gather(di, (int)(g.size() / 3), C.st), "gather(exchange)");
    ++C.launches;
  }
  C.flush();
  std::vector<long long> ob(P + 1);
  for (int i = 0; i <= P; ++i) ob[i] = off[i] * (long long)sizeof(double);
  if (C.comm.fn(C.comm.user, C.channel, buf, ob.data(), P, C.st) != 0)
    throw CudaFailure("all-gather of the partitioned results failed");
  for (size_t i = 0; i < items.size(); ++i)
    if (items[i].owner != me) *items[i].dst = pos[i];
}

void exchange_p2p(Ctx& C, Arena& ar, const std::vector<PItem>& items) {
  if (!C.comm.on() || items.empty()) return;
  const int P = C.comm.size, me = C.comm.rank;
  if (!C.comm.a2a) {  // no all-to-all: every rank receives every item
    std::vector<XItem> x;
    x.reserve(items.size());
    for (const PItem& it : items) x.push_back(XItem{it.src, it.len, it.ptr});
    exchange(C, ar, x);
    return;
  }
  std::vector<long long> soff(P + 1, 0), roff(P + 1, 0);
  for (const PItem& it : items) {
    if (it.src < 0 || it.src >= P || it.dst < 0 || it.dst >= P || it.src == it.dst)
      throw StructureErr("exchange_p2p: item without a valid source and destination");
    if (it.src == me) soff[it.dst + 1] += it.len;
    if (it.dst == me) roff[it.src + 1] += it.len;
  }
  for (int i = 0; i < P; ++i) {
    soff[i + 1] += soff[i];
    roff[i + 1] += roff[i];
  }
  double* sbuf = soff[P] > 0 ? ar.alloc(soff[P]) : nullptr;
  double* rbuf = roff[P] > 0 ? ar.alloc(roff[P]) : nullptr;
  std::vector<long long> srun(soff.begin(), soff.end() - 1), rrun(roff.begin(), roff.end() - 1), g;
  std::vector<std::pair<double**, double*>> recv;
  for (const PItem& it : items) {
    if (it.src == me && it.len > 0) {
      if (!*it.ptr) throw StructureErr("exchange_p2p: item to send was not computed");
      g.push_back((long long)*it.ptr);
      g.push_back(it.len);
      g.push_back((long long)(sbuf + srun[it.dst]));
      srun[it.dst] += it.len;
    }
    if (it.dst == me) {
      recv.emplace_back(it.ptr, rbuf + rrun[it.src]);
      rrun[it.src] += it.len;
    }
  }
  if (!g.empty()) {  // pack the outgoing blocks, grouped by destination
    long long* di = C.push(g);
    C.flush();
    cuda_check(launch_gather(di, (int)(g.size() / 3), C.st), "gather(exchange_p2p)");
    ++C.launches;
  }
  C.flush();
  std::vector<long long> sb(P + 1), rb(P + 1);
  for (int i = 0; i <= P; ++i) {
    sb[i] = soff[i] * (long long)sizeof(double);
    rb[i] = roff[i] * (long long)sizeof(double);
  }
  if (C.comm.a2a(C.comm.a2a_user, C.channel, sbuf, sb.data(), rbuf, rb.data(), P, C.st) != 0)
    throw CudaFailure("all-to-all of the partitioned results failed");
  for (auto& r : recv) *r.first = r.second;
}

void gather_rows(Ctx& C, H2& h) {
  if (!h.dist_rows) return;
  if (!C.comm.on()) throw InvalidInput("a partitioned matrix needs its communicator to be gathered");
  const Blocks& B = *h.bt;
  const Part part = make_part(*B.rows, C.comm);
  std::vector<XItem> items;
  for (int b = 0; b < B.nb; ++b) {
    if (!B.leaf(b)) continue;
    const int t = B.row[b], s = B.col[b];
    if (part.top(t)) continue;
    if (B.adm[b]) items.push_back(XItem{part.owner[t], (long long)h.rb->rank[t] * h.cb->rank[s], &h.coup[b]});
    else items.push_back(XItem{part.owner[t], (long long)B.rows->size(t) * B.cols->size(s), &h.near[b]});
  }
  auto ar = std::make_shared<Arena>(C.st);
  exchange(C, *ar, items);
  h.owned.push_back(ar);
  h.dist_rows = false;
  h.dist_halo = false;
}

void need_whole(Ctx& C, H2& h) { gather_rows(C, h); }
void need_rows_halo(Ctx& C, H2& h) {
  if (h.dist_rows && !h.dist_halo) gather_rows(C, h);
}

void exchange_ints(Ctx& C, const Part& part, const std::vector<int>& ids, std::vector<int>& v) {
  if (!C.comm.on() || !part.on() || ids.empty()) return;
  const int P = C.comm.size, me = C.comm.rank;
  std::vector<long long> off(P + 1, 0);
  for (int t : ids) {
    if (part.owner[t] < 0) throw StructureErr("exchange_ints: replicated cluster listed");
    ++off[part.owner[t] + 1];
  }
  for (int i = 0; i < P; ++i) off[i + 1] += off[i];
  const long long total = off[P];
  std::vector<long long> run(off.begin(), off.end() - 1), pos(ids.size());
  std::vector<double> hb(total, 0.0);
  for (size_t i = 0; i < ids.size(); ++i) {
    const int o = part.owner[ids[i]];
    pos[i] = run[o]++;
    if (o == me) hb[pos[i]] = (double)v[ids[i]];
  }
  Arena tmp(C.st);
  double* d = tmp.alloc(total);
  C.flush();
  cuda_check(cudaMemcpyAsync(d, hb.data(), total * sizeof(double), cudaMemcpyHostToDevice, C.st), "upload");
  std::vector<long long> ob(P + 1);
  for (int i = 0; i <= P; ++i) ob[i] = off[i] * (long long)sizeof(double);
  if (C.comm.fn(C.comm.user, C.channel, d, ob.data(), P, C.st) != 0)
    throw CudaFailure("all-gather of the partitioned ranks failed");
  const std::vector<double> back = C.read(d, total);
  for (size_t i = 0; i < ids.size(); ++i)
    if (part.owner[ids[i]] != me) v[ids[i]] = (int)back[pos[i]];
}

}  // namespace h2g
