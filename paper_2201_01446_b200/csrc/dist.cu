// Spatial domain decomposition across GPUs (one process per GPU) with NCCL over NVLink.
//
// Reference semantics: partition_domain (domain.cpp:21-82) -- 1-D slabs along the axis with the
// largest plane spacing (first wins), atoms ranked by wrapped fractional coordinate (ties by id)
// and split into equal-count chunks; ghosts are the non-owned atoms whose circular fractional
// distance to the owned extent is <= (r_cut + buffer) / spacing. run_md rebuilds the partition
// and the lists every rebuild_every steps (md.cpp:70-102, 210).
//
// Per rank the local system is owned + ghost atoms in ascending global id (so local index order
// is global order and the neighbour list reproduces the global canonical order). Only owned
// atoms are centres. Per step:
//   forward halo   owned positions -> the ranks that hold them as ghosts   (ncclSend/ncclRecv)
//   evaluate       local kernels; ghost rows only gather the reverse pair gradients
//   reverse halo   ghost force partials -> owners, accumulated in peer order (deterministic)
// At a rebuild every rank all-gathers the owned (id, x, v), repartitions identically and
// rebuilds its local system. No collective touches the data path except these exchanges.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "engine.hpp"

namespace dpb {

#define DPB_NCCL(x)                                                                        \
  do {                                                                                     \
    ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) throw ::dpb::CudaErr(std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

struct Dist {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  // global state (refreshed at every rebuild)
  int64_t N = 0;
  std::vector<double> gpos, gvel;
  std::vector<int32_t> gtypes;
  double box[9];
  uint8_t pbc[3];
  double margin = 0.0;
  // local system
  std::vector<int64_t> lgid;
  std::vector<uint8_t> lcenter;
  int64_t n_own = 0;
  int64_t max_own = 0;
  // exchange maps: for peer p, send = my owned atoms that p holds as ghosts, recv = my ghosts
  // owned by p; both in ascending global id, so the two sides agree entry by entry
  std::vector<int64_t> soff, roff;
  DevBuf<int32_t> sidx, ridx;
  DevBuf<double> sbuf, rbuf, gbuf_send, gbuf_all;
};

namespace {

void host_cell(const double* h, double* hinv, double& vol) {
  const double* a = h;
  const double* b = h + 3;
  const double* c = h + 6;
  const double bxc[3] = {b[1] * c[2] - b[2] * c[1], b[2] * c[0] - b[0] * c[2], b[0] * c[1] - b[1] * c[0]};
  vol = a[0] * bxc[0] + a[1] * bxc[1] + a[2] * bxc[2];
  const double cxa[3] = {c[1] * a[2] - c[2] * a[1], c[2] * a[0] - c[0] * a[2], c[0] * a[1] - c[1] * a[0]};
  const double axb[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
  for (int x = 0; x < 3; ++x) {
    hinv[3 * x + 0] = bxc[x] / vol;
    hinv[3 * x + 1] = cxa[x] / vol;
    hinv[3 * x + 2] = axb[x] / vol;
  }
  if (vol < 0) vol = -vol;
}

double spacing(const double* h, double vol, int k) {
  const double* u = h + 3 * ((k + 1) % 3);
  const double* v = h + 3 * ((k + 2) % 3);
  const double cr[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
  return vol / std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
}

double circ_dist(double x, double lo, double hi, bool periodic) {
  if (x >= lo && x <= hi) return 0.0;
  const double d1 = (x < lo) ? lo - x : x - hi;
  if (!periodic) return d1;
  const double d2 = (x < lo) ? x + 1.0 - hi : lo + 1.0 - x;
  return std::min(d1, d2);
}

} // namespace

// partition_domain (domain.cpp:21-82): owner[i] and, per worker, its ghost ids (ascending).
void partition(const Dist& D, std::vector<int>& owner, std::vector<std::vector<int64_t>>& ghosts) {
  const int64_t n = D.N;
  const int W = static_cast<int>(std::min<int64_t>(D.world, n));
  double hinv[9], vol;
  host_cell(D.box, hinv, vol);
  int ax = 0;
  double best = -1.0;
  for (int k = 0; k < 3; ++k) {
    const double sp = spacing(D.box, vol, k);
    if (sp > best) {
      best = sp;
      ax = k;
    }
  }
  const bool per = D.pbc[ax] != 0;
  const double mf = D.margin / spacing(D.box, vol, ax);
  std::vector<double> fw(n);
  for (int64_t i = 0; i < n; ++i) {
    const double* r = &D.gpos[3 * i];
    const double f = r[0] * hinv[ax] + r[1] * hinv[3 + ax] + r[2] * hinv[6 + ax];
    fw[i] = per ? f - std::floor(f) : f;
  }
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (fw[a] != fw[b]) return fw[a] < fw[b];
    return a < b;
  });
  owner.assign(n, 0);
  std::vector<double> lo(D.world, 0.0), hi(D.world, -1.0);
  const int64_t base = n / W, extra = n % W;
  int64_t at = 0;
  for (int w = 0; w < W; ++w) {
    const int64_t cnt = base + (w < extra ? 1 : 0);
    double l = 2.0, hh = -2.0;
    for (int64_t k = at; k < at + cnt; ++k) {
      owner[order[k]] = w;
      l = std::min(l, fw[order[k]]);
      hh = std::max(hh, fw[order[k]]);
    }
    lo[w] = l;
    hi[w] = hh;
    at += cnt;
  }
  ghosts.assign(D.world, {});
  for (int w = 0; w < W; ++w)
    for (int64_t j = 0; j < n; ++j)
      if (owner[j] != w && circ_dist(fw[j], lo[w], hi[w], per) <= mf) ghosts[w].push_back(j);
}

namespace {

__global__ void k_pack3(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ src,
                        double* __restrict__ dst) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const int64_t i = idx[k];
  dst[3 * k] = src[3 * i];
  dst[3 * k + 1] = src[3 * i + 1];
  dst[3 * k + 2] = src[3 * i + 2];
}

__global__ void k_unpack_pos(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ src,
                             double* __restrict__ pos3, double4* __restrict__ pos4) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const int64_t i = idx[k];
  const double x = src[3 * k], y = src[3 * k + 1], z = src[3 * k + 2];
  pos3[3 * i] = x;
  pos3[3 * i + 1] = y;
  pos3[3 * i + 2] = z;
  pos4[i] = make_double4(x, y, z, 0.0);
}

__global__ void k_accum3(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ src,
                         double* __restrict__ dst) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const int64_t i = idx[k];
  dst[3 * i] += src[3 * k];
  dst[3 * i + 1] += src[3 * k + 1];
  dst[3 * i + 2] += src[3 * k + 2];
}

__global__ void k_pack_state(int64_t n, const uint8_t* __restrict__ center, const int64_t* __restrict__ gid,
                             const int64_t* __restrict__ slot, const double* __restrict__ x,
                             const double* __restrict__ v, double* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !center[i]) return;
  double* o = out + 7 * slot[i];
  o[0] = static_cast<double>(gid[i]);
  for (int c = 0; c < 3; ++c) {
    o[1 + c] = x[3 * i + c];
    o[4 + c] = v[3 * i + c];
  }
}

// Host plan of one rank: local atoms (owned + ghosts, ascending global id), centre mask and the
// exchange lists (local indices) per peer: s = my owned atoms that peer p holds as ghosts,
// rv = my ghosts owned by p, both ascending in global id.
struct Plan {
  std::vector<int64_t> lgid;
  std::vector<uint8_t> lcenter;
  std::vector<int64_t> soff, roff;
  std::vector<int32_t> s, rv;
};

void make_plan(const Dist& D, int r, Plan& P) {
  std::vector<int> owner;
  std::vector<std::vector<int64_t>> ghosts;
  partition(D, owner, ghosts);
  std::vector<uint8_t> is_ghost(D.N, 0);
  for (int64_t j : ghosts[r]) is_ghost[j] = 1;
  P.lgid.clear();
  P.lcenter.clear();
  for (int64_t j = 0; j < D.N; ++j) {
    if (owner[j] == r || is_ghost[j]) {
      P.lgid.push_back(j);
      P.lcenter.push_back(owner[j] == r ? 1 : 0);
    }
  }
  const int64_t nl = static_cast<int64_t>(P.lgid.size());
  std::vector<int64_t> lidx(D.N, -1);
  for (int64_t k = 0; k < nl; ++k) lidx[P.lgid[k]] = k;
  P.soff.assign(D.world + 1, 0);
  P.roff.assign(D.world + 1, 0);
  P.s.clear();
  P.rv.clear();
  for (int p = 0; p < D.world; ++p) {
    P.soff[p] = static_cast<int64_t>(P.s.size());
    P.roff[p] = static_cast<int64_t>(P.rv.size());
    if (p == r) continue;
    for (int64_t j : ghosts[p])
      if (owner[j] == r) P.s.push_back(static_cast<int32_t>(lidx[j]));
    for (int64_t j : ghosts[r])
      if (owner[j] == p) P.rv.push_back(static_cast<int32_t>(lidx[j]));
  }
  P.soff[D.world] = static_cast<int64_t>(P.s.size());
  P.roff[D.world] = static_cast<int64_t>(P.rv.size());
}

// Build the local system for this rank from the global state and upload it.
void build_local(Engine& E) {
  static const bool trace = std::getenv("DPB_TRACE") != nullptr;
  auto now = [&] {
    if (trace) cudaStreamSynchronize(E.stream);
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  Dist& D = *E.dist;
  Plan P;
  make_plan(D, D.rank, P);
  const auto t1 = now();
  D.lgid.swap(P.lgid);
  D.lcenter.swap(P.lcenter);
  D.soff = P.soff;
  D.roff = P.roff;
  const std::vector<int32_t>& s = P.s;
  const std::vector<int32_t>& rv = P.rv;
  const int64_t nl = static_cast<int64_t>(D.lgid.size());
  D.n_own = 0;
  for (auto c : D.lcenter) D.n_own += c;
  D.sidx.ensure(s.size() + 1);
  D.ridx.ensure(rv.size() + 1);
  const size_t mx = std::max(s.size(), rv.size()) + 1;
  D.sbuf.ensure(3 * mx);
  D.rbuf.ensure(3 * mx);
  if (!s.empty()) DPB_CUDA(cudaMemcpyAsync(D.sidx.p, s.data(), s.size() * 4, cudaMemcpyHostToDevice, E.stream));
  if (!rv.empty()) DPB_CUDA(cudaMemcpyAsync(D.ridx.p, rv.data(), rv.size() * 4, cudaMemcpyHostToDevice, E.stream));
  // local arrays
  std::vector<double> lp(3 * nl), lv(3 * nl);
  std::vector<int32_t> lt(nl);
  for (int64_t k = 0; k < nl; ++k) {
    const int64_t j = D.lgid[k];
    for (int c = 0; c < 3; ++c) {
      lp[3 * k + c] = D.gpos[3 * j + c];
      lv[3 * k + c] = D.gvel[3 * j + c];
    }
    lt[k] = D.gtypes[j];
  }
  const auto t2 = now();
  E.set_config(nl, lp.data(), lt.data(), D.box, D.pbc, D.lcenter.data());
  const auto t3 = now();
  E.md_upload_atoms(lv.data());
  const auto t4 = now();
  E.build_list(E.r_cut + E.md.buffer);
  const auto t5 = now();
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[dpb rank %d] local: plan %.2f, arrays %.2f, set_config %.2f, upload %.2f, list %.2f ms\n",
                 D.rank, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5));
  }
}

void exchange(Engine& E, const std::vector<int64_t>& out_off, const std::vector<int64_t>& in_off) {
  Dist& D = *E.dist;
  DPB_NCCL(ncclGroupStart());
  for (int p = 0; p < D.world; ++p) {
    const int64_t so = out_off[p], sc = out_off[p + 1] - so;
    const int64_t ro = in_off[p], rc = in_off[p + 1] - ro;
    if (sc > 0) DPB_NCCL(ncclSend(D.sbuf.p + 3 * so, 3 * sc, ncclDouble, p, D.comm, E.stream));
    if (rc > 0) DPB_NCCL(ncclRecv(D.rbuf.p + 3 * ro, 3 * rc, ncclDouble, p, D.comm, E.stream));
  }
  DPB_NCCL(ncclGroupEnd());
}

} // namespace

void dist_init(Engine& E, int rank, int world, const void* uid) {
  if (world < 1 || rank < 0 || rank >= world) throw InputErr("bad rank/world");
  if (!E.dist) E.dist = new Dist();
  Dist& D = *E.dist;
  D.rank = rank;
  D.world = world;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  DPB_CUDA(cudaSetDevice(E.device));
  DPB_NCCL(ncclCommInitRank(&D.comm, world, id, rank));
}

void dist_destroy(Engine& E) {
  if (!E.dist) return;
  if (E.dist->comm) ncclCommDestroy(E.dist->comm);
  E.dist->sidx.release();
  E.dist->ridx.release();
  E.dist->sbuf.release();
  E.dist->rbuf.release();
  E.dist->gbuf_send.release();
  E.dist->gbuf_all.release();
  delete E.dist;
  E.dist = nullptr;
}

int64_t dist_n_total(const Engine& E) { return E.dist->N; }

void dist_allreduce_sum(Engine& E, double* dev, int count) {
  if (count > 0) DPB_NCCL(ncclAllReduce(dev, dev, count, ncclDouble, ncclSum, E.dist->comm, E.stream));
}

void dist_md_begin(Engine& E, int64_t N, const double* pos, const double* vel, const int32_t* types,
                   const double* box, const uint8_t* pbc, const dp_md_config* cfg) {
  Dist& D = *E.dist;
  if (N < 1) throw InputErr("configuration has no atoms");
  for (int64_t i = 0; i < N; ++i)
    if (types[i] < 0 || types[i] >= E.n_types) throw InputErr("atom type id out of range");
  D.N = N;
  D.gpos.assign(pos, pos + 3 * N);
  D.gvel.assign(vel, vel + 3 * N);
  D.gtypes.assign(types, types + N);
  std::memcpy(D.box, box, sizeof(D.box));
  std::memcpy(D.pbc, pbc, sizeof(D.pbc));
  D.margin = E.r_cut + cfg->buffer;
  D.max_own = N / std::min<int64_t>(D.world, N) + 1;
  E.md = *cfg;
  build_local(E);
}

// Positions of my ghosts from their owners.
void dist_halo_forward(Engine& E) {
  Dist& D = *E.dist;
  const int64_t ns = D.soff[D.world], nr = D.roff[D.world];
  if (ns) k_pack3<<<ceil_div(ns, 256), 256, 0, E.stream>>>(ns, D.sidx.p, E.pos3.p, D.sbuf.p);
  exchange(E, D.soff, D.roff);
  if (nr) k_unpack_pos<<<ceil_div(nr, 256), 256, 0, E.stream>>>(nr, D.ridx.p, D.rbuf.p, E.pos3.p, E.pos4.p);
  E.launches += 2;
}

// Ghost force partials (minus the pair gradients landing on them) back to their owners.
void dist_halo_reverse(Engine& E) {
  Dist& D = *E.dist;
  const int64_t ns = D.soff[D.world], nr = D.roff[D.world];
  if (nr) k_pack3<<<ceil_div(nr, 256), 256, 0, E.stream>>>(nr, D.ridx.p, E.forces.p, D.sbuf.p);
  exchange(E, D.roff, D.soff);
  for (int p = 0; p < D.world; ++p) {
    const int64_t o = D.soff[p], c = D.soff[p + 1] - o;
    if (c) k_accum3<<<ceil_div(c, 256), 256, 0, E.stream>>>(c, D.sidx.p + o, D.rbuf.p + 3 * o, E.forces.p);
  }
  E.launches += 1 + D.world;
}

// All-gather of the owned (id, x, v) into the global arrays on every rank.
static void gather_global(Engine& E) {
  Dist& D = *E.dist;
  const int64_t nl = E.n;
  std::vector<int64_t> slot(nl, 0);
  int64_t k = 0;
  for (int64_t i = 0; i < nl; ++i)
    if (D.lcenter[i]) slot[i] = k++;
  DevBuf<int64_t> dgid, dslot;
  dgid.ensure(nl);
  dslot.ensure(nl);
  DPB_CUDA(cudaMemcpyAsync(dgid.p, D.lgid.data(), nl * 8, cudaMemcpyHostToDevice, E.stream));
  DPB_CUDA(cudaMemcpyAsync(dslot.p, slot.data(), nl * 8, cudaMemcpyHostToDevice, E.stream));
  D.gbuf_send.ensure(7 * D.max_own);
  D.gbuf_all.ensure(7 * D.max_own * D.world);
  DPB_CUDA(cudaMemsetAsync(D.gbuf_send.p, 0xff, 7 * D.max_own * sizeof(double), E.stream)); // NaN ids
  k_pack_state<<<ceil_div(nl, 256), 256, 0, E.stream>>>(nl, E.center.p, dgid.p, dslot.p, E.pos3.p,
                                                        E.vel3.p, D.gbuf_send.p);
  DPB_NCCL(ncclAllGather(D.gbuf_send.p, D.gbuf_all.p, 7 * D.max_own, ncclDouble, D.comm, E.stream));
  std::vector<double> all(7 * D.max_own * D.world);
  DPB_CUDA(cudaMemcpyAsync(all.data(), D.gbuf_all.p, all.size() * 8, cudaMemcpyDeviceToHost, E.stream));
  DPB_CUDA(cudaStreamSynchronize(E.stream));
  dgid.release();
  dslot.release();
  for (int64_t q = 0; q < D.max_own * D.world; ++q) {
    const double* o = &all[7 * q];
    if (!(o[0] >= 0.0)) continue;
    const int64_t j = static_cast<int64_t>(o[0]);
    for (int c = 0; c < 3; ++c) {
      D.gpos[3 * j + c] = o[1 + c];
      D.gvel[3 * j + c] = o[4 + c];
    }
  }
}

void dist_rebuild(Engine& E) {
  static const bool trace = std::getenv("DPB_TRACE") != nullptr;
  auto now = [&] {
    if (trace) cudaStreamSynchronize(E.stream);
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  gather_global(E);
  const auto t1 = now();
  build_local(E);
  const auto t2 = now();
  if (trace)
    std::fprintf(stderr, "[dpb rank %d] rebuild: gather %.2f ms, local %.2f ms\n", E.dist->rank,
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(t2 - t1).count());
}

void dist_md_end(Engine& E, double* gpos, double* gvel) {
  Dist& D = *E.dist;
  gather_global(E);
  if (gpos) std::memcpy(gpos, D.gpos.data(), 3 * D.N * 8);
  if (gvel) std::memcpy(gvel, D.gvel.data(), 3 * D.N * 8);
  // counters summed over ranks, largest drift over ranks
  DPB_NCCL(ncclAllReduce(E.counters.p, E.counters.p, 3, ncclUint64, ncclSum, D.comm, E.stream));
  DPB_NCCL(ncclAllReduce(E.red.p + 11, E.red.p + 11, 1, ncclDouble, ncclMax, D.comm, E.stream));
}

} // namespace dpb

extern "C" {

int dp_partition_domain(int64_t n, const double* pos, const double* box, const uint8_t* pbc,
                        int n_workers, double margin, int32_t* owner, uint8_t* ghost_mask) {
  return dpb::guard_call(nullptr, [&] {
    if (n_workers < 1) throw dpb::InputErr("worker count must be at least 1");
    dpb::Dist D;
    D.world = n_workers;
    D.N = n;
    D.gpos.assign(pos, pos + 3 * n);
    std::memcpy(D.box, box, sizeof(D.box));
    std::memcpy(D.pbc, pbc, sizeof(D.pbc));
    D.margin = margin;
    std::vector<int> own;
    std::vector<std::vector<int64_t>> gh;
    dpb::partition(D, own, gh);
    for (int64_t i = 0; i < n; ++i) owner[i] = own[i];
    std::memset(ghost_mask, 0, static_cast<size_t>(n_workers) * n);
    for (int w = 0; w < n_workers; ++w)
      for (int64_t j : gh[w]) ghost_mask[static_cast<int64_t>(w) * n + j] = 1;
  });
}

// Host-side plan of one rank (for tests of the decomposition logic without GPUs). Arrays sized
// n (lgid, center, send, recv) and n_workers+1 (offsets); send/recv hold GLOBAL ids.
int dp_dist_plan(int64_t n, const double* pos, const double* box, const uint8_t* pbc, int n_workers,
                 int rank, double margin, int64_t* n_local, int64_t* lgid, uint8_t* center,
                 int64_t* send_off, int64_t* send_gid, int64_t* recv_off, int64_t* recv_gid) {
  return dpb::guard_call(nullptr, [&] {
    if (n_workers < 1 || rank < 0 || rank >= n_workers) throw dpb::InputErr("bad rank/world");
    dpb::Dist D;
    D.world = n_workers;
    D.N = n;
    D.gpos.assign(pos, pos + 3 * n);
    std::memcpy(D.box, box, sizeof(D.box));
    std::memcpy(D.pbc, pbc, sizeof(D.pbc));
    D.margin = margin;
    dpb::Plan P;
    dpb::make_plan(D, rank, P);
    *n_local = static_cast<int64_t>(P.lgid.size());
    for (size_t k = 0; k < P.lgid.size(); ++k) {
      lgid[k] = P.lgid[k];
      center[k] = P.lcenter[k];
    }
    for (int p = 0; p <= n_workers; ++p) {
      send_off[p] = P.soff[p];
      recv_off[p] = P.roff[p];
    }
    for (size_t k = 0; k < P.s.size(); ++k) send_gid[k] = P.lgid[P.s[k]];
    for (size_t k = 0; k < P.rv.size(); ++k) recv_gid[k] = P.lgid[P.rv[k]];
  });
}

int dp_nccl_unique_id(void* out, int len) {
  return dpb::guard_call(nullptr, [&] {
    if (!out || len < static_cast<int>(sizeof(ncclUniqueId))) throw dpb::InputErr("buffer too small");
    ncclUniqueId id;
    DPB_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

} // extern "C"
