// Spatial domain decomposition across GPUs (one process per GPU) with NCCL over NVLink.
//
// Reference semantics: partition_domain (domain.cpp:21-82) -- 1-D slabs along the axis with the
// largest plane spacing (first wins), atoms ranked by wrapped fractional coordinate (ties by id)
// and split into equal-count chunks; ghosts are the non-owned atoms whose circular fractional
// distance to the owned extent is <= (r_cut + buffer) / spacing. run_md rebuilds the partition
// and the lists every rebuild_every steps (md.cpp:70-102, 210).
//
// Per rank the local system is the owned atoms (ascending global id) followed by the ghosts
// (ascending global id): the centres are one contiguous range, so the evaluation chunks never
// span ghost rows. Rows are built and sorted in global-id space (pairs evaluated from the lower
// global id, keys sorted by (type, global id, shift), then mapped back to local indices), so every
// row equals the global row entry for entry and in order. Only owned atoms are centres. Per step:
//   forward halo   owned positions -> the ranks that hold them as ghosts   (ncclSend/ncclRecv)
//   evaluate       local kernels (centres = owned atoms)
//   pair halo      for each ghost j and each entry (j -> i) with i owned here, the pair gradient
//                  g(i -> j) -> j's owner, which sums it into F_j in its own row order
// so each owned atom's force is summed in exactly the order one GPU sums it: forces, positions
// and velocities are bitwise independent of the GPU count (tests/test_gpu_dist.py).
// At a rebuild every rank all-gathers the owned (id, x, v), repartitions identically and
// rebuilds its local system. No collective touches the data path except these exchanges.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <nccl.h>

#include <cub/cub.cuh>

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
  // device-side repartition (every rebuild): global state, sort keys, owners, plans
  DevBuf<double> d_gpos, d_gvel, d_fw, d_lohi, d_lpos, d_lvel;
  DevBuf<int32_t> d_gtypes, d_owner, d_ids, d_ids2, d_flag, d_scan, d_lidx, d_lgid, d_slot, d_ltypes;
  DevBuf<uint64_t> d_keys, d_keys2;
  DevBuf<uint8_t> d_smask, d_lcenter;
  DevBuf<int64_t> d_counts; // [0] n_local, [1 .. W] send counts, [W+1 .. 2W] recv counts
  // pair-gradient halo (per step, after the backward pass): for every ghost j of this rank and
  // every entry (j -> i) of its row with i owned here, the gradient g of the reverse pair
  // (i -> j) goes to j's owner, which sums it into F_j in its own row order -- the force
  // summation order of one GPU. Slots are fixed per rebuild (NaN marks a non-real pair).
  DevBuf<int64_t> gs_base;   // [ghost list] first send slot of each ghost (ridx order)
  DevBuf<int64_t> gr_base;   // [owned list] first receive slot of each owned atom (sidx order)
  DevBuf<int32_t> rslot;     // [E] receive slot of an owned row's entry with a ghost neighbour, else -1
  DevBuf<int64_t> d_gcnt;    // scratch counts
  DevBuf<double> gsend, grecv;
  std::vector<int64_t> gsoff, groff; // slot offsets per peer (send / receive)
  // owned atoms without / with a ghost neighbour: the first set's forces run while the pair
  // halo is in flight
  DevBuf<int32_t> f_inner, f_bound, d_tflag, d_tscan;
  int64_t n_inner = 0, n_bound = 0;
  DevBuf<unsigned char> d_tmp;
  bool host_global_valid = true; // gpos/gvel (host) reflect the last gather
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

// Per ghost j of the list (t-th): number of entries of its row whose neighbour is owned here.
__global__ void k_ghost_slots(int64_t m, const int32_t* __restrict__ list, const int64_t* __restrict__ row_off,
                              const uint64_t* __restrict__ keys, const uint8_t* __restrict__ center,
                              int64_t* __restrict__ cnt) {
  const int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= m) return;
  const int j = list[t];
  int c = 0;
  for (int64_t e = row_off[j] + lane; e < row_off[j + 1]; e += 32) c += center[key_j(keys[e])] ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[t] = c;
}

// Per owned atom j of peer p's list (t-th): entries of its row whose neighbour is owned by p;
// with fill != 0 also their receive slots, in row order (= the order p packs them in).
__global__ void k_owned_slots(int64_t m, const int32_t* __restrict__ list, int p, const int64_t* __restrict__ row_off,
                              const uint64_t* __restrict__ keys, const int32_t* __restrict__ gid,
                              const int32_t* __restrict__ owner, int64_t* __restrict__ cnt,
                              const int64_t* __restrict__ base, int64_t off, int32_t* __restrict__ rslot) {
  const int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= m) return;
  const int j = list[t];
  int c = 0;
  for (int64_t b = row_off[j]; b < row_off[j + 1]; b += 32) {
    const int64_t e = b + lane;
    const bool mine = e < row_off[j + 1] && owner[gid[key_j(keys[e])]] == p;
    const unsigned mk = __ballot_sync(0xffffffffu, mine);
    if (rslot && mine) rslot[e] = static_cast<int32_t>(off + base[t] + c + __popc(mk & ((1u << lane) - 1u)));
    c += __popc(mk);
  }
  if (!rslot && lane == 0) cnt[t] = c;
}

// Pack: for ghost j (t-th of the list) and every entry (j -> i) with i owned here, the gradient
// of the reverse pair (i -> j) -- g[realoff[i] + k] when that pair is real (rank k), else NaN.
__global__ void k_pack_pair_g(int64_t m, const int32_t* __restrict__ list, const int64_t* __restrict__ row_off,
                              const uint64_t* __restrict__ keys, const uint16_t* __restrict__ rev,
                              const int16_t* __restrict__ rank, const int64_t* __restrict__ realoff,
                              const uint8_t* __restrict__ center, const double* __restrict__ g,
                              const int64_t* __restrict__ base, double* __restrict__ out) {
  const int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= m) return;
  const int j = list[t];
  int64_t slot = base[t];
  for (int64_t b = row_off[j]; b < row_off[j + 1]; b += 32) {
    const int64_t e = b + lane;
    int i = 0;
    bool own = false;
    if (e < row_off[j + 1]) {
      i = key_j(keys[e]);
      own = center[i] != 0;
    }
    const unsigned mk = __ballot_sync(0xffffffffu, own);
    if (own) {
      const int k = rank[row_off[i] + rev[e]];
      double* o = out + 3 * (slot + __popc(mk & ((1u << lane) - 1u)));
      if (k >= 0) {
        const double* gi = g + 3 * (realoff[i] + k);
        o[0] = gi[0];
        o[1] = gi[1];
        o[2] = gi[2];
      } else {
        o[0] = o[1] = o[2] = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
    slot += __popc(mk);
  }
}

// Owned atom i touches a ghost (some neighbour of its row is not a centre here): flag 1.
__global__ void k_touch_ghost(int64_t n_own, const int64_t* __restrict__ row_off, const uint64_t* __restrict__ keys,
                              const uint8_t* __restrict__ center, int32_t* __restrict__ flag) {
  const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_own) return;
  bool t = false;
  for (int64_t e = row_off[i] + lane; e < row_off[i + 1]; e += 32) t |= center[key_j(keys[e])] == 0;
  t = __any_sync(0xffffffffu, t);
  if (lane == 0) flag[i] = t ? 1 : 0;
}

__global__ void k_split_atoms(int64_t n_own, const int32_t* __restrict__ flag, const int32_t* __restrict__ scan,
                              int32_t* __restrict__ inner, int32_t* __restrict__ bound) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n_own) return;
  if (flag[i]) bound[scan[i]] = static_cast<int32_t>(i);
  else inner[i - scan[i]] = static_cast<int32_t>(i);
}

// Chunk classification: flag[k] = 1 when a centre of chunk k (atoms [cka[k], cka[k+1])) has a
// ghost in its neighbour row. Thread per atom, chunk found by binary search.
__global__ void k_chunk_ghost(int64_t n, int nk, const int64_t* __restrict__ cka, const uint8_t* __restrict__ center,
                              const int64_t* __restrict__ row_off, const uint64_t* __restrict__ keys,
                              int* __restrict__ flag) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !center[i]) return;
  int lo = 0, hi = nk - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cka[mid] <= i) lo = mid; else hi = mid - 1;
  }
  for (int64_t e = row_off[i]; e < row_off[i + 1]; ++e)
    if (!center[key_j(keys[e])]) {
      flag[lo] = 1;
      return;
    }
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


__device__ __forceinline__ double circ_dist_d(double x, double lo, double hi, bool periodic) {
  if (x >= lo && x <= hi) return 0.0;
  const double d1 = (x < lo) ? lo - x : x - hi;
  if (!periodic) return d1;
  const double d2 = (x < lo) ? x + 1.0 - hi : lo + 1.0 - x;
  return fmin(d1, d2);
}

__global__ void k_unpack_global(int64_t nrec, const double* __restrict__ all, double* __restrict__ gpos,
                                double* __restrict__ gvel) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (q >= nrec) return;
  const double* o = all + 7 * q;
  if (!(o[0] >= 0.0)) return;
  const int64_t j = static_cast<int64_t>(o[0]);
  for (int c = 0; c < 3; ++c) {
    gpos[3 * j + c] = o[1 + c];
    gvel[3 * j + c] = o[4 + c];
  }
}

// Wrapped fractional coordinate along the slab axis (domain.cpp:38-45) and an order-preserving
// integer key (stable radix sort over ids 0..N-1 = the reference's (fw, id) ordering).
__global__ void k_fw_keys(int64_t N, const double* __restrict__ gpos, double h0, double h1, double h2, int per,
                          double* __restrict__ fw, uint64_t* __restrict__ keys, int32_t* __restrict__ ids) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= N) return;
  const double* r = gpos + 3 * i;
  const double f = __dadd_rn(__dadd_rn(__dmul_rn(r[0], h0), __dmul_rn(r[1], h1)), __dmul_rn(r[2], h2));
  const double w = per ? __dsub_rn(f, floor(f)) : f;
  fw[i] = w;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(w));
  keys[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
  ids[i] = static_cast<int32_t>(i);
}

// Equal-count chunks of the sorted order (domain.cpp:49-63): owner and [lo, hi] per worker.
__global__ void k_owner(int64_t N, int W, const int32_t* __restrict__ sorted_ids, const double* __restrict__ fw,
                        int32_t* __restrict__ owner, double* __restrict__ lohi) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= N) return;
  const int64_t base = N / W, extra = N % W;
  const int64_t big = extra * (base + 1);
  const int w = k < big ? static_cast<int>(k / (base + 1)) : static_cast<int>(extra + (k - big) / base);
  const int64_t start = w < extra ? w * (base + 1) : big + (w - extra) * base;
  const int64_t cnt = base + (w < extra ? 1 : 0);
  const int id = sorted_ids[k];
  owner[id] = w;
  if (k == start) lohi[2 * w] = fw[id];
  if (k == start + cnt - 1) lohi[2 * w + 1] = fw[id];
}

// Local membership (owned or ghost of rank r) and, per peer p, "I own it and p holds it as a
// ghost" as a bit mask (domain.cpp:64-80 ghost rule).
__global__ void k_flags(int64_t N, int r, int W, const int32_t* __restrict__ owner, const double* __restrict__ fw,
                        const double* __restrict__ lohi, double mf, int per, int32_t* __restrict__ local,
                        uint8_t* __restrict__ smask, int32_t* __restrict__ oflag) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= N) return;
  const int o = owner[id];
  const double x = fw[id];
  const bool own = o == r;
  const bool ghost = !own && circ_dist_d(x, lohi[2 * r], lohi[2 * r + 1], per) <= mf;
  local[id] = (own || ghost) ? 1 : 0;
  oflag[id] = own ? 1 : 0;
  uint8_t m = 0;
  if (own)
    for (int p = 0; p < W; ++p)
      if (p != r && circ_dist_d(x, lohi[2 * p], lohi[2 * p + 1], per) <= mf) m |= static_cast<uint8_t>(1u << p);
  smask[id] = m;
}

// Local order: the owned atoms first (ascending global id), then the ghosts (ascending global
// id), so the centres are one contiguous range and the evaluation chunks hold no ghost rows.
__global__ void k_local_index(int64_t N, const int32_t* __restrict__ local, const int32_t* __restrict__ scan,
                              const int32_t* __restrict__ oflag, const int32_t* __restrict__ oscan,
                              int32_t* __restrict__ lidx, int32_t* __restrict__ lgid, int64_t* __restrict__ counts) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= N) return;
  if (local[id]) {
    const int n_own = oscan[N - 1] + oflag[N - 1];
    const int l = oflag[id] ? oscan[id] : n_own + (scan[id] - oscan[id]);
    lidx[id] = l;
    lgid[l] = static_cast<int32_t>(id);
  } else {
    lidx[id] = -1;
  }
  if (id == N - 1) counts[0] = scan[id] + local[id];
}

// Flag of peer p: send (mode 0: owned, p holds it as a ghost) or recv (mode 1: my ghost owned by p).
__global__ void k_peer_flag(int64_t N, int r, int p, int mode, const uint8_t* __restrict__ smask,
                            const int32_t* __restrict__ local, const int32_t* __restrict__ owner,
                            int32_t* __restrict__ flag) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= N) return;
  flag[id] = mode == 0 ? ((smask[id] >> p) & 1) : ((local[id] && owner[id] == p && owner[id] != r) ? 1 : 0);
}

// Ascending-id compaction of the flagged local indices into dst (+ count into counts[slot]).
__global__ void k_peer_scatter(int64_t N, const int32_t* __restrict__ flag, const int32_t* __restrict__ scan,
                               const int32_t* __restrict__ lidx, int32_t* __restrict__ dst,
                               int64_t* __restrict__ counts, int slot) {
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= N) return;
  if (flag[id]) dst[scan[id]] = lidx[id];
  if (id == N - 1) counts[slot] = scan[id] + flag[id];
}

__global__ void k_local_arrays(int64_t nl, int r, const int32_t* __restrict__ lgid, const double* __restrict__ gpos,
                               const double* __restrict__ gvel, const int32_t* __restrict__ gtypes,
                               const int32_t* __restrict__ owner, double* __restrict__ lp, double* __restrict__ lv,
                               int32_t* __restrict__ lt, uint8_t* __restrict__ lc) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k >= nl) return;
  const int64_t j = lgid[k];
  for (int c = 0; c < 3; ++c) {
    lp[3 * k + c] = gpos[3 * j + c];
    lv[3 * k + c] = gvel[3 * j + c];
  }
  lt[k] = gtypes[j];
  lc[k] = owner[j] == r ? 1 : 0;
}

__global__ void k_slot_of_center(int64_t nl, const uint8_t* __restrict__ center, const int32_t* __restrict__ scan,
                                 int32_t* __restrict__ slot) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < nl) slot[k] = center[k] ? scan[k] : -1;
}

__global__ void k_pack_state_d(int64_t n, const int32_t* __restrict__ slot, const int32_t* __restrict__ gid,
                               const double* __restrict__ x, const double* __restrict__ v, double* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || slot[i] < 0) return;
  double* o = out + 7 * static_cast<int64_t>(slot[i]);
  o[0] = static_cast<double>(gid[i]);
  for (int c = 0; c < 3; ++c) {
    o[1 + c] = x[3 * i + c];
    o[4 + c] = v[3 * i + c];
  }
}

__global__ void k_u8_to_i32(int64_t n, const uint8_t* __restrict__ a, int32_t* __restrict__ b) {
  const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (k < n) b[k] = a[k];
}

template <class T>
void excl_scan(Dist& D, const T* in, T* out, int64_t n, cudaStream_t st) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, n, st);
  D.d_tmp.ensure(b + 1);
  cub::DeviceScan::ExclusiveSum(D.d_tmp.p, b, in, out, n, st);
}

// The partition and exchange plan of this rank, computed on the device from d_gpos (identical
// on every rank after the all-gather). Produces D.sidx / D.ridx (device), D.soff / D.roff and the
// local arrays (host copies for set_config), with one small read-back of the counts.
void device_plan(Engine& E, std::vector<double>& lp, std::vector<double>& lv, std::vector<int32_t>& lt,
                 std::vector<uint8_t>& lc) {
  Dist& D = *E.dist;
  cudaStream_t st = E.stream;
  const int64_t N = D.N;
  const int W = static_cast<int>(std::min<int64_t>(D.world, N));
  if (D.world > 8) throw InputErr("the device partition supports up to 8 ranks");
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
  const int per = D.pbc[ax] != 0;
  const double mf = D.margin / spacing(D.box, vol, ax);
  D.d_fw.ensure(N);
  D.d_keys.ensure(N);
  D.d_keys2.ensure(N);
  D.d_ids.ensure(N);
  D.d_ids2.ensure(N);
  D.d_owner.ensure(N);
  D.d_lohi.ensure(2 * D.world);
  D.d_flag.ensure(N);
  D.d_scan.ensure(N);
  D.d_lidx.ensure(N);
  D.d_lgid.ensure(N);
  D.d_smask.ensure(N);
  D.d_counts.ensure(2 * D.world + 2);
  const int nb = static_cast<int>(ceil_div(N, 256));
  k_fw_keys<<<nb, 256, 0, st>>>(N, D.d_gpos.p, hinv[ax], hinv[3 + ax], hinv[6 + ax], per, D.d_fw.p, D.d_keys.p,
                                D.d_ids.p);
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, D.d_keys.p, D.d_keys2.p, D.d_ids.p, D.d_ids2.p, static_cast<int>(N), 0, 64,
                                  st);
  D.d_tmp.ensure(b + 1);
  cub::DeviceRadixSort::SortPairs(D.d_tmp.p, b, D.d_keys.p, D.d_keys2.p, D.d_ids.p, D.d_ids2.p, static_cast<int>(N), 0,
                                  64, st);
  k_owner<<<nb, 256, 0, st>>>(N, W, D.d_ids2.p, D.d_fw.p, D.d_owner.p, D.d_lohi.p);
  // (d_ids / d_ids2 are free after k_owner: owned flag and its scan)
  k_flags<<<nb, 256, 0, st>>>(N, D.rank, W, D.d_owner.p, D.d_fw.p, D.d_lohi.p, mf, per, D.d_flag.p, D.d_smask.p,
                              D.d_ids.p);
  excl_scan(D, D.d_flag.p, D.d_scan.p, N, st);
  excl_scan(D, D.d_ids.p, D.d_ids2.p, N, st);
  k_local_index<<<nb, 256, 0, st>>>(N, D.d_flag.p, D.d_scan.p, D.d_ids.p, D.d_ids2.p, D.d_lidx.p, D.d_lgid.p,
                                    D.d_counts.p);
  // exchange lists per peer, ascending global id; staged at offset p * N, packed after the counts
  D.sidx.ensure(static_cast<size_t>(N) * D.world + 1);
  D.ridx.ensure(static_cast<size_t>(N) * D.world + 1);
  DevBuf<int32_t>& pf = D.d_ids;  // reuse (free after the sort) as the per-peer flag
  DevBuf<int32_t>& ps = D.d_ids2; // scan of the peer flag (the sorted ids are no longer needed)
  for (int mode = 0; mode < 2; ++mode)
    for (int p = 0; p < D.world; ++p) {
      if (p == D.rank) {
        DPB_CUDA(cudaMemsetAsync(D.d_counts.p + 1 + mode * D.world + p, 0, sizeof(int64_t), st));
        continue;
      }
      k_peer_flag<<<nb, 256, 0, st>>>(N, D.rank, p, mode, D.d_smask.p, D.d_flag.p, D.d_owner.p, pf.p);
      excl_scan(D, pf.p, ps.p, N, st);
      int32_t* dst = (mode == 0 ? D.sidx.p : D.ridx.p) + static_cast<size_t>(p) * N;
      k_peer_scatter<<<nb, 256, 0, st>>>(N, pf.p, ps.p, D.d_lidx.p, dst, D.d_counts.p, 1 + mode * D.world + p);
    }
  std::vector<int64_t> cnt(2 * D.world + 1);
  DPB_CUDA(cudaMemcpyAsync(cnt.data(), D.d_counts.p, cnt.size() * 8, cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaStreamSynchronize(st));
  const int64_t nl = cnt[0];
  D.soff.assign(D.world + 1, 0);
  D.roff.assign(D.world + 1, 0);
  for (int p = 0; p < D.world; ++p) {
    D.soff[p + 1] = D.soff[p] + cnt[1 + p];
    D.roff[p + 1] = D.roff[p] + cnt[1 + D.world + p];
  }
  // pack the per-peer lists contiguously (device to device)
  for (int mode = 0; mode < 2; ++mode) {
    DevBuf<int32_t>& L = mode == 0 ? D.sidx : D.ridx;
    const std::vector<int64_t>& off = mode == 0 ? D.soff : D.roff;
    for (int p = 0; p < D.world; ++p) {
      const int64_t c = off[p + 1] - off[p];
      if (c && p > 0)
        DPB_CUDA(cudaMemcpyAsync(L.p + off[p], L.p + static_cast<size_t>(p) * N, c * sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, st));
    }
  }
  const size_t mx = std::max(D.soff[D.world], D.roff[D.world]) + 1;
  D.sbuf.ensure(3 * mx);
  D.rbuf.ensure(3 * mx);
  // local arrays (owned, then ghosts, each ascending in global id)
  D.d_lpos.ensure(3 * nl + 3);
  D.d_lvel.ensure(3 * nl + 3);
  D.d_ltypes.ensure(nl + 1);
  D.d_lcenter.ensure(nl + 1);
  k_local_arrays<<<ceil_div(nl, 256), 256, 0, st>>>(nl, D.rank, D.d_lgid.p, D.d_gpos.p, D.d_gvel.p, D.d_gtypes.p,
                                                    D.d_owner.p, D.d_lpos.p, D.d_lvel.p, D.d_ltypes.p, D.d_lcenter.p);
  lp.resize(3 * nl);
  lv.resize(3 * nl);
  lt.resize(nl);
  lc.resize(nl);
  DPB_CUDA(cudaMemcpyAsync(lp.data(), D.d_lpos.p, 3 * nl * 8, cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaMemcpyAsync(lv.data(), D.d_lvel.p, 3 * nl * 8, cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaMemcpyAsync(lt.data(), D.d_ltypes.p, nl * 4, cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaMemcpyAsync(lc.data(), D.d_lcenter.p, nl, cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaStreamSynchronize(st));
  D.lcenter.assign(lc.begin(), lc.end());
  D.n_own = 0;
  for (auto c : lc) D.n_own += c;
}

// Host plan of one rank: local atoms (owned, then ghosts, each ascending in global id), centre mask and the
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
  // owned atoms first, then the ghosts, each in ascending global id
  for (int64_t j = 0; j < D.N; ++j)
    if (owner[j] == r) {
      P.lgid.push_back(j);
      P.lcenter.push_back(1);
    }
  for (int64_t j = 0; j < D.N; ++j)
    if (owner[j] != r && is_ghost[j]) {
      P.lgid.push_back(j);
      P.lcenter.push_back(0);
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

// Slots of the pair-gradient halo (see Dist): send slots per ghost (ridx order) and receive
// slots per entry of the owned rows that have a ghost neighbour, with one read-back of the
// per-peer totals. Both sides count the same set -- the entries (j -> i) of j's row with i
// owned by the sender -- because every rank's rows equal the global rows.
void pair_plan(Engine& E) {
  Dist& D = *E.dist;
  cudaStream_t st = E.stream;
  const int W = D.world;
  const int64_t ng = D.roff[W], no = D.soff[W];
  D.d_gcnt.ensure(std::max(ng, no) + 2);
  D.gs_base.ensure(ng + 2);
  D.gr_base.ensure(no + 2);
  std::vector<int64_t> tot(2 * (W + 1), 0);
  // send side: ghosts in ridx order, per-peer segments are contiguous
  DPB_CUDA(cudaMemsetAsync(D.d_gcnt.p, 0, (ng + 1) * sizeof(int64_t), st));
  if (ng) k_ghost_slots<<<ceil_div(ng * 32, 256), 256, 0, st>>>(ng, D.ridx.p, E.row_off.p, E.keys.p, E.center.p,
                                                                D.d_gcnt.p);
  excl_scan(D, D.d_gcnt.p, D.gs_base.p, ng + 1, st);
  for (int p = 0; p <= W; ++p)
    DPB_CUDA(cudaMemcpyAsync(&tot[p], D.gs_base.p + D.roff[p], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  // receive side: owned atoms in sidx order (peer p's segment = p's ghosts owned here)
  DPB_CUDA(cudaMemsetAsync(D.d_gcnt.p, 0, (no + 1) * sizeof(int64_t), st));
  for (int p = 0; p < W; ++p) {
    const int64_t o = D.soff[p], c = D.soff[p + 1] - o;
    if (c) k_owned_slots<<<ceil_div(c * 32, 256), 256, 0, st>>>(c, D.sidx.p + o, p, E.row_off.p, E.keys.p, D.d_lgid.p,
                                                                D.d_owner.p, D.d_gcnt.p + o, nullptr, 0, nullptr);
  }
  excl_scan(D, D.d_gcnt.p, D.gr_base.p, no + 1, st);
  D.rslot.ensure(E.e_cap + 1);
  DPB_CUDA(cudaMemsetAsync(D.rslot.p, 0xff, (E.e_cap + 1) * sizeof(int32_t), st));
  for (int p = 0; p < W; ++p) {
    const int64_t o = D.soff[p], c = D.soff[p + 1] - o;
    if (c) k_owned_slots<<<ceil_div(c * 32, 256), 256, 0, st>>>(c, D.sidx.p + o, p, E.row_off.p, E.keys.p, D.d_lgid.p,
                                                                D.d_owner.p, nullptr, D.gr_base.p + o, 0, D.rslot.p);
  }
  for (int p = 0; p <= W; ++p)
    DPB_CUDA(cudaMemcpyAsync(&tot[W + 1 + p], D.gr_base.p + D.soff[p], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  DPB_CUDA(cudaStreamSynchronize(st));
  D.gsoff.assign(tot.begin(), tot.begin() + W + 1);
  D.groff.assign(tot.begin() + W + 1, tot.end());
  // interior / boundary owned atoms (local owned range [0, n_own))
  const int64_t no_ = E.n_centers;
  D.d_tflag.ensure(no_ + 1);
  D.d_tscan.ensure(no_ + 1);
  D.f_inner.ensure(no_ + 1);
  D.f_bound.ensure(no_ + 1);
  DPB_CUDA(cudaMemsetAsync(D.d_tflag.p + no_, 0, sizeof(int32_t), st));
  if (no_) k_touch_ghost<<<ceil_div(no_ * 32, 256), 256, 0, st>>>(no_, E.row_off.p, E.keys.p, E.center.p, D.d_tflag.p);
  excl_scan(D, D.d_tflag.p, D.d_tscan.p, no_ + 1, st);
  if (no_) k_split_atoms<<<ceil_div(no_, 256), 256, 0, st>>>(no_, D.d_tflag.p, D.d_tscan.p, D.f_inner.p, D.f_bound.p);
  int32_t nb = 0;
  DPB_CUDA(cudaMemcpyAsync(&nb, D.d_tscan.p + no_, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  D.gsend.ensure(3 * D.gsoff[W] + 3);
  D.grecv.ensure(3 * D.groff[W] + 3);
  DPB_CUDA(cudaStreamSynchronize(st));
  D.n_bound = nb;
  D.n_inner = no_ - nb;
  E.launches += 4 + 2 * W;
}

// Build the local system for this rank from the global state and upload it.
void build_local(Engine& E) {
  static const bool trace = std::getenv("DPB_TRACE") != nullptr;
  static const bool check = std::getenv("DPB_CHECK_PLAN") != nullptr;
  auto now = [&] {
    if (trace) cudaStreamSynchronize(E.stream);
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  Dist& D = *E.dist;
  std::vector<double> lp, lv;
  std::vector<int32_t> lt;
  std::vector<uint8_t> lc;
  device_plan(E, lp, lv, lt, lc);
  const int64_t nl = static_cast<int64_t>(lt.size());
  if (check) {
    // the host restatement of partition_domain must agree entry by entry
    if (!D.host_global_valid) {
      D.gpos.resize(3 * D.N);
      D.gvel.resize(3 * D.N);
      DPB_CUDA(cudaMemcpy(D.gpos.data(), D.d_gpos.p, 3 * D.N * 8, cudaMemcpyDeviceToHost));
      DPB_CUDA(cudaMemcpy(D.gvel.data(), D.d_gvel.p, 3 * D.N * 8, cudaMemcpyDeviceToHost));
      D.host_global_valid = true;
    }
    Plan P;
    make_plan(D, D.rank, P);
    std::vector<int32_t> s(D.soff[D.world]), rv(D.roff[D.world]);
    if (!s.empty()) DPB_CUDA(cudaMemcpy(s.data(), D.sidx.p, s.size() * 4, cudaMemcpyDeviceToHost));
    if (!rv.empty()) DPB_CUDA(cudaMemcpy(rv.data(), D.ridx.p, rv.size() * 4, cudaMemcpyDeviceToHost));
    if (P.lcenter != lc || P.soff != D.soff || P.roff != D.roff || P.s != s || P.rv != rv)
      throw CudaErr("device partition differs from the host restatement of partition_domain");
  }
  const auto t1 = now();
  E.set_config(nl, lp.data(), lt.data(), D.box, D.pbc, lc.data());
  const auto t2 = now();
  E.md_upload_atoms(lv.data());
  E.gid_of = D.d_lgid.p;  // rows in global-id order, pairs evaluated from the lower global id
  E.local_of = D.d_lidx.p;
  E.build_list(E.r_cut + E.md.buffer);
  E.classify_chunks();
  pair_plan(E);
  const auto t3 = now();
  if (trace) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[dpb rank %d] local: device plan %.2f, set_config %.2f, upload+list %.2f ms\n", D.rank,
                 ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
}

void exchange(Engine& E, const std::vector<int64_t>& out_off, const std::vector<int64_t>& in_off,
              cudaStream_t st) {
  Dist& D = *E.dist;
  DPB_NCCL(ncclGroupStart());
  for (int p = 0; p < D.world; ++p) {
    const int64_t so = out_off[p], sc = out_off[p + 1] - so;
    const int64_t ro = in_off[p], rc = in_off[p + 1] - ro;
    if (sc > 0) DPB_NCCL(ncclSend(D.sbuf.p + 3 * so, 3 * sc, ncclDouble, p, D.comm, st));
    if (rc > 0) DPB_NCCL(ncclRecv(D.rbuf.p + 3 * ro, 3 * rc, ncclDouble, p, D.comm, st));
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
  for (auto* b : {&E.dist->gs_base, &E.dist->gr_base, &E.dist->d_gcnt}) b->release();
  E.dist->rslot.release();
  E.dist->gsend.release();
  E.dist->grecv.release();
  Dist& D = *E.dist;
  for (auto* b : {&D.d_gpos, &D.d_gvel, &D.d_fw, &D.d_lohi, &D.d_lpos, &D.d_lvel}) b->release();
  for (auto* b : {&D.d_gtypes, &D.d_owner, &D.d_ids, &D.d_ids2, &D.d_flag, &D.d_scan, &D.d_lidx, &D.d_lgid,
                  &D.d_slot, &D.d_ltypes})
    b->release();
  D.d_keys.release();
  D.d_keys2.release();
  D.d_smask.release();
  D.d_lcenter.release();
  D.d_counts.release();
  D.d_tmp.release();
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
  D.d_gpos.ensure(3 * N);
  D.d_gvel.ensure(3 * N);
  D.d_gtypes.ensure(N);
  DPB_CUDA(cudaMemcpyAsync(D.d_gpos.p, pos, 3 * N * 8, cudaMemcpyHostToDevice, E.stream));
  DPB_CUDA(cudaMemcpyAsync(D.d_gvel.p, vel, 3 * N * 8, cudaMemcpyHostToDevice, E.stream));
  DPB_CUDA(cudaMemcpyAsync(D.d_gtypes.p, types, N * 4, cudaMemcpyHostToDevice, E.stream));
  D.host_global_valid = true;
  E.md = *cfg;
  build_local(E);
}

// Positions of my ghosts from their owners.
// Forward halo: owned positions -> the peers' ghosts. With overlap on, it runs on st_comm after
// the drift (ev_kd); the evaluation makes only the chunks with ghost neighbours (and the force
// kernel) wait for it (ev_halo). Every NCCL call on st_comm is ordered after the stream's
// earlier NCCL calls through the event it waits on, and the stream's later ones wait for
// ev_rx / ev_halo, so one communicator never has two operations in flight.
void dist_halo_forward(Engine& E) {
  Dist& D = *E.dist;
  const int64_t ns = D.soff[D.world], nr = D.roff[D.world];
  cudaStream_t st = E.stream;
  if (E.halo_overlap) {
    DPB_CUDA(cudaEventRecord(E.ev_kd, E.stream));
    DPB_CUDA(cudaStreamWaitEvent(E.st_comm, E.ev_kd, 0));
    st = E.st_comm;
  }
  if (ns) k_pack3<<<ceil_div(ns, 256), 256, 0, st>>>(ns, D.sidx.p, E.pos3.p, D.sbuf.p);
  exchange(E, D.soff, D.roff, st);
  if (nr) k_unpack_pos<<<ceil_div(nr, 256), 256, 0, st>>>(nr, D.ridx.p, D.rbuf.p, E.pos3.p, E.pos4.p);
  E.launches += 2;
  if (E.halo_overlap) {
    DPB_CUDA(cudaEventRecord(E.ev_halo, st));
    E.halo_pending = true;
  }
}

// Pair-gradient halo (every evaluation, before the force kernel): pack the reverse gradients of
// my ghosts' rows, exchange them with the peers (grouped send/recv, slot counts fixed at the
// rebuild), and hand the receive buffer and slot map to the force kernel.
// With overlap (default) the pack and the exchange run on the communication stream, ordered after
// the evaluation by ev_kd; ev_halo marks the received gradients. Returns the interior / boundary
// owned-atom lists for the split force launch.
void dist_exchange_g(Engine& E, const int32_t** rslot, const double** grecv, const int32_t** inner,
                     int64_t* n_inner, const int32_t** bound, int64_t* n_bound) {
  Dist& D = *E.dist;
  const int W = D.world;
  const int64_t ng = D.roff[W];
  cudaStream_t st = E.stream;
  if (E.halo_overlap) {
    DPB_CUDA(cudaEventRecord(E.ev_kd, E.stream));
    DPB_CUDA(cudaStreamWaitEvent(E.st_comm, E.ev_kd, 0));
    st = E.st_comm;
  }
  if (ng)
    k_pack_pair_g<<<ceil_div(ng * 32, 256), 256, 0, st>>>(ng, D.ridx.p, E.row_off.p, E.keys.p, E.rev.p, E.ridx.p,
                                                         E.realoff.p, E.center.p, E.g.p, D.gs_base.p, D.gsend.p);
  DPB_NCCL(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    const int64_t so = D.gsoff[p], sc = D.gsoff[p + 1] - so;
    const int64_t ro = D.groff[p], rc = D.groff[p + 1] - ro;
    if (sc > 0) DPB_NCCL(ncclSend(D.gsend.p + 3 * so, 3 * sc, ncclDouble, p, D.comm, st));
    if (rc > 0) DPB_NCCL(ncclRecv(D.grecv.p + 3 * ro, 3 * rc, ncclDouble, p, D.comm, st));
  }
  DPB_NCCL(ncclGroupEnd());
  if (E.halo_overlap) DPB_CUDA(cudaEventRecord(E.ev_halo, st));
  E.launches += 1;
  *rslot = D.rslot.p;
  *grecv = D.grecv.p;
  *inner = D.f_inner.p;
  *n_inner = D.n_inner;
  *bound = D.f_bound.p;
  *n_bound = D.n_bound;
}

// All-gather of the owned (id, x, v) into the global arrays on every rank (device resident).
static void gather_global(Engine& E) {
  Dist& D = *E.dist;
  const int64_t nl = E.n;
  D.d_slot.ensure(nl + 1);
  D.d_flag.ensure(nl + 1);
  // slot of each owned atom = its rank among the local centres (ascending global id)
  DevBuf<int32_t>& cflag = D.d_ids;
  cflag.ensure(nl + 1);
  k_u8_to_i32<<<ceil_div(nl, 256), 256, 0, E.stream>>>(nl, E.center.p, cflag.p);
  excl_scan(D, cflag.p, D.d_flag.p, nl, E.stream);
  k_slot_of_center<<<ceil_div(nl, 256), 256, 0, E.stream>>>(nl, E.center.p, D.d_flag.p, D.d_slot.p);
  D.gbuf_send.ensure(7 * D.max_own);
  D.gbuf_all.ensure(7 * D.max_own * D.world);
  DPB_CUDA(cudaMemsetAsync(D.gbuf_send.p, 0xff, 7 * D.max_own * sizeof(double), E.stream)); // NaN ids
  k_pack_state_d<<<ceil_div(nl, 256), 256, 0, E.stream>>>(nl, D.d_slot.p, D.d_lgid.p, E.pos3.p, E.vel3.p,
                                                          D.gbuf_send.p);
  DPB_NCCL(ncclAllGather(D.gbuf_send.p, D.gbuf_all.p, 7 * D.max_own, ncclDouble, D.comm, E.stream));
  const int64_t nrec = D.max_own * D.world;
  k_unpack_global<<<ceil_div(nrec, 256), 256, 0, E.stream>>>(nrec, D.gbuf_all.p, D.d_gpos.p, D.d_gvel.p);
  E.launches += 5;
  D.host_global_valid = false;
}

void Engine::classify_chunks() {
  if (!dist || n_chunks < 2) return;
  DevBuf<int64_t> cka;
  DevBuf<int> flag;
  cka.ensure(n_chunks + 1);
  flag.ensure(n_chunks);
  DPB_CUDA(cudaMemcpyAsync(cka.p, ck_a.data(), (n_chunks + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
  DPB_CUDA(cudaMemsetAsync(flag.p, 0, n_chunks * sizeof(int), stream));
  k_chunk_ghost<<<ceil_div(n, 256), 256, 0, stream>>>(n, n_chunks, cka.p, center.p, row_off.p, keys.p, flag.p);
  ++launches;
  std::vector<int> f(n_chunks);
  DPB_CUDA(cudaMemcpyAsync(f.data(), flag.p, n_chunks * sizeof(int), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  cka.release();
  flag.release();
  ck_order.clear();
  for (int k = 0; k < n_chunks; ++k) {
    ck_ghost[k] = f[k] ? 1 : 0;
    if (!f[k]) ck_order.push_back(k);
  }
  for (int k = 0; k < n_chunks; ++k)
    if (f[k]) ck_order.push_back(k);
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

void dist_agree_err(Engine& E) {
  DPB_NCCL(ncclAllReduce(E.err.p, E.err.p, 1, ncclInt32, ncclMax, E.dist->comm, E.stream));
}

void dist_md_end(Engine& E, double* gpos, double* gvel) {
  Dist& D = *E.dist;
  gather_global(E);
  if (gpos) DPB_CUDA(cudaMemcpyAsync(gpos, D.d_gpos.p, 3 * D.N * 8, cudaMemcpyDeviceToHost, E.stream));
  if (gvel) DPB_CUDA(cudaMemcpyAsync(gvel, D.d_gvel.p, 3 * D.N * 8, cudaMemcpyDeviceToHost, E.stream));
  DPB_CUDA(cudaStreamSynchronize(E.stream));
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
