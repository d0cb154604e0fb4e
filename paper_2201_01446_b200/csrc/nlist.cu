// nlist_build: bit-exact GPU neighbour list.
//
// Reference: build_neighbor_list neighbor.cpp:162-179, brute scan :63-84 with scan_images
// :23-48, linked cells :88-158, canonical sort :10-17. Both reference paths accept exactly the
// images (j, s) with |d|^2 <= cutoff^2 where d is evaluated ONCE per pair from the lower index
// (cells: q > i half walk; brute: i <= j) and mirrored with -s into the other row. This kernel
// reproduces that rule: every candidate pair is evaluated from min(i, j) with the reference's
// image range and un-fused arithmetic, so entries are bitwise identical whatever the binning.
// Rows are sorted by the packed key (type_j, j, shift) -- the stable type partition of the
// canonical order, which is the env-mat slot order (env_mat.cpp:25, 36-41).
#include <cub/cub.cuh>

#include "engine.hpp"

namespace dpb {

namespace {

struct NlParams {
  DevCell c;
  double cut2;
  double rc2; // model cutoff^2: the count pass also counts the entries inside it (g capacity)
  double margin[3];
  int nb[3];
  int full[3]; // 1: visit every bin along the axis (fewer than 3 bins), 0: 3-bin stencil
  int n;
};

__device__ __forceinline__ void frac_exact(const DevCell& c, double3 r, double* f) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    f[k] = __dadd_rn(__dadd_rn(__dmul_rn(r.x, c.hinv[k]), __dmul_rn(r.y, c.hinv[3 + k])),
                     __dmul_rn(r.z, c.hinv[6 + k]));
}

__global__ void k_frac_bin(NlParams p, const double4* __restrict__ pos, double* __restrict__ frac,
                           int* __restrict__ bin_of, int* __restrict__ bin_count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  double f[3];
  frac_exact(p.c, ld_pos(pos, i), f);
  int b[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    frac[3 * i + k] = f[k];
    if (p.c.per[k] && p.nb[k] > 1) {
      const double fl = floor(f[k]);
      int bk = static_cast<int>(__dmul_rn(__dsub_rn(f[k], fl), static_cast<double>(p.nb[k])));
      b[k] = min(max(bk, 0), p.nb[k] - 1);
    } else {
      b[k] = 0;
    }
  }
  const int bin = (b[0] * p.nb[1] + b[1]) * p.nb[2] + b[2];
  bin_of[i] = bin;
  atomicAdd(bin_count + bin, 1);
}

__global__ void k_bin_fill(int n, const int* __restrict__ bin_of, const int* __restrict__ bin_start,
                           int* __restrict__ bin_fill, int* __restrict__ bin_atoms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = bin_of[i];
  bin_atoms[bin_start[b] + atomicAdd(bin_fill + b, 1)] = i;
}

__device__ __forceinline__ int warp_excl_scan_nl(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Warp per centre (lanes over the candidates of each neighbouring bin): same acceptance rule,
// image range and arithmetic as the reference's scan (one evaluation per pair from min(i, j)). Row order before the sort is
// (bin, candidate, image) with lanes interleaved; rows are sorted afterwards, so the list is
// identical. WRITE=false counts, WRITE=true emits keys at warp-scanned positions.
template <bool WRITE>
__global__ void __launch_bounds__(256) k_nlist_warp(NlParams p, const double4* __restrict__ pos,
                                                    const double* __restrict__ frac, const int32_t* __restrict__ types,
                                                    const int* __restrict__ bin_of, const int* __restrict__ bin_start,
                                                    const int* __restrict__ bin_atoms, int64_t* __restrict__ row_len,
                                                    const int64_t* __restrict__ row_off, uint64_t* __restrict__ keys,
                                                    unsigned long long* __restrict__ n_inner, int* err, int64_t e_cap,
                                                    const int32_t* __restrict__ gid) {
  const int lane = threadIdx.x & 31;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= p.n) return;
  if (WRITE && row_off[i + 1] > e_cap) {
    if (lane == 0) raise_err(err, DEV_LIST_CAP);
    return;
  }
  const int bi = bin_of[i];
  const int bc[3] = {bi / (p.nb[1] * p.nb[2]), (bi / p.nb[2]) % p.nb[1], bi % p.nb[2]};
  int cnt[3], first[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (p.full[k]) {
      cnt[k] = p.nb[k];
      first[k] = 0;
    } else {
      cnt[k] = 3;
      first[k] = bc[k] - 1;
    }
  }
  const double3 ri = ld_pos(pos, i);
  const double fi[3] = {frac[3 * i], frac[3 * i + 1], frac[3 * i + 2]};
  int64_t count = 0;
  int inner = 0;
  const int64_t base = WRITE ? row_off[i] : 0;
  for (int o0 = 0; o0 < cnt[0]; ++o0) {
    const int q0 = (first[0] + o0 + p.nb[0]) % p.nb[0];
    for (int o1 = 0; o1 < cnt[1]; ++o1) {
      const int q1 = (first[1] + o1 + p.nb[1]) % p.nb[1];
      for (int o2 = 0; o2 < cnt[2]; ++o2) {
        const int q2 = (first[2] + o2 + p.nb[2]) % p.nb[2];
        const int q = (q0 * p.nb[1] + q1) * p.nb[2] + q2;
        const int qs = bin_start[q], qe = bin_start[q + 1];
        for (int idx0 = qs; idx0 < qe; idx0 += 32) {
          const int idx = idx0 + lane;
          int mine = 0;
          int j = 0, a = 0, b = 0, lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
          bool i_low = true;
          double3 ra, rb;
          if (idx < qe) {
            j = bin_atoms[idx];
            // every pair is evaluated once from its lower GLOBAL index (a decomposed run's
            // local order differs), so all ranks and one GPU accept exactly the same entries
            i_low = gid ? gid[i] <= gid[j] : i <= j;
            a = i_low ? i : j;
            b = i_low ? j : i;
            const double3 rj = ld_pos(pos, j);
            ra = i_low ? ri : rj;
            rb = i_low ? rj : ri;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              if (p.c.per[k]) {
                const double fa = i_low ? fi[k] : frac[3 * a + k];
                const double fb = i_low ? frac[3 * b + k] : fi[k];
                const double df = __dsub_rn(fb, fa);
                lo[k] = static_cast<int>(ceil(__dsub_rn(__dsub_rn(-df, p.margin[k]), 1e-12)));
                hi[k] = static_cast<int>(floor(__dadd_rn(__dadd_rn(-df, p.margin[k]), 1e-12)));
              } else {
                lo[k] = hi[k] = 0;
              }
            }
            for (int s0 = lo[0]; s0 <= hi[0]; ++s0)
              for (int s1 = lo[1]; s1 <= hi[1]; ++s1)
                for (int s2 = lo[2]; s2 <= hi[2]; ++s2) {
                  if (a == b && s0 == 0 && s1 == 0 && s2 == 0) continue;
                  double d[3];
                  disp_exact(p.c, ra, rb, s0, s1, s2, d);
                  const double r2 = norm2_exact(d);
                  if (r2 <= p.cut2) ++mine;
                  if (!WRITE && r2 < p.rc2) ++inner;
                }
          }
          int tot;
          const int ex = warp_excl_scan_nl(mine, lane, &tot);
          if (WRITE && mine) {
            int w = 0;
            for (int s0 = lo[0]; s0 <= hi[0]; ++s0)
              for (int s1 = lo[1]; s1 <= hi[1]; ++s1)
                for (int s2 = lo[2]; s2 <= hi[2]; ++s2) {
                  if (a == b && s0 == 0 && s1 == 0 && s2 == 0) continue;
                  double d[3];
                  disp_exact(p.c, ra, rb, s0, s1, s2, d);
                  if (norm2_exact(d) <= p.cut2) {
                    const int e0 = i_low ? s0 : -s0, e1 = i_low ? s1 : -s1, e2 = i_low ? s2 : -s2;
                    if (e0 < -511 || e0 > 511 || e1 < -511 || e1 > 511 || e2 < -511 || e2 > 511)
                      raise_err(err, DEV_SHIFT_RANGE);
                    const int64_t at = base + count + ex + w;
                    keys[at] = make_key(types[j], j, e0, e1, e2);
                    ++w;
                  }
                }
          }
          count += tot;
        }
      }
    }
  }
  if (!WRITE) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) inner += __shfl_xor_sync(0xffffffffu, inner, o);
    if (lane == 0) {
      row_len[i] = count;
      atomicAdd(n_inner, static_cast<unsigned long long>(inner));
    }
  }
}

// Rows of non-centre atoms (ghosts of a decomposed run) hold no real entry: ridx = -1 once per
// list build (the per-step kernels only visit the centres' rows). Warp per row.
__global__ void k_mark_ghost_rows(int n, const uint8_t* __restrict__ center, const int64_t* __restrict__ row_off,
                                  int16_t* __restrict__ ridx) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n || center[i]) return;
  for (int64_t e = row_off[i] + (threadIdx.x & 31); e < row_off[i + 1]; e += 32) ridx[e] = -1;
}

// Neighbour field of every key through a map (local index <-> global id of a decomposed run).
__global__ void k_keys_map(const int64_t* __restrict__ row_off, int n, uint64_t* __restrict__ keys,
                           const int32_t* __restrict__ map) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= row_off[n]) return;
  const uint64_t k = keys[e];
  keys[e] = with_key_j(k, map[key_j(k)]);
}

// Reverse entry of every list entry, warp per row: the position of (j -> i, -s) inside row j
// (rows are at most 8192 long, so 16 bits; the entry is row_off[j] + rev[e]). Decomposed runs
// sort their rows with global ids in the keys (gid/lidx map them), like one GPU does.
__global__ void k_reverse_rows(const int64_t* __restrict__ row_off, int n, const uint64_t* __restrict__ keys,
                               const int32_t* __restrict__ types, uint16_t* __restrict__ rev, int* err,
                               const int32_t* __restrict__ gid, const int32_t* __restrict__ lidx) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int ti = types[i];
  for (int64_t e = row_off[i] + (threadIdx.x & 31); e < row_off[i + 1]; e += 32) {
    const uint64_t k = keys[e];
    const int j = lidx ? lidx[key_j(k)] : key_j(k);
    const uint64_t want = reverse_key(k, ti, gid ? gid[i] : i);
    const int64_t r0 = row_off[j], r1 = row_off[j + 1];
    int64_t lo = r0, hi = r1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < want)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo >= r1 || keys[lo] != want) {
      raise_err(err, DEV_ASYMMETRIC); // the list is not symmetric (a supplied list can be)
      rev[e] = 0;
    } else {
      rev[e] = static_cast<uint16_t>(lo - r0);
    }
  }
}

// One block per row: bitonic sort of the row's keys in shared memory.
__global__ void k_sort_rows(int n, const int64_t* __restrict__ row_off, uint64_t* __restrict__ keys,
                            int cap, int* err) {
  extern __shared__ uint64_t sk[];
  const int i = blockIdx.x;
  if (i >= n) return;
  const int64_t off = row_off[i];
  const int len = static_cast<int>(row_off[i + 1] - off);
  if (len > cap) {
    if (threadIdx.x == 0) raise_err(err, DEV_ROW_CAP);
    return;
  }
  if (len < 2) return;
  int P = 2;
  while (P < len) P <<= 1;
  for (int t = threadIdx.x; t < P; t += blockDim.x) sk[t] = t < len ? keys[off + t] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = threadIdx.x; t < P; t += blockDim.x) {
        const int u = t ^ jj;
        if (u > t) {
          const uint64_t x = sk[t], y = sk[u];
          const bool up = (t & k) == 0;
          if ((x > y) == up) {
            sk[t] = y;
            sk[u] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < len; t += blockDim.x) keys[off + t] = sk[t];
}

__global__ void k_max_len(int n, const int64_t* __restrict__ row_len, int* out) {
  int m = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    m = max(m, static_cast<int>(row_len[i]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

double host_spacing(const DevCell& c, int k) {
  const double* u = c.h + 3 * ((k + 1) % 3);
  const double* v = c.h + 3 * ((k + 2) % 3);
  const double cr[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                        u[0] * v[1] - u[1] * v[0]};
  return c.vol / std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
}

} // namespace

void Engine::launch_nlist(double cutoff) {
  if (!(cutoff > 0.0)) throw InputErr("neighbor cutoff must be positive");
  if (n >= (1ll << 28)) throw InputErr("too many atoms for the packed neighbour key (2^28)");
  NlParams p;
  p.c = cell;
  p.cut2 = cutoff * cutoff;
  p.n = static_cast<int>(n);
  int64_t nbins = 1;
  for (int k = 0; k < 3; ++k) {
    p.margin[k] = cutoff / host_spacing(cell, k);
    int nb = 1;
    if (cell.per[k]) {
      const double want = std::floor(host_spacing(cell, k) / cutoff);
      nb = static_cast<int>(std::min(want, 1024.0));
      if (nb < 1) nb = 1;
    }
    p.nb[k] = nb;
    p.full[k] = nb < 3 ? 1 : 0;
    nbins *= nb;
  }
  const int N = p.n;
  frac.ensure(3 * n);
  bin_of.ensure(n);
  bin_atoms.ensure(n);
  bin_start.ensure(nbins + 1);
  bin_fill.ensure(nbins + 1);
  DevBuf<int64_t>& lens = nl_len;
  lens.ensure(n + 1);
  row_off.ensure(n + 1);
  row_len.ensure(1);
  DPB_CUDA(cudaMemsetAsync(bin_fill.p, 0, (nbins + 1) * sizeof(int), stream));
  k_frac_bin<<<ceil_div(N, 256), 256, 0, stream>>>(p, pos4.p, frac.p, bin_of.p, bin_fill.p);
  ++launches;
  // exclusive scan of bin counts -> bin_start
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, bin_fill.p, bin_start.p, nbins + 1, stream);
  DevBuf<unsigned char>& tmp = scan_tmp;
  tmp.ensure(tmp_bytes + 1);
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, bin_fill.p, bin_start.p, nbins + 1, stream);
  ++launches;
  DPB_CUDA(cudaMemsetAsync(bin_fill.p, 0, (nbins + 1) * sizeof(int), stream));
  k_bin_fill<<<ceil_div(N, 256), 256, 0, stream>>>(N, bin_of.p, bin_start.p, bin_fill.p, bin_atoms.p);
  ++launches;
  inner_cnt.ensure(1);
  DPB_CUDA(cudaMemsetAsync(inner_cnt.p, 0, sizeof(unsigned long long), stream));
  p.rc2 = r_cut * r_cut;
  k_nlist_warp<false><<<ceil_div(static_cast<int64_t>(N) * 32, 256), 256, 0, stream>>>(
      p, pos4.p, frac.p, types.p, bin_of.p, bin_start.p, bin_atoms.p, lens.p, nullptr, nullptr, inner_cnt.p, err.p, 0,
      gid_of);
  ++launches;
  DPB_CUDA(cudaMemsetAsync(lens.p + n, 0, sizeof(int64_t), stream));
  size_t tmp2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, lens.p, row_off.p, n + 1, stream);
  tmp.ensure(tmp2 + 1);
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp2, lens.p, row_off.p, n + 1, stream);
  ++launches;
  DPB_CUDA(cudaMemsetAsync(row_len.p, 0, sizeof(int), stream));
  k_max_len<<<std::min(ceil_div(N, 256), 1024), 256, 0, stream>>>(N, lens.p, row_len.p);
  ++launches;
  // Sizing: the total, the longest row and the number of entries inside r_cut are read back (one
  // sync per build; MD rebuilds every rebuild_every steps) and every per-entry buffer is sized
  // for this list, so no kernel can index past a capacity.
  int64_t total = 0;
  int mx = 0;
  unsigned long long inner = 0;
  DPB_CUDA(cudaMemcpyAsync(&total, row_off.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaMemcpyAsync(&mx, row_len.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaMemcpyAsync(&inner, inner_cnt.p, sizeof(inner), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  n_entries = total;
  max_row = mx;
  if (total + 1 > e_cap) e_cap = total + total / 16 + 1024;
  int rc = 2;
  while (rc < mx + mx / 8) rc <<= 1;
  if (rc > row_cap) row_cap = rc;
  // pair gradients are stored for real pairs only (compact, realoff[i] + rank): the pairs inside
  // r_cut at build time + 12.5 % for their drift until the next rebuild (checked on the device)
  set_gcap(static_cast<int64_t>(inner), static_cast<int64_t>(inner) + static_cast<int64_t>(inner / 8) + 4096);
  keys.ensure(e_cap + 1);
  k_nlist_warp<true><<<ceil_div(static_cast<int64_t>(N) * 32, 256), 256, 0, stream>>>(
      p, pos4.p, frac.p, types.p, bin_of.p, bin_start.p, bin_atoms.p, nullptr, row_off.p, keys.p, nullptr, err.p,
      e_cap, gid_of);
  ++launches;
  finish_list(cutoff);
}

// Grow only when the pairs inside r_cut at this build exceed the capacity (a rebuild in an MD
// run must not reallocate tens of GB for a 0.1 % change); shrink when far too large.
void Engine::set_gcap(int64_t need, int64_t want) {
  want = std::min<int64_t>(want, e_cap);
  if (need > g_cap || want < g_cap / 2) {
    g.release();
    g.ensure(3 * want + 3);
    g_cap = static_cast<int64_t>((g.n - 3) / 3); // the allocation's growth slack included
  }
}

// Rows are filled (keys, row_off, capacities): sort them into the type-sectored canonical
// order, index the reverse entries, mark ghost rows, snapshot the positions.
void Engine::finish_list(double cutoff) {
  const int N = static_cast<int>(n);
  const int cap = row_cap;
  if (cap > 8192) throw NumErr("neighbour row longer than 8192 entries");
  rev.ensure(e_cap + 1);
  ridx.ensure(e_cap + 1);
  // decomposed runs: rows sorted in global-id order (the single-GPU order), then back to local j
  const int64_t ne = n_entries > 0 ? n_entries : 1;
  if (gid_of) {
    k_keys_map<<<ceil_div(ne, 256), 256, 0, stream>>>(row_off.p, N, keys.p, gid_of);
    ++launches;
  }
  smem_optin(k_sort_rows, cap * sizeof(uint64_t));
  k_sort_rows<<<N, 256, cap * sizeof(uint64_t), stream>>>(N, row_off.p, keys.p, cap, err.p);
  ++launches;
  k_reverse_rows<<<ceil_div(static_cast<int64_t>(N) * 32, 256), 256, 0, stream>>>(row_off.p, N, keys.p, types.p,
                                                                                  rev.p, err.p, gid_of, local_of);
  ++launches;
  if (gid_of) {
    k_keys_map<<<ceil_div(ne, 256), 256, 0, stream>>>(row_off.p, N, keys.p, local_of);
    ++launches;
  }
  if (n_centers < n) {
    k_mark_ghost_rows<<<ceil_div(N, 8), 256, 0, stream>>>(N, center.p, row_off.p, ridx.p);
    ++launches;
  }
  ref_pos.ensure(3 * n);
  DPB_CUDA(cudaMemcpyAsync(ref_pos.p, pos3.p, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  list_cutoff = cutoff;
  list_valid = true;
  if (pbuf_cap > 0) grow_pbuf();
  if (plan_dirty) apply_plan();
  ensure_entry_step_buffers();
}

// A caller-supplied NeighborList (neighbor.hpp:18-23: full, symmetric, rows canonical or not),
// as compute_energy_forces_virial_tabulated takes it (fused.hpp:70-73). Validated on the host,
// packed into keys, then sorted and reverse-indexed on the device like a built list.
void Engine::import_list(const int64_t* off, const int32_t* jj, const int32_t* sh) {
  if (!off || !jj || !sh) throw InputErr("null neighbour list array");
  if (off[0] != 0) throw InputErr("neighbour list offsets must start at 0");
  int mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (off[i + 1] < off[i]) throw InputErr("neighbour list offsets must be non-decreasing");
    mx = std::max<int64_t>(mx, off[i + 1] - off[i]);
  }
  const int64_t total = off[n];
  std::vector<uint64_t> k(total + 1);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t e = off[i]; e < off[i + 1]; ++e) {
      const int j = jj[e];
      if (j < 0 || j >= n) throw InputErr("neighbour index out of range");
      for (int x = 0; x < 3; ++x)
        if (sh[3 * e + x] < -511 || sh[3 * e + x] > 511) throw InputErr("neighbour shift outside +-511 cells");
      k[e] = make_key(h_types[j], j, sh[3 * e], sh[3 * e + 1], sh[3 * e + 2]);
    }
  n_entries = total;
  max_row = mx;
  if (total + 1 > e_cap) e_cap = total + total / 8 + 1024;
  int rc = 2;
  while (rc < mx + mx / 8) rc <<= 1;
  row_cap = std::max(row_cap, rc);
  set_gcap(total + 1, total + 1);
  row_off.ensure(n + 1);
  keys.ensure(e_cap + 1);
  DPB_CUDA(cudaMemcpyAsync(row_off.p, off, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
  DPB_CUDA(cudaMemcpyAsync(keys.p, k.data(), total * sizeof(uint64_t), cudaMemcpyHostToDevice, stream));
  finish_list(0.0);
  DPB_CUDA(cudaStreamSynchronize(stream)); // host staging buffers go out of scope
}

void Engine::download_list(int64_t* offsets, int32_t* jout, int32_t* shift) {
  sync_entry_count();
  std::vector<int64_t> off(n + 1);
  std::vector<uint64_t> k(n_entries);
  DPB_CUDA(cudaMemcpyAsync(off.data(), row_off.p, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  if (n_entries)
    DPB_CUDA(cudaMemcpyAsync(k.data(), keys.p, n_entries * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  // Rows are stored type-sectored; the canonical order drops the type bits (neighbor.cpp:10-17).
  for (int64_t i = 0; i < n; ++i) {
    offsets[i] = off[i];
    std::vector<uint64_t> row(k.begin() + off[i], k.begin() + off[i + 1]);
    for (auto& x : row) x &= ~(63ull << 58);
    std::sort(row.begin(), row.end());
    for (size_t e = 0; e < row.size(); ++e) {
      jout[off[i] + e] = key_j(row[e]);
      key_shift(row[e], shift + 3 * (off[i] + e));
    }
  }
  offsets[n] = off[n];
}

void Engine::sync_entry_count() {
  if (n_entries >= 0) return;
  DPB_CUDA(cudaMemcpyAsync(&n_entries, row_off.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
}

} // namespace dpb
