// prod_force / prod_virial with scatter-free ownership, fixed-order reductions, and the
// device-resident velocity-Verlet pieces.
//
// Reference scatter (exact.cpp:22-38): for every centre i and real slot k with neighbour j,
//   F_i += g, F_j -= g, Xi[3x+y] += d_x g_y.
// Every list entry (i -> j, s) has its mirror (j -> i, -s) in row j (the list is symmetric,
// neighbor.cpp:76-79, :147-150). The pair gradient of the k-th real entry of row i (list order)
// is stored compactly at g[realoff[i] + k]; ridx[e] = k (or -1 when the env-mat filter dropped
// the entry), so each atom can GATHER its force without atomics:
//   F_i = sum_{real e in row i} g(e) - sum_{e in row i, rev(e) real} g(rev(e))
// in a fixed order.
#include "engine.hpp"

namespace dpb {

namespace {

// One warp per atom. The k-th own term of the row (list order, which filtering by cutoff
// preserves) and the k-th reverse term are always summed by lane k mod 32, so the result is
// bitwise independent of the list cutoff, as the reference's is (SURVEY.md §8.1 pitfall 1).
// VIR: also the per-centre virial sum_k d_k (x) g_k with d re-evaluated exactly as the env-mat
// did (exact path; the tabulated path forms it in k_tab_bwd_g from its records).
#ifndef FORCES_MINB
#define FORCES_MINB 3 // 3 CTAs (24 warps) per SM
#endif

template <bool VIR>
__device__ __forceinline__ void force_row(int64_t w, int n, DevCell c, const double4* __restrict__ pos,
                                                const int64_t* __restrict__ row_off,
                                                const uint64_t* __restrict__ keys,
                                                const uint16_t* __restrict__ rev,
                                                const int16_t* __restrict__ ridx,
                                                const int64_t* __restrict__ realoff,
                                                const double* __restrict__ g,
                                                double* __restrict__ f, double* __restrict__ vpart,
                                                const uint8_t* __restrict__ center,
                                                const int32_t* __restrict__ rslot,
                                                const double* __restrict__ grecv,
                                                const int32_t* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const int i = list ? list[w] : static_cast<int>(w); // list: a subset of the atoms (decomposed runs)
  if (!center[i]) return; // ghosts of a decomposed run: their owners compute their forces
  double3 ri;
  if (VIR) ri = ld_pos(pos, i);
  constexpr int NACC = VIR ? 15 : 6;
  double acc[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
  const int64_t e0 = row_off[i], e1 = row_off[i + 1];
  const double* gi = g + 3 * (center[i] ? realoff[i] : 0);
  int co = 0, cr = 0;
  // the next 32 entries' key / reverse position / own rank are loaded one iteration ahead
  uint64_t key_n = 0;
  int rv_n = 0, ko_n = -1;
  if (e0 + lane < e1) {
    key_n = keys[e0 + lane];
    rv_n = rev[e0 + lane];
    ko_n = ridx[e0 + lane];
  }
  for (int64_t base = e0; base < e1; base += 32) {
    const int64_t e = base + lane;
    const bool valid = e < e1;
    double go[3] = {0.0, 0.0, 0.0}, gr[3] = {0.0, 0.0, 0.0}, d[3] = {0.0, 0.0, 0.0};
    bool fo = false, fr = false;
    const uint64_t key = key_n;
    const int rv = rv_n, ko = ko_n;
    if (e + 32 < e1) {
      key_n = keys[e + 32];
      rv_n = rev[e + 32];
      ko_n = ridx[e + 32];
    }
    if (valid) {
      const int j = key_j(key);
      const int64_t m = row_off[j] + rv; // reverse entry (j -> i, -s)
      const int kr = ridx[m];
      fo = ko >= 0;
      fr = kr >= 0;
      if (fo) {
        go[0] = gi[3 * ko];
        go[1] = gi[3 * ko + 1];
        go[2] = gi[3 * ko + 2];
        if (VIR) {
          int sh[3];
          key_shift(key, sh);
          disp_exact(c, ri, ld_pos(pos, j), sh[0], sh[1], sh[2], d);
        }
      }
      if (fr) {
        const double* gj = g + 3 * (realoff[j] + kr);
        gr[0] = gj[0];
        gr[1] = gj[1];
        gr[2] = gj[2];
      }
      if (rslot && !center[j]) {
        // ghost neighbour: g(j -> i) was computed by j's owner and received in the pair halo
        // (NaN: that pair is not real from j's side)
        const double* gj = grecv + 3 * static_cast<int64_t>(rslot[e]);
        gr[0] = gj[0];
        gr[1] = gj[1];
        gr[2] = gj[2];
        fr = !isnan(gr[0]);
      }
    }
    const unsigned mo = __ballot_sync(0xffffffffu, fo);
    const unsigned mr = __ballot_sync(0xffffffffu, fr);
    {
      const int k = (lane - co) & 31;
      const bool take = k < __popc(mo);
      const int src = take ? static_cast<int>(__fns(mo, 0, k + 1)) : lane;
      double v[6];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        v[x] = __shfl_sync(0xffffffffu, go[x], src);
        if (VIR) v[3 + x] = __shfl_sync(0xffffffffu, d[x], src);
      }
      if (take) {
#pragma unroll
        for (int x = 0; x < 3; ++x) acc[x] += v[x];
        if (VIR)
#pragma unroll
          for (int x = 0; x < 3; ++x)
#pragma unroll
            for (int y = 0; y < 3; ++y) acc[(6 + 3 * x + y) % NACC] += v[3 + x] * v[y];
      }
    }
    {
      const int k = (lane - cr) & 31;
      const bool take = k < __popc(mr);
      const int src = take ? static_cast<int>(__fns(mr, 0, k + 1)) : lane;
      double v[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) v[x] = __shfl_sync(0xffffffffu, gr[x], src);
      if (take)
#pragma unroll
        for (int x = 0; x < 3; ++x) acc[3 + x] += v[x];
    }
    co += __popc(mo);
    cr += __popc(mr);
  }
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = warp_sum(acc[k]);
  if (lane == 0) {
#pragma unroll
    for (int x = 0; x < 3; ++x) f[3 * i + x] = acc[x] - acc[3 + x];
    if (VIR)
#pragma unroll
      for (int k = 0; k < 9; ++k) vpart[9 * static_cast<int64_t>(i) + k] = acc[(6 + k) % NACC];
  }
}

// persistent: one resident wave of CTAs, a warp per atom striding over the atoms
template <bool VIR>
__global__ void __launch_bounds__(256, FORCES_MINB) k_forces(int n, DevCell c, const double4* __restrict__ pos,
                                                const int64_t* __restrict__ row_off,
                                                const uint64_t* __restrict__ keys,
                                                const uint16_t* __restrict__ rev,
                                                const int16_t* __restrict__ ridx,
                                                const int64_t* __restrict__ realoff,
                                                const double* __restrict__ g,
                                                double* __restrict__ f, double* __restrict__ vpart,
                                                const uint8_t* __restrict__ center,
                                                const int32_t* __restrict__ rslot,
                                                const double* __restrict__ grecv,
                                                const int32_t* __restrict__ list) {
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t w = blockIdx.x * wpb + (threadIdx.x >> 5); w < n; w += gridDim.x * wpb)
    force_row<VIR>(w, n, c, pos, row_off, keys, rev, ridx, realoff, g, f, vpart, center, rslot, grecv, list);
}

// Deterministic two-level reduction of `width` interleaved columns over n rows.
constexpr int RED_BLOCKS = 256;
constexpr int RED_THREADS = 256;

__global__ void k_reduce_cols(int64_t n, int width, const double* __restrict__ x, int ld,
                              double* __restrict__ partial) {
  __shared__ double sh[RED_THREADS];
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * chunk;
  const int64_t hi = min(n, lo + chunk);
  for (int c = 0; c < width; ++c) {
    double s = 0.0;
    for (int64_t r = lo + threadIdx.x; r < hi; r += blockDim.x) s += x[r * ld + c];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x * width + c] = sh[0];
    __syncthreads();
  }
}

__global__ void k_reduce_final(int nb, int width, const double* __restrict__ partial,
                               double* __restrict__ out) {
  __shared__ double sh[RED_BLOCKS];
  for (int c = 0; c < width; ++c) {
    sh[threadIdx.x] = threadIdx.x < nb ? partial[threadIdx.x * width + c] : 0.0;
    __syncthreads();
    for (int o = blockDim.x >> 1; o > 0; o >>= 1) {
      if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = sh[0];
    __syncthreads();
  }
}

__global__ void k_pos4(int64_t n, const double* __restrict__ p3, double4* __restrict__ p4) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  p4[i] = make_double4(p3[3 * i], p3[3 * i + 1], p3[3 * i + 2], 0.0);
}

// First half kick and drift (md.cpp:205-208): v += (dt/2 F) acc, x += dt v.
__global__ void k_kick_drift(int64_t n, double half, double dt, const double* __restrict__ f,
                             const double* __restrict__ accf, double* __restrict__ v,
                             double* __restrict__ x, double4* __restrict__ p4,
                             const uint8_t* __restrict__ center) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !center[i]) return;
  double r[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double vv = __dadd_rn(v[3 * i + c], __dmul_rn(__dmul_rn(half, f[3 * i + c]), accf[i]));
    v[3 * i + c] = vv;
    r[c] = __dadd_rn(x[3 * i + c], __dmul_rn(dt, vv));
    x[3 * i + c] = r[c];
  }
  p4[i] = make_double4(r[0], r[1], r[2], 0.0);
}

// Second half kick (md.cpp:220-222).
__global__ void k_kick(int64_t n, double half, const double* __restrict__ f,
                       const double* __restrict__ accf, double* __restrict__ v,
                       const uint8_t* __restrict__ center) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n || !center[i]) return;
#pragma unroll
  for (int c = 0; c < 3; ++c)
    v[3 * i + c] = __dadd_rn(v[3 * i + c], __dmul_rn(__dmul_rn(half, f[3 * i + c]), accf[i]));
}

// max_i |x_i - x_i^ref|^2 (md.cpp:136-147) via integer max on the non-negative bit pattern.
__global__ void k_drift2(int64_t n, const double* __restrict__ x, const double* __restrict__ ref,
                         const uint8_t* __restrict__ center, unsigned long long* out) {
  unsigned long long best = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!center[i]) continue;
    double d2 = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double d = __dsub_rn(x[3 * i + c], ref[3 * i + c]);
      d2 = __dadd_rn(d2, __dmul_rn(d, d));
    }
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d2));
    best = b > best ? b : best;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
    best = t > best ? t : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// Staleness guard (md.cpp:211-217): drift = sqrt(max d2); track the maximum; flag if stale.
__global__ void k_stale_check(const unsigned long long* d2bits, double half_buffer,
                              double* max_seen, int* err) {
  const double drift = sqrt(__longlong_as_double(static_cast<long long>(*d2bits)));
  if (drift > *max_seen) *max_seen = drift;
  if (drift > half_buffer) raise_err(err, DEV_STALE);
}

// Kinetic energy per atom: 0.5 m v^2 MVV (md.cpp:172-178).
__global__ void k_ke_atoms(int64_t n, const double* __restrict__ v, const double* __restrict__ mass,
                           double mvv, const uint8_t* __restrict__ center, double* __restrict__ ke) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  if (!center[i]) {
    ke[i] = 0.0;
    return;
  }
  const double v2 = v[3 * i] * v[3 * i] + v[3 * i + 1] * v[3 * i + 1] + v[3 * i + 2] * v[3 * i + 2];
  ke[i] = 0.5 * mass[i] * v2 * mvv;
}

// Thermo record (md.cpp:179-189) from device reductions: red = [E, Xi(9)], ke_sum.
__global__ void k_thermo(int64_t step, int64_t n, double vol, const double* __restrict__ red,
                         const double* __restrict__ ke_sum, dp_thermo* out) {
  const double kB = 8.617333262e-5;
  const double bar = 1.602176634e6;
  dp_thermo t;
  t.step = step;
  t.ke = ke_sum[0];
  t.pe = red[0];
  t.temperature = 2.0 * t.ke / (3.0 * static_cast<double>(n) * kB);
  const double trv = red[1] + red[5] + red[9];
  t.pressure = (2.0 * t.ke + trv) / (3.0 * vol) * bar;
  *out = t;
}

__global__ void k_zero_ghost_vpart(int64_t n, const uint8_t* __restrict__ center, double* __restrict__ vpart) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n && !center[i])
#pragma unroll
    for (int k = 0; k < 9; ++k) vpart[9 * i + k] = 0.0;
}

} // namespace

// ghosts are no centres: no virial partial (the tabulated path writes the centres' in k_tab_bwd_g)
void Engine::zero_ghost_vpart() {
  k_zero_ghost_vpart<<<ceil_div(n, 256), 256, 0, stream>>>(n, center.p, vpart.p);
  ++launches;
}

void Engine::launch_forces() {
  const int N = static_cast<int>(n);
  forces.ensure(3 * n);
  // the exact path has no per-real records: its virial is formed here from the re-evaluated d
  auto kf = virial_in_forces ? k_forces<true> : k_forces<false>;
  int per_sm = 1;
  DPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, 256, 0));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t fmax = static_cast<int64_t>(sms > 0 ? sms : 148) * std::max(per_sm, 1);
  auto fgrid = [&](int64_t m) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 8), fmax))); };
  if (dist) {
    if (virial_in_forces) throw InputErr("the exact path is single-GPU");
    // pair halo in flight (communication stream) while the owned atoms without ghost neighbours
    // get their forces; the boundary atoms wait for the received gradients
    const int32_t *rslot = nullptr, *inner = nullptr, *bound = nullptr;
    const double* grecv = nullptr;
    int64_t ni = 0, nb = 0;
    dist_exchange_g(*this, &rslot, &grecv, &inner, &ni, &bound, &nb);
    if (ni)
      kf<<<fgrid(ni), 256, 0, stream>>>(static_cast<int>(ni), cell, pos4.p, row_off.p, keys.p, rev.p, ridx.p,
                                               realoff.p, g.p, forces.p, vpart.p, center.p, rslot, grecv, inner);
    if (halo_overlap) DPB_CUDA(cudaStreamWaitEvent(stream, ev_halo, 0));
    if (nb)
      kf<<<fgrid(nb), 256, 0, stream>>>(static_cast<int>(nb), cell, pos4.p, row_off.p, keys.p, rev.p, ridx.p,
                                               realoff.p, g.p, forces.p, vpart.p, center.p, rslot, grecv, bound);
    launches += 2;
  } else {
    kf<<<fgrid(N), 256, 0, stream>>>(N, cell, pos4.p, row_off.p, keys.p, rev.p, ridx.p, realoff.p, g.p,
                                            forces.p, vpart.p, center.p, nullptr, nullptr, nullptr);
    ++launches;
  }
  if (n_centers < n && !virial_in_forces) zero_ghost_vpart();
  // energy (1 column) then virial (9 columns) with fixed-order tree reductions
  red.ensure(RED_BLOCKS * 10 + 64);
  double* partial = red.p + 64;
  const int nb = static_cast<int>(std::min<int64_t>(RED_BLOCKS, std::max<int64_t>(1, n / 64)));
  k_reduce_cols<<<nb, RED_THREADS, 0, stream>>>(n, 1, e_atom.p, 1, partial);
  k_reduce_final<<<1, RED_BLOCKS, 0, stream>>>(nb, 1, partial, red.p);
  k_reduce_cols<<<nb, RED_THREADS, 0, stream>>>(n, 9, vpart.p, 9, partial);
  k_reduce_final<<<1, RED_BLOCKS, 0, stream>>>(nb, 9, partial, red.p + 1);
  launches += 4;
}

void launch_pos4(Engine& E) {
  k_pos4<<<ceil_div(E.n, 256), 256, 0, E.stream>>>(E.n, E.pos3.p, E.pos4.p);
  ++E.launches;
}

void launch_kick_drift(Engine& E, double half, double dt) {
  k_kick_drift<<<ceil_div(E.n, 256), 256, 0, E.stream>>>(E.n, half, dt, E.forces.p, E.acc_fac.p,
                                                         E.vel3.p, E.pos3.p, E.pos4.p, E.center.p);
  ++E.launches;
}

void launch_kick(Engine& E, double half) {
  k_kick<<<ceil_div(E.n, 256), 256, 0, E.stream>>>(E.n, half, E.forces.p, E.acc_fac.p, E.vel3.p,
                                                   E.center.p);
  ++E.launches;
}

// red layout: [0] E, [1..9] virial, [10] ke, [11] max drift seen, [12..13] drift bits scratch,
// [14..63] free; partials after 64.
void launch_stale_check(Engine& E, double half_buffer) {
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(E.red.p + 12);
  DPB_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), E.stream));
  const int blocks = std::max(1, std::min(ceil_div(E.n, 256), 1184));
  k_drift2<<<blocks, 256, 0, E.stream>>>(E.n, E.pos3.p, E.ref_pos.p, E.center.p, bits);
  k_stale_check<<<1, 1, 0, E.stream>>>(bits, half_buffer, E.red.p + 11, E.err.p);
  E.launches += 2;
}

double host_max_drift(Engine& E) {
  E.red.ensure(RED_BLOCKS * 10 + 64);
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(E.red.p + 12);
  DPB_CUDA(cudaMemsetAsync(bits, 0, sizeof(unsigned long long), E.stream));
  const int blocks = std::max(1, std::min(ceil_div(E.n, 256), 1184));
  k_drift2<<<blocks, 256, 0, E.stream>>>(E.n, E.pos3.p, E.ref_pos.p, E.center.p, bits);
  ++E.launches;
  unsigned long long h = 0;
  DPB_CUDA(cudaMemcpyAsync(&h, bits, sizeof(h), cudaMemcpyDeviceToHost, E.stream));
  DPB_CUDA(cudaStreamSynchronize(E.stream));
  double d2;
  std::memcpy(&d2, &h, sizeof(d2));
  return std::sqrt(d2);
}

void launch_thermo(Engine& E, int64_t step, dp_thermo* dst, double* mass_atom, double* ke_scratch) {
  k_ke_atoms<<<ceil_div(E.n, 256), 256, 0, E.stream>>>(E.n, E.vel3.p, mass_atom, units::MVV_TO_EV,
                                                       E.center.p, ke_scratch);
  double* partial = E.red.p + 64;
  const int nb = static_cast<int>(std::min<int64_t>(RED_BLOCKS, std::max<int64_t>(1, E.n / 64)));
  k_reduce_cols<<<nb, RED_THREADS, 0, E.stream>>>(E.n, 1, ke_scratch, 1, partial);
  k_reduce_final<<<1, RED_BLOCKS, 0, E.stream>>>(nb, 1, partial, E.red.p + 10);
  E.launches += 3;
  const int64_t n_total = E.dist ? dist_n_total(E) : E.n;
  if (E.dist) {
    // energy, virial and kinetic energy summed over ranks (in scratch, red[0..10] stays local)
    DPB_CUDA(cudaMemcpyAsync(E.red.p + 32, E.red.p, 11 * sizeof(double), cudaMemcpyDeviceToDevice, E.stream));
    dist_allreduce_sum(E, E.red.p + 32, 11);
    k_thermo<<<1, 1, 0, E.stream>>>(step, n_total, E.cell.vol, E.red.p + 32, E.red.p + 42, dst);
  } else {
    k_thermo<<<1, 1, 0, E.stream>>>(step, n_total, E.cell.vol, E.red.p, E.red.p + 10, dst);
  }
  ++E.launches;
}

} // namespace dpb
