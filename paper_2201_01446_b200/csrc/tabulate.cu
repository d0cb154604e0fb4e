// prod_env_mat + tabulate_fusion, forward and backward.
//
// Reference, per centre (fused.cpp:182-243):
//   env-mat       env_mat.cpp:10-74  d, r^2 < r_c^2 filter, s = w(r)/r, R = (s, s d/r), dR/dd
//   forward       fused.cpp:13-37    T[a][p] += R[a] * G_p(s) over real slots, G = quintic table
//   descriptor    contract.hpp:9-17  D[q][p] = sum_a T[a][q] T[a][p], q < m_lt
//   adjoint       contract.hpp:21-38 dT from dD
//   gradient pass fused.cpp:203-242  drow[a] = dT[a].G, ds = sum_p (sum_a R[a] dT[a][p]) G'_p,
//                                    g = sum_a drow[a] dR[a]/dd  (= dE_i/dd_ij)
//
// B200 formulation: the table is piecewise polynomial, G_p(s) = sum_m C[t][th][m][p]
// u^m with u = s - node(th). Grouping a centre's real neighbours by (type, interval) turns both
// passes into small dense contractions against the coefficient block of each touched interval:
//   forward   T[a][p] = sum_groups sum_m W[a][m] C[m][p],   W[a][m] = sum_{k in group} R_k[a] u_k^m
//   backward  P[a][m] = sum_p dT[a][p] C[m][p] per group,  then per neighbour
//             drow[a] = sum_m u^m P[a][m],  H'[a] = sum_m m u^(m-1) P[a][m],  ds = sum_a R[a] H'[a]
// so the embedding matrix G is never formed (not even one row at a time), and each touched
// coefficient block (6 x M doubles) is read once per centre instead of once per neighbour.
//
// Kernels (per evaluation):
//   k_env_fwd    one thread per list entry: env-mat, real filter, interval, (R, u)   [parallel]
//   k_tab_fwd    one warp per centre: stable counting sort of reals by (type, interval),
//                group moments, T = W . C, D = T<^T T
//   k_tab_bwd_P  one warp per centre: dT from dD, interval projections P per group
//   k_tab_bwd_g  one thread per list entry: dE_i/dd_ij from P, written at the entry   [parallel]
// All reductions have a fixed order, so results are bitwise reproducible run to run.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "tab_common.cuh"
#include "tc_common.cuh"

namespace dpb {

namespace {

// ---------------------------------------------------------------- k_env_fwd (thread per entry)
__global__ void __launch_bounds__(256) k_env_fwd(TabParams p) {
  // entries of the centre range [i0, i1); chunk-local arrays at el = e - row_off[i0]
  const int64_t eb = p.row_off[p.i0];
  const int64_t el = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t e = eb + el;
  bool ext = false;
  const bool in_range = e < p.E && e < p.row_off[p.i1];
  if (in_range && el >= p.es) raise_err(p.err, DEV_LIST_CAP); // chunk entry capacity (never expected)
  const bool live = in_range && el < p.es;
  // owner and key loaded together (independent), then the centre flag and the positions
  const int i = live ? p.eown[e] : 0;
  const uint64_t key = live ? p.keys[e] : 0;
  const bool cen = live && p.center[i];
  if (live && !cen) p.ebin[e] = -1;
  if (cen) {
    int sh[3];
    key_shift(key, sh);
    double d[3];
    disp_exact(p.c, ld_pos(p.pos, i), ld_pos(p.pos, key_j(key)), sh[0], sh[1], sh[2], d);
    const double r2 = norm2_exact(d);
    int bin = -1;
    if (r2 < 1e-12) {
      raise_err(p.err, DEV_OVERLAP); // env_mat.cpp:33 throws before any table lookup
    } else if (r2 < p.rc2 && p.tn == 0) {
      // exact path: no table; the real entry is tagged with its neighbour type
      const double r = sqrt(r2);
      const double ir = 1.0 / r;
      const double s = switch_fn(r, p.rs, p.rc) * ir;
      bin = key_type(key);
      p.erc[el] = s;
      p.erc[p.es + el] = s * (d[0] * ir);
      p.erc[2 * p.es + el] = s * (d[1] * ir);
      p.erc[3 * p.es + el] = s * (d[2] * ir);
    } else if (r2 < p.rc2) {
      const double r = sqrt(r2);
      const double ir = 1.0 / r;
      const double s = switch_fn(r, p.rs, p.rc) * ir;
      const int th = locate(p, s, ext, p.err);
      bin = key_type(key) * p.tn + th;
      p.erc[el] = s;
      p.erc[p.es + el] = s * (d[0] * ir);
      p.erc[2 * p.es + el] = s * (d[1] * ir);
      p.erc[3 * p.es + el] = s * (d[2] * ir);
      p.erc[4 * p.es + el] = s - node_x(p.x0, p.h, th);
    }
    p.ebin[e] = bin;
  }
  const unsigned m = __ballot_sync(0xffffffffu, ext);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(p.counters + 2, static_cast<unsigned long long>(__popc(m)));
}

// ---------------------------------------------------------------- per-warp shared memory
constexpr int HCAP = 256; // counting-sort bins; wider (type, interval) ranges use a bitonic sort
constexpr int GB = 8;     // groups per batch
#ifndef TAB_FWD_MINB
#define TAB_FWD_MINB 8 // 2-warp CTAs per SM: 128 registers, 16 warps per SM
#endif
#ifndef TAB_EBIN_PREFETCH
#define TAB_EBIN_PREFETCH 1
#endif
#ifndef TAB_L2_PREFETCH
#define TAB_L2_PREFETCH 0 // bulk L2 prefetch of the next centre's rows: measured 0.03 ms/step slower
#endif
#ifndef TAB_MOMENT_PAIR
#define TAB_MOMENT_PAIR 1 // members per lane iteration of the moment sums (2: two gathers in flight, measured neutral)
#endif

struct FwdSmem {
  uint32_t* rk; // [scap] bin of real k (list order)
  uint16_t* ex; // [scap] entry of real k
  uint16_t* rn; // [scap] stable rank of real k inside its bin
  uint16_t* od; // [scap] sorted position -> k
  int* hs;      // [HCAP + 1] bin counts -> bin starts
  int* gs;      // [gcap + 1] group start (sorted position)
  int* gb;      // [gcap] group bin
  int* tc;      // [64] per-type real counts
  double* W;    // [GB][24] moments of one batch
  double* ts;   // [4][Mp] copy of T (aliases rk/rn/hs after the sort)
};

__host__ __device__ __forceinline__ size_t align16(size_t b) { return (b + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ int gcap_of(int scap) { return scap > HCAP ? scap : HCAP; }

__host__ __device__ __forceinline__ size_t fwd_front_bytes(int scap, int Mp) {
  const size_t front = static_cast<size_t>(scap) * (4 + 2) + (HCAP + 1) * 4;
  const size_t tsb = static_cast<size_t>(4) * Mp * 8;
  return align16(front > tsb ? front : tsb);
}

__host__ __device__ __forceinline__ size_t fwd_smem_bytes(int scap, int Mp) {
  return align16(fwd_front_bytes(scap, Mp) + GB * 24 * 8 + static_cast<size_t>(scap) * 4 +
                 static_cast<size_t>(2 * gcap_of(scap) + 1) * 4 + 64 * 4);
}

__device__ __forceinline__ FwdSmem carve_fwd(unsigned char* base, int scap, int Mp) {
  FwdSmem w;
  w.ts = reinterpret_cast<double*>(base);
  w.rk = reinterpret_cast<uint32_t*>(base);
  w.hs = reinterpret_cast<int*>(base + static_cast<size_t>(scap) * 4);
  w.rn = reinterpret_cast<uint16_t*>(base + static_cast<size_t>(scap) * 4 + (HCAP + 1) * 4);
  unsigned char* q = base + fwd_front_bytes(scap, Mp);
  w.W = reinterpret_cast<double*>(q);
  q += GB * 24 * 8;
  w.gs = reinterpret_cast<int*>(q);
  q += (gcap_of(scap) + 1) * 4;
  w.gb = reinterpret_cast<int*>(q);
  q += gcap_of(scap) * 4;
  w.tc = reinterpret_cast<int*>(q);
  q += 64 * 4;
  w.od = reinterpret_cast<uint16_t*>(q);
  q += static_cast<size_t>(scap) * 2;
  w.ex = reinterpret_cast<uint16_t*>(q);
  return w;
}

// Global-memory warp sort of a[0..n) ascending (fallback for wide bin ranges; rare). Bitonic
// network in its all-ascending form (mirror stage + half cleaners), so the implicit +inf padding
// up to the next power of two never moves and its comparisons can simply be skipped.
__device__ void warp_sort_global(uint64_t* a, int n, int lane) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int t = lane; t < P; t += 32) {
      const int u = t ^ (k - 1);
      if (u > t && u < n) {
        const uint64_t x = a[t], y = a[u];
        if (x > y) {
          a[t] = y;
          a[u] = x;
        }
      }
    }
    __syncwarp();
    for (int j = k >> 2; j > 0; j >>= 1) {
      for (int t = lane; t < P; t += 32) {
        const int u = t ^ j;
        if (u > t && u < n) {
          const uint64_t x = a[t], y = a[u];
          if (x > y) {
            a[t] = y;
            a[u] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Stable sort of the reals by bin: od[j] = real index at sorted position j, plus the group
// table (gs, gb). Counting sort over [kmin, kmax] when it fits HCAP bins, else bitonic.
__device__ int sort_and_group(const FwdSmem& w, uint64_t* scratch, int nreal, int kmin, int kmax,
                              int lane) {
  if (nreal == 0) return 0;
  const int range = kmax - kmin + 1;
  int G = 0;
  if (range <= HCAP) {
    for (int b = lane; b <= range; b += 32) w.hs[b] = 0;
    __syncwarp();
    for (int base = 0; base < nreal; base += 32) {
      const int k = base + lane;
      const bool act = k < nreal;
      const unsigned b = act ? w.rk[k] - kmin : 0xffffffffu;
      const unsigned mm = __match_any_sync(0xffffffffu, b);
      const int below = __popc(mm & ((1u << lane) - 1u));
      const int cnt = act ? w.hs[b] : 0;
      __syncwarp();
      if (act) {
        w.rn[k] = static_cast<uint16_t>(cnt + below);
        if (below == 0) w.hs[b] = cnt + __popc(mm);
      }
      __syncwarp();
    }
    const int seg = (range + 31) / 32;
    const int b0 = min(lane * seg, range), b1 = min(b0 + seg, range);
    int sum = 0, ne = 0;
    for (int b = b0; b < b1; ++b) {
      sum += w.hs[b];
      ne += w.hs[b] > 0;
    }
    int tot, gtot;
    int run = warp_excl_scan(sum, lane, &tot);
    int gr = warp_excl_scan(ne, lane, &gtot);
    __syncwarp();
    for (int b = b0; b < b1; ++b) {
      const int c = w.hs[b];
      if (c > 0) {
        w.gs[gr] = run;
        w.gb[gr] = b + kmin;
        ++gr;
      }
      w.hs[b] = run;
      run += c;
    }
    G = gtot;
    if (lane == 0) w.gs[G] = nreal;
    __syncwarp();
    for (int k = lane; k < nreal; k += 32) w.od[w.hs[w.rk[k] - kmin] + w.rn[k]] = static_cast<uint16_t>(k);
  } else {
    for (int k = lane; k < nreal; k += 32) scratch[k] = (static_cast<uint64_t>(w.rk[k]) << 32) | k;
    __syncwarp();
    warp_sort_global(scratch, nreal, lane);
    for (int base = 0; base < nreal; base += 32) {
      const int j = base + lane;
      bool head = false;
      uint64_t v = 0;
      if (j < nreal) {
        v = scratch[j];
        head = (j == 0) || ((v >> 32) != (scratch[j - 1] >> 32));
      }
      const unsigned m = __ballot_sync(0xffffffffu, head);
      if (head) {
        const int at = G + __popc(m & ((1u << lane) - 1u));
        w.gs[at] = j;
        w.gb[at] = static_cast<int>(v >> 32);
      }
      G += __popc(m);
      if (j < nreal) w.od[j] = static_cast<uint16_t>(v & 0xffffffffu);
    }
    if (lane == 0) w.gs[G] = nreal;
  }
  __syncwarp();
  return G;
}

// ---------------------------------------------------------------- k_tab_fwd (warp per centre)
// Features are owned in contiguous runs: lane l holds f = F*l .. F*l + F-1.
// F32 (mixed mode, SURVEY §8d C3 "mixed-precision tabulate_fusion"): the contraction T += W . C
// runs on FP32 coefficients and accumulators (half the coefficient traffic, 2x the FP64 rate);
// the moments W stay FP64. FP64 mode (F32 = false) is the parity path.
// WM (FP64 W-mode): the kernel stops after the sort and the group moments, which it
// writes to Pbuf[wbase[i] + g][a][m] (groups allocated per centre from p.wcnt); k_tab_fwd_T2 then
// contracts them with the coefficients on the FP64 tensor pipe and forms T and D. p.count_only:
// n_grp only (first evaluation of a system, to size Pbuf).
template <int F, bool F32 = false, bool WM = false>
__global__ void __launch_bounds__(64, TAB_FWD_MINB) k_tab_fwd(TabParams p) {
  using acc_t = typename std::conditional<F32, float, double>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const FwdSmem w = carve_fwd(smem + wid * fwd_smem_bytes(p.scap, p.Mp), p.scap, p.Mp);
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  const int f0 = F * lane;
  const int64_t eb = p.row_off[p.i0];
  for (int i = p.i0 + blockIdx.x * wpb + wid; i < p.i1; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int64_t loff = off - eb; // chunk-local entry offset
    const int len = static_cast<int>(p.row_off[i + 1] - off);
#if TAB_L2_PREFETCH
    {
      // the warp's next centre: its bins (lane 0) and the five (R, u) slices (lanes 1-5)
      const int in = i + gridDim.x * wpb;
      if (in < p.i1 && lane < 6) {
        const int64_t o2 = p.row_off[in];
        const int64_t l2 = p.row_off[in + 1] - o2;
        if (lane == 0) l2_prefetch(p.ebin + o2, static_cast<size_t>(l2) * 4);
        else l2_prefetch(p.erc + static_cast<size_t>(lane - 1) * p.es + (o2 - eb), static_cast<size_t>(l2) * 8);
      }
    }
#endif
    for (int t = lane; t < 64; t += 32) w.tc[t] = 0;
    __syncwarp();
    // --- compaction of the reals (list order), per-type counts ---
    int nreal = 0, kmin = 0x7fffffff, kmax = -1;
#if TAB_EBIN_PREFETCH
    int bin_nx = lane < len ? p.ebin[off + lane] : -1; // next 32 bins in flight
#endif
    for (int base = 0; base < len; base += 32) {
      const int e = base + lane;
#if TAB_EBIN_PREFETCH
      const int bin = bin_nx;
      if (base + 32 < len) bin_nx = e + 32 < len ? p.ebin[off + e + 32] : -1;
#else
      const int bin = e < len ? p.ebin[off + e] : -1;
#endif
      const bool real = bin >= 0;
      const unsigned m = __ballot_sync(0xffffffffu, real);
      const int t = real ? bin / p.tn : -1;
      if (real) {
        const int at = nreal + __popc(m & ((1u << lane) - 1u));
        w.rk[at] = static_cast<uint32_t>(bin);
        w.ex[at] = static_cast<uint16_t>(e);
        kmin = min(kmin, bin);
        kmax = max(kmax, bin);
      }
      const unsigned tm = __match_any_sync(0xffffffffu, t);
      if (real && (tm & ((1u << lane) - 1u)) == 0) w.tc[t] += __popc(tm);
      nreal += __popc(m);
      __syncwarp();
    }
    kmin = warp_min(kmin);
    kmax = warp_max(kmax);
    for (int t = lane; t < p.n_types; t += 32)
      if (w.tc[t] > p.max_nbr[t]) raise_err(p.err, DEV_OVERFLOW);
    const int G = sort_and_group(w, p.skeys + loff, nreal, kmin, kmax, lane);
    if (lane == 0) {
      if (!WM || !p.count_only) atomicAdd(p.counters + 0, static_cast<unsigned long long>(nreal));
      p.n_real[i] = nreal;
      p.n_grp[i] = G;
    }
    int64_t wb = -1;
    if constexpr (WM) {
      if (p.count_only) {
        __syncwarp();
        continue;
      }
      if (lane == 0) {
        const int64_t b = static_cast<int64_t>(atomicAdd(p.wcnt, static_cast<unsigned long long>(G)));
        if (b + G > p.pcap) raise_err(p.err, DEV_PBUF);
        else wb = b;
        p.wbase[i] = wb;
      }
      wb = __shfl_sync(0xffffffffu, wb, 0);
    }
    for (int j = lane; j < nreal; j += 32) {
      const int k = w.od[j];
      p.skeys[loff + j] = (static_cast<uint64_t>(w.rk[k]) << 32) | w.ex[k];
    }
    for (int g = lane; g < G; g += 32) {
      p.gbin[loff + g] = w.gb[g];
      for (int j = w.gs[g]; j < w.gs[g + 1]; ++j) p.egrp[loff + w.ex[w.od[j]]] = g;
    }
    if constexpr (WM) {
      if (wb < 0) {
        __syncwarp();
        continue;
      }
    }
    // --- moments of each (type, interval) group, then T += W . C[interval] ---
    acc_t tacc[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) tacc[a][q] = acc_t(0);
    // coefficient rows of one group (a register prefetch of the next group was measured: it
    // raised the kernel to 168 registers, 12 instead of 16 warps per SM, and ran 3 % slower)
    auto load_c = [&](int gidx, acc_t (&cn)[6][F]) {
      if constexpr (F32) {
        const float* C = p.tab32 + static_cast<size_t>(w.gb[gidx]) * istride + f0;
#pragma unroll
        for (int mm = 0; mm < 6; ++mm) {
          if constexpr (F % 4 == 0) {
#pragma unroll
            for (int q = 0; q < F; q += 4) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(C + mm * p.Mp + q));
              cn[mm][q] = v.x;
              cn[mm][q + 1] = v.y;
              cn[mm][q + 2] = v.z;
              cn[mm][q + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int q = 0; q < F; ++q) cn[mm][q] = __ldg(C + mm * p.Mp + q);
          }
        }
        return;
      }
      const double* C = reinterpret_cast<const double*>(p.tab) + static_cast<size_t>(w.gb[gidx]) * istride + f0;
#pragma unroll
      for (int mm = 0; mm < 6; ++mm) {
        if constexpr (F % 2 == 0) {
#pragma unroll
          for (int q = 0; q < F; q += 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(C + mm * p.Mp + q));
            cn[mm][q] = static_cast<acc_t>(v.x);
            cn[mm][q + 1] = static_cast<acc_t>(v.y);
          }
        } else {
#pragma unroll
          for (int q = 0; q < F; ++q) cn[mm][q] = static_cast<acc_t>(__ldg(C + mm * p.Mp + q));
        }
      }
    };
    for (int g0 = 0; g0 < G; g0 += GB) {
      {
        // 4 lanes per group split its members; reduce-scatter leaves lane r with W[a = r][0..5]
        const int gl = lane >> 2, r = lane & 3;
        const int g = g0 + gl;
        double Wv[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) Wv[k] = 0.0;
        if (g < G) {
          const int j1 = w.gs[g + 1];
          // members j, j + 4 of this lane loaded together (two gathers in flight), accumulated in
          // member order
          for (int j = w.gs[g] + r; j < j1; j += 4 * TAB_MOMENT_PAIR) {
            const bool two = TAB_MOMENT_PAIR == 2 && j + 4 < j1;
            const int64_t e = loff + w.ex[w.od[j]];
            const int64_t e2 = two ? loff + w.ex[w.od[j + 4]] : e;
            const double R[4] = {p.erc[e], p.erc[p.es + e], p.erc[2 * p.es + e], p.erc[3 * p.es + e]};
            const double uu = p.erc[4 * p.es + e];
            const double R2[4] = {p.erc[e2], p.erc[p.es + e2], p.erc[2 * p.es + e2], p.erc[3 * p.es + e2]};
            const double uu2 = p.erc[4 * p.es + e2];
            double um = 1.0;
#pragma unroll
            for (int mm = 0; mm < 6; ++mm) {
#pragma unroll
              for (int a = 0; a < 4; ++a) Wv[a * 6 + mm] += R[a] * um;
              um *= uu;
            }
            if (two) {
              um = 1.0;
#pragma unroll
              for (int mm = 0; mm < 6; ++mm) {
#pragma unroll
                for (int a = 0; a < 4; ++a) Wv[a * 6 + mm] += R2[a] * um;
                um *= uu2;
              }
            }
          }
        }
        {
          const bool hi = lane & 2;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            const double send = hi ? Wv[k] : Wv[k + 12];
            const double keep = hi ? Wv[k + 12] : Wv[k];
            Wv[k] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
          }
        }
        {
          const bool hi = lane & 1;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const double send = hi ? Wv[k] : Wv[k + 6];
            const double keep = hi ? Wv[k + 6] : Wv[k];
            Wv[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
          }
        }
        if constexpr (WM) {
          if (g < G) {
            double* Wg = p.Pbuf + (wb + g) * 24 + r * 6;
#pragma unroll
            for (int mm = 0; mm < 6; mm += 2) *reinterpret_cast<double2*>(Wg + mm) = make_double2(Wv[mm], Wv[mm + 1]);
          }
          continue;
        }
        if (g < G)
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) w.W[gl * 24 + r * 6 + mm] = Wv[mm];
      }
      __syncwarp();
      const int gn = min(GB, G - g0);
      for (int gg = 0; gg < gn; ++gg) {
        const double* Wg = w.W + gg * 24;
        acc_t c[6][F];
        load_c(g0 + gg, c);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) {
            const acc_t wa = static_cast<acc_t>(Wg[a * 6 + mm]);
#pragma unroll
            for (int q = 0; q < F; ++q) tacc[a][q] += wa * c[mm][q];
          }
        }
      }
      __syncwarp();
    }
    if constexpr (WM) {
      __syncwarp();
      continue;
    }
    // --- T out, D = T<^T T (contract.hpp:9-17) ---
    double* ts = w.ts;
    double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) {
        Ti[a * p.Mp + f0 + q] = tacc[a][q];
        ts[a * p.Mp + f0 + q] = tacc[a][q];
      }
    __syncwarp();
    const int slot = p.slot_of[i];
    double* Drow = p.D + static_cast<size_t>(slot < 0 ? 0 : slot) * p.K0p;
    if (slot >= 0 && f0 < p.M) {
      for (int qq = 0; qq < p.mlt; ++qq) {
        const double t0 = ts[qq], t1 = ts[p.Mp + qq], t2 = ts[2 * p.Mp + qq], t3 = ts[3 * p.Mp + qq];
        double dv[F];
#pragma unroll
        for (int q = 0; q < F; ++q) {
          double acc = t0 * tacc[0][q];
          acc += t1 * tacc[1][q];
          acc += t2 * tacc[2][q];
          acc += t3 * tacc[3][q];
          dv[q] = acc;
        }
        if (p.D2) {
          float* d2 = p.D2 + static_cast<size_t>(slot) * 2 * p.K0p + qq * p.M + f0;
#pragma unroll
          for (int q = 0; q < F; ++q) {
            const float x = static_cast<float>(dv[q]);
            const float hi = tf32_rna(x);
            d2[q] = hi;
            d2[p.K0p + q] = tf32_rna(x - hi);
          }
          continue;
        }
        double* dst = Drow + qq * p.M + f0;
        if constexpr (F % 2 == 0) {
          if ((p.M & 1) == 0) {
#pragma unroll
            for (int q = 0; q < F; q += 2) *reinterpret_cast<double2*>(dst + q) = make_double2(dv[q], dv[q + 1]);
            continue;
          }
        }
#pragma unroll
        for (int q = 0; q < F; ++q) dst[q] = dv[q];
      }
    }
    __syncwarp();
  }
}

// Reduce-scatter of 16 per-lane partials: afterwards lane l holds the warp sum of entry l & 15.
__device__ __forceinline__ double rs16(double* v, int lane) {
#pragma unroll
  for (int lvl = 8; lvl >= 1; lvl >>= 1) {
    const bool hi = lane & lvl;
#pragma unroll
    for (int i = 0; i < lvl; ++i) {
      const double send = hi ? v[i] : v[i + lvl];
      const double keep = hi ? v[i + lvl] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, lvl);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// ---------------------------------------------------------------- k_tab_dT (warp per centre)
// dT = adjoint of D = T<^T T (contract.hpp:21-38): dT[a][p] = sum_{q<mlt} dD[q][p] T[a][q]
// + [p < mlt] sum_r dD[p][r] T[a][r]. Written to dTg[i][4][Mp] for the projection kernels.
template <int F>
__global__ void __launch_bounds__(256, 2) k_tab_dT(TabParams p, double* __restrict__ dTg) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  double* ts = reinterpret_cast<double*>(smem) + wid * (4 * p.Mp + 4 * p.mlt);
  double* S = ts + 4 * p.Mp;
  const int f0 = F * lane;
  for (int i = p.i0 + blockIdx.x * wpb + wid; i < p.i1; i += gridDim.x * wpb) {
    double* out = dTg + static_cast<size_t>(i) * 4 * p.Mp;
    if (!p.center[i]) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < F; ++q) out[a * p.Mp + f0 + q] = 0.0;
      continue;
    }
#if TAB_L2_PREFETCH
    {
      // the warp's next centre: its dD row (lane 0) and T rows (lane 1)
      const int in = i + gridDim.x * wpb;
      if (in < p.i1 && lane < 2 && p.center[in]) {
        if (lane == 1) {
          l2_prefetch(p.T + static_cast<size_t>(in) * 4 * p.Mp, static_cast<size_t>(4) * p.Mp * 8);
        } else {
          const int s2 = p.slot_of[in];
          if (s2 >= 0) l2_prefetch(p.dD + static_cast<size_t>(s2) * p.K0p, static_cast<size_t>(p.mlt) * p.M * 8);
        }
      }
    }
#endif
    const double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
    double tv[4][F], dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) {
        tv[a][q] = Ti[a * p.Mp + f0 + q];
        ts[a * p.Mp + f0 + q] = tv[a][q];
        dT[a][q] = 0.0;
      }
    __syncwarp();
    const int slot = p.slot_of[i];
    const double* dDrow = p.dD + static_cast<size_t>(slot < 0 ? 0 : slot) * p.K0p;
    const bool fon = f0 < p.M && slot >= 0;
    const bool vec = ((p.M | p.K0p) & 1) == 0; // 16-byte aligned dD pairs
    for (int q0 = 0; q0 < p.mlt; q0 += 4) {
      double part[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) part[k] = 0.0;
#pragma unroll
      for (int ql = 0; ql < 4; ++ql) {
        const int qq = q0 + ql;
        if (qq < p.mlt) {
          double dq[F];
          if constexpr (F % 2 == 0) {
            if (vec) {
#pragma unroll
              for (int q = 0; q < F; q += 2) {
                const double2 v = fon ? *reinterpret_cast<const double2*>(dDrow + qq * p.M + f0 + q)
                                      : make_double2(0.0, 0.0);
                dq[q] = v.x;
                dq[q + 1] = v.y;
              }
            } else {
#pragma unroll
              for (int q = 0; q < F; ++q) dq[q] = fon ? dDrow[qq * p.M + f0 + q] : 0.0;
            }
          } else {
#pragma unroll
            for (int q = 0; q < F; ++q) dq[q] = fon ? dDrow[qq * p.M + f0 + q] : 0.0;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const double ta = ts[a * p.Mp + qq];
#pragma unroll
            for (int q = 0; q < F; ++q) {
              dT[a][q] += dq[q] * ta;
              part[ql * 4 + a] += dq[q] * tv[a][q];
            }
          }
        }
      }
      const double s = rs16(part, lane);
      if (lane < 16 && q0 + (lane >> 2) < p.mlt) S[(q0 + (lane >> 2)) * 4 + (lane & 3)] = s;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < F; ++q) {
      const int f = f0 + q;
      if (f < p.mlt)
#pragma unroll
        for (int a = 0; a < 4; ++a) dT[a][q] += S[f * 4 + a];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) out[a * p.Mp + f0 + q] = dT[a][q];
    __syncwarp();
    if (lane == 0) atomicAdd(p.counters + 1, static_cast<unsigned long long>(p.n_real[i]));
  }
}

// ---------------------------------------------------------------- k_tab_bwd_P (warp per centre)
// Per-warp projections P[a][m] = sum_p dT[a][p] C[th][m][p] of every group of a centre (FMA +
// reduce-scatter). Used for the atom blocks whose interval union is too wide for the tensor-core
// kernel below (fb_list, e.g. fine tables), or for feature widths above 128.
template <int F>
__global__ void __launch_bounds__(64, 6) k_tab_bwd_P(TabParams p, const double* __restrict__ dTg,
                                                     const int* __restrict__ fb_list, const int* __restrict__ fb_count,
                                                     int na) {
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  const int f0 = F * lane;
  const int total = fb_list ? *fb_count * na : p.i1 - p.i0;
  const int64_t eb = p.row_off[p.i0];
  for (int idx = blockIdx.x * wpb + wid; idx < total; idx += gridDim.x * wpb) {
    const int i = fb_list ? fb_list[idx / na] + idx % na : p.i0 + idx; // fb_list holds block starts
    if (i >= p.i1) continue;
    const int64_t off = p.row_off[i];
    const int nreal = p.n_real[i];
    int G = p.n_grp[i];
    if (p.goff[i] + G > p.pcap) {
      if (lane == 0) raise_err(p.err, DEV_PBUF);
      G = 0;
    }
    const uint64_t* sk = p.skeys + (off - eb);
    double* Pout = p.Pbuf + p.goff[i] * 24;
    const double* dTi = dTg + static_cast<size_t>(i) * 4 * p.Mp;
    double dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) dT[a][q] = dTi[a * p.Mp + f0 + q];
    // --- P[a][m] = sum_p dT[a][p] C[m][p] per group (reduce-scatter over the feature lanes) ---
    int g = 0;
    for (int base = 0; base < nreal && g < G; base += 32) {
      const int k = base + lane;
      bool head = false;
      uint64_t v = 0;
      if (k < nreal) {
        v = sk[k];
        head = (k == 0) || ((v >> 32) != (sk[k - 1] >> 32));
      }
      unsigned m = __ballot_sync(0xffffffffu, head);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const int bin = static_cast<int>(__shfl_sync(0xffffffffu, v, src) >> 32);
        const double* C = p.tab + static_cast<size_t>(bin) * istride + f0;
        double c[6][F];
#pragma unroll
        for (int mm = 0; mm < 6; ++mm) {
          if constexpr (F % 2 == 0) {
#pragma unroll
            for (int q = 0; q < F; q += 2) {
              const double2 cv = __ldg(reinterpret_cast<const double2*>(C + mm * p.Mp + q));
              c[mm][q] = cv.x;
              c[mm][q + 1] = cv.y;
            }
          } else {
#pragma unroll
            for (int q = 0; q < F; ++q) c[mm][q] = __ldg(C + mm * p.Mp + q);
          }
        }
        double part[24];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < F; ++q) acc += dT[a][q] * c[mm][q];
            part[a * 6 + mm] = acc;
          }
        const int b = rs24(part, lane);
        if ((lane & 3) == 0) {
          Pout[g * 24 + b] = part[0];
          Pout[g * 24 + b + 1] = part[1];
          Pout[g * 24 + b + 2] = part[2];
        }
        ++g;
      }
    }
  }
}

// ---------------------------------------------------------------- k_tab_bwd_P2 (CTA, FP64 tensor pipe)
// The projections of 32 consecutive centres at once: every interval touched by any of them (the
// union, ~44 for Cu at h = 0.01 vs ~29 per centre) is staged ONCE in shared memory (cp.async,
// double-buffered, 4 intervals = 24 coefficient rows per stage) and contracted with the 128 dT rows
// (32 centres x 4) on DMMA.8x8x4: P[(i,a)][(th,m)] = sum_p dT[i][a][p] C[th][m][p]. The per-warp
// kernel re-read 6 KB of coefficients per (centre, interval) through L1 and reduced with shuffles;
// here coefficient traffic drops by ~20x and the MACs run on the tensor pipe. Only the (centre,
// interval) pairs the centre really has are written (Pbuf, same layout as the per-warp kernel).
constexpr int P2_NA = 32, P2_CB = 4, P2_UCAP = 128, P2_UW = P2_UCAP / 32, P2_BMW = 256;
constexpr int P2_THREADS = 512; // 16 warps, one m-tile (2 centres x 4 rows) each

__host__ __device__ inline size_t p2_smem_bytes(int Mp) {
  const int pitch = Mp + 4;
  return static_cast<size_t>(4 * P2_NA + 2 * 6 * P2_CB) * pitch * sizeof(double) +
         (2 * P2_BMW + P2_UCAP + P2_NA / 2 * P2_UW + 4) * sizeof(int) + P2_NA * P2_UCAP * sizeof(int16_t);
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int F>
__global__ void __launch_bounds__(P2_THREADS, 1) k_tab_bwd_P2(TabParams p, const double* __restrict__ dTg,
                                                       int* __restrict__ fb_list, int* __restrict__ fb_count) {
  constexpr int Mp = 32 * F, pitch = Mp + 4, units = Mp / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  double* dTs = reinterpret_cast<double*>(smem);                         // [128][pitch]
  double* Cs = dTs + 4 * P2_NA * pitch;                                  // [2][24][pitch]
  uint32_t* bm = reinterpret_cast<uint32_t*>(Cs + 2 * 6 * P2_CB * pitch); // [BMW] union bitmap
  int* wpre = reinterpret_cast<int*>(bm + P2_BMW);                       // [BMW] popcount prefix
  int* ubin = wpre + P2_BMW;                                             // [UCAP] union bins
  uint32_t* mtmask = reinterpret_cast<uint32_t*>(ubin + P2_UCAP);        // [NA/2][UW] per m-tile union
  int* misc = reinterpret_cast<int*>(mtmask + P2_NA / 2 * P2_UW);        // bmin, bmax, U
  int16_t* gidx = reinterpret_cast<int16_t*>(misc + 4);                  // [NA][UCAP] group of slot or -1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int nblk = (p.i1 - p.i0 + P2_NA - 1) / P2_NA;
  const int64_t eb = p.row_off[p.i0];
  // output columns of this thread inside a chunk: c = 8 nt + 2 tig + h -> (slot c / 6, m = c % 6)
  int cslot[6], cm[6];
#pragma unroll
  for (int nt = 0; nt < 3; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = nt * 8 + 2 * tig + h;
      cslot[nt * 2 + h] = c / 6;
      cm[nt * 2 + h] = c % 6;
    }
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int i0 = p.i0 + blk * P2_NA;
#if TAB_L2_PREFETCH
    {
      // the CTA's next block: its 32 centres' dT rows (contiguous), in 16 KB pieces
      const int n0 = i0 + gridDim.x * P2_NA;
      const int nc = min(P2_NA, p.i1 - n0);
      if (nc > 0) {
        const size_t bytes = static_cast<size_t>(nc) * 4 * Mp * sizeof(double);
        const size_t piece = size_t(16384) * tid;
        if (piece < bytes)
          l2_prefetch(dTg + static_cast<size_t>(n0) * 4 * Mp + piece / sizeof(double),
                      bytes - piece < 16384 ? bytes - piece : 16384);
      }
    }
#endif
    // dT rows of the 32 centres (contiguous in dTg)
    for (int q = tid; q < 4 * P2_NA * units; q += P2_THREADS) {
      const int row = q / units, c2 = q % units;
      double* dst = dTs + row * pitch + 2 * c2;
      if (i0 + (row >> 2) < p.i1)
        tc::cp_async16(dst, dTg + (static_cast<size_t>(i0) * 4 + row) * Mp + 2 * c2);
      else
        dst[0] = dst[1] = 0.0;
    }
    tc::cp_commit();
    if (tid == 0) {
      misc[0] = 0x7fffffff;
      misc[1] = -1;
    }
    for (int q = tid; q < P2_NA * P2_UCAP / 2; q += P2_THREADS) reinterpret_cast<int32_t*>(gidx)[q] = -1;
    for (int q = tid; q < P2_NA / 2 * P2_UW; q += P2_THREADS) mtmask[q] = 0u;
    __syncthreads();
    // interval range of the block: each centre's group bins are sorted (gbin, written by k_tab_fwd)
    if (tid < P2_NA && i0 + tid < p.i1) {
      const int i = i0 + tid;
      const int G = p.n_grp[i];
      if (G > 0) {
        const int32_t* gb = p.gbin + (p.row_off[i] - eb);
        atomicMin(misc, gb[0]);
        atomicMax(misc + 1, gb[G - 1]);
      }
    }
    __syncthreads();
    const int bmin = misc[0], bmax = misc[1];
    const int range = bmax < 0 ? 0 : bmax - bmin + 1;
    const int nw = (range + 31) >> 5;
    const bool wide = nw > P2_BMW;
    if (!wide)
      for (int w = tid; w < nw; w += P2_THREADS) bm[w] = 0u;
    __syncthreads();
    if (!wide) {
      for (int al = warp * 2; al < warp * 2 + 2; ++al) {
        const int i = i0 + al;
        if (i >= p.i1) break;
        const int G = p.n_grp[i];
        const int32_t* gb = p.gbin + (p.row_off[i] - eb);
        for (int g = lane; g < G; g += 32) {
          const int b = gb[g] - bmin;
          atomicOr(bm + (b >> 5), 1u << (b & 31));
        }
      }
    }
    __syncthreads();
    if (!wide && warp == 0) {
      // exclusive prefix of the bitmap popcounts -> union list in ascending bin order
      constexpr int PER = P2_BMW / 32;
      int c[PER], s = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int w = lane * PER + k;
        c[k] = w < nw ? __popc(bm[w]) : 0;
        s += c[k];
      }
      int tot;
      int ex = warp_excl_scan(s, lane, &tot);
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int w = lane * PER + k;
        if (w < nw) {
          wpre[w] = ex;
          uint32_t bits = bm[w];
          int at = ex;
          while (bits) {
            const int bit = __ffs(bits) - 1;
            bits &= bits - 1;
            if (at < P2_UCAP) ubin[at] = bmin + 32 * w + bit;
            ++at;
          }
        }
        ex += c[k];
      }
      if (lane == 0) misc[2] = tot;
    }
    __syncthreads();
    const int U = range == 0 ? 0 : misc[2];
    if (wide || U > P2_UCAP) {
      if (tid == 0) fb_list[atomicAdd(fb_count, 1)] = i0;
      tc::cp_wait<0>();
      __syncthreads();
      continue;
    }
    // slot -> group of each centre, and the union each m-tile (2 centres) really needs
    for (int al = warp * 2; al < warp * 2 + 2; ++al) {
      const int i = i0 + al;
      if (i >= p.i1) break;
      const int G = p.n_grp[i];
      const int32_t* gb = p.gbin + (p.row_off[i] - eb);
      for (int g = lane; g < G; g += 32) {
        const int b = gb[g] - bmin;
        const int u = wpre[b >> 5] + __popc(bm[b >> 5] & ((1u << (b & 31)) - 1u));
        gidx[al * P2_UCAP + u] = static_cast<int16_t>(g);
        atomicOr(mtmask + (al >> 1) * P2_UW + (u >> 5), 1u << (u & 31));
      }
    }
    // this thread's output row (the warp's m-tile): centre, component, group base
    int r_al[1], r_a[1];
    int64_t r_base[1];
    bool r_ok[1];
#pragma unroll
    for (int mt = 0; mt < 1; ++mt) {
      const int r = warp * 8 + gid;
      r_al[mt] = r >> 2;
      r_a[mt] = r & 3;
      const int i = i0 + r_al[mt];
      r_ok[mt] = i < p.i1;
      r_base[mt] = r_ok[mt] ? p.goff[i] : 0;
      if (r_ok[mt] && r_base[mt] + p.n_grp[i] > p.pcap) {
        if (r_a[mt] == 0 && tig == 0) raise_err(p.err, DEV_PBUF);
        r_ok[mt] = false;
      }
    }
    // coefficient chunks: CB intervals x 6 rows, double-buffered
    const int nch = (U + P2_CB - 1) / P2_CB;
    auto stage = [&](int ch, int buf) {
      double* dst0 = Cs + buf * 6 * P2_CB * pitch;
      for (int q = tid; q < 6 * P2_CB * units; q += P2_THREADS) {
        const int row = q / units, c2 = q % units;
        const int u = ch * P2_CB + row / 6, m = row % 6;
        double* dst = dst0 + row * pitch + 2 * c2;
        if (u < U)
          tc::cp_async16(dst, p.tab + static_cast<size_t>(ubin[u]) * 6 * Mp + m * Mp + 2 * c2);
        else
          dst[0] = dst[1] = 0.0;
      }
      tc::cp_commit();
    };
    if (nch > 0) stage(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
      if (ch + 1 < nch) {
        stage(ch + 1, (ch + 1) & 1);
        tc::cp_wait<1>();
      } else {
        tc::cp_wait<0>();
      }
      __syncthreads();
      const double* cs = Cs + (ch & 1) * 6 * P2_CB * pitch;
      double acc[1][3][2];
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) acc[0][nt][0] = acc[0][nt][1] = 0.0;
      const double* a0 = dTs + (warp * 8 + gid) * pitch + tig;
      const double* b0 = cs + gid * pitch + tig;
      // n-tile nt covers chunk slots {nt, nt+1} (columns 8 nt .. 8 nt + 7 of 6 per slot); the
      // m-tile needs it only if one of its two centres has one of those intervals
      const int sh = (ch * P2_CB) & 31, wd = (ch * P2_CB) >> 5;
      const unsigned n0 = (mtmask[warp * P2_UW + wd] >> sh) & 15u;
      const unsigned use = ((n0 & 3u) ? 1u : 0u) | ((n0 & 6u) ? 2u : 0u) | ((n0 & 12u) ? 4u : 0u);
      if (use == 7u) {
#pragma unroll 4
        for (int k = 0; k < Mp; k += 4) {
          const double av0 = a0[k];
          const double bv0 = b0[k], bv1 = b0[8 * pitch + k], bv2 = b0[16 * pitch + k];
          dmma884(acc[0][0][0], acc[0][0][1], av0, bv0);
          dmma884(acc[0][1][0], acc[0][1][1], av0, bv1);
          dmma884(acc[0][2][0], acc[0][2][1], av0, bv2);
        }
      } else if (use) {
#pragma unroll 2
        for (int k = 0; k < Mp; k += 4) {
          const double av0 = a0[k];
          const double bv0 = b0[k], bv1 = b0[8 * pitch + k], bv2 = b0[16 * pitch + k];
          if (use & 1u) dmma884(acc[0][0][0], acc[0][0][1], av0, bv0);
          if (use & 2u) dmma884(acc[0][1][0], acc[0][1][1], av0, bv1);
          if (use & 4u) dmma884(acc[0][2][0], acc[0][2][1], av0, bv2);
        }
      }
      // scatter the (centre, interval) pairs that exist into Pbuf
#pragma unroll
      for (int mt = 0; mt < 1; ++mt) {
        if (!r_ok[mt]) continue;
        const int16_t* gi = gidx + r_al[mt] * P2_UCAP + ch * P2_CB;
        double* pb = p.Pbuf + r_base[mt] * 24 + r_a[mt] * 6;
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const int u = ch * P2_CB + cslot[k];
          const int g = u < U ? gi[cslot[k]] : -1;
          if (g >= 0) pb[static_cast<int64_t>(g) * 24 + cm[k]] = acc[mt][k >> 1][k & 1];
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- k_tab_fwd_T2 (CTA, staged union)
// The forward contraction T[i][a][p] = sum_groups sum_m W[i][g][a][m] C[bin(g)][m][p] of 32
// consecutive centres per CTA: the union of their intervals is staged once in shared memory
// (cp.async, double-buffered, 4 intervals per stage, 8 rows each) together with the matching
// slice of the moments written by k_tab_fwd<WM>; each warp then contracts its two centres from
// shared memory with lanes owning features. The per-warp k_tab_fwd streams 6 KB of coefficients
// per (centre, interval) from L2 (the hot table does not fit the L1 left beside its shared
// memory); here each staged interval serves all 32 centres. Per accumulator the FMA chain is the
// per-warp kernel's (intervals ascending, m ascending), so T and D are bitwise identical to it.
// (A first version contracted on DMMA with rows = (centre, a), k = (interval, m): slower, see
// DESIGN.md §9.) Blocks whose union exceeds T2_UCAP intervals contract per warp from the moments.
constexpr int T2_NA = 32, T2_CB = 4, T2_UCAP = 128, T2_UW = T2_UCAP / 32, T2_BMW = 256, T2_AP = 36;
constexpr int T2_THREADS = 512; // 16 warps, one m-tile (2 centres x 4 rows) each

__host__ __device__ inline size_t t2_region_bytes(int Mp) {
  const int pitch = Mp + 4;
  const size_t stg = (static_cast<size_t>(2) * 8 * T2_CB * pitch + static_cast<size_t>(2) * 4 * T2_NA * T2_AP) * 8;
  const size_t ts = static_cast<size_t>(T2_THREADS / 32) * 4 * (pitch - 4) * 8; // per-warp T (wide blocks)
  return stg > ts ? stg : ts;
}

__host__ __device__ inline size_t t2_smem_bytes(int Mp) {
  return t2_region_bytes(Mp) + T2_NA * sizeof(int64_t) +
         (2 * T2_BMW + T2_UCAP + T2_NA / 2 * T2_UW + 4) * sizeof(int) + T2_NA * T2_UCAP * sizeof(int16_t);
}

template <int F>
__global__ void __launch_bounds__(T2_THREADS, 1) k_tab_fwd_T2(TabParams p) {
  constexpr int Mp = 32 * F, pitch = Mp + 4, units = Mp / 2, NT = Mp / 8, CR = 8 * T2_CB;
  extern __shared__ __align__(16) unsigned char smem[];
  double* Cs = reinterpret_cast<double*>(smem);          // [2][CR][pitch] coefficient rows (k x features)
  double* As = Cs + 2 * CR * pitch;                      // [2][128][AP] moments (rows x k)
  int64_t* wb_s = reinterpret_cast<int64_t*>(smem + t2_region_bytes(Mp)); // [NA] first group in Pbuf
  uint32_t* bm = reinterpret_cast<uint32_t*>(wb_s + T2_NA);              // [BMW] union bitmap
  int* wpre = reinterpret_cast<int*>(bm + T2_BMW);                       // [BMW] popcount prefix
  int* ubin = wpre + T2_BMW;                                             // [UCAP] union bins
  uint32_t* mtmask = reinterpret_cast<uint32_t*>(ubin + T2_UCAP);        // [NA/2][UW] per m-tile union
  int* misc = reinterpret_cast<int*>(mtmask + T2_NA / 2 * T2_UW);        // bmin, bmax, U
  int16_t* gidx = reinterpret_cast<int16_t*>(misc + 4);                  // [NA][UCAP] group of slot or -1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;         // warp = m-tile = centres 2w, 2w+1
  const int gid = lane >> 2, tig = lane & 3;
  const int nblk = (p.i1 - p.i0 + T2_NA - 1) / T2_NA;
  const int64_t eb = p.row_off[p.i0];
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int i0 = p.i0 + blk * T2_NA;
    const int na = min(T2_NA, p.i1 - i0);
    if (tid == 0) {
      misc[0] = 0x7fffffff;
      misc[1] = -1;
    }
    for (int q = tid; q < T2_NA * T2_UCAP / 2; q += T2_THREADS) reinterpret_cast<int32_t*>(gidx)[q] = -1;
    for (int q = tid; q < T2_NA / 2 * T2_UW; q += T2_THREADS) mtmask[q] = 0u;
    if (tid < T2_NA) wb_s[tid] = tid < na ? p.wbase[i0 + tid] : -1;
    __syncthreads();
    if (tid < na) {
      const int i = i0 + tid;
      const int G = p.n_grp[i];
      if (G > 0) {
        const int32_t* gb = p.gbin + (p.row_off[i] - eb);
        atomicMin(misc, gb[0]);
        atomicMax(misc + 1, gb[G - 1]);
      }
    }
    __syncthreads();
    const int bmin = misc[0], bmax = misc[1];
    const int range = bmax < 0 ? 0 : bmax - bmin + 1;
    const int nw = (range + 31) >> 5;
    const bool wide = nw > T2_BMW;
    if (!wide)
      for (int w = tid; w < nw; w += T2_THREADS) bm[w] = 0u;
    __syncthreads();
    if (!wide) {
      for (int al = warp * 2; al < warp * 2 + 2 && al < na; ++al) {
        const int i = i0 + al;
        const int G = p.n_grp[i];
        const int32_t* gb = p.gbin + (p.row_off[i] - eb);
        for (int g = lane; g < G; g += 32) {
          const int b = gb[g] - bmin;
          atomicOr(bm + (b >> 5), 1u << (b & 31));
        }
      }
    }
    __syncthreads();
    if (!wide && warp == 0) {
      constexpr int PER = T2_BMW / 32;
      int c[PER], s = 0;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int w = lane * PER + k;
        c[k] = w < nw ? __popc(bm[w]) : 0;
        s += c[k];
      }
      int tot;
      int ex = warp_excl_scan(s, lane, &tot);
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int w = lane * PER + k;
        if (w < nw) {
          wpre[w] = ex;
          uint32_t bits = bm[w];
          int at = ex;
          while (bits) {
            const int bit = __ffs(bits) - 1;
            bits &= bits - 1;
            if (at < T2_UCAP) ubin[at] = bmin + 32 * w + bit;
            ++at;
          }
        }
        ex += c[k];
      }
      if (lane == 0) misc[2] = tot;
    }
    __syncthreads();
    const int U = range == 0 ? 0 : misc[2];
    if (wide || U > T2_UCAP) {
      // per-warp contraction from the moments (groups ascending, then a, m as k_tab_fwd); lanes
      // own features f0 .. f0 + F - 1; T[a][0..Mp) of the centre staged per warp for D
      const int f0 = F * lane;
      double* ts = Cs + warp * 4 * Mp;
      for (int al = warp * 2; al < warp * 2 + 2 && al < na; ++al) {
        double tacc[4][F];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < F; ++q) tacc[a][q] = 0.0;
        const int i = i0 + al;
        const int64_t wb = wb_s[al];
        if (wb >= 0) {
          const int G = p.n_grp[i];
          const int32_t* gb = p.gbin + (p.row_off[i] - eb);
          for (int g = 0; g < G; ++g) {
            const double* C = p.tab + static_cast<size_t>(gb[g]) * 6 * Mp + f0;
            const double* Wg = p.Pbuf + (wb + g) * 24;
            double c[6][F];
#pragma unroll
            for (int mm = 0; mm < 6; ++mm)
#pragma unroll
              for (int q = 0; q < F; ++q) c[mm][q] = __ldg(C + mm * Mp + q);
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int mm = 0; mm < 6; ++mm) {
                const double wa = Wg[a * 6 + mm];
#pragma unroll
                for (int q = 0; q < F; ++q) tacc[a][q] += wa * c[mm][q];
              }
          }
        }
        double* Ti = p.T + static_cast<size_t>(i) * 4 * Mp;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < F; ++q) {
            Ti[a * Mp + f0 + q] = tacc[a][q];
            ts[a * Mp + f0 + q] = tacc[a][q];
          }
        __syncwarp();
        const int slot = p.slot_of[i];
        if (slot >= 0 && f0 < p.M) {
          double* Drow = p.D + static_cast<size_t>(slot) * p.K0p;
          for (int qq = 0; qq < p.mlt; ++qq) {
            const double t0 = ts[qq], t1 = ts[Mp + qq], t2 = ts[2 * Mp + qq], t3 = ts[3 * Mp + qq];
#pragma unroll
            for (int q = 0; q < F; ++q) {
              double v = t0 * tacc[0][q];
              v += t1 * tacc[1][q];
              v += t2 * tacc[2][q];
              v += t3 * tacc[3][q];
              Drow[qq * p.M + f0 + q] = v;
            }
          }
        }
        __syncwarp();
      }
      __syncthreads();
      continue;
    }
    // slot -> group of each centre, and the union each m-tile (2 centres) really needs
    for (int al = warp * 2; al < warp * 2 + 2 && al < na; ++al) {
      const int i = i0 + al;
      const int G = p.n_grp[i];
      const int32_t* gb = p.gbin + (p.row_off[i] - eb);
      for (int g = lane; g < G; g += 32) {
        const int b = gb[g] - bmin;
        const int u = wpre[b >> 5] + __popc(bm[b >> 5] & ((1u << (b & 31)) - 1u));
        gidx[al * T2_UCAP + u] = static_cast<int16_t>(g);
        atomicOr(mtmask + (al >> 1) * T2_UW + (u >> 5), 1u << (u & 31));
      }
    }
    __syncthreads();
    const int nch = (U + T2_CB - 1) / T2_CB;
    auto stage = [&](int ch, int buf) {
      double* cdst = Cs + buf * CR * pitch;
      for (int q = tid; q < CR * units; q += T2_THREADS) {
        const int row = q / units, c2 = q % units;
        const int u = ch * T2_CB + (row >> 3), m = row & 7;
        double* dst = cdst + row * pitch + 2 * c2;
        if (m < 6 && u < U)
          tc::cp_async16(dst, p.tab + static_cast<size_t>(ubin[u]) * 6 * Mp + m * Mp + 2 * c2);
        else
          dst[0] = dst[1] = 0.0;
      }
      double* adst = As + buf * 4 * T2_NA * T2_AP;
      for (int q = tid; q < 4 * T2_NA * T2_CB * 4; q += T2_THREADS) {
        const int row = q >> 4, ul = (q >> 2) & 3, piece = q & 3;
        const int al = row >> 2, a = row & 3;
        const int u = ch * T2_CB + ul;
        const int g = u < U ? gidx[al * T2_UCAP + u] : -1;
        const int64_t wb = wb_s[al];
        double* dst = adst + row * T2_AP + ul * 8 + piece * 2;
        if (piece < 3 && g >= 0 && wb >= 0)
          tc::cp_async16(dst, p.Pbuf + (wb + g) * 24 + a * 6 + piece * 2);
        else
          dst[0] = dst[1] = 0.0;
      }
      tc::cp_commit();
    };
    // per-warp contraction of its two centres from the staged slice, lanes own features
    // f0 .. f0 + F - 1: for each of the centre's intervals (ascending), for m, for a,
    // T[a][f] += W[a][m] C[m][f] -- per accumulator the same FMA chain as k_tab_fwd, so T and D
    // are bitwise those of the per-warp kernel
    const int f0 = F * lane;
    double tacc[2][4][F];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < F; ++q) tacc[c][a][q] = 0.0;
    if (nch > 0) stage(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
      if (ch + 1 < nch) {
        stage(ch + 1, (ch + 1) & 1);
        tc::cp_wait<1>();
      } else {
        tc::cp_wait<0>();
      }
      __syncthreads();
      const double* cs = Cs + (ch & 1) * CR * pitch + f0;
      const double* as = As + (ch & 1) * 4 * T2_NA * T2_AP;
      const bool ok0 = warp * 2 < na && wb_s[warp * 2] >= 0;
      const bool ok1 = warp * 2 + 1 < na && wb_s[warp * 2 + 1] >= 0;
      const int16_t* g0 = gidx + (warp * 2) * T2_UCAP + ch * T2_CB;
      const double* w0 = as + (warp * 2) * 4 * T2_AP;
      const double* w1 = w0 + 4 * T2_AP;
      for (int ul = 0; ul < T2_CB && ch * T2_CB + ul < U; ++ul) {
        // both centres of the warp share the staged coefficient rows of an interval they both have
        const bool h0 = ok0 && g0[ul] >= 0, h1 = ok1 && g0[T2_UCAP + ul] >= 0;
        if (!(h0 || h1)) continue;
        const double* cr = cs + ul * 8 * pitch;
        const double* wr0 = w0 + ul * 8;
        const double* wr1 = w1 + ul * 8;
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          double cm[F];
          if constexpr (F % 2 == 0) {
#pragma unroll
            for (int q = 0; q < F; q += 2) {
              const double2 v = *reinterpret_cast<const double2*>(cr + m * pitch + q);
              cm[q] = v.x;
              cm[q + 1] = v.y;
            }
          } else {
#pragma unroll
            for (int q = 0; q < F; ++q) cm[q] = cr[m * pitch + q];
          }
          if (h0) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const double wa = wr0[a * T2_AP + m];
#pragma unroll
              for (int q = 0; q < F; ++q) tacc[0][a][q] += wa * cm[q];
            }
          }
          if (h1) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const double wa = wr1[a * T2_AP + m];
#pragma unroll
              for (int q = 0; q < F; ++q) tacc[1][a][q] += wa * cm[q];
            }
          }
        }
      }
      __syncthreads();
    }
    // T out, D = T<^T T (contract.hpp:9-17) as in k_tab_fwd (T of the centre staged per warp)
    double* ts = Cs + warp * 4 * Mp;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int al = warp * 2 + c;
      if (al >= na) break;
      const int i = i0 + al;
      double* Ti = p.T + static_cast<size_t>(i) * 4 * Mp;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int q = 0; q < F; ++q) {
          Ti[a * Mp + f0 + q] = tacc[c][a][q];
          ts[a * Mp + f0 + q] = tacc[c][a][q];
        }
      __syncwarp();
      const int slot = p.slot_of[i];
      if (slot >= 0 && f0 < p.M) {
        double* Drow = p.D + static_cast<size_t>(slot) * p.K0p;
        for (int qq = 0; qq < p.mlt; ++qq) {
          const double t0 = ts[qq], t1 = ts[Mp + qq], t2 = ts[2 * Mp + qq], t3 = ts[3 * Mp + qq];
          double dv[F];
#pragma unroll
          for (int q = 0; q < F; ++q) {
            double v = t0 * tacc[c][0][q];
            v += t1 * tacc[c][1][q];
            v += t2 * tacc[c][2][q];
            v += t3 * tacc[c][3][q];
            dv[q] = v;
          }
          double* dst = Drow + qq * p.M + f0;
          if constexpr (F % 2 == 0) {
            if ((p.M & 1) == 0) {
#pragma unroll
              for (int q = 0; q < F; q += 2) *reinterpret_cast<double2*>(dst + q) = make_double2(dv[q], dv[q + 1]);
              continue;
            }
          }
#pragma unroll
          for (int q = 0; q < F; ++q) dst[q] = dv[q];
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- k_tab_bwd_g (thread per entry)
__global__ void __launch_bounds__(256) k_tab_bwd_g(TabParams p) {
  const int64_t eo = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t eb = p.row_off[p.i0];
  const int64_t e = eb + eo;
  if (e >= p.E || e >= p.row_off[p.i1]) return;
  // bin, owner, group and key loaded together (independent; egrp is unset for non-real entries
  // but inside the chunk buffer), so a real entry waits for one latency, not three
  const int bin = p.ebin[e];
  const int i = p.eown[e];
  const int grp = p.egrp[e - eb];
  const uint64_t key = p.keys[e];
  double* ge = p.g + 3 * e;
  if (bin < 0) return; // never read: k_forces gathers only real entries (own and reverse)
  const int64_t gi = p.goff[i] + grp;
  Env ev;
  env_of(p, ld_pos(p.pos, i), key, ev);
  const int th = bin % p.tn;
  if (gi >= p.pcap) {
    raise_err(p.err, DEV_PBUF);
    ge[0] = ge[1] = ge[2] = 0.0;
    return;
  }
  // the group's 24 projections as 12 16-byte loads (a Pbuf row is 192 B, 16-byte aligned)
  const double2* P2 = reinterpret_cast<const double2*>(p.Pbuf + gi * 24);
  double P[24];
#pragma unroll
  for (int q = 0; q < 12; ++q) {
    const double2 v = __ldg(P2 + q);
    P[2 * q] = v.x;
    P[2 * q + 1] = v.y;
  }
  const double R[4] = {ev.s, ev.s * ev.u[0], ev.s * ev.u[1], ev.s * ev.u[2]};
  const double uu = ev.s - node_x(p.x0, p.h, th);
  double drow[4], dsum = 0.0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const double* Pa = P + a * 6;
    drow[a] = ((((Pa[5] * uu + Pa[4]) * uu + Pa[3]) * uu + Pa[2]) * uu + Pa[1]) * uu + Pa[0];
    const double h1 = (((5.0 * Pa[5] * uu + 4.0 * Pa[4]) * uu + 3.0 * Pa[3]) * uu + 2.0 * Pa[2]) * uu + Pa[1];
    dsum += R[a] * h1;
  }
  drow[0] += dsum;
  double dd[12];
#pragma unroll
  for (int x = 0; x < 3; ++x) dd[x] = ev.sd * ev.u[x];
#pragma unroll
  for (int y = 0; y < 3; ++y)
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      double v = ev.sd * ev.u[x] * ev.u[y] - ev.s * ev.ir * ev.u[x] * ev.u[y];
      if (x == y) v += ev.s * ev.ir;
      dd[3 * (1 + y) + x] = v;
    }
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    double acc = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a) acc += drow[a] * dd[3 * a + x];
    ge[x] = acc;
  }
}

// ---------------------------------------------------------------- host side
int sm_count(int dev) {
  int s = 0;
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

template <int F, bool F32>
void launch_fwd_warp2(const TabParams& p, cudaStream_t st, int sms) {
  const size_t bytes = 2 * fwd_smem_bytes(p.scap, p.Mp);
  if (bytes > 227 * 1024) throw NumErr("neighbour rows too long for the tabulate kernel");
  DPB_CUDA(cudaFuncSetAttribute(k_tab_fwd<F, F32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  const int blocks = std::max(1, std::min(ceil_div(p.i1 - p.i0, 2), sms * 32));
  k_tab_fwd<F, F32><<<blocks, 64, bytes, st>>>(p);
  DPB_CUDA(cudaGetLastError());
}

template <int F>
void launch_fwd_warp(const TabParams& p, cudaStream_t st, int sms) {
  if (p.tab32) launch_fwd_warp2<F, true>(p, st, sms);
  else launch_fwd_warp2<F, false>(p, st, sms);
}

__global__ void k_to_f32(int64_t n, const double* __restrict__ x, float* __restrict__ y) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) y[i] = static_cast<float>(x[i]);
}

template <int F>
void launch_bwd_warp(const TabParams& p, const double* dTg, const int* fb_list, const int* fb_count, int na,
                     cudaStream_t st, int sms) {
  const int blocks = fb_list ? sms * 8 : std::max(1, std::min(ceil_div(p.i1 - p.i0, 2), sms * 32));
  k_tab_bwd_P<F><<<blocks, 64, 0, st>>>(p, dTg, fb_list, fb_count, na);
  DPB_CUDA(cudaGetLastError());
}

template <int F>
void launch_dT(const TabParams& p, double* dTg, cudaStream_t st, int sms) {
  const size_t bytes = 8 * (4 * static_cast<size_t>(p.Mp) + 4 * p.mlt) * sizeof(double);
  DPB_CUDA(cudaFuncSetAttribute(k_tab_dT<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  const int blocks = std::max(1, std::min(ceil_div(p.i1 - p.i0, 8), sms * 8));
  k_tab_dT<F><<<blocks, 256, bytes, st>>>(p, dTg);
  DPB_CUDA(cudaGetLastError());
}

} // namespace

// Parameters of the centre range [i0, i1) of the current chunk (Engine::use_chunk): window
// pointers of its buffer set, its Pbuf region.
TabParams chunk_params(Engine& E, int64_t i0, int64_t i1) {
  TabParams p = make_params(E);
  p.i0 = static_cast<int>(i0);
  p.i1 = static_cast<int>(i1);
  p.Pbuf = E.Pbuf.p + static_cast<size_t>(E.cur_set) * E.pbuf_cap * 24;
  return p;
}

// Total groups of a centre range (for the Pbuf capacity of its chunk).
__global__ void k_group_total(const int32_t* __restrict__ n_grp, const int64_t* __restrict__ goff, int i0, int i1,
                              int64_t* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = i1 > i0 ? goff[i1 - 1] + n_grp[i1 - 1] : 0;
}

// env-mat of every entry of the rows [i0, i1): grid bound = the chunk's entry capacity
void env_range(Engine& E, const TabParams& p, cudaStream_t st) {
  const int64_t ne = std::min<int64_t>(p.es, p.E);
  if (ne > 0) {
    k_env_fwd<<<ceil_div(ne, 256), 256, 0, st>>>(p);
    ++E.launches;
  }
}

// env + k_tab_fwd over centres [i0, i1) of chunk k, then the group offsets of the chunk
// (goff[i0..i1) start at 0; the chunk's buffer set owns Pbuf[set * pbuf_cap ...]).
// FP32 copy of the coefficient table for the mixed-mode forward contraction
void Engine::ensure_tab32() {
  if (precision != 1 || tab32_ver == tab_ver) return;
  const int64_t cnt = static_cast<int64_t>(n_types) * static_cast<int64_t>(tab_n) * 6 * Mp;
  tab32.ensure(cnt);
  k_to_f32<<<ceil_div(cnt, 256), 256, 0, stream>>>(cnt, tab.p, tab32.p);
  DPB_CUDA(cudaStreamSynchronize(stream));
  tab32_ver = tab_ver;
}

// Opt-in (DPB_T2=1), results bitwise equal to the default path: measured at C2 the moments kernel
// + k_tab_fwd_T2 take 0.19 + 0.40 ms per 16k-centre chunk against 0.42 ms for the per-warp
// k_tab_fwd (step 5.33 vs 5.01 ms); DESIGN.md §9.
bool Engine::t2_ok() const {
  static const bool on = std::getenv("DPB_T2") != nullptr && std::getenv("DPB_T2")[0] == '1';
  return on && precision == 0 && Mp <= 128;
}

template <int F>
void launch_fwd_wm(const TabParams& p, cudaStream_t st, int sms) {
  const size_t bytes = 2 * fwd_smem_bytes(p.scap, p.Mp);
  if (bytes > 227 * 1024) throw NumErr("neighbour rows too long for the tabulate kernel");
  DPB_CUDA(cudaFuncSetAttribute(k_tab_fwd<F, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  const int blocks = std::max(1, std::min(ceil_div(p.i1 - p.i0, 2), sms * 32));
  k_tab_fwd<F, false, true><<<blocks, 64, bytes, st>>>(p);
  DPB_CUDA(cudaGetLastError());
}

template <int F>
void launch_fwd_t2(const TabParams& p, cudaStream_t st, int sms) {
  const size_t bytes = t2_smem_bytes(32 * F);
  DPB_CUDA(cudaFuncSetAttribute(k_tab_fwd_T2<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  const int nblk = ceil_div(p.i1 - p.i0, T2_NA);
  k_tab_fwd_T2<F><<<std::max(1, std::min(nblk, sms)), T2_THREADS, bytes, st>>>(p);
  DPB_CUDA(cudaGetLastError());
}

void Engine::tab_fwd_range(int k, int64_t i0, int64_t i1, cudaStream_t st) {
  ensure_tab32();
  TabParams p = chunk_params(*this, i0, i1);
  env_range(*this, p, st);
  const int sms = sm_count(device);
  // group offsets of the chunk -> goff, its total -> h_gtotal[k] (pinned, read at Pbuf sizing)
  auto scan_groups = [&] {
    DevBuf<unsigned char>& tmp = cur_set == 0 ? scan_tmp : scan_tmp2;
    const int cnt = static_cast<int>(i1 - i0);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, n_grp.p + i0, goff.p + i0, cnt, st);
    tmp.ensure(tb + 1);
    cub::DeviceScan::ExclusiveSum(tmp.p, tb, n_grp.p + i0, goff.p + i0, cnt, st);
    gtot.ensure(MAX_CHUNKS);
    k_group_total<<<1, 32, 0, st>>>(n_grp.p, goff.p, static_cast<int>(i0), static_cast<int>(i1), gtot.p + k);
    if (!h_gtotal) {
      DPB_CUDA(cudaMallocHost(&h_gtotal, MAX_CHUNKS * sizeof(int64_t)));
      std::memset(h_gtotal, 0, MAX_CHUNKS * sizeof(int64_t));
    }
    DPB_CUDA(cudaMemcpyAsync(h_gtotal + k, gtot.p + k, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    launches += 2;
  };
  if (t2_ok()) {
    // moments (k_tab_fwd<WM>) into this chunk's Pbuf region, then the tensor-pipe contraction
    auto wm = [&](const TabParams& q) {
      switch (Mp / 32) {
#define DPB_WM(F) case F: launch_fwd_wm<F>(q, st, sms); break;
        DPB_WM(1) DPB_WM(2) DPB_WM(3) DPB_WM(4)
#undef DPB_WM
      }
      ++launches;
    };
    if (pbuf_cap == 0) {
      // first evaluation of this system/plan: exact group total of this chunk (one sync)
      p.count_only = 1;
      wm(p);
      scan_groups();
      DPB_CUDA(cudaStreamSynchronize(st));
      grow_pbuf();
      p = chunk_params(*this, i0, i1);
    }
    wcnt.ensure(2);
    p.wcnt = wcnt.p + cur_set;
    DPB_CUDA(cudaMemsetAsync(p.wcnt, 0, sizeof(unsigned long long), st));
    wm(p);
    switch (Mp / 32) {
#define DPB_T2(F) case F: launch_fwd_t2<F>(p, st, sms); break;
      DPB_T2(1) DPB_T2(2) DPB_T2(3) DPB_T2(4)
#undef DPB_T2
    }
    ++launches;
    scan_groups();
    return;
  }
  switch (Mp / 32) {
    case 1: launch_fwd_warp<1>(p, st, sms); break;
    case 2: launch_fwd_warp<2>(p, st, sms); break;
    case 3: launch_fwd_warp<3>(p, st, sms); break;
    case 4: launch_fwd_warp<4>(p, st, sms); break;
    case 5: launch_fwd_warp<5>(p, st, sms); break;
    case 6: launch_fwd_warp<6>(p, st, sms); break;
    case 7: launch_fwd_warp<7>(p, st, sms); break;
    case 8: launch_fwd_warp<8>(p, st, sms); break;
    default: throw InputErr("feature width 4*d1 must be at most 256");
  }
  ++launches;
  scan_groups();
}

void Engine::launch_tab_fwd() {
  tab_fwd_range(0, 0, n, stream);
  size_pbuf_if_needed();
}

// Pbuf capacity: exact (one sync) on the first evaluation of a system; afterwards the previous
// totals + 50 % slack, grown at list rebuilds (MD) or by the retry of a single evaluation; the
// backward kernels refuse to write past it (DEV_PBUF).
void Engine::size_pbuf_if_needed() {
  if (pbuf_cap != 0) return;
  DPB_CUDA(cudaDeviceSynchronize());
  grow_pbuf();
}

void Engine::launch_env_exact() {
  TabParams p = make_params(*this);
  p.tn = 0;
  p.counters = exact_ctr.p;
  if (p.E > 0) {
    k_env_fwd<<<ceil_div(p.E, 256), 256, 0, stream>>>(p);
    ++launches;
  }
}

void Engine::grow_pbuf() {
  if (!h_gtotal) return;
  // one region per buffer set, each sized for the largest chunk seen (+50 %)
  int64_t tot = 0;
  for (int c = 0; c < n_chunks; ++c) tot = std::max(tot, h_gtotal[c]);
  const int64_t want = tot + tot / 2 + 1024;
  if (want > pbuf_cap) {
    Pbuf.ensure(static_cast<size_t>(want) * 24 * ck_sets);
    pbuf_cap = want;
  }
}

void Engine::tab_bwd_range(int, int64_t i0, int64_t i1, cudaStream_t st) {
  TabParams p = chunk_params(*this, i0, i1);
  const int sms = sm_count(device);
  double* dTw = wa(dTbuf, 4 * Mp);
  const int nblk_all = ceil_div(ck_cap_a, P2_NA);
  fb_list.ensure(2 * (nblk_all + 1));
  int* fbl = fb_list.p + cur_set * (nblk_all + 1);
  const int nblk = ceil_div(i1 - i0, P2_NA);
  switch (Mp / 32) {
#define DPB_DT(F) case F: launch_dT<F>(p, dTw, st, sms); break;
    DPB_DT(1) DPB_DT(2) DPB_DT(3) DPB_DT(4) DPB_DT(5) DPB_DT(6) DPB_DT(7) DPB_DT(8)
#undef DPB_DT
    default: throw InputErr("feature width 4*d1 must be at most 256");
  }
  ++launches;
  const bool tensor = Mp <= 128;
  const int* fl = nullptr;
  const int* fc = nullptr;
  if (tensor) {
    // 32-centre blocks on the FP64 tensor pipe; blocks with a too wide interval union are listed
    // and done by the per-warp kernel
    DPB_CUDA(cudaMemsetAsync(fbl + nblk_all, 0, sizeof(int), st));
    const size_t bytes = p2_smem_bytes(Mp);
    switch (Mp / 32) {
#define DPB_P2(F)                                                                                             \
  case F:                                                                                                     \
    DPB_CUDA(cudaFuncSetAttribute(k_tab_bwd_P2<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,              \
                                  static_cast<int>(bytes)));                                                  \
    k_tab_bwd_P2<F><<<std::max(1, std::min(nblk, sms)), P2_THREADS, bytes, st>>>(p, dTw, fbl, fbl + nblk_all);   \
    break;
      DPB_P2(1) DPB_P2(2) DPB_P2(3) DPB_P2(4)
#undef DPB_P2
    }
    DPB_CUDA(cudaGetLastError());
    ++launches;
    fl = fbl;
    fc = fbl + nblk_all;
  }
  switch (Mp / 32) {
#define DPB_BW(F) case F: launch_bwd_warp<F>(p, dTw, fl, fc, P2_NA, st, sms); break;
    DPB_BW(1) DPB_BW(2) DPB_BW(3) DPB_BW(4) DPB_BW(5) DPB_BW(6) DPB_BW(7) DPB_BW(8)
#undef DPB_BW
    default: throw InputErr("feature width 4*d1 must be at most 256");
  }
  ++launches;
  const int64_t ne = std::min<int64_t>(p.es, p.E);
  if (ne > 0) {
    k_tab_bwd_g<<<ceil_div(ne, 256), 256, 0, st>>>(p);
    ++launches;
  }
}

void Engine::launch_tab_bwd() { tab_bwd_range(0, 0, n, stream); }


} // namespace dpb
