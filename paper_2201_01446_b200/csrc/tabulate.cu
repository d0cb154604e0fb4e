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
// Kernels (per evaluation chunk):
//   k_tab_fwd    one warp per centre: env-mat of the row (list order), real filter, interval,
//                compact per-real records (R, u, d) + list ranks (ridx), stable counting sort of
//                the reals by (type, interval), group moments, T = W . C, D = T<^T T
//   k_tab_dT2    two warps per centre: dT from dD (contract.hpp:21-38), dD and T rows streamed into
//                shared memory by bulk copies (k_tab_dT: the register-load version, fallback)
//   k_tab_bwd_P2 32 centres per CTA: interval projections P per group on DMMA (k_tab_bwd_P per
//                warp for blocks with a too wide interval union)
//   k_tab_bwd_g  one warp per centre: dE_i/dd_ij from P and the records, written compactly at
//                g[realoff[i] + k], and the centre's virial
// All reductions have a fixed order, so results are bitwise reproducible run to run.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "tab_common.cuh"
#include "tc_common.cuh"

namespace dpb {

namespace {

// ---------------------------------------------------------------- per-warp shared memory
constexpr int HCAP = 256; // counting-sort bins; wider (type, interval) ranges use a bitonic sort
constexpr int GB = 8;     // groups per batch
#ifndef TAB_FWD_MINB
#define TAB_FWD_MINB 8 // 2-warp CTAs per SM: 128 registers, 16 warps per SM
#endif

struct FwdSmem {
  uint32_t* rk; // [scap] bin of real k (list order)
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
// prod_env_mat + tabulate_fusion forward in one pass over the centre's row (fused.cpp:182-202):
//  A  entries in list order, 32 per step: key, neighbour position (one 32-byte gather), exact
//     displacement and r^2, the env-mat filter r^2 < r_c^2 (env_mat.cpp:32), s = w(r)/r, the
//     table interval (locate), R = (s, s d/r) and u = s - node. Every real entry gets its list
//     rank k (ridx, 16 bits) and a 64-byte record rec[k] = (R0..R3, u, d0..d2) -- written
//     densely, in rank order, into the chunk's record buffer, which the moments below and the
//     backward pass (k_tab_bwd_g) read back; nothing else per entry reaches HBM.
//  B  stable counting sort of the reals by (type, interval) -> groups (sort_and_group)
//  C  group moments W[a][m] = sum_k R_k[a] u_k^m (members in sorted order), then
//     T += W . C[interval] with lanes owning features
//  D  T out, D = T<^T T (contract.hpp:9-17) as the fitting input
// Features are owned in contiguous runs: lane l holds f = F*l .. F*l + F-1.
// F32 (mixed mode, SURVEY §8d C3 "mixed-precision tabulate_fusion"): the contraction T += W . C
// runs on FP32 coefficients and accumulators (half the coefficient traffic, 2x the FP64 rate);
// the moments W stay FP64. FP64 mode (F32 = false) is the parity path.
template <int F, bool F32 = false>
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
    if (!p.center[i]) {
      for (int e = lane; e < len; e += 32) p.ridx[off + e] = -1;
      if (lane == 0) {
        p.n_real[i] = 0;
        p.n_grp[i] = 0;
      }
      continue;
    }
    if (loff + len > p.es) { // chunk record capacity (sized from the list; never expected)
      if (lane == 0) raise_err(p.err, DEV_LIST_CAP);
      continue;
    }
    for (int t = lane; t < 64; t += 32) w.tc[t] = 0;
    __syncwarp();
    const double3 ri = ld_pos(p.pos, i);
    double* recs = p.rec + loff * 8;
    // --- A: env-mat of the row, compaction of the reals (list order) ---
    int nreal = 0, kmin = 0x7fffffff, kmax = -1;
    // software pipeline over 32-entry steps: keys two steps ahead, neighbour positions one
    uint64_t key_nx = lane < len ? p.keys[off + lane] : 0;
    uint64_t key_nx2 = 32 + lane < len ? p.keys[off + 32 + lane] : 0;
    double3 pj_nx = lane < len ? ld_pos(p.pos, key_j(key_nx)) : ri;
    for (int base = 0; base < len; base += 32) {
      const int e = base + lane;
      const bool valid = e < len;
      const uint64_t key = key_nx;
      const double3 pj = pj_nx;
      if (base + 32 < len) {
        key_nx = key_nx2;
        if (e + 32 < len) pj_nx = ld_pos(p.pos, key_j(key_nx));
        if (base + 64 < len) key_nx2 = e + 64 < len ? p.keys[off + e + 64] : 0;
      }
      double d[3] = {0.0, 0.0, 0.0};
      double r2 = 0.0;
      if (valid) {
        int sh[3];
        key_shift(key, sh);
        disp_exact(p.c, ri, pj, sh[0], sh[1], sh[2], d);
        r2 = norm2_exact(d);
        if (r2 < 1e-12) raise_err(p.err, DEV_OVERLAP); // env_mat.cpp:33
      }
      const bool real = valid && r2 >= 1e-12 && r2 < p.rc2;
      bool ext = false;
      int bin = -1;
      double R[4] = {0.0, 0.0, 0.0, 0.0}, uu = 0.0;
      if (real) {
        const double r = sqrt(r2);
        const double ir = 1.0 / r;
        const double s = switch_fn(r, p.rs, p.rc) * ir;
        const int th = locate(p, s, ext, p.err);
        bin = key_type(key) * p.tn + th;
        R[0] = s;
        R[1] = s * (d[0] * ir);
        R[2] = s * (d[1] * ir);
        R[3] = s * (d[2] * ir);
        uu = s - node_x(p.x0, p.h, th);
      }
      const unsigned m = __ballot_sync(0xffffffffu, real);
      const int k = nreal + __popc(m & ((1u << lane) - 1u));
      if (valid) p.ridx[off + e] = static_cast<int16_t>(real ? k : -1);
      const int t = real ? bin / p.tn : -1;
      if (real) {
        w.rk[k] = static_cast<uint32_t>(bin);
        double* rp = recs + static_cast<int64_t>(k) * 8;
        st4(rp, R[0], R[1], R[2], R[3]);
        st4(rp + 4, uu, d[0], d[1], d[2]);
        kmin = min(kmin, bin);
        kmax = max(kmax, bin);
      }
      const unsigned tm = __match_any_sync(0xffffffffu, t);
      if (real && (tm & ((1u << lane) - 1u)) == 0) w.tc[t] += __popc(tm);
      const unsigned xm = __ballot_sync(0xffffffffu, ext);
      if (lane == 0 && xm) atomicAdd(p.counters + 2, static_cast<unsigned long long>(__popc(xm)));
      nreal += __popc(m);
      __syncwarp();
    }
    kmin = warp_min(kmin);
    kmax = warp_max(kmax);
    for (int t = lane; t < p.n_types; t += 32)
      if (w.tc[t] > p.max_nbr[t]) raise_err(p.err, DEV_OVERFLOW); // env_mat.cpp:37-39
    // --- B: groups ---
    const int G = sort_and_group(w, p.sscr + loff, nreal, kmin, kmax, lane);
    if (lane == 0) {
      atomicAdd(p.counters + 0, static_cast<unsigned long long>(nreal));
      p.n_real[i] = nreal;
      p.n_grp[i] = G;
    }
    for (int g = lane; g < G; g += 32) {
      p.gbin[loff + g] = w.gb[g];
      for (int j = w.gs[g]; j < w.gs[g + 1]; ++j) p.egrp[loff + w.od[j]] = g;
    }
    __syncwarp(); // the records written above are read back by other lanes below
    // --- C: moments of each (type, interval) group, then T += W . C[interval] ---
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
        if constexpr (F % 4 == 0) {
#pragma unroll
          for (int q = 0; q < F; q += 4) {
            const double4 v = ldg4(C + mm * p.Mp + q);
            cn[mm][q] = static_cast<acc_t>(v.x);
            cn[mm][q + 1] = static_cast<acc_t>(v.y);
            cn[mm][q + 2] = static_cast<acc_t>(v.z);
            cn[mm][q + 3] = static_cast<acc_t>(v.w);
          }
        } else if constexpr (F % 2 == 0) {
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
          // members j, j + 4 (, j + 8, ...) of this lane in order; the records of two members
          // are requested before either is used
          for (int j = w.gs[g] + r; j < j1; j += 8) {
            const bool two = j + 4 < j1;
            const double* rp = recs + static_cast<int64_t>(w.od[j]) * 8;
            const double* rq = recs + static_cast<int64_t>(w.od[two ? j + 4 : j]) * 8;
            const double4 rv = ldc4(rp);
            const double uu = rp[4];
            const double4 rw = ldc4(rq);
            const double uw = rq[4];
            {
              const double R[4] = {rv.x, rv.y, rv.z, rv.w};
              double um = 1.0;
#pragma unroll
              for (int mm = 0; mm < 6; ++mm) {
#pragma unroll
                for (int a = 0; a < 4; ++a) Wv[a * 6 + mm] += R[a] * um;
                um *= uu;
              }
            }
            if (two) {
              const double R[4] = {rw.x, rw.y, rw.z, rw.w};
              double um = 1.0;
#pragma unroll
              for (int mm = 0; mm < 6; ++mm) {
#pragma unroll
                for (int a = 0; a < 4; ++a) Wv[a * 6 + mm] += R[a] * um;
                um *= uw;
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
        if (g < G)
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) w.W[gl * 24 + r * 6 + mm] = Wv[mm];
      }
      __syncwarp();
      const int gn = min(GB, G - g0);
      for (int gg = 0; gg < gn; ++gg) {
        const double2* Wg2 = reinterpret_cast<const double2*>(w.W + gg * 24); // 16-byte broadcasts
        acc_t c[6][F];
        load_c(g0 + gg, c);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int mp = 0; mp < 3; ++mp) {
            const double2 wv = Wg2[a * 3 + mp];
            const acc_t w0 = static_cast<acc_t>(wv.x), w1 = static_cast<acc_t>(wv.y);
#pragma unroll
            for (int q = 0; q < F; ++q) tacc[a][q] += w0 * c[2 * mp][q];
#pragma unroll
            for (int q = 0; q < F; ++q) tacc[a][q] += w1 * c[2 * mp + 1][q];
          }
        }
      }
      __syncwarp();
    }
    // --- D: T out, D = T<^T T (contract.hpp:9-17) ---
    double* ts = w.ts;
    double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if constexpr (F % 4 == 0) {
#pragma unroll
        for (int q = 0; q < F; q += 4) st4(Ti + a * p.Mp + f0 + q, tacc[a][q], tacc[a][q + 1], tacc[a][q + 2], tacc[a][q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < F; ++q) Ti[a * p.Mp + f0 + q] = tacc[a][q];
      }
#pragma unroll
      for (int q = 0; q < F; ++q) ts[a * p.Mp + f0 + q] = tacc[a][q];
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
        if constexpr (F % 4 == 0) {
          if ((p.M & 3) == 0) {
#pragma unroll
            for (int q = 0; q < F; q += 4) st4(dst + q, dv[q], dv[q + 1], dv[q + 2], dv[q + 3]);
            continue;
          }
        }
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
__global__ void __launch_bounds__(256, 1) k_tab_dT(TabParams p, double* __restrict__ dTg) {
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
    const double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
    double tv[4][F], dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      if constexpr (F % 4 == 0) {
#pragma unroll
        for (int q = 0; q < F; q += 4) {
          const double4 v = ldg4(Ti + a * p.Mp + f0 + q);
          tv[a][q] = v.x;
          tv[a][q + 1] = v.y;
          tv[a][q + 2] = v.z;
          tv[a][q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < F; ++q) tv[a][q] = Ti[a * p.Mp + f0 + q];
      }
#pragma unroll
      for (int q = 0; q < F; ++q) {
        ts[a * p.Mp + f0 + q] = tv[a][q];
        dT[a][q] = 0.0;
      }
    }
    __syncwarp();
    const int slot = p.slot_of[i];
    const double* dDrow = p.dD + static_cast<size_t>(slot < 0 ? 0 : slot) * p.K0p;
    const bool fon = f0 < p.M && slot >= 0;
    const bool vec = ((p.M | p.K0p) & 1) == 0; // 16-byte aligned dD pairs
    const bool vec4 = ((p.M | p.K0p) & 3) == 0; // 32-byte aligned dD quads
    // the dD rows of up to QB features q are loaded together (all 16 rows of the Cu model at F = 4:
    // 16 KB in flight per warp, so HBM sees enough requests), then contracted in ascending q
    constexpr int QB = (64 / F) < 16 ? (64 / F) : 16;
    for (int q0 = 0; q0 < p.mlt; q0 += QB) {
      double dq[QB][F];
#pragma unroll
      for (int ql = 0; ql < QB; ++ql) {
        const int qq = q0 + ql;
        const bool on = fon && qq < p.mlt;
        if constexpr (F % 4 == 0) {
          if (vec4) {
#pragma unroll
            for (int q = 0; q < F; q += 4) {
              const double4 v = on ? ldg4(dDrow + qq * p.M + f0 + q) : make_double4(0.0, 0.0, 0.0, 0.0);
              dq[ql][q] = v.x;
              dq[ql][q + 1] = v.y;
              dq[ql][q + 2] = v.z;
              dq[ql][q + 3] = v.w;
            }
            continue;
          }
        }
        if constexpr (F % 2 == 0) {
          if (vec) {
#pragma unroll
            for (int q = 0; q < F; q += 2) {
              const double2 v = on ? __ldg(reinterpret_cast<const double2*>(dDrow + qq * p.M + f0 + q))
                                   : make_double2(0.0, 0.0);
              dq[ql][q] = v.x;
              dq[ql][q + 1] = v.y;
            }
            continue;
          }
        }
#pragma unroll
        for (int q = 0; q < F; ++q) dq[ql][q] = on ? dDrow[qq * p.M + f0 + q] : 0.0;
      }
#pragma unroll
      for (int qb = 0; qb < QB; qb += 4) {
        double part[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) part[k] = 0.0;
#pragma unroll
        for (int ql = 0; ql < 4; ++ql) {
          const int qq = q0 + qb + ql;
          if (qb + ql < QB && qq < p.mlt) {
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const double ta = ts[a * p.Mp + qq];
#pragma unroll
              for (int q = 0; q < F; ++q) {
                dT[a][q] += dq[qb + ql][q] * ta;
                part[ql * 4 + a] += dq[qb + ql][q] * tv[a][q];
              }
            }
          }
        }
        const double sv = rs16(part, lane);
        if (lane < 16 && q0 + qb + (lane >> 2) < p.mlt) S[(q0 + qb + (lane >> 2)) * 4 + (lane & 3)] = sv;
      }
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
    for (int a = 0; a < 4; ++a) {
      if constexpr (F % 4 == 0) {
#pragma unroll
        for (int q = 0; q < F; q += 4) st4(out + a * p.Mp + f0 + q, dT[a][q], dT[a][q + 1], dT[a][q + 2], dT[a][q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < F; ++q) out[a * p.Mp + f0 + q] = dT[a][q];
      }
    }
    __syncwarp();
    if (lane == 0) atomicAdd(p.counters + 1, static_cast<unsigned long long>(p.n_real[i]));
  }
}

// ---------------------------------------------------------------- k_tab_dT2 (bulk-copy stream)
// k_tab_dT with the centre's dD row (mlt x M) and T row (4 x Mp) brought into shared memory by
// one bulk copy each (cp.async.bulk + mbarrier), double-buffered per CTA: the copies of the next
// centre are in flight while the current one is contracted. DT2_W warps per centre, each summing
// its share of the q rows of dT[a][p] = sum_q dD[q][p] T[a][q] (shares combined in warp order)
// and the S[q][a] = sum_p dD[q][p] T[a][p] of its own q; lane owns features p = lane + 32 f.
constexpr int DT2_W = 2;
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   tc::smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(tc::smem_u32(mbar))
               : "memory");
}

__host__ __device__ inline size_t dt2_cta_doubles(int M, int Mp, int mlt) {
  // two buffers (dD row + T row), S, the dT shares of warps 1.., two mbarriers
  return 2 * (static_cast<size_t>(mlt) * M + 4 * static_cast<size_t>(Mp)) + 4 * static_cast<size_t>(mlt) +
         (DT2_W - 1) * 4 * static_cast<size_t>(Mp) + 2;
}

template <int F>
__global__ void __launch_bounds__(32 * DT2_W) k_tab_dT2(TabParams p, double* __restrict__ dTg) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const size_t bufd = static_cast<size_t>(p.mlt) * p.M + 4 * static_cast<size_t>(p.Mp);
  double* base = reinterpret_cast<double*>(smem);
  double* S = base + 2 * bufd;       // [mlt][4]
  double* H = S + 4 * p.mlt;         // [W - 1][4][Mp] dT shares of warps 1..
  uint64_t* mbar = reinterpret_cast<uint64_t*>(H + (DT2_W - 1) * 4 * p.Mp);
  const uint32_t dbytes = static_cast<uint32_t>(p.mlt) * p.M * 8, tbytes = 4u * p.Mp * 8;
  if (threadIdx.x == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  const int qh = (((p.mlt + DT2_W - 1) / DT2_W) + 3) & ~3; // multiple of 4 (rs16 blocks)
  const int qa = wid * qh, qb = min(p.mlt, qa + qh); // this warp's q rows
  const int stride = gridDim.x;
  auto issue = [&](int i, int b, bool cen, int slot) {
    if (threadIdx.x == 0 && cen) {
      double* db = base + b * bufd;
      tc::mbar_expect_tx(&mbar[b], dbytes + tbytes);
      bulk_g2s(db, p.dD + static_cast<size_t>(slot) * p.K0p, dbytes, &mbar[b]);
      bulk_g2s(db + static_cast<size_t>(p.mlt) * p.M, p.T + static_cast<size_t>(i) * 4 * p.Mp, tbytes, &mbar[b]);
    }
  };
  uint32_t phase[2] = {0u, 0u};
  // centre flag, slot and real count of the centre after next are loaded one step ahead
  int i = p.i0 + blockIdx.x;
  bool cen_c = false, cen_n = false;
  int slot_n = 0, nr_c = 0, nr_n = 0;
  unsigned long long rows = 0; // rows_backward of this CTA's centres, added once at the end
  if (i < p.i1) {
    cen_c = p.center[i];
    nr_c = p.n_real[i];
    issue(i, 0, cen_c, p.slot_of[i]);
  }
  if (i + stride < p.i1) {
    cen_n = p.center[i + stride];
    slot_n = p.slot_of[i + stride];
    nr_n = p.n_real[i + stride];
  }
  for (int n = 0; i < p.i1; ++n, i += stride) {
    const int b = n & 1;
    const bool cen = cen_c;
    const int nr = nr_c;
    if (i + stride < p.i1) issue(i + stride, b ^ 1, cen_n, slot_n);
    cen_c = cen_n;
    nr_c = nr_n;
    if (i + 2 * stride < p.i1) {
      cen_n = p.center[i + 2 * stride];
      slot_n = p.slot_of[i + 2 * stride];
      nr_n = p.n_real[i + 2 * stride];
    }
    double* out = dTg + static_cast<size_t>(i) * 4 * p.Mp;
    if (!cen) {
      if (wid == 0)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int f = 0; f < F; ++f) out[a * p.Mp + lane + 32 * f] = 0.0;
      continue;
    }
    tc::mbar_wait(&mbar[b], phase[b]);
    phase[b] ^= 1u;
    const double* db = base + b * bufd;
    const double* tb = db + static_cast<size_t>(p.mlt) * p.M;
    double tv[4][F], dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int f = 0; f < F; ++f) {
        tv[a][f] = tb[a * p.Mp + lane + 32 * f];
        dT[a][f] = 0.0;
      }
    for (int q0 = qa; q0 < qb; q0 += 4) {
      double part[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) part[k] = 0.0;
#pragma unroll
      for (int ql = 0; ql < 4; ++ql) {
        const int qq = q0 + ql;
        if (qq < qb) {
          double dq[F];
#pragma unroll
          for (int f = 0; f < F; ++f) dq[f] = lane + 32 * f < p.M ? db[qq * p.M + lane + 32 * f] : 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const double ta = tb[a * p.Mp + qq];
#pragma unroll
            for (int f = 0; f < F; ++f) {
              dT[a][f] += dq[f] * ta;
              part[ql * 4 + a] += dq[f] * tv[a][f];
            }
          }
        }
      }
      const double sv = rs16(part, lane);
      if (lane < 16 && q0 + (lane >> 2) < qb) S[(q0 + (lane >> 2)) * 4 + (lane & 3)] = sv;
    }
    if (wid > 0)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int f = 0; f < F; ++f) H[((wid - 1) * 4 + a) * p.Mp + lane + 32 * f] = dT[a][f];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        const int pp = lane + 32 * f;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          double v = dT[a][f];
#pragma unroll
          for (int w = 1; w < DT2_W; ++w) v += H[((w - 1) * 4 + a) * p.Mp + pp];
          if (pp < p.mlt) v += S[pp * 4 + a];
          out[a * p.Mp + pp] = v;
        }
      }
      rows += static_cast<unsigned long long>(nr);
    }
    // shared-memory reads of this buffer (and of S, H) are done before they are overwritten
    tc::fence_proxy_async();
    __syncthreads();
  }
  if (threadIdx.x == 0 && rows) atomicAdd(p.counters + 1, rows);
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
    int G = p.n_grp[i];
    if (p.goff[i] + G > p.pcap) {
      if (lane == 0) raise_err(p.err, DEV_PBUF);
      G = 0;
    }
    const int32_t* gbins = p.gbin + (off - eb); // the centre's group bins, ascending
    double* Pout = p.Pbuf + p.goff[i] * 24;
    const double* dTi = dTg + static_cast<size_t>(i) * 4 * p.Mp;
    double dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) dT[a][q] = dTi[a * p.Mp + f0 + q];
    // --- P[a][m] = sum_p dT[a][p] C[m][p] per group (reduce-scatter over the feature lanes) ---
    for (int g = 0; g < G; ++g) {
      {
        const int bin = gbins[g];
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
constexpr int P2_NA = 16, P2_CB = 4, P2_UCAP = 128, P2_UW = P2_UCAP / 32, P2_BMW = 256;
// 8 warps, one m-tile (2 centres x 4 rows) each, whose dT rows live in registers as DMMA A
// fragments; two CTAs per SM, so one block's union set-up overlaps the other's MMAs
constexpr int P2_THREADS = 256;

__host__ __device__ inline size_t p2_smem_bytes(int Mp) {
  const int pitch = Mp + 4;
  return static_cast<size_t>(2 * 6 * P2_CB) * pitch * sizeof(double) +
         (2 * P2_BMW + P2_UCAP + P2_NA / 2 * P2_UW + 4) * sizeof(int) + P2_NA * P2_UCAP * sizeof(int16_t);
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int F>
__global__ void __launch_bounds__(P2_THREADS, 2) k_tab_bwd_P2(TabParams p, const double* __restrict__ dTg,
                                                       int* __restrict__ fb_list, int* __restrict__ fb_count) {
  constexpr int Mp = 32 * F, pitch = Mp + 4, units = Mp / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  double* Cs = reinterpret_cast<double*>(smem);                          // [2][24][pitch]
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
    // this warp's m-tile of dT (rows warp*8 + gid, contiguous in dTg) as DMMA A fragments:
    // afr[j] = dT[row][4 j + tig]; in flight during the union set-up below
    double afr[Mp / 4];
    {
      const int r = warp * 8 + gid;
      const bool ok = i0 + (r >> 2) < p.i1;
      const double* src = dTg + (static_cast<size_t>(i0) * 4 + r) * Mp + tig;
#pragma unroll
      for (int j = 0; j < Mp / 4; ++j) afr[j] = ok ? __ldg(src + 4 * j) : 0.0;
    }
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
      const double* b0 = cs + gid * pitch + tig;
      // n-tile nt covers chunk slots {nt, nt+1} (columns 8 nt .. 8 nt + 7 of 6 per slot); the
      // m-tile needs it only if one of its two centres has one of those intervals
      const int sh = (ch * P2_CB) & 31, wd = (ch * P2_CB) >> 5;
      const unsigned n0 = (mtmask[warp * P2_UW + wd] >> sh) & 15u;
      const unsigned use = ((n0 & 3u) ? 1u : 0u) | ((n0 & 6u) ? 2u : 0u) | ((n0 & 12u) ? 4u : 0u);
      if (use == 7u) {
#pragma unroll
        for (int j = 0; j < Mp / 4; ++j) {
          const int k = 4 * j;
          const double av0 = afr[j];
          const double bv0 = b0[k], bv1 = b0[8 * pitch + k], bv2 = b0[16 * pitch + k];
          dmma884(acc[0][0][0], acc[0][0][1], av0, bv0);
          dmma884(acc[0][1][0], acc[0][1][1], av0, bv1);
          dmma884(acc[0][2][0], acc[0][2][1], av0, bv2);
        }
      } else if (use) {
#pragma unroll
        for (int j = 0; j < Mp / 4; ++j) {
          const int k = 4 * j;
          const double av0 = afr[j];
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
        // columns 2 tig, 2 tig + 1 of an n-tile are (slot, m), (slot, m + 1) with m even: one
        // 16-byte store per n-tile (P rows are 192 B, m pairs 16-byte aligned)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt) {
          const int u = ch * P2_CB + cslot[2 * nt];
          const int g = u < U ? gi[cslot[2 * nt]] : -1;
          if (g >= 0)
            *reinterpret_cast<double2*>(pb + static_cast<int64_t>(g) * 24 + cm[2 * nt]) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------- k_tab_bwd_g (warp per centre)
// Gradient pass of fused_atom_energy (fused.cpp:203-242) per real neighbour k (lane k mod 32),
// from its record (R, u, d) and its group's projections P:
//   drow[a] = sum_m u^m P[a][m],  ds = sum_a R[a] sum_m m u^(m-1) P[a][m],  drow[0] += ds,
//   g = sum_a drow[a] dR[a]/dd   (= dE_i/dd_ij, env_mat.cpp:55-71 derivatives)
// written compactly at g[realoff[i] + k], plus the centre's virial sum_k d_k (x) g_k (the
// reference scatter, exact.cpp:34) reduced in a fixed order: lane k mod 32, then a warp tree.
__global__ void __launch_bounds__(256) k_tab_bwd_g(TabParams p) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int64_t eb = p.row_off[p.i0];
  for (int i = p.i0 + blockIdx.x * wpb + (threadIdx.x >> 5); i < p.i1; i += gridDim.x * wpb) {
    if (!p.center[i]) continue;
    const int nreal = p.n_real[i];
    const int64_t loff = p.row_off[i] - eb;
    const int64_t ro = p.realoff[i];
    const int64_t gb0 = p.goff[i];
    double vir[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) vir[k] = 0.0;
    const bool fits = ro + nreal <= p.gcap && gb0 + p.n_grp[i] <= p.pcap;
    if (!fits && lane == 0) raise_err(p.err, ro + nreal > p.gcap ? DEV_GCAP : DEV_PBUF);
    for (int k = lane; fits && k < nreal; k += 32) {
      const double* rp = p.rec + (loff + k) * 8;
      const int grp = p.egrp[loff + k];
      const double4 ra = ldg4(rp), rb = ldg4(rp + 4);
      const double R[4] = {ra.x, ra.y, ra.z, ra.w};
      const double uu = rb.x;
      const double d[3] = {rb.y, rb.z, rb.w};
      // the group's 24 projections as 6 32-byte loads (a Pbuf row is 192 B, 32-byte aligned)
      const double* Pg = p.Pbuf + (gb0 + grp) * 24;
      double P[24];
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double4 v = ldg4(Pg + 4 * q);
        P[4 * q] = v.x;
        P[4 * q + 1] = v.y;
        P[4 * q + 2] = v.z;
        P[4 * q + 3] = v.w;
      }
      // env-mat derivative terms from d, exactly as the forward pass evaluated them
      const double r = sqrt(norm2_exact(d));
      const double wv = switch_fn(r, p.rs, p.rc);
      const double ir = 1.0 / r;
      const double s = wv * ir;
      const double sd = switch_deriv(r, p.rs, p.rc) * ir - wv * ir * ir;
      const double u[3] = {d[0] * ir, d[1] * ir, d[2] * ir};
      double drow[4], dsum = 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double* Pa = P + a * 6;
        drow[a] = ((((Pa[5] * uu + Pa[4]) * uu + Pa[3]) * uu + Pa[2]) * uu + Pa[1]) * uu + Pa[0];
        const double h1 = (((5.0 * Pa[5] * uu + 4.0 * Pa[4]) * uu + 3.0 * Pa[3]) * uu + 2.0 * Pa[2]) * uu + Pa[1];
        dsum += R[a] * h1;
      }
      drow[0] += dsum;
      double dR[12];
#pragma unroll
      for (int x = 0; x < 3; ++x) dR[x] = sd * u[x];
#pragma unroll
      for (int y = 0; y < 3; ++y)
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          double v = sd * u[x] * u[y] - s * ir * u[x] * u[y];
          if (x == y) v += s * ir;
          dR[3 * (1 + y) + x] = v;
        }
      double gv[3];
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) acc += drow[a] * dR[3 * a + x];
        gv[x] = acc;
      }
      double* ge = p.g + 3 * (ro + k);
      ge[0] = gv[0];
      ge[1] = gv[1];
      ge[2] = gv[2];
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) vir[3 * x + y] += d[x] * gv[y];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) vir[k] = warp_sum(vir[k]);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 9; ++k) p.vpart[9 * static_cast<int64_t>(i) + k] = vir[k];
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
  static const bool legacy = std::getenv("DPB_DT_LEGACY") != nullptr;
  const size_t b2 = dt2_cta_doubles(p.M, p.Mp, p.mlt) * sizeof(double);
  if (!legacy && b2 <= 110 * 1024 && (p.M & 1) == 0 && (p.Mp & 1) == 0 && (p.K0p & 1) == 0) {
    smem_optin(k_tab_dT2<F>, b2);
    int per_sm = 1;
    DPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tab_dT2<F>, 32 * DT2_W, b2));
    const int blocks = std::max(1, std::min(p.i1 - p.i0, sms * std::max(per_sm, 1)));
    k_tab_dT2<F><<<blocks, 32 * DT2_W, b2, st>>>(p, dTg);
    DPB_CUDA(cudaGetLastError());
    return;
  }
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

// Pair-gradient base of the chunk after this one (evaluation order): its base + its real pairs.
__global__ void k_real_end(const int32_t* __restrict__ n_real, const int64_t* __restrict__ realoff, int i0, int i1,
                           const int64_t* __restrict__ base, int64_t* __restrict__ next) {
  if (threadIdx.x == 0 && blockIdx.x == 0) *next = i1 > i0 ? realoff[i1 - 1] + n_real[i1 - 1] : *base;
}

// FP32 copy of the coefficient table for the mixed-mode forward contraction
void Engine::ensure_tab32() {
  if (precision != 1 || tab32_ver == tab_ver) return;
  const int64_t cnt = static_cast<int64_t>(n_types) * static_cast<int64_t>(tab_n) * 6 * Mp;
  tab32.ensure(cnt);
  k_to_f32<<<ceil_div(cnt, 256), 256, 0, stream>>>(cnt, tab.p, tab32.p);
  DPB_CUDA(cudaStreamSynchronize(stream));
  tab32_ver = tab_ver;
}

// k_tab_fwd over centres [i0, i1) of chunk k (q-th in evaluation order), then the chunk's group
// offsets (goff[i0..i1) start at 0; the chunk's buffer set owns Pbuf[set * pbuf_cap ...]) and its
// compact pair-gradient offsets realoff[i0..i1) = rbase[q] + exclusive scan of n_real.
void Engine::tab_fwd_range(int k, int q, int64_t i0, int64_t i1, cudaStream_t st) {
  ensure_tab32();
  TabParams p = chunk_params(*this, i0, i1);
  const int sms = sm_count(device);
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
  DevBuf<unsigned char>& tmp = cur_set == 0 ? scan_tmp : scan_tmp2;
  const int cnt = static_cast<int>(i1 - i0);
  size_t tb = 0, tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, n_grp.p + i0, goff.p + i0, cnt, st);
  cub::DeviceScan::ExclusiveScan(nullptr, tb2, n_real.p + i0, realoff.p + i0, cuda::std::plus<int64_t>(),
                                 cub::FutureValue<int64_t>(rbase.p + q), cnt, st);
  tmp.ensure(std::max(tb, tb2) + 1);
  // group offsets of the chunk -> goff, its total -> h_gtotal[k] (pinned, read at Pbuf sizing)
  cub::DeviceScan::ExclusiveSum(tmp.p, tb, n_grp.p + i0, goff.p + i0, cnt, st);
  gtot.ensure(MAX_CHUNKS);
  k_group_total<<<1, 32, 0, st>>>(n_grp.p, goff.p, static_cast<int>(i0), static_cast<int>(i1), gtot.p + k);
  if (!h_gtotal) {
    DPB_CUDA(cudaMallocHost(&h_gtotal, MAX_CHUNKS * sizeof(int64_t)));
    std::memset(h_gtotal, 0, MAX_CHUNKS * sizeof(int64_t));
  }
  DPB_CUDA(cudaMemcpyAsync(h_gtotal + k, gtot.p + k, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  // compact pair-gradient slots: realoff = base of this chunk + exclusive scan of n_real
  cub::DeviceScan::ExclusiveScan(tmp.p, tb2, n_real.p + i0, realoff.p + i0, cuda::std::plus<int64_t>(),
                                 cub::FutureValue<int64_t>(rbase.p + q), cnt, st);
  k_real_end<<<1, 32, 0, st>>>(n_real.p, realoff.p, static_cast<int>(i0), static_cast<int>(i1), rbase.p + q,
                               rbase.p + q + 1);
  launches += 4;
}

void Engine::launch_tab_fwd() {
  DPB_CUDA(cudaMemsetAsync(rbase.p, 0, sizeof(int64_t), stream));
  tab_fwd_range(0, 0, 0, n, stream);
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

void Engine::grow_pbuf() {
  if (!h_gtotal) return;
  // one region per buffer set, sized for the largest chunk: the highest groups-per-centre rate
  // seen in any evaluated chunk x the largest chunk's centres, +50 %
  double rate = 0.0;
  int64_t cmax = 0;
  for (int c = 0; c < n_chunks; ++c) {
    const int64_t cc = ck_s[c + 1] - ck_s[c];
    cmax = std::max(cmax, cc);
    if (cc > 0 && h_gtotal[c] > 0) rate = std::max(rate, static_cast<double>(h_gtotal[c]) / static_cast<double>(cc));
  }
  const int64_t tot = static_cast<int64_t>(std::ceil(rate * static_cast<double>(cmax)));
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
    k_tab_bwd_P2<F><<<std::max(1, std::min(nblk, 2 * sms)), P2_THREADS, bytes, st>>>(p, dTw, fbl, fbl + nblk_all);   \
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
  if (i1 > i0) {
    // persistent: one resident wave of CTAs striding over the centres (non-persistent 8-centre
    // CTAs: C2 4.244 -> 4.227 ms/step)
    int per_sm = 1;
    DPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tab_bwd_g, 256, 0));
    k_tab_bwd_g<<<std::max(1, std::min(ceil_div(i1 - i0, 8), sms * std::max(per_sm, 1))), 256, 0, st>>>(p);
    ++launches;
  }
}

void Engine::launch_tab_bwd() { tab_bwd_range(0, 0, n, stream); }


} // namespace dpb
