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
// One warp per centre; lanes own features in the contraction and neighbours in the env-mat.
#include "engine.hpp"

namespace dpb {

namespace {

struct TabParams {
  const double4* pos;
  const int64_t* row_off;
  const uint64_t* keys;
  uint64_t* skeys;
  int32_t* n_real;
  const double* tab; // [type][interval][6][Mp]
  const int* max_nbr;
  DevCell c;
  double rc2, rs, rc;
  double x0, h, x_end;
  long tn;
  int n, n_types, M, Mp, mlt, K0p;
  const int32_t* slot_of;
  double* T;  // [n][4][Mp]
  double* D;  // [slots][K0p]
  const double* dD;
  double* g;        // [E][3]
  double* fcenter;  // [n][3]
  double* vpart;    // [n][9]
  unsigned long long* counters;
  int* err;
  int scap;
};

__device__ __forceinline__ double node_x(double x0, double h, long th) {
  return __dadd_rn(x0, __dmul_rn(static_cast<double>(th), h));
}

// locate (table.cpp:20-32): floor, then nudge so node(th) <= x < node(th+1) in the exact
// arithmetic of the nodes; clamp past the end and flag extrapolation.
__device__ __forceinline__ long locate(const TabParams& p, double x, bool& ext, int* err) {
  if (!(x >= p.x0)) {
    raise_err(err, DEV_TABLE_LOW);
    ext = false;
    return 0;
  }
  const double tf = floor(__ddiv_rn(__dsub_rn(x, p.x0), p.h));
  if (!(tf < static_cast<double>(p.tn) + 2.0)) {  // far past the end (or inf): clamp directly
    ext = true;
    return p.tn - 1;
  }
  long th = static_cast<long>(tf);
  while (node_x(p.x0, p.h, th + 1) <= x) ++th;
  while (th > 0 && node_x(p.x0, p.h, th) > x) --th;
  ext = false;
  if (th >= p.tn) {
    th = p.tn - 1;
    ext = x > p.x_end;
  }
  return th;
}

__device__ __forceinline__ double switch_fn(double r, double rs, double rc) {
  if (r >= rc) return 0.0;
  if (r <= rs) return 1.0;
  const double u = (r - rs) / (rc - rs);
  const double uu = u * u;
  return fmax(0.0, uu * u * (-6.0 * uu + 15.0 * u - 10.0) + 1.0);
}

__device__ __forceinline__ double switch_deriv(double r, double rs, double rc) {
  if (r >= rc || r <= rs) return 0.0;
  const double inv = 1.0 / (rc - rs);
  const double u = (r - rs) * inv;
  const double um1 = u - 1.0;
  return -30.0 * u * u * um1 * um1 * inv;
}

// Environment of one real neighbour (env_mat.cpp:29-71).
struct Env {
  double d[3], r, ir, s, sd, u[3];
};

__device__ __forceinline__ void env_of(const TabParams& p, double3 ri, uint64_t key, Env& e) {
  int sh[3];
  key_shift(key, sh);
  disp_exact(p.c, ri, ld_pos(p.pos, key_j(key)), sh[0], sh[1], sh[2], e.d);
  const double r2 = norm2_exact(e.d);
  e.r = sqrt(r2);
  const double w = switch_fn(e.r, p.rs, p.rc);
  e.ir = 1.0 / e.r;
  e.s = w * e.ir;
  e.sd = switch_deriv(e.r, p.rs, p.rc) * e.ir - w * e.ir * e.ir;
#pragma unroll
  for (int x = 0; x < 3; ++x) e.u[x] = e.d[x] * e.ir;
}

// ---------------------------------------------------------------- per-warp shared memory
// Forward: reals in list order (bin, entry, stable rank), sorted order, bin histogram, groups,
// a cache of (R[4], u) for the first NC reals, one batch of group moments, and T for D.
// Backward: sorted (bin, entry) keys, groups, one batch of interval projections P, T.
constexpr int NC = 256;   // cached reals per centre (the rest are recomputed)
constexpr int HCAP = 512; // counting-sort bins; wider ranges fall back to a bitonic sort
constexpr int GB = 8;     // groups per batch

struct FwdSmem {
  uint32_t* rk;  // [scap] global bin t*tn + interval of real k
  uint16_t* ex;  // [scap] list entry of real k
  uint16_t* rn;  // [scap] stable rank of real k inside its bin
  uint16_t* od;  // [scap] sorted position -> k
  int* hs;       // [HCAP + 1] bin counts -> bin starts
  int* gs;       // [gcap + 1] group start (sorted positions)
  int* gb;       // [gcap] group bin
  int* tc;       // [64] per-type real counts
  double* W;     // [GB][24] moments of one batch
  double* cache; // [5][NC] R0..R3, u  (aliased: bitonic scratch, then T copy)
};

__host__ __device__ __forceinline__ size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ __forceinline__ size_t fwd_cache_bytes(int scap, int Mp) {
  size_t c = static_cast<size_t>(5) * NC * 8;
  if (static_cast<size_t>(scap) * 8 > c) c = static_cast<size_t>(scap) * 8;
  if (static_cast<size_t>(4) * Mp * 8 > c) c = static_cast<size_t>(4) * Mp * 8;
  return c;
}

__host__ __device__ __forceinline__ int gcap_of(int scap) { return scap > HCAP ? scap : HCAP; }

__host__ __device__ __forceinline__ size_t fwd_smem_bytes(int scap, int Mp) {
  const int gcap = gcap_of(scap);
  size_t b = fwd_cache_bytes(scap, Mp) + GB * 24 * 8;
  b += static_cast<size_t>(scap) * (4 + 2 + 2 + 2);
  b += static_cast<size_t>(HCAP + 1) * 4 + static_cast<size_t>(2 * gcap + 1) * 4 + 64 * 4;
  return align16(b);
}

__device__ __forceinline__ FwdSmem carve_fwd(unsigned char* base, int scap, int Mp) {
  FwdSmem w;
  w.cache = reinterpret_cast<double*>(base);
  unsigned char* p = base + fwd_cache_bytes(scap, Mp);
  w.W = reinterpret_cast<double*>(p);
  p += GB * 24 * 8;
  w.rk = reinterpret_cast<uint32_t*>(p);
  p += static_cast<size_t>(scap) * 4;
  w.hs = reinterpret_cast<int*>(p);
  p += (HCAP + 1) * 4;
  const int gcap = gcap_of(scap);
  w.gs = reinterpret_cast<int*>(p);
  p += (gcap + 1) * 4;
  w.gb = reinterpret_cast<int*>(p);
  p += gcap * 4;
  w.tc = reinterpret_cast<int*>(p);
  p += 64 * 4;
  w.ex = reinterpret_cast<uint16_t*>(p);
  p += static_cast<size_t>(scap) * 2;
  w.rn = reinterpret_cast<uint16_t*>(p);
  p += static_cast<size_t>(scap) * 2;
  w.od = reinterpret_cast<uint16_t*>(p);
  return w;
}

struct BwdSmem {
  uint64_t* sk; // [scap] sorted (bin << 32 | entry)
  int* gs;      // [gcap + 1]
  int* gb;      // [gcap]
  double* P;    // [GB][24]
  double* S;    // [m_lt <= 256][4] second term of dT
  double* ts;   // [4][Mp]
};

__host__ __device__ __forceinline__ size_t bwd_smem_bytes(int scap, int Mp) {
  const int gcap = gcap_of(scap);
  size_t b = static_cast<size_t>(scap) * 8 + GB * 24 * 8 + 256 * 4 * 8 + static_cast<size_t>(4) * Mp * 8;
  b += static_cast<size_t>(2 * gcap + 1) * 4;
  return align16(b);
}

__device__ __forceinline__ BwdSmem carve_bwd(unsigned char* base, int scap, int Mp) {
  BwdSmem w;
  w.sk = reinterpret_cast<uint64_t*>(base);
  unsigned char* p = base + static_cast<size_t>(scap) * 8;
  w.P = reinterpret_cast<double*>(p);
  p += GB * 24 * 8;
  w.S = reinterpret_cast<double*>(p);
  p += 256 * 4 * 8;
  w.ts = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(4) * Mp * 8;
  const int gcap = gcap_of(scap);
  w.gs = reinterpret_cast<int*>(p);
  p += (gcap + 1) * 4;
  w.gb = reinterpret_cast<int*>(p);
  return w;
}

// Warp bitonic sort of sk[0..n) ascending (pads to a power of two with ~0). Fallback only.
__device__ void warp_sort(uint64_t* sk, int n, int lane) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int t = n + lane; t < P; t += 32) sk[t] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < P; t += 32) {
        const int u = t ^ j;
        if (u > t) {
          const uint64_t x = sk[t], y = sk[u];
          if ((x > y) == ((t & k) == 0)) {
            sk[t] = y;
            sk[u] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Exclusive warp scan of non-negative ints.
__device__ __forceinline__ int warp_excl_scan(int v, int lane, int* total) {
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Reduce-scatter of 24 per-lane partials: afterwards every lane holds the full warp sums of
// entries base..base+2 with base = 12*b4 + 6*b3 + 3*b2 (b = lane bits). Deterministic.
__device__ __forceinline__ int rs24(double* v, int lane) {
  {
    const bool hi = lane & 16;
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const double send = hi ? v[i] : v[i + 12];
      const double keep = hi ? v[i + 12] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
  }
  {
    const bool hi = lane & 8;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const double send = hi ? v[i] : v[i + 6];
      const double keep = hi ? v[i + 6] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
  }
  {
    const bool hi = lane & 4;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double send = hi ? v[i] : v[i + 3];
      const double keep = hi ? v[i + 3] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    v[i] += __shfl_xor_sync(0xffffffffu, v[i], 2);
    v[i] += __shfl_xor_sync(0xffffffffu, v[i], 1);
  }
  return ((lane >> 4) & 1) * 12 + ((lane >> 3) & 1) * 6 + ((lane >> 2) & 1) * 3;
}

// Reduce-scatter of 32 per-lane partials: afterwards lane l holds the warp sum of entry l.
__device__ __forceinline__ double rs32(double* v, int lane) {
#pragma unroll
  for (int lvl = 16; lvl >= 1; lvl >>= 1) {
    const bool hi = lane & lvl;
#pragma unroll
    for (int i = 0; i < lvl; ++i) {
      const double send = hi ? v[i] : v[i + lvl];
      const double keep = hi ? v[i + lvl] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, lvl);
    }
  }
  return v[0];
}

// Sort the nreal reals by bin (stable: list order inside a bin) and build the groups.
// Returns the group count. Counting sort over [kmin, kmax] when it fits HCAP bins, otherwise
// a bitonic sort of (bin, k) keys in the cache region (the cache is then unusable: *cache_ok=0).
__device__ int sort_and_group(const FwdSmem& w, int nreal, int kmin, int kmax, int lane,
                              bool* cache_ok) {
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
    // exclusive scan of counts, segment per lane; groups = non-empty bins
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
    __syncwarp();
  } else {
    *cache_ok = false;
    uint64_t* sk = reinterpret_cast<uint64_t*>(w.cache);
    for (int k = lane; k < nreal; k += 32) sk[k] = (static_cast<uint64_t>(w.rk[k]) << 16) | k;
    warp_sort(sk, nreal, lane);
    for (int base = 0; base < nreal; base += 32) {
      const int k = base + lane;
      bool head = false;
      if (k < nreal) {
        w.od[k] = static_cast<uint16_t>(sk[k] & 0xffff);
        head = (k == 0) || ((sk[k] >> 16) != (sk[k - 1] >> 16));
      }
      const unsigned m = __ballot_sync(0xffffffffu, head);
      if (head) {
        const int at = G + __popc(m & ((1u << lane) - 1u));
        w.gs[at] = k;
        w.gb[at] = static_cast<int>(sk[k] >> 16);
      }
      G += __popc(m);
    }
    if (lane == 0) w.gs[G] = nreal;
    __syncwarp();
  }
  return G;
}

template <int F>
__global__ void __launch_bounds__(64) k_tab_fwd(TabParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const FwdSmem w = carve_fwd(smem + wid * fwd_smem_bytes(p.scap, p.Mp), p.scap, p.Mp);
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  const int nc = NC < p.scap ? NC : p.scap;
  double* cR = w.cache;  // [4][NC]
  double* cU = w.cache + 4 * NC;
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    const double3 ri = ld_pos(p.pos, i);
    for (int t = lane; t < 64; t += 32) w.tc[t] = 0;
    __syncwarp();
    // --- pass 1: env-mat of every list entry, compaction of the reals ---
    int nreal = 0, next = 0, kmin = 0x7fffffff, kmax = -1;
    for (int base = 0; base < len; base += 32) {
      const int e = base + lane;
      bool real = false, ext = false;
      int bin = 0, t = 0;
      double R0 = 0, R1 = 0, R2 = 0, R3 = 0, ul = 0;
      if (e < len) {
        const uint64_t key = p.keys[off + e];
        int sh[3];
        key_shift(key, sh);
        double d[3];
        disp_exact(p.c, ri, ld_pos(p.pos, key_j(key)), sh[0], sh[1], sh[2], d);
        const double r2 = norm2_exact(d);
        if (r2 < 1e-12) {
          raise_err(p.err, DEV_OVERLAP); // env_mat.cpp:33 throws before any table lookup
        } else if (r2 < p.rc2) {
          real = true;
          const double r = sqrt(r2);
          const double ir = 1.0 / r;
          const double s = switch_fn(r, p.rs, p.rc) * ir;
          const long th = locate(p, s, ext, p.err);
          t = key_type(key);
          bin = static_cast<int>(t * p.tn + th);
          R0 = s;
          R1 = s * (d[0] * ir);
          R2 = s * (d[1] * ir);
          R3 = s * (d[2] * ir);
          ul = s - node_x(p.x0, p.h, th);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, real);
      const int at = nreal + __popc(m & ((1u << lane) - 1u));
      if (real) {
        w.rk[at] = static_cast<uint32_t>(bin);
        w.ex[at] = static_cast<uint16_t>(e);
        if (at < nc) {
          cR[at] = R0;
          cR[NC + at] = R1;
          cR[2 * NC + at] = R2;
          cR[3 * NC + at] = R3;
          cU[at] = ul;
        }
        kmin = min(kmin, bin);
        kmax = max(kmax, bin);
      }
      const unsigned tm = __match_any_sync(0xffffffffu, real ? t : -1);
      if (real && (tm & ((1u << lane) - 1u)) == 0) w.tc[t] += __popc(tm);
      nreal += __popc(m);
      next += __popc(__ballot_sync(0xffffffffu, ext));
      __syncwarp();
    }
    kmin = warp_min(kmin);
    kmax = warp_max(kmax);
    __syncwarp();
    for (int t = lane; t < p.n_types; t += 32)
      if (w.tc[t] > p.max_nbr[t]) raise_err(p.err, DEV_OVERFLOW);
    if (lane == 0) {
      atomicAdd(p.counters + 0, static_cast<unsigned long long>(nreal));
      if (next) atomicAdd(p.counters + 2, static_cast<unsigned long long>(next));
      p.n_real[i] = nreal;
    }
    bool cache_ok = true;
    const int G = sort_and_group(w, nreal, kmin, kmax, lane, &cache_ok);
    for (int j = lane; j < nreal; j += 32) {
      const int k = w.od[j];
      p.skeys[off + j] = (static_cast<uint64_t>(w.rk[k]) << 32) | w.ex[k];
    }
    // --- moments of each (type, interval) group, then T += W . C[interval] ---
    double tacc[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) tacc[a][q] = 0.0;
    for (int g0 = 0; g0 < G; g0 += GB) {
      {
        const int g = g0 + (lane >> 2), a = lane & 3;
        if (g < G) {
          double Wm[6] = {0, 0, 0, 0, 0, 0};
          const int j1 = w.gs[g + 1];
          const int th = w.gb[g] % static_cast<int>(p.tn);
          for (int j = w.gs[g]; j < j1; ++j) {
            const int k = w.od[j];
            double Ra, uu;
            if (cache_ok && k < nc) {
              Ra = cR[a * NC + k];
              uu = cU[k];
            } else {
              Env ev;
              env_of(p, ri, p.keys[off + w.ex[k]], ev);
              Ra = a == 0 ? ev.s : ev.s * ev.u[a - 1];
              uu = ev.s - node_x(p.x0, p.h, th);
            }
            double um = Ra;
#pragma unroll
            for (int mm = 0; mm < 6; ++mm) {
              Wm[mm] += um;
              um *= uu;
            }
          }
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) w.W[(lane >> 2) * 24 + a * 6 + mm] = Wm[mm];
        }
      }
      __syncwarp();
      const int gn = min(GB, G - g0);
      for (int gg = 0; gg < gn; ++gg) {
        const double* C = p.tab + static_cast<size_t>(w.gb[g0 + gg]) * istride;
        const double* Wg = w.W + gg * 24;
        double c[F][6];
#pragma unroll
        for (int q = 0; q < F; ++q)
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) c[q][mm] = __ldg(C + mm * p.Mp + lane + 32 * q);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          double wa[6];
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) wa[mm] = Wg[a * 6 + mm];
#pragma unroll
          for (int q = 0; q < F; ++q) {
            double acc = tacc[a][q];
#pragma unroll
            for (int mm = 0; mm < 6; ++mm) acc += wa[mm] * c[q][mm];
            tacc[a][q] = acc;
          }
        }
      }
      __syncwarp();
    }
    // --- T out, D = T<^T T (contract.hpp:9-17) ---
    double* ts = w.cache;
    double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) {
        Ti[a * p.Mp + lane + 32 * q] = tacc[a][q];
        ts[a * p.Mp + lane + 32 * q] = tacc[a][q];
      }
    __syncwarp();
    double* Drow = p.D + static_cast<size_t>(p.slot_of[i]) * p.K0p;
    for (int qq = 0; qq < p.mlt; ++qq) {
      const double t0 = ts[qq], t1 = ts[p.Mp + qq], t2 = ts[2 * p.Mp + qq], t3 = ts[3 * p.Mp + qq];
#pragma unroll
      for (int q = 0; q < F; ++q) {
        const int f = lane + 32 * q;
        if (f < p.M) {
          double acc = t0 * tacc[0][q];
          acc += t1 * tacc[1][q];
          acc += t2 * tacc[2][q];
          acc += t3 * tacc[3][q];
          Drow[qq * p.M + f] = acc;
        }
      }
    }
    __syncwarp();
  }
}

template <int F>
__global__ void __launch_bounds__(64) k_tab_bwd(TabParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const BwdSmem w = carve_bwd(smem + wid * bwd_smem_bytes(p.scap, p.Mp), p.scap, p.Mp);
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    const double3 ri = ld_pos(p.pos, i);
    for (int e = lane; e < 3 * len; e += 32) p.g[3 * off + e] = 0.0;
    const int nreal = p.n_real[i];
    for (int k = lane; k < nreal; k += 32) w.sk[k] = p.skeys[off + k];
    // --- dT = adjoint of D = T<^T T (contract.hpp:21-38) ---
    const double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
    double tv[4][F], dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) {
        tv[a][q] = Ti[a * p.Mp + lane + 32 * q];
        w.ts[a * p.Mp + lane + 32 * q] = tv[a][q];
        dT[a][q] = 0.0;
      }
    __syncwarp();
    const double* dDrow = p.dD + static_cast<size_t>(p.slot_of[i]) * p.K0p;
    for (int q0 = 0; q0 < p.mlt; q0 += 8) {
      double part[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) part[k] = 0.0;
#pragma unroll
      for (int ql = 0; ql < 8; ++ql) {
        const int qq = q0 + ql;
        if (qq < p.mlt) {
          double dq[F];
#pragma unroll
          for (int q = 0; q < F; ++q) {
            const int f = lane + 32 * q;
            dq[q] = f < p.M ? dDrow[qq * p.M + f] : 0.0;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const double ta = w.ts[a * p.Mp + qq];
#pragma unroll
            for (int q = 0; q < F; ++q) {
              dT[a][q] += dq[q] * ta;
              part[ql * 4 + a] += dq[q] * tv[a][q];
            }
          }
        }
      }
      const double s = rs32(part, lane);
      if (q0 + (lane >> 2) < p.mlt) w.S[(q0 + (lane >> 2)) * 4 + (lane & 3)] = s;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < F; ++q) {
      const int f = lane + 32 * q;
      if (f < p.mlt)
#pragma unroll
        for (int a = 0; a < 4; ++a) dT[a][q] += w.S[f * 4 + a];
    }
    // --- groups of the sorted reals (written by the forward pass) ---
    int G = 0;
    for (int base = 0; base < nreal; base += 32) {
      const int k = base + lane;
      bool head = false;
      if (k < nreal) head = (k == 0) || ((w.sk[k] >> 32) != (w.sk[k - 1] >> 32));
      const unsigned m = __ballot_sync(0xffffffffu, head);
      if (head) {
        const int at = G + __popc(m & ((1u << lane) - 1u));
        w.gs[at] = k;
        w.gb[at] = static_cast<int>(w.sk[k] >> 32);
      }
      G += __popc(m);
    }
    if (lane == 0) {
      w.gs[G] = nreal;
      atomicAdd(p.counters + 1, static_cast<unsigned long long>(nreal));
    }
    __syncwarp();
    double fc[3] = {0.0, 0.0, 0.0};
    double vir[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) vir[k] = 0.0;
    for (int g0 = 0; g0 < G; g0 += GB) {
      const int gn = min(GB, G - g0);
      // P[a][m] = sum_p dT[a][p] C[m][p] per group (reduce-scatter over the feature lanes)
      for (int gg = 0; gg < gn; ++gg) {
        const double* C = p.tab + static_cast<size_t>(w.gb[g0 + gg]) * istride;
        double part[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) part[k] = 0.0;
#pragma unroll
        for (int q = 0; q < F; ++q) {
#pragma unroll
          for (int mm = 0; mm < 6; ++mm) {
            const double c = __ldg(C + mm * p.Mp + lane + 32 * q);
#pragma unroll
            for (int a = 0; a < 4; ++a) part[a * 6 + mm] += dT[a][q] * c;
          }
        }
        const int b = rs24(part, lane);
        if ((lane & 3) == 0) {
          w.P[gg * 24 + b] = part[0];
          w.P[gg * 24 + b + 1] = part[1];
          w.P[gg * 24 + b + 2] = part[2];
        }
      }
      __syncwarp();
      // members of the batch: one lane per real neighbour
      const int j0 = w.gs[g0], j1 = w.gs[g0 + gn];
      for (int j = j0 + lane; j < j1; j += 32) {
        const uint64_t sk = w.sk[j];
        const int e = static_cast<int>(sk & 0xffffffffu);
        const int bin = static_cast<int>(sk >> 32);
        const long th = bin % p.tn;
        int gg = 0;
        while (gg + 1 < gn && w.gs[g0 + gg + 1] <= j) ++gg;
        const double* P = w.P + gg * 24;
        Env ev;
        env_of(p, ri, p.keys[off + e], ev);
        const double R[4] = {ev.s, ev.s * ev.u[0], ev.s * ev.u[1], ev.s * ev.u[2]};
        const double uu = ev.s - node_x(p.x0, p.h, th);
        double drow[4], dsum = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double* Pa = P + a * 6;
          drow[a] = ((((Pa[5] * uu + Pa[4]) * uu + Pa[3]) * uu + Pa[2]) * uu + Pa[1]) * uu + Pa[0];
          const double h1 =
              (((5.0 * Pa[5] * uu + 4.0 * Pa[4]) * uu + 3.0 * Pa[3]) * uu + 2.0 * Pa[2]) * uu + Pa[1];
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
        double gx[3];
#pragma unroll
        for (int x = 0; x < 3; ++x) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) acc += drow[a] * dd[3 * a + x];
          gx[x] = acc;
          p.g[3 * (off + e) + x] = acc;
          fc[x] += acc;
        }
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int y = 0; y < 3; ++y) vir[3 * x + y] += ev.d[x] * gx[y];
      }
      __syncwarp();
    }
#pragma unroll
    for (int x = 0; x < 3; ++x) fc[x] = warp_sum(fc[x]);
#pragma unroll
    for (int k = 0; k < 9; ++k) vir[k] = warp_sum(vir[k]);
    if (lane == 0) {
#pragma unroll
      for (int x = 0; x < 3; ++x) p.fcenter[3 * i + x] = fc[x];
#pragma unroll
      for (int k = 0; k < 9; ++k) p.vpart[9 * static_cast<size_t>(i) + k] = vir[k];
    }
    __syncwarp();
  }
}

template <int F>
void launch_tab(bool fwd, const TabParams& p, int n, cudaStream_t st, int sms) {
  const size_t per = fwd ? fwd_smem_bytes(p.scap, p.Mp) : bwd_smem_bytes(p.scap, p.Mp);
  const int wpb = 2;
  const size_t bytes = per * wpb;
  if (bytes > 227 * 1024) throw NumErr("neighbour rows too long for the tabulate kernel");
  auto kern = fwd ? k_tab_fwd<F> : k_tab_bwd<F>;
  DPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  const int blocks = std::max(1, std::min(ceil_div(n, wpb), sms * 32));
  kern<<<blocks, wpb * 32, bytes, st>>>(p);
  DPB_CUDA(cudaGetLastError());
}

TabParams make_params(Engine& E) {
  TabParams p{};
  p.pos = E.pos4.p;
  p.row_off = E.row_off.p;
  p.keys = E.keys.p;
  p.skeys = E.skeys.p;
  p.n_real = E.n_real.p;
  p.tab = E.tab.p;
  p.max_nbr = E.d_max_nbr.p;
  p.c = E.cell;
  p.rc2 = E.r_cut * E.r_cut;
  p.rs = E.r_smooth;
  p.rc = E.r_cut;
  p.x0 = E.tab_x0;
  p.h = E.tab_h;
  p.x_end = E.tab_x0 + E.tab_h * static_cast<double>(E.tab_n);
  p.tn = static_cast<long>(E.tab_n);
  p.n = static_cast<int>(E.n);
  p.n_types = E.n_types;
  p.M = E.M;
  p.Mp = E.Mp;
  p.mlt = E.mlt;
  p.K0p = E.K0p;
  p.slot_of = E.slot_of.p;
  p.T = E.T.p;
  p.D = E.D.p;
  p.dD = E.dD.p;
  p.g = E.g.p;
  p.fcenter = E.fcenter.p;
  p.vpart = E.vpart.p;
  p.counters = E.counters.p;
  p.err = E.err.p;
  int scap = 32;
  while (scap < E.max_row) scap <<= 1;
  p.scap = scap;
  return p;
}

int sm_count(int dev) {
  int s = 0;
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

void dispatch(Engine& E, bool fwd) {
  TabParams p = make_params(E);
  const int sms = sm_count(E.device);
  switch (E.Mp / 32) {
    case 1: launch_tab<1>(fwd, p, p.n, E.stream, sms); break;
    case 2: launch_tab<2>(fwd, p, p.n, E.stream, sms); break;
    case 3: launch_tab<3>(fwd, p, p.n, E.stream, sms); break;
    case 4: launch_tab<4>(fwd, p, p.n, E.stream, sms); break;
    case 5: launch_tab<5>(fwd, p, p.n, E.stream, sms); break;
    case 6: launch_tab<6>(fwd, p, p.n, E.stream, sms); break;
    case 7: launch_tab<7>(fwd, p, p.n, E.stream, sms); break;
    case 8: launch_tab<8>(fwd, p, p.n, E.stream, sms); break;
    default: throw InputErr("feature width 4*d1 must be at most 256");
  }
  ++E.launches;
}

} // namespace

void Engine::launch_tab_fwd() { dispatch(*this, true); }
void Engine::launch_tab_bwd() { dispatch(*this, false); }

} // namespace dpb
