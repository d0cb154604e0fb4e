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

// Per-warp shared memory carve-up.
struct WarpSmem {
  uint64_t* sk;   // scap sorted (type, interval, entry) keys
  int* gstart;    // scap + 1 group starts
  int* grp;       // scap member -> group id
  double* wb;     // 32 x 24 moments / interval projections of one group batch
  double* red;    // 32 x 25 transpose-reduce scratch
  double* ts;     // 4 x Mp copy of T
  int* tcnt;      // 64 per-type counters
};

__host__ __device__ __forceinline__ size_t warp_smem_bytes(int scap, int Mp) {
  const size_t b = static_cast<size_t>(scap) * 8 + 32 * 24 * 8 + 32 * 25 * 8 + 4 * Mp * 8 +
                   (static_cast<size_t>(scap) * 2 + 1 + 64) * 4;
  return (b + 15) & ~static_cast<size_t>(15);
}

__device__ __forceinline__ WarpSmem carve(unsigned char* base, int scap, int Mp) {
  WarpSmem w;
  w.sk = reinterpret_cast<uint64_t*>(base);
  w.wb = reinterpret_cast<double*>(w.sk + scap);
  w.red = w.wb + 32 * 24;
  w.ts = w.red + 32 * 25;
  w.gstart = reinterpret_cast<int*>(w.ts + 4 * Mp);
  w.grp = w.gstart + scap + 1;
  w.tcnt = w.grp + scap;
  return w;
}

// Warp bitonic sort of sk[0..n) ascending (pads to a power of two with ~0).
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

// Group heads of the sorted (type, interval) keys -> gstart[0..G], grp[k]. Returns G.
__device__ int make_groups(const WarpSmem& w, int nreal, int lane) {
  int G = 0;
  for (int base = 0; base < nreal; base += 32) {
    const int k = base + lane;
    bool head = false;
    if (k < nreal) head = (k == 0) || ((w.sk[k] >> 32) != (w.sk[k - 1] >> 32));
    const unsigned m = __ballot_sync(0xffffffffu, head);
    const unsigned lt = (1u << lane) - 1u;
    if (head) w.gstart[G + __popc(m & lt)] = k;
    if (k < nreal) w.grp[k] = G + __popc(m & (lt | (1u << lane))) - 1;
    G += __popc(m);
  }
  if (lane == 0) w.gstart[G] = nreal;
  __syncwarp();
  return G;
}

template <int F>
__global__ void __launch_bounds__(128) k_tab_fwd(TabParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const WarpSmem w = carve(smem + wid * warp_smem_bytes(p.scap, p.Mp), p.scap, p.Mp);
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    const double3 ri = ld_pos(p.pos, i);
    for (int t = lane; t < 64; t += 32) w.tcnt[t] = 0;
    __syncwarp();
    // --- env-mat scan: real neighbours -> (type, interval, entry) keys ---
    int nreal = 0, next = 0;
    for (int base = 0; base < len; base += 32) {
      const int e = base + lane;
      bool real = false, ext = false;
      uint64_t sk = 0;
      if (e < len) {
        const uint64_t key = p.keys[off + e];
        int sh[3];
        key_shift(key, sh);
        double d[3];
        disp_exact(p.c, ri, ld_pos(p.pos, key_j(key)), sh[0], sh[1], sh[2], d);
        const double r2 = norm2_exact(d);
        if (r2 < 1e-12) {
          raise_err(p.err, DEV_OVERLAP);  // env_mat.cpp:33 throws before any table lookup
        } else if (r2 < p.rc2) {
          real = true;
          const double r = sqrt(r2);
          const double s = switch_fn(r, p.rs, p.rc) * (1.0 / r);
          const long th = locate(p, s, ext, p.err);
          const int t = key_type(key);
          atomicAdd(w.tcnt + t, 1);
          sk = (static_cast<uint64_t>(t) << 58) | (static_cast<uint64_t>(th) << 32) |
               static_cast<uint64_t>(e);
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, real);
      const int at = nreal + __popc(m & ((1u << lane) - 1u));
      if (real) {
        if (at < p.scap) w.sk[at] = sk;
        else raise_err(p.err, DEV_ROW_CAP);
      }
      nreal += __popc(m);
      next += __popc(__ballot_sync(0xffffffffu, ext));
    }
    nreal = min(nreal, p.scap);
    __syncwarp();
    for (int t = lane; t < p.n_types; t += 32)
      if (w.tcnt[t] > p.max_nbr[t]) raise_err(p.err, DEV_OVERFLOW);
    if (lane == 0) {
      atomicAdd(p.counters + 0, static_cast<unsigned long long>(nreal));
      if (next) atomicAdd(p.counters + 2, static_cast<unsigned long long>(next));
    }
    warp_sort(w.sk, nreal, lane);
    for (int k = lane; k < nreal; k += 32) p.skeys[off + k] = w.sk[k];
    if (lane == 0) p.n_real[i] = nreal;
    const int G = make_groups(w, nreal, lane);
    // --- moments per group, then T += W . C[interval] ---
    double tacc[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) tacc[a][q] = 0.0;
    for (int gb = 0; gb < G; gb += 32) {
      const int g = gb + lane;
      if (g < G) {
        double W[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) W[k] = 0.0;
        const int k1 = w.gstart[g + 1];
        for (int k = w.gstart[g]; k < k1; ++k) {
          const uint64_t sk = w.sk[k];
          const long th = static_cast<long>((sk >> 32) & 0x3ffffffull);
          Env ev;
          env_of(p, ri, p.keys[off + static_cast<int>(sk & 0xffffffffu)], ev);
          const double R[4] = {ev.s, ev.s * ev.u[0], ev.s * ev.u[1], ev.s * ev.u[2]};
          const double uu = ev.s - node_x(p.x0, p.h, th);
          double um = 1.0;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
#pragma unroll
            for (int a = 0; a < 4; ++a) W[a * 6 + m] += R[a] * um;
            um *= uu;
          }
        }
#pragma unroll
        for (int k = 0; k < 24; ++k) w.wb[lane * 24 + k] = W[k];
      }
      __syncwarp();
      const int gn = min(32, G - gb);
      for (int gg = 0; gg < gn; ++gg) {
        const uint64_t sk = w.sk[w.gstart[gb + gg]];
        const int t = key_type(sk);
        const long th = static_cast<long>((sk >> 32) & 0x3ffffffull);
        const double* C = p.tab + (static_cast<size_t>(t) * p.tn + th) * istride;
        const double* Wg = w.wb + gg * 24;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          const int f = lane + 32 * q;
          double c[6];
#pragma unroll
          for (int m = 0; m < 6; ++m) c[m] = __ldg(C + m * p.Mp + f);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            double acc = tacc[a][q];
#pragma unroll
            for (int m = 0; m < 6; ++m) acc += Wg[a * 6 + m] * c[m];
            tacc[a][q] = acc;
          }
        }
      }
      __syncwarp();
    }
    // --- T out, D = T<^T T ---
    double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < F; ++q) {
        Ti[a * p.Mp + lane + 32 * q] = tacc[a][q];
        w.ts[a * p.Mp + lane + 32 * q] = tacc[a][q];
      }
    __syncwarp();
    double* Drow = p.D + static_cast<size_t>(p.slot_of[i]) * p.K0p;
    for (int qq = 0; qq < p.mlt; ++qq) {
      const double t0 = w.ts[qq], t1 = w.ts[p.Mp + qq], t2 = w.ts[2 * p.Mp + qq],
                   t3 = w.ts[3 * p.Mp + qq];
#pragma unroll
      for (int q = 0; q < F; ++q) {
        const int f = lane + 32 * q;
        if (f < p.M) {
          double acc = 0.0;
          acc += t0 * tacc[0][q];
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
__global__ void __launch_bounds__(128) k_tab_bwd(TabParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const WarpSmem w = carve(smem + wid * warp_smem_bytes(p.scap, p.Mp), p.scap, p.Mp);
  const size_t istride = static_cast<size_t>(6) * p.Mp;
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    const double3 ri = ld_pos(p.pos, i);
    for (int e = lane; e < 3 * len; e += 32) p.g[3 * off + e] = 0.0;
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
    for (int qq = 0; qq < p.mlt; ++qq) {
      double dq[F];
#pragma unroll
      for (int q = 0; q < F; ++q) {
        const int f = lane + 32 * q;
        dq[q] = f < p.M ? dDrow[qq * p.M + f] : 0.0;
      }
      double S[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double ta = w.ts[a * p.Mp + qq];
        double part = 0.0;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          dT[a][q] += dq[q] * ta;
          part += dq[q] * tv[a][q];
        }
        S[a] = warp_sum(part);
      }
      if (lane == (qq & 31)) {
#pragma unroll
        for (int q = 0; q < F; ++q)
          if (q == (qq >> 5))
#pragma unroll
            for (int a = 0; a < 4; ++a) dT[a][q] += S[a];
      }
    }
    // --- groups of this centre's real neighbours (sorted in the forward pass) ---
    const int nreal = p.n_real[i];
    for (int k = lane; k < nreal; k += 32) w.sk[k] = p.skeys[off + k];
    __syncwarp();
    const int G = make_groups(w, nreal, lane);
    if (lane == 0) atomicAdd(p.counters + 1, static_cast<unsigned long long>(nreal));
    double fc[3] = {0.0, 0.0, 0.0};
    double vir[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) vir[k] = 0.0;
    for (int gb = 0; gb < G; gb += 32) {
      const int gn = min(32, G - gb);
      // P[a][m] = sum_p dT[a][p] C[m][p] for each group of the batch.
      for (int gg = 0; gg < gn; ++gg) {
        const uint64_t sk = w.sk[w.gstart[gb + gg]];
        const int t = key_type(sk);
        const long th = static_cast<long>((sk >> 32) & 0x3ffffffull);
        const double* C = p.tab + (static_cast<size_t>(t) * p.tn + th) * istride;
        double part[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) part[k] = 0.0;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          const int f = lane + 32 * q;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            const double c = __ldg(C + m * p.Mp + f);
#pragma unroll
            for (int a = 0; a < 4; ++a) part[a * 6 + m] += dT[a][q] * c;
          }
        }
#pragma unroll
        for (int k = 0; k < 24; ++k) w.red[lane * 25 + k] = part[k];
        __syncwarp();
        if (lane < 24) {
          double s = 0.0;
#pragma unroll 8
          for (int l = 0; l < 32; ++l) s += w.red[l * 25 + lane];
          w.wb[gg * 24 + lane] = s;
        }
        __syncwarp();
      }
      // Members of the batch: one lane per real neighbour.
      const int k0 = w.gstart[gb], k1 = w.gstart[gb + gn];
      for (int k = k0 + lane; k < k1; k += 32) {
        const uint64_t sk = w.sk[k];
        const int e = static_cast<int>(sk & 0xffffffffu);
        const long th = static_cast<long>((sk >> 32) & 0x3ffffffull);
        const double* P = w.wb + (w.grp[k] - gb) * 24;
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
  const size_t per = warp_smem_bytes(p.scap, p.Mp);
  int wpb = 4;
  while (wpb > 1 && per * wpb > 200 * 1024) wpb >>= 1;
  if (per * wpb > 220 * 1024) throw NumErr("neighbour rows too long for the tabulate kernel");
  const size_t bytes = per * wpb;
  auto kern = fwd ? k_tab_fwd<F> : k_tab_bwd<F>;
  DPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  const int blocks = std::max(1, std::min(ceil_div(n, wpb), sms * 16));
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
