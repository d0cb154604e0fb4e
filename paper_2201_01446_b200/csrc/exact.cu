// Exact (untabulated) DP-SE evaluation and the GPU table builder.
//
// Reference:
//   embedding net      model.cpp:60-149   1 -> d1 -> 2 d1 -> 4 d1, tanh, "concatenate the input
//                                         with itself" shortcuts; value, d/ds, d2/ds2 forward mode
//   exact energy/force exact.cpp:77-173   T = sum_slots R (x) G(s), D, fitting, dT, then per slot
//                                         drow[a] = dT[a].G, ds = sum_p (sum_a R[a] dT[a][p]) G'_p
//   table build        table.cpp:77-162   node values / derivatives, quintic Hermite coefficients,
//                                         node verification at 1e-10
//   rmse tooling       rmse.cpp:48-118    exact vs tabulated energies / forces (host, api.cpp)
//
// B200 formulation: one warp per centre evaluates the embedding net for NP neighbours at a time
// (lane = output feature v = lane + 32 k, weights read coalesced through L1, activations in the
// warp's shared scratch); the embedding matrix is never stored. The backward kernel recomputes
// G and G' instead of keeping 2 x 128 doubles per pair in HBM, so any system size runs in the
// same memory as the tabulated path. The fitting net and the force gather are shared with the
// tabulated path.
#include <cub/cub.cuh>

#include "tab_common.cuh"

namespace dpb {

namespace {

constexpr int NP = 4; // neighbours per embedding step

// Embedding net of NP scalars (warp-cooperative). ORD 0: values, 1: + d/ds, 2: + d2/ds2.
// Outputs: feature v = lane + 32 k for k < F (zero beyond 4 d1).
template <int F, int ORD>
__device__ void embed_warp(const EmbPtrs& w, int d1, const double (&s)[NP], double* sc, int lane,
                           double (&g)[NP][F], double (&g1)[NP][F], double (&g2)[NP][F]) {
  const int d2 = 2 * d1, d4 = 4 * d1;
  double* a = sc;
  double* ag = a + NP * d1;
  double* agg = ag + NP * d1;
  double* b = agg + NP * d1;
  double* bg = b + NP * d2;
  double* bgg = bg + NP * d2;
  for (int u = lane; u < d1; u += 32) {
    const double w0 = w.w0[u], b0 = w.b0[u];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double t = tanh(s[p] * w0 + b0);
      const double dt = 1.0 - t * t;
      a[p * d1 + u] = t;
      if (ORD >= 1) ag[p * d1 + u] = dt * w0;
      if (ORD >= 2) agg[p * d1 + u] = -2.0 * t * dt * w0 * w0;
    }
  }
  __syncwarp();
  constexpr int F1 = (F + 1) / 2;
#pragma unroll
  for (int k = 0; k < F1; ++k) {
    const int v = lane + 32 * k;
    if (v < d2) {
      double z[NP], zg[NP], zgg[NP];
      const double bias = w.b1[v];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        z[p] = bias;
        zg[p] = 0.0;
        zgg[p] = 0.0;
      }
      for (int u = 0; u < d1; ++u) {
        const double wv = __ldg(w.w1 + static_cast<size_t>(u) * d2 + v);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          z[p] += a[p * d1 + u] * wv;
          if (ORD >= 1) zg[p] += ag[p * d1 + u] * wv;
          if (ORD >= 2) zgg[p] += agg[p * d1 + u] * wv;
        }
      }
      const int s0 = v % d1;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double t = tanh(z[p]);
        const double dt = 1.0 - t * t;
        b[p * d2 + v] = a[p * d1 + s0] + t;
        if (ORD >= 1) bg[p * d2 + v] = ag[p * d1 + s0] + dt * zg[p];
        if (ORD >= 2) bgg[p * d2 + v] = agg[p * d1 + s0] + dt * zgg[p] - 2.0 * t * dt * zg[p] * zg[p];
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < F; ++k) {
    const int v = lane + 32 * k;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      g[p][k] = 0.0;
      if (ORD >= 1) g1[p][k] = 0.0;
      if (ORD >= 2) g2[p][k] = 0.0;
    }
    if (v < d4) {
      double z[NP], zg[NP], zgg[NP];
      const double bias = w.b2[v];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        z[p] = bias;
        zg[p] = 0.0;
        zgg[p] = 0.0;
      }
      for (int u = 0; u < d2; ++u) {
        const double wv = __ldg(w.w2 + static_cast<size_t>(u) * d4 + v);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          z[p] += b[p * d2 + u] * wv;
          if (ORD >= 1) zg[p] += bg[p * d2 + u] * wv;
          if (ORD >= 2) zgg[p] += bgg[p * d2 + u] * wv;
        }
      }
      const int s0 = v % d2;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double t = tanh(z[p]);
        const double dt = 1.0 - t * t;
        g[p][k] = b[p * d2 + s0] + t;
        if (ORD >= 1) g1[p][k] = bg[p * d2 + s0] + dt * zg[p];
        if (ORD >= 2) g2[p][k] = bgg[p * d2 + s0] + dt * zgg[p] - 2.0 * t * dt * zg[p] * zg[p];
      }
    }
  }
  __syncwarp();
}

__host__ __device__ __forceinline__ int emb_scratch(int d1) { return 3 * NP * (d1 + 2 * d1); }

// ---------------------------------------------------------------- env-mat (thread per entry)
// prod_env_mat for the exact path (env_mat.cpp:29-71): real filter and R = (s, s d/r) per list
// entry; xbin = neighbour type of a real entry, -1 otherwise (the exact path evaluates the
// embedding net itself, so there is no table interval).
__global__ void __launch_bounds__(256) k_env_exact(TabParams p) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= p.E || e >= p.row_off[p.n]) return;
  // owner of the entry: binary search of row_off (the exact path is a validation path)
  int lo = 0, hi = p.n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (p.row_off[mid] <= e) lo = mid;
    else hi = mid;
  }
  const int i = lo;
  const uint64_t key = p.keys[e];
  int bin = -1;
  if (p.center[i]) {
    int sh[3];
    key_shift(key, sh);
    double d[3];
    disp_exact(p.c, ld_pos(p.pos, i), ld_pos(p.pos, key_j(key)), sh[0], sh[1], sh[2], d);
    const double r2 = norm2_exact(d);
    if (r2 < 1e-12) {
      raise_err(p.err, DEV_OVERLAP); // env_mat.cpp:33
    } else if (r2 < p.rc2) {
      const double r = sqrt(r2);
      const double ir = 1.0 / r;
      const double s = switch_fn(r, p.rs, p.rc) * ir;
      bin = key_type(key);
      p.xrc[e] = s;
      p.xrc[p.E + e] = s * (d[0] * ir);
      p.xrc[2 * p.E + e] = s * (d[1] * ir);
      p.xrc[3 * p.E + e] = s * (d[2] * ir);
    }
  }
  const_cast<int32_t*>(p.xbin)[e] = bin;
}

// List ranks of the real entries of every row (ridx, -1 otherwise) and their count: the
// compact pair-gradient layout the force kernel gathers from (force.cu). Warp per row.
__global__ void k_exact_rank(TabParams p) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= p.n) return;
  const int64_t off = p.row_off[i];
  const int len = static_cast<int>(p.row_off[i + 1] - off);
  int cnt = 0;
  for (int base = 0; base < len; base += 32) {
    const int e = base + lane;
    const bool real = e < len && p.xbin[off + e] >= 0;
    const unsigned m = __ballot_sync(0xffffffffu, real);
    if (e < len) p.ridx[off + e] = static_cast<int16_t>(real ? cnt + __popc(m & ((1u << lane) - 1u)) : -1);
    cnt += __popc(m);
  }
  if (lane == 0) p.n_real[i] = cnt;
}

// Compact the real entries of neighbour type t of row [off, off+len) into idx (list order).
__device__ __forceinline__ int compact_type(const TabParams& p, int64_t off, int len, int t, int* idx,
                                            int lane) {
  int cnt = 0;
  for (int base = 0; base < len; base += 32) {
    const int e = base + lane;
    const int bin = e < len ? p.xbin[off + e] : -1;
    const bool take = bin >= 0 && bin == t;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (take) idx[cnt + __popc(m & ((1u << lane) - 1u))] = e;
    cnt += __popc(m);
  }
  __syncwarp();
  return cnt;
}

// ---------------------------------------------------------------- forward: T, D (warp per centre)
template <int F>
__global__ void __launch_bounds__(128) k_exact_fwd(TabParams p, const EmbPtrs* nets, int d1) {
  extern __shared__ __align__(16) double xsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int per_warp = emb_scratch(d1) + 4 * p.Mp + p.scap / 2 + 2;
  double* sc = xsm + wid * per_warp;
  double* ts = sc + emb_scratch(d1);
  int* idx = reinterpret_cast<int*>(ts + 4 * p.Mp);
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    if (!p.center[i]) continue;
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    double T[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < F; ++k) T[a][k] = 0.0;
    for (int t = 0; t < p.n_types; ++t) {
      const int cnt = compact_type(p, off, len, t, idx, lane);
      if (cnt > p.max_nbr[t] && lane == 0) raise_err(p.err, DEV_OVERFLOW); // env_mat.cpp:37-39
      for (int c0 = 0; c0 < cnt; c0 += NP) {
        double s[NP], R[NP][4];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const bool ok = c0 + q < cnt;
          const int64_t e = off + (ok ? idx[c0 + q] : 0);
#pragma unroll
          for (int a = 0; a < 4; ++a) R[q][a] = ok ? p.xrc[a * p.E + e] : 0.0;
          s[q] = R[q][0];
        }
        double g[NP][F], g1[NP][F], g2[NP][F];
        embed_warp<F, 0>(nets[t], d1, s, sc, lane, g, g1, g2);
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int k = 0; k < F; ++k) T[a][k] += R[q][a] * g[q][k];
      }
    }
    // T and D = T<^T T (contract.hpp:9-17)
    double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < F; ++k) {
        Ti[a * p.Mp + lane + 32 * k] = T[a][k];
        ts[a * p.Mp + lane + 32 * k] = T[a][k];
      }
    __syncwarp();
    const int slot = p.slot_of[i];
    if (slot >= 0) {
      for (int qq = 0; qq < p.mlt; ++qq) {
        const double t0 = ts[qq], t1 = ts[p.Mp + qq], t2 = ts[2 * p.Mp + qq], t3 = ts[3 * p.Mp + qq];
#pragma unroll
        for (int k = 0; k < F; ++k) {
          const int f = lane + 32 * k;
          if (f >= p.M) continue;
          double acc = t0 * T[0][k];
          acc += t1 * T[1][k];
          acc += t2 * T[2][k];
          acc += t3 * T[3][k];
          if (p.D2) {
            const float x = static_cast<float>(acc);
            const float hi = tf32_rna(x);
            float* d2 = p.D2 + static_cast<size_t>(slot) * 2 * p.K0p + qq * p.M + f;
            d2[0] = hi;
            d2[p.K0p] = tf32_rna(x - hi);
          } else {
            p.D[static_cast<size_t>(slot) * p.K0p + qq * p.M + f] = acc;
          }
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- backward: g per entry
template <int F>
__global__ void __launch_bounds__(128) k_exact_bwd(TabParams p, const EmbPtrs* nets, int d1) {
  extern __shared__ __align__(16) double xsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int per_warp = emb_scratch(d1) + 4 * p.Mp + 4 * p.mlt + p.scap / 2 + 2;
  double* sc = xsm + wid * per_warp;
  double* ts = sc + emb_scratch(d1);
  double* S = ts + 4 * p.Mp;
  int* idx = reinterpret_cast<int*>(S + 4 * p.mlt);
  for (int i = blockIdx.x * wpb + wid; i < p.n; i += gridDim.x * wpb) {
    const int64_t off = p.row_off[i];
    const int len = static_cast<int>(p.row_off[i + 1] - off);
    if (!p.center[i]) continue;
    const int64_t ro = p.realoff[i];
    if (ro + p.n_real[i] > p.gcap) {
      if (lane == 0) raise_err(p.err, DEV_GCAP);
      continue;
    }
    // dT = adjoint of D (contract.hpp:21-38), lane features f = lane + 32 k
    const double* Ti = p.T + static_cast<size_t>(i) * 4 * p.Mp;
    double tv[4][F], dT[4][F];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int k = 0; k < F; ++k) {
        tv[a][k] = Ti[a * p.Mp + lane + 32 * k];
        ts[a * p.Mp + lane + 32 * k] = tv[a][k];
        dT[a][k] = 0.0;
      }
    __syncwarp();
    const int slot = p.slot_of[i];
    const double* dDrow = p.dD + static_cast<size_t>(slot < 0 ? 0 : slot) * p.K0p;
    for (int q0 = 0; q0 < p.mlt; q0 += 8) {
      double part[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) part[k] = 0.0;
#pragma unroll
      for (int ql = 0; ql < 8; ++ql) {
        const int qq = q0 + ql;
        if (qq < p.mlt && slot >= 0) {
#pragma unroll
          for (int k = 0; k < F; ++k) {
            const int f = lane + 32 * k;
            const double dq = f < p.M ? dDrow[qq * p.M + f] : 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              dT[a][k] += dq * ts[a * p.Mp + qq];
              part[ql * 4 + a] += dq * tv[a][k];
            }
          }
        }
      }
      const double sv = rs32(part, lane);
      if (q0 + (lane >> 2) < p.mlt) S[(q0 + (lane >> 2)) * 4 + (lane & 3)] = sv;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < F; ++k) {
      const int f = lane + 32 * k;
      if (f < p.mlt)
#pragma unroll
        for (int a = 0; a < 4; ++a) dT[a][k] += S[f * 4 + a];
    }
    __syncwarp();
    const double3 ri = ld_pos(p.pos, i);
    for (int t = 0; t < p.n_types; ++t) {
      const int cnt = compact_type(p, off, len, t, idx, lane);
      for (int c0 = 0; c0 < cnt; c0 += NP) {
        double s[NP], R[NP][4];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const bool ok = c0 + q < cnt;
          const int64_t e = off + (ok ? idx[c0 + q] : 0);
#pragma unroll
          for (int a = 0; a < 4; ++a) R[q][a] = ok ? p.xrc[a * p.E + e] : 0.0;
          s[q] = R[q][0];
        }
        double g[NP][F], g1[NP][F], g2[NP][F];
        embed_warp<F, 1>(nets[t], d1, s, sc, lane, g, g1, g2);
        // per pair: drow[a] = dT[a].G, ds = sum_p (sum_a R[a] dT[a][p]) G'_p (exact.cpp:116-129)
        double red[NP][5];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          double ds = 0.0;
#pragma unroll
          for (int a = 0; a < 4; ++a) red[q][a] = 0.0;
#pragma unroll
          for (int k = 0; k < F; ++k) {
            double dg = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              red[q][a] += dT[a][k] * g[q][k];
              dg += R[q][a] * dT[a][k];
            }
            ds += dg * g1[q][k];
          }
          red[q][4] = ds;
        }
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
          for (int c = 0; c < 5; ++c) red[q][c] = warp_sum(red[q][c]);
        if (lane < NP && c0 + lane < cnt) {
          double rr[5];
#pragma unroll
          for (int q = 0; q < NP; ++q)
            if (q == lane)
#pragma unroll
              for (int c = 0; c < 5; ++c) rr[c] = red[q][c];
          const int64_t e = off + idx[c0 + lane];
          Env ev;
          env_of(p, ri, p.keys[e], ev);
          double drow[4] = {rr[0] + rr[4], rr[1], rr[2], rr[3]};
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
          double* ge = p.g + 3 * (ro + p.ridx[e]); // compact slot of the real pair
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) acc += drow[a] * dd[3 * a + x];
            ge[x] = acc;
          }
        }
        __syncwarp();
      }
    }
  }
}

// ---------------------------------------------------------------- table builder
// Node values and derivatives (table.cpp:93-97): one warp per NP nodes.
template <int F>
__global__ void __launch_bounds__(128) k_table_nodes(EmbPtrs net, int d1, double x0, double h, int n_nodes,
                                                     double* val, double* dv1, double* dv2) {
  extern __shared__ __align__(16) double xsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  double* sc = xsm + wid * emb_scratch(d1);
  const int m = 4 * d1;
  for (int k0 = (blockIdx.x * wpb + wid) * NP; k0 < n_nodes; k0 += gridDim.x * wpb * NP) {
    double s[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) s[q] = node_x(x0, h, min(k0 + q, n_nodes - 1));
    double g[NP][F], g1[NP][F], g2[NP][F];
    embed_warp<F, 2>(net, d1, s, sc, lane, g, g1, g2);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (k0 + q >= n_nodes) break;
#pragma unroll
      for (int k = 0; k < F; ++k) {
        const int f = lane + 32 * k;
        if (f < m) {
          const size_t o = static_cast<size_t>(k0 + q) * m + f;
          val[o] = g[q][k];
          dv1[o] = g1[q][k];
          dv2[o] = g2[q][k];
        }
      }
    }
  }
}

// Quintic Hermite coefficients per (interval, feature) (table.cpp:99-130); written both in the
// reference layout [interval][block][k][f] and in the engine layout [interval][k][Mp].
__global__ void k_table_coeffs(int n, int m, int B, int Mp, double x0, double h, const double* __restrict__ val,
                               const double* __restrict__ dv1, const double* __restrict__ dv2,
                               double* __restrict__ ref, double* __restrict__ eng) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(n) * m) return;
  const int th = static_cast<int>(idx / m);
  const int pf = static_cast<int>(idx % m);
  const double hl = node_x(x0, h, th + 1) - node_x(x0, h, th);
  const size_t o = static_cast<size_t>(th) * m + pf;
  const double a0 = val[o];
  const double a1 = dv1[o];
  const double a2 = 0.5 * dv2[o];
  const double dv = val[o + m] - (a0 + a1 * hl + a2 * hl * hl);
  const double dg = dv1[o + m] - (a1 + 2.0 * a2 * hl);
  const double dc = dv2[o + m] - 2.0 * a2;
  const double h2 = hl * hl;
  const double h3 = h2 * hl;
  const double a3 = (10.0 * dv - 4.0 * hl * dg + 0.5 * h2 * dc) / h3;
  const double a4 = (-15.0 * dv + 7.0 * hl * dg - h2 * dc) / (h3 * hl);
  const double a5 = (6.0 * dv - 3.0 * hl * dg + 0.5 * h2 * dc) / (h3 * h2);
  const double cs[6] = {a0, a1, a2, a3, a4, a5};
  const int nb = (m + B - 1) / B;
  double* c = ref + static_cast<size_t>(th) * nb * 6 * B + static_cast<size_t>(pf / B) * 6 * B + (pf % B);
  double* e = eng + static_cast<size_t>(th) * 6 * Mp + pf;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    c[k * B] = cs[k];
    e[k * Mp] = cs[k];
  }
}

// Node verification (table.cpp:133-147): the table must reproduce the net at every node.
__global__ void k_table_verify(int n, int m, int Mp, double x0, double h, const double* __restrict__ val,
                               const double* __restrict__ eng, int* err) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(n + 1) * m) return;
  const int k = static_cast<int>(idx / m);
  const int pf = static_cast<int>(idx % m);
  const double x = node_x(x0, h, k);
  // locate (table.cpp:20-32) of a node: its own interval, the last node in the last interval
  int th = static_cast<int>(floor((x - x0) / h));
  while (node_x(x0, h, th + 1) <= x) ++th;
  while (th > 0 && node_x(x0, h, th) > x) --th;
  if (th >= n) th = n - 1;
  const double u = x - node_x(x0, h, th);
  const double* c = eng + static_cast<size_t>(th) * 6 * Mp + pf;
  const double row = ((((c[5 * Mp] * u + c[4 * Mp]) * u + c[3 * Mp]) * u + c[2 * Mp]) * u + c[Mp]) * u + c[0];
  const double f = val[static_cast<size_t>(k) * m + pf];
  const double e = fabs(row - f);
  if (!(e <= 1e-10 * fmax(1.0, fabs(f)))) raise_err(err, DEV_TABLE_VERIFY);
}

int sm_count_x(int dev) {
  int s = 0;
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

template <int F>
void launch_exact(const TabParams& p, const EmbPtrs* nets, int d1, bool fwd, cudaStream_t st, int sms) {
  const size_t per_warp =
      static_cast<size_t>(emb_scratch(d1) + 4 * p.Mp + 4 * p.mlt + p.scap / 2 + 2) * sizeof(double);
  const size_t bytes = 4 * per_warp;
  if (bytes > 227 * 1024) throw NumErr("neighbour rows too long for the exact-path kernel");
  if (fwd) {
    DPB_CUDA(cudaFuncSetAttribute(k_exact_fwd<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
    k_exact_fwd<F><<<std::max(1, std::min(ceil_div(p.n, 4), sms * 16)), 128, bytes, st>>>(p, nets, d1);
  } else {
    DPB_CUDA(cudaFuncSetAttribute(k_exact_bwd<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
    k_exact_bwd<F><<<std::max(1, std::min(ceil_div(p.n, 4), sms * 16)), 128, bytes, st>>>(p, nets, d1);
  }
  DPB_CUDA(cudaGetLastError());
}

void dispatch_exact(const TabParams& p, const EmbPtrs* nets, int d1, bool fwd, cudaStream_t st, int sms) {
  switch (p.Mp / 32) {
    case 1: launch_exact<1>(p, nets, d1, fwd, st, sms); break;
    case 2: launch_exact<2>(p, nets, d1, fwd, st, sms); break;
    case 3: launch_exact<3>(p, nets, d1, fwd, st, sms); break;
    case 4: launch_exact<4>(p, nets, d1, fwd, st, sms); break;
    case 5: launch_exact<5>(p, nets, d1, fwd, st, sms); break;
    case 6: launch_exact<6>(p, nets, d1, fwd, st, sms); break;
    case 7: launch_exact<7>(p, nets, d1, fwd, st, sms); break;
    case 8: launch_exact<8>(p, nets, d1, fwd, st, sms); break;
    default: throw InputErr("feature width 4*d1 must be at most 256");
  }
}

template <int F>
void launch_nodes(const EmbPtrs& net, int d1, double x0, double h, int n_nodes, double* val, double* d1v,
                  double* d2v, cudaStream_t st) {
  const size_t bytes = 4 * static_cast<size_t>(emb_scratch(d1)) * sizeof(double);
  DPB_CUDA(cudaFuncSetAttribute(k_table_nodes<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bytes)));
  const int blocks = std::max(1, ceil_div(n_nodes, 4 * NP));
  k_table_nodes<F><<<blocks, 128, bytes, st>>>(net, d1, x0, h, n_nodes, val, d1v, d2v);
  DPB_CUDA(cudaGetLastError());
}

} // namespace

void Engine::set_embedding(const dp_embedding_desc* nets) {
  if (!nets) throw InputErr("null embedding description");
  const size_t per = static_cast<size_t>(d1) * (1 + 1 + 2 * d1 + 2 + 8 * d1 + 4);
  std::vector<double> buf(per * n_types);
  for (int t = 0; t < n_types; ++t) {
    const dp_embedding_desc& e = nets[t];
    if (e.d1 != d1) throw InputErr("all embedding nets must share d1 with the model");
    if (!e.w0 || !e.b0 || !e.w1 || !e.b1 || !e.w2 || !e.b2) throw InputErr("null embedding weights");
    double* o = buf.data() + per * t;
    auto put = [&](const double* src, size_t cnt) {
      std::copy(src, src + cnt, o);
      o += cnt;
    };
    put(e.w0, d1);
    put(e.b0, d1);
    put(e.w1, static_cast<size_t>(2) * d1 * d1);
    put(e.b1, 2 * d1);
    put(e.w2, static_cast<size_t>(8) * d1 * d1);
    put(e.b2, 4 * d1);
  }
  emb_w.ensure(buf.size());
  DPB_CUDA(cudaMemcpy(emb_w.p, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice));
  std::vector<EmbPtrs> ptrs(n_types);
  for (int t = 0; t < n_types; ++t) {
    const double* b = emb_w.p + per * t;
    EmbPtrs& q = ptrs[t];
    q.w0 = b;
    q.b0 = q.w0 + d1;
    q.w1 = q.b0 + d1;
    q.b1 = q.w1 + 2 * d1 * d1;
    q.w2 = q.b1 + 2 * d1;
    q.b2 = q.w2 + 8 * d1 * d1;
  }
  emb_ptrs_host = ptrs;
  emb_ptrs.ensure(n_types);
  DPB_CUDA(cudaMemcpy(emb_ptrs.p, ptrs.data(), n_types * sizeof(EmbPtrs), cudaMemcpyHostToDevice));
  has_embedding = true;
}

void Engine::evaluate_exact() {
  if (!has_embedding) throw InputErr("the exact path needs the embedding nets (dp_set_embedding)");
  if (!list_valid) throw InputErr("no neighbour list");
  if (n_chunks > 1 || plan_dirty) {
    // the exact kernels index every list entry: whole system in one chunk for this call
    force_single_chunk = true;
    apply_plan();
    force_single_chunk = false;
    plan_dirty = true; // the tabulated path re-plans its chunks at its next evaluation
  }
  use_chunk(0);
  TabParams p = make_params(*this);
  p.tn = 0;                     // env-mat only: xbin = neighbour type of a real entry
  p.counters = exact_ctr.p;     // the exact path does not touch the tabulation counters
  const int sms = sm_count_x(device);
  xbin.ensure(e_cap + 1);
  xrc.ensure(4 * e_cap + 4);
  p.xbin = xbin.p;
  p.xrc = xrc.p;
  phase_begin(1);
  k_env_exact<<<ceil_div(e_cap, 256), 256, 0, stream>>>(p);
  k_exact_rank<<<ceil_div(static_cast<int64_t>(n) * 32, 256), 256, 0, stream>>>(p);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, n_real.p, realoff.p, static_cast<int>(n), stream);
    scan_tmp.ensure(tb + 1);
    cub::DeviceScan::ExclusiveSum(scan_tmp.p, tb, n_real.p, realoff.p, static_cast<int>(n), stream);
  }
  launches += 3;
  dispatch_exact(p, emb_ptrs.p, d1, true, stream, sms);
  ++launches;
  phase_begin(2);
  if (precision == 1)
    launch_fitting_mixed();
  else
    launch_fitting();
  phase_begin(3);
  dispatch_exact(p, emb_ptrs.p, d1, false, stream, sms);
  ++launches;
  phase_begin(4);
  virial_in_forces = true; // no per-real records on this path: d is re-evaluated there
  launch_forces();
  virial_in_forces = false;
  phase_end();
}

void Engine::build_tables_gpu(double step, uint64_t* n_out, double* x_end_out, double* coeffs_out, bool install) {
  if (!has_embedding) throw InputErr("building tables needs the embedding nets (dp_set_embedding)");
  if (!(step > 0.0)) throw InputErr("table step must be positive");
  // table_domain_end (table.cpp:151-153) with r_min = 0.5
  const double x_end = switch_w(0.5, r_smooth, r_cut) / 0.5;
  const double x0 = 0.0;
  if (!(x_end > x0)) throw InputErr("table domain end is not positive");
  uint64_t n = static_cast<uint64_t>(std::ceil((x_end - x0) / step - 1e-9));
  if (n == 0) n = 1;
  if (n_out) *n_out = n;
  if (x_end_out) *x_end_out = x_end;
  if (!coeffs_out && !install) return;
  if (n > (1u << 24)) throw InputErr("table step too small");
  const int m = M, B = 16, nb = (m + B - 1) / B;
  const size_t nodes = n + 1;
  DevBuf<double> val, dv1, dv2, ref, eng;
  val.ensure(nodes * m);
  dv1.ensure(nodes * m);
  dv2.ensure(nodes * m);
  ref.ensure(static_cast<size_t>(n_types) * n * nb * 6 * B);
  eng.ensure(static_cast<size_t>(n_types) * n * 6 * Mp);
  DPB_CUDA(cudaMemsetAsync(ref.p, 0, ref.n * sizeof(double), stream));
  DPB_CUDA(cudaMemsetAsync(eng.p, 0, eng.n * sizeof(double), stream));
  DPB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
  for (int t = 0; t < n_types; ++t) {
    const EmbPtrs& net = emb_ptrs_host[t];
    switch (Mp / 32) {
      case 1: launch_nodes<1>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 2: launch_nodes<2>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 3: launch_nodes<3>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 4: launch_nodes<4>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 5: launch_nodes<5>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 6: launch_nodes<6>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 7: launch_nodes<7>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      case 8: launch_nodes<8>(net, d1, x0, step, static_cast<int>(nodes), val.p, dv1.p, dv2.p, stream); break;
      default: throw InputErr("feature width 4*d1 must be at most 256");
    }
    const int64_t tot = static_cast<int64_t>(n) * m;
    double* refp = ref.p + static_cast<size_t>(t) * n * nb * 6 * B;
    double* engp = eng.p + static_cast<size_t>(t) * n * 6 * Mp;
    k_table_coeffs<<<ceil_div(tot, 256), 256, 0, stream>>>(static_cast<int>(n), m, B, Mp, x0, step, val.p, dv1.p,
                                                          dv2.p, refp, engp);
    k_table_verify<<<ceil_div(tot + m, 256), 256, 0, stream>>>(static_cast<int>(n), m, Mp, x0, step, val.p, engp,
                                                               err.p);
    launches += 3;
  }
  check_err();
  if (coeffs_out)
    DPB_CUDA(cudaMemcpy(coeffs_out, ref.p, static_cast<size_t>(n_types) * n * nb * 6 * B * sizeof(double),
                        cudaMemcpyDeviceToHost));
  if (install) {
    tab.ensure(static_cast<size_t>(n_types) * n * 6 * Mp);
    ++tab_ver;
    DPB_CUDA(cudaMemcpyAsync(tab.p, eng.p, static_cast<size_t>(n_types) * n * 6 * Mp * sizeof(double),
                             cudaMemcpyDeviceToDevice, stream));
    tab_x0 = x0;
    tab_h = step;
    tab_n = n;
    tab_block = B;
    pbuf_cap = 0; // group counts change with the interval width
  }
  DPB_CUDA(cudaStreamSynchronize(stream));
}

} // namespace dpb
