// Device-side building blocks shared by the tabulated (tabulate.cu) and exact (exact.cu)
// environment / embedding kernels: kernel parameter block, env-mat of one entry
// (env_mat.cpp:29-71), switching function (switch_fn.hpp:11-25), table locate (table.cpp:20-32)
// and deterministic warp reductions.
#pragma once

#include "engine.hpp"

namespace dpb {
namespace {

struct TabParams {
  const double4* pos;
  const int64_t* row_off;
  const uint64_t* keys;
  const uint8_t* center; // [n] 1 = evaluated centre, 0 = ghost
  int16_t* ridx;        // [E] list rank of a real entry within its row, -1 otherwise
  double* rec;          // [Ec][8] per-real records R0..R3, u, d0..d2 (chunk-local, rank order)
  uint64_t* sscr;       // [Ec] sort scratch (wide bin ranges)
  int32_t* egrp;        // [Ec] group index of real k of a centre (chunk-local, rank order)
  int32_t* gbin;        // [Ec] per row: the centre's group bins, ascending (first n_grp entries)
  int32_t* n_real;      // [n]
  int32_t* n_grp;       // [n+1] groups per centre -> (scanned) offsets into Pbuf
  const int64_t* goff;  // [n+1] exclusive scan of n_grp
  const int64_t* realoff; // [n+1] first compact pair-gradient slot of each centre
  double* Pbuf;         // [sum groups][24]
  int64_t pcap;         // groups Pbuf can hold
  const int32_t* xbin;  // exact path: [E] neighbour type of a real entry, -1 otherwise
  double* xrc;          // exact path: [4][E] R0..R3 per entry
  const double* tab;    // [type][interval][6][Mp]
  const float* tab32;   // the same in FP32 (mixed mode forward contraction) or null
  const int* max_nbr;
  DevCell c;
  double rc2, rs, rc;
  double x0, h, x_end, ih; // ih = 1 / h (first guess of locate only)
  int tn;
  int n, n_types, M, Mp, mlt, K0p;
  int i0, i1;           // centre range of this launch (pipelined halves); [0, n) otherwise
  int64_t E;            // global entry capacity
  int64_t es;           // capacity of the chunk-local entry arrays (rec, egrp, gbin, sscr)
  const int32_t* slot_of;
  double* T;            // [n][4][Mp]
  double* D;            // [slots][K0p] (FP64 mode)
  float* D2;            // [slots][2*K0p] mixed mode: tf32 split (hi | lo) of D, the tcgen05 operand
  const double* dD;
  double* g;            // [gcap][3] compact pair gradients
  int64_t gcap;
  double* vpart;        // [n][9] per-centre virial partials
  unsigned long long* counters;
  int* err;
  int scap;
};

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ double node_x(double x0, double h, int th) {
  return __dadd_rn(x0, __dmul_rn(static_cast<double>(th), h));
}

// locate (table.cpp:20-32): floor, then nudge so node(th) <= x < node(th+1) in the exact
// arithmetic of the nodes; clamp past the end and flag extrapolation.
__device__ __forceinline__ int locate(const TabParams& p, double x, bool& ext, int* err) {
  if (!(x >= p.x0)) {
    raise_err(err, DEV_TABLE_LOW);
    ext = false;
    return 0;
  }
  // first guess by a multiply (at most one interval off); the nudge loops below fix th exactly
  const double tf = floor(__dmul_rn(__dsub_rn(x, p.x0), p.ih));
  if (!(tf < static_cast<double>(p.tn) + 2.0)) {  // far past the end (or inf): clamp directly
    ext = true;
    return p.tn - 1;
  }
  int th = static_cast<int>(tf);
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



inline TabParams make_params(Engine& E) {
  TabParams p{};
  p.pos = E.pos4.p;
  p.row_off = E.row_off.p;
  p.keys = E.keys.p;
  p.center = E.center.p;
  p.ridx = E.ridx.p;
  p.rec = E.we(E.rec, 8); // chunk-local entry arrays of the current buffer set
  p.sscr = E.we(E.sscr);
  p.egrp = E.we(E.egrp);
  p.gbin = E.we(E.gbin);
  p.n_real = E.n_real.p;
  p.n_grp = E.n_grp.p;
  p.goff = E.goff.p;
  p.realoff = E.realoff.p;
  p.Pbuf = E.Pbuf.p;
  p.pcap = E.pbuf_cap;
  p.xbin = E.xbin.p;
  p.xrc = E.xrc.p;
  p.tab = E.tab.p;
  p.tab32 = E.precision == 1 ? E.tab32.p : nullptr;
  p.max_nbr = E.d_max_nbr.p;
  p.c = E.cell;
  p.rc2 = E.r_cut * E.r_cut;
  p.rs = E.r_smooth;
  p.rc = E.r_cut;
  p.x0 = E.tab_x0;
  p.h = E.tab_h;
  p.ih = 1.0 / E.tab_h;
  p.x_end = E.tab_x0 + E.tab_h * static_cast<double>(E.tab_n);
  p.tn = static_cast<int>(E.tab_n);
  p.n = static_cast<int>(E.n);
  p.i0 = 0;
  p.i1 = static_cast<int>(E.n);
  p.n_types = E.n_types;
  p.M = E.M;
  p.Mp = E.Mp;
  p.mlt = E.mlt;
  p.K0p = E.K0p;
  p.E = E.e_cap;
  p.es = E.ck_cap_e; // chunk-local entry arrays are indexed e - row_off[i0] (see chunk_params)
  p.slot_of = E.slot_of.p;
  p.T = E.wa(E.T, 4 * E.Mp); // per-centre windows of the current chunk (Engine::use_chunk)
  p.D = E.precision == 1 ? nullptr : E.ws(E.D, E.K0p);
  p.D2 = E.precision == 1 ? E.ws(E.tc_d2, 2 * E.K0p) : nullptr;
  p.dD = E.ws(E.dD, E.K0p);
  p.g = E.g.p;
  p.gcap = E.g_cap;
  p.vpart = E.vpart.p;
  p.counters = E.counters.p;
  p.err = E.err.p;
  int scap = 32;
  while (scap < E.row_cap) scap <<= 1;
  p.scap = scap;
  return p;
}


} // namespace
} // namespace dpb
