// Host-side fixture generators and table compression for the dp_b200 C-ABI.
//
// These produce the inputs the hot path consumes (model weights, compression tables, FCC
// configurations, initial velocities) and must be bit-identical to the reference generators so
// that GPU results can be compared against the reference on identical inputs:
//   Rng / mix_seed                    /root/reference/proj/include/dpmd/rng.hpp:12-49
//   presets, gen_model, gen_config    /root/reference/proj/src/model_io.cpp:16-61, 129-224
//   make_test_model, make_random_config /root/reference/proj/tests/helpers.hpp:21-99
//   embedding_derivatives             /root/reference/proj/src/model.cpp:109-149
//   build_table / build_tables        /root/reference/proj/src/table.cpp:77-162
//   init_velocities                   /root/reference/proj/src/md.cpp:14-55
//   DPTB container                    /root/reference/proj/src/table_io.cpp:32-89
//   TanhTable                         /root/reference/proj/src/tanh_table.cpp:5-21
// Compiled with -ffp-contract=off: the reference is built without -march, so x86-64 codegen
// never fuses multiply-add and every expression below is evaluated as written.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dp_b200.h"
#include "host_common.hpp"

namespace dpb {

namespace {

// ---- deterministic stream (rng.hpp:12-41) ----
struct Stream {
  std::mt19937_64 eng;
  double spare = 0.0;
  bool has_spare = false;
  explicit Stream(uint64_t seed) : eng(seed) {}
  double uni() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uni();
    double u2 = uni();
    while (u1 <= 0.0) u1 = uni();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 6.283185307179586476925286766559 * u2;
    spare = rad * std::sin(ang);
    has_spare = true;
    return rad * std::cos(ang);
  }
};

void draw_normal(Stream& st, double* dst, std::size_t count, double sigma) {
  for (std::size_t k = 0; k < count; ++k) dst[k] = sigma * st.normal();
}

struct PresetRow {
  const char* name;
  dp_preset p;
  double fit_input_scale, fit_out_scale, embed_w_sigma, embed_center_hi;
};

// model_io.cpp:20-58 (copper-like and water-like).
const PresetRow* find_preset(const char* name) {
  static PresetRow rows[2];
  static bool init = false;
  if (!init) {
    std::memset(rows, 0, sizeof(rows));
    PresetRow& cu = rows[0];
    cu.name = "copper-like";
    cu.p.n_types = 1;
    cu.p.masses[0] = 63.546;
    cu.p.max_nbr[0] = 512;
    cu.p.r_cut = 8.0;
    cu.p.r_smooth = 7.5;
    cu.p.d1 = 32;
    cu.p.m_lt = 16;
    cu.p.fit_width = 240;
    cu.p.fit_hidden = 3;
    cu.p.lattice_a = 3.634;
    cu.p.site_pattern[0] = 0;
    cu.p.n_sites = 1;
    cu.fit_input_scale = 2.0e-3;
    cu.fit_out_scale = 0.1;
    cu.embed_w_sigma = 12.0;
    cu.embed_center_hi = 0.55;
    PresetRow& w = rows[1];
    w.name = "water-like";
    w.p.n_types = 2;
    w.p.masses[0] = 15.999;
    w.p.masses[1] = 1.008;
    w.p.max_nbr[0] = 46;
    w.p.max_nbr[1] = 92;
    w.p.r_cut = 6.0;
    w.p.r_smooth = 5.5;
    w.p.d1 = 32;
    w.p.m_lt = 16;
    w.p.fit_width = 240;
    w.p.fit_hidden = 3;
    w.p.lattice_a = 4.6;
    w.p.site_pattern[0] = 0;
    w.p.site_pattern[1] = 1;
    w.p.site_pattern[2] = 1;
    w.p.n_sites = 3;
    w.fit_input_scale = 2.0e-3;
    w.fit_out_scale = 0.1;
    w.embed_w_sigma = 12.0;
    w.embed_center_hi = 0.5;
    init = true;
  }
  for (auto& r : rows) {
    if (std::strcmp(r.name, name) == 0) return &r;
  }
  throw InputErr(std::string("unknown preset: ") + name);
}

// Weight scales of one generator family.
struct Scales {
  double emb_w0, emb_center_hi, fit_first, fit_out;
  bool test_family; // helpers.hpp:21-72 draws b0 ~ N(0,1) and w_out ~ N(0, 1/width)
};

void fill_model(const dp_preset& s, const Scales& sc, uint64_t seed, double* blob) {
  Stream st(seed);
  ModelLayout lay(s);
  const int d1 = s.d1;
  for (int t = 0; t < s.n_types; ++t) {
    double* e = blob + lay.emb_off[t];
    double* w0 = e;
    double* b0 = w0 + d1;
    double* w1 = b0 + d1;
    double* b1 = w1 + 2 * d1 * d1;
    double* w2 = b1 + 2 * d1;
    double* b2 = w2 + 8 * d1 * d1;
    draw_normal(st, w0, d1, sc.emb_w0);
    if (sc.emb_center_hi > 0.0) {
      for (int k = 0; k < d1; ++k) b0[k] = -w0[k] * (sc.emb_center_hi * st.uni());
    } else {
      draw_normal(st, b0, d1, 1.0);
    }
    draw_normal(st, w1, static_cast<std::size_t>(d1) * 2 * d1, 1.0 / std::sqrt(double(d1)));
    draw_normal(st, b1, 2 * d1, 1.0);
    draw_normal(st, w2, static_cast<std::size_t>(2 * d1) * 4 * d1,
                1.0 / std::sqrt(double(2 * d1)));
    draw_normal(st, b2, 4 * d1, 1.0);
  }
  for (int t = 0; t < s.n_types; ++t) {
    int cur = s.m_lt * 4 * d1;
    for (int k = 0; k < s.fit_hidden; ++k) {
      double* w = blob + lay.fit_w_off[t][k];
      double* b = blob + lay.fit_b_off[t][k];
      double sigma = 1.0 / std::sqrt(double(cur));
      if (k == 0) sigma *= sc.fit_first;
      draw_normal(st, w, static_cast<std::size_t>(cur) * s.fit_width, sigma);
      draw_normal(st, b, s.fit_width, 0.1);
      cur = s.fit_width;
    }
    double* wo = blob + lay.fit_wout_off[t];
    draw_normal(st, wo, cur, sc.fit_out / std::sqrt(double(cur)));
    blob[lay.fit_bout_off[t]] = 0.0;
  }
}

// Value, first and second derivative of one embedding net at input x, forward mode
// (model.cpp:109-149). Widths d1 -> 2 d1 -> 4 d1, doubling layers add their input repeated.
void embed_d012(const double* e, int d1, double x, double* g, double* g1, double* g2,
                std::vector<double>& scratch) {
  const int d2 = 2 * d1;
  const int d4 = 4 * d1;
  const double* w0 = e;
  const double* b0 = w0 + d1;
  const double* w1 = b0 + d1;
  const double* b1 = w1 + 2 * d1 * d1;
  const double* w2 = b1 + d2;
  const double* b2 = w2 + 8 * d1 * d1;
  scratch.resize(6 * static_cast<std::size_t>(d2));
  double* a = scratch.data();
  double* ag = a + d2;
  double* agg = ag + d2;
  double* h = agg + d2;
  double* hg = h + d2;
  double* hgg = hg + d2;
  for (int u = 0; u < d1; ++u) {
    const double t = std::tanh(x * w0[u] + b0[u]);
    const double dt = 1.0 - t * t;
    a[u] = t;
    ag[u] = dt * w0[u];
    agg[u] = -2.0 * t * dt * w0[u] * w0[u];
  }
  for (int v = 0; v < d2; ++v) {
    double z = b1[v], zg = 0.0, zgg = 0.0;
    for (int u = 0; u < d1; ++u) {
      const double w = w1[u * d2 + v];
      z += a[u] * w;
      zg += ag[u] * w;
      zgg += agg[u] * w;
    }
    const double t = std::tanh(z);
    const double dt = 1.0 - t * t;
    h[v] = a[v % d1] + t;
    hg[v] = ag[v % d1] + dt * zg;
    hgg[v] = agg[v % d1] + dt * zgg - 2.0 * t * dt * zg * zg;
  }
  for (int v = 0; v < d4; ++v) {
    double z = b2[v], zg = 0.0, zgg = 0.0;
    for (int u = 0; u < d2; ++u) {
      const double w = w2[u * d4 + v];
      z += h[u] * w;
      zg += hg[u] * w;
      zgg += hgg[u] * w;
    }
    const double t = std::tanh(z);
    const double dt = 1.0 - t * t;
    g[v] = h[v % d2] + t;
    g1[v] = hg[v % d2] + dt * zg;
    g2[v] = hgg[v % d2] + dt * zgg - 2.0 * t * dt * zg * zg;
  }
}

// Horner value of all m features at x on a blocked table (table.cpp:20-32, 57-75).
void table_values(const double* coeffs, std::size_t n, double x0, double hstep, int m, int blk,
                  double x, double* row) {
  const int nb = (m + blk - 1) / blk;
  const std::size_t stride = static_cast<std::size_t>(nb) * 6 * blk;
  if (!(x >= x0)) throw InputErr("table input below domain start");
  long th = static_cast<long>(std::floor((x - x0) / hstep));
  while (x0 + static_cast<double>(th + 1) * hstep <= x) ++th;
  while (th > 0 && x0 + static_cast<double>(th) * hstep > x) --th;
  if (th >= static_cast<long>(n)) th = static_cast<long>(n) - 1;
  const double u = x - (x0 + static_cast<double>(th) * hstep);
  const double* iv = coeffs + static_cast<std::size_t>(th) * stride;
  for (int p = 0; p < m; ++p) {
    const double* c = iv + static_cast<std::size_t>(p / blk) * 6 * blk + (p % blk);
    row[p] = ((((c[5 * blk] * u + c[4 * blk]) * u + c[3 * blk]) * u + c[2 * blk]) * u +
              c[blk]) * u + c[0];
  }
}

} // namespace

ModelLayout::ModelLayout(const dp_preset& s) {
  const int d1 = s.d1;
  std::size_t off = 0;
  const std::size_t emb = static_cast<std::size_t>(d1) * (2 + 2 * d1 + 2 + 8 * d1 + 4);
  for (int t = 0; t < s.n_types; ++t) {
    emb_off.push_back(off);
    off += emb;
  }
  fit_w_off.resize(s.n_types);
  fit_b_off.resize(s.n_types);
  for (int t = 0; t < s.n_types; ++t) {
    int cur = s.m_lt * 4 * d1;
    for (int k = 0; k < s.fit_hidden; ++k) {
      fit_w_off[t].push_back(off);
      off += static_cast<std::size_t>(cur) * s.fit_width;
      fit_b_off[t].push_back(off);
      off += s.fit_width;
      cur = s.fit_width;
    }
    fit_wout_off.push_back(off);
    off += cur;
    fit_bout_off.push_back(off);
    off += 1;
  }
  total = off;
}

void check_shape(const dp_preset& s) {
  if (s.n_types < 1 || s.n_types > 8) throw InputErr("n_types must lie in [1, 8]");
  if (s.d1 < 1) throw InputErr("embedding width must be positive");
  if (s.m_lt < 1 || s.m_lt > 4 * s.d1) throw InputErr("m_lt must lie in [1, 4*d1]");
  if (s.fit_hidden < 1 || s.fit_width < 1) throw InputErr("fitting net needs hidden layers");
  if (!(s.r_cut > 0.0) || !(s.r_smooth >= 0.0) || !(s.r_smooth < s.r_cut))
    throw InputErr("model cutoffs must satisfy 0 <= r_smooth < r_cut");
  for (int t = 0; t < s.n_types; ++t)
    if (s.max_nbr[t] <= 0) throw InputErr("model max_nbr entries must be positive");
}

double domain_end(double r_smooth, double r_cut) {
  const double r_min = 0.5; // table.hpp:52-54 default closest approach
  return switch_w(r_min, r_smooth, r_cut) / r_min;
}

} // namespace dpb

using namespace dpb;

extern "C" {

int dp_preset_get(const char* name, dp_preset* out) {
  return guard_call(nullptr, [&] {
    if (!name || !out) throw InputErr("null argument");
    *out = find_preset(name)->p;
  });
}

int64_t dp_model_blob_size(const dp_preset* shape) {
  if (!shape) return -1;
  try {
    check_shape(*shape);
    return static_cast<int64_t>(ModelLayout(*shape).total);
  } catch (...) {
    return -1;
  }
}

int dp_gen_model(const char* preset, uint64_t seed, double* blob) {
  return guard_call(nullptr, [&] {
    const PresetRow* r = find_preset(preset);
    Scales sc{r->embed_w_sigma, r->embed_center_hi, r->fit_input_scale, r->fit_out_scale, false};
    fill_model(r->p, sc, seed, blob);
  });
}

int dp_gen_test_model(const dp_preset* shape, uint64_t seed, double fit_scale, double* blob) {
  return guard_call(nullptr, [&] {
    check_shape(*shape);
    Scales sc{1.0, 0.0, fit_scale, 1.0, true};
    fill_model(*shape, sc, seed, blob);
  });
}

int dp_build_tables(const dp_preset* shape, const double* blob, double h, uint64_t* n_intervals,
                    double* x_end_out, double* coeffs) {
  return guard_call(nullptr, [&] {
    check_shape(*shape);
    const double x0 = 0.0;
    const double x_end = domain_end(shape->r_smooth, shape->r_cut);
    if (!(x_end > 0.0)) throw InputErr("table domain end is not positive");
    if (!(h > 0.0)) throw InputErr("table step must be positive");
    std::size_t n = static_cast<std::size_t>(std::ceil((x_end - x0) / h - 1e-9));
    if (n == 0) n = 1;
    if (n_intervals) *n_intervals = n;
    if (x_end_out) *x_end_out = x_end;
    if (!coeffs) return;
    const int d1 = shape->d1;
    const int m = 4 * d1;
    const int blk = 16;
    const int nb = (m + blk - 1) / blk;
    const std::size_t stride = static_cast<std::size_t>(nb) * 6 * blk;
    ModelLayout lay(*shape);
    for (int t = 0; t < shape->n_types; ++t) {
      const double* e = blob + lay.emb_off[t];
      double* tab = coeffs + static_cast<std::size_t>(t) * n * stride;
      std::memset(tab, 0, n * stride * sizeof(double));
      const std::size_t nn = n + 1;
      std::vector<double> f0(nn * m), f1(nn * m), f2(nn * m);
#pragma omp parallel
      {
        std::vector<double> scratch;
#pragma omp for schedule(static)
        for (long k = 0; k < static_cast<long>(nn); ++k) {
          const std::size_t o = static_cast<std::size_t>(k) * m;
          embed_d012(e, d1, x0 + static_cast<double>(k) * h, &f0[o], &f1[o], &f2[o], scratch);
        }
      }
      // Quintic Hermite per interval: match value, slope and curvature at both nodes.
#pragma omp parallel for schedule(static)
      for (long th = 0; th < static_cast<long>(n); ++th) {
        const double hl = (x0 + static_cast<double>(th + 1) * h) - (x0 + static_cast<double>(th) * h);
        const std::size_t lo = static_cast<std::size_t>(th) * m;
        const std::size_t hi = lo + m;
        double* iv = tab + static_cast<std::size_t>(th) * stride;
        for (int p = 0; p < m; ++p) {
          const double c0 = f0[lo + p];
          const double c1 = f1[lo + p];
          const double c2 = 0.5 * f2[lo + p];
          const double dv = f0[hi + p] - (c0 + c1 * hl + c2 * hl * hl);
          const double dg = f1[hi + p] - (c1 + 2.0 * c2 * hl);
          const double dc = f2[hi + p] - 2.0 * c2;
          const double h2 = hl * hl;
          const double h3 = h2 * hl;
          double* c = iv + static_cast<std::size_t>(p / blk) * 6 * blk + (p % blk);
          c[0] = c0;
          c[blk] = c1;
          c[2 * blk] = c2;
          c[3 * blk] = (10.0 * dv - 4.0 * hl * dg + 0.5 * h2 * dc) / h3;
          c[4 * blk] = (-15.0 * dv + 7.0 * hl * dg - h2 * dc) / (h3 * hl);
          c[5 * blk] = (6.0 * dv - 3.0 * hl * dg + 0.5 * h2 * dc) / (h3 * h2);
        }
      }
      // Node verification (table.cpp:136-147).
      std::vector<double> row(m);
      for (std::size_t k = 0; k < nn; ++k) {
        table_values(tab, n, x0, h, m, blk, x0 + static_cast<double>(k) * h, row.data());
        for (int p = 0; p < m; ++p) {
          const double ref = f0[k * m + p];
          const double err = std::fabs(row[p] - ref);
          const double scale = std::max(1.0, std::fabs(ref));
          if (!(err <= 1e-10 * scale)) throw NumErr("table verification failed at a node");
        }
      }
    }
  });
}

int dp_gen_config(const char* preset, int nx, int ny, int nz, double jitter, uint64_t seed,
                  double* pos, int32_t* types, double box[9]) {
  return guard_call(nullptr, [&] {
    const PresetRow* r = find_preset(preset);
    if (nx < 1 || ny < 1 || nz < 1) throw InputErr("cell repeat counts must be positive");
    if (jitter < 0.0) throw InputErr("jitter must be non-negative");
    static const double sites[4][3] = {{0, 0, 0}, {0, 0.5, 0.5}, {0.5, 0, 0.5}, {0.5, 0.5, 0}};
    const double a = r->p.lattice_a;
    for (int k = 0; k < 9; ++k) box[k] = 0.0;
    box[0] = a * nx;
    box[4] = a * ny;
    box[8] = a * nz;
    Stream st(seed);
    std::size_t at = 0;
    for (int ix = 0; ix < nx; ++ix)
      for (int iy = 0; iy < ny; ++iy)
        for (int iz = 0; iz < nz; ++iz)
          for (int b = 0; b < 4; ++b) {
            const double base[3] = {a * (ix + sites[b][0]), a * (iy + sites[b][1]),
                                    a * (iz + sites[b][2])};
            for (int x = 0; x < 3; ++x) {
              const double off = jitter > 0.0 ? jitter * (2.0 * st.uni() - 1.0) : 0.0;
              pos[3 * at + x] = base[x] + off;
            }
            types[at] = r->p.site_pattern[at % r->p.n_sites];
            ++at;
          }
  });
}

int dp_gen_random_config(int n, int n_types, double L, double min_sep, uint64_t seed, double* pos,
                         int32_t* types) {
  return guard_call(nullptr, [&] {
    if (n < 1 || n_types < 1) throw InputErr("bad random config request");
    Stream st(seed);
    int have = 0;
    while (have < n) {
      const double p[3] = {L * st.uni(), L * st.uni(), L * st.uni()};
      bool ok = true;
      for (int i = 0; i < have && ok; ++i) {
        double d2 = 0.0;
        for (int x = 0; x < 3; ++x) {
          double d = p[x] - pos[3 * i + x];
          d -= L * std::round(d / L);
          d2 += d * d;
        }
        if (d2 < min_sep * min_sep) ok = false;
      }
      if (!ok) continue;
      for (int x = 0; x < 3; ++x) pos[3 * have + x] = p[x];
      types[have] = static_cast<int32_t>(st.eng() % static_cast<uint64_t>(n_types));
      ++have;
    }
  });
}

int dp_init_velocities(int64_t n, const int32_t* types, const double* masses, double t_init,
                       uint64_t seed, double* vel) {
  return guard_call(nullptr, [&] {
    if (n < 2) throw InputErr("velocity initialization needs at least two atoms");
    if (t_init < 0.0) throw InputErr("temperature must be non-negative");
    for (int64_t k = 0; k < 3 * n; ++k) vel[k] = 0.0;
    if (t_init == 0.0) return;
    Stream st(seed);
    for (int64_t i = 0; i < n; ++i) {
      const double mass = masses[types[i]];
      const double sigma = std::sqrt(units::K_B * t_init / (mass * units::MVV_TO_EV));
      for (int x = 0; x < 3; ++x) vel[3 * i + x] = sigma * st.normal();
    }
    double p[3] = {0.0, 0.0, 0.0};
    double mtot = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double mass = masses[types[i]];
      mtot += mass;
      for (int x = 0; x < 3; ++x) p[x] += mass * vel[3 * i + x];
    }
    for (int64_t i = 0; i < n; ++i)
      for (int x = 0; x < 3; ++x) vel[3 * i + x] -= p[x] / mtot;
    double ke = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double mass = masses[types[i]];
      const double v2 = vel[3 * i] * vel[3 * i] + vel[3 * i + 1] * vel[3 * i + 1] +
                        vel[3 * i + 2] * vel[3 * i + 2];
      ke += 0.5 * mass * v2 * units::MVV_TO_EV;
    }
    const double t_cur = 2.0 * ke / (3.0 * static_cast<double>(n) * units::K_B);
    const double scale = std::sqrt(t_init / t_cur);
    for (int64_t k = 0; k < 3 * n; ++k) vel[k] *= scale;
  });
}

uint64_t dp_mix_seed(uint64_t seed, uint64_t k) {
  uint64_t z = seed + (k + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int dp_write_tables(const char* path, const dp_table_desc* t) {
  return guard_call(nullptr, [&] {
    if (!t || t->n_tables < 1) throw InputErr("no tables to write");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw InputErr(std::string("cannot open table file for writing: ") + path);
    const uint32_t hdr[4] = {1u, static_cast<uint32_t>(t->n_tables), static_cast<uint32_t>(t->m),
                             static_cast<uint32_t>(t->block)};
    const uint64_t n = t->n;
    bool ok = std::fwrite("DPTB", 1, 4, f) == 4 && std::fwrite(hdr, 4, 4, f) == 4 &&
              std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&t->x0, 8, 1, f) == 1 &&
              std::fwrite(&t->h, 8, 1, f) == 1;
    const std::size_t stride =
        static_cast<std::size_t>((t->m + t->block - 1) / t->block) * 6 * t->block;
    for (int k = 0; ok && k < t->n_tables; ++k)
      ok = std::fwrite(t->coeffs[k], 8, n * stride, f) == n * stride;
    std::fclose(f);
    if (!ok) throw InputErr(std::string("short write to table file: ") + path);
  });
}

int dp_read_tables_header(const char* path, int* n_tables, int* m, int* block, uint64_t* n,
                          double* x0, double* h) {
  return guard_call(nullptr, [&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw InputErr(std::string("cannot open table file: ") + path);
    char magic[4];
    uint32_t hdr[4];
    uint64_t nn;
    double xs[2];
    bool ok = std::fread(magic, 1, 4, f) == 4;
    if (!ok || std::memcmp(magic, "DPTB", 4) != 0) {
      std::fclose(f);
      throw InputErr(std::string("not a table file (bad magic): ") + path);
    }
    ok = std::fread(hdr, 4, 4, f) == 4 && std::fread(&nn, 8, 1, f) == 1 &&
         std::fread(xs, 8, 2, f) == 2;
    std::fclose(f);
    if (!ok) throw InputErr("table file truncated");
    if (hdr[0] != 1) throw InputErr("unsupported table file version");
    if (hdr[1] == 0 || hdr[2] == 0 || hdr[3] == 0 || nn == 0 || !(xs[1] > 0.0))
      throw InputErr("table file header is inconsistent");
    *n_tables = static_cast<int>(hdr[1]);
    *m = static_cast<int>(hdr[2]);
    *block = static_cast<int>(hdr[3]);
    *n = nn;
    *x0 = xs[0];
    *h = xs[1];
  });
}

int dp_read_tables(const char* path, double* coeffs) {
  int nt, m, blk;
  uint64_t n;
  double x0, h;
  int rc = dp_read_tables_header(path, &nt, &m, &blk, &n, &x0, &h);
  if (rc) return rc;
  return guard_call(nullptr, [&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw InputErr(std::string("cannot open table file: ") + path);
    std::fseek(f, 4 + 16 + 8 + 16, SEEK_SET);
    const std::size_t count =
        static_cast<std::size_t>(nt) * n * static_cast<std::size_t>((m + blk - 1) / blk) * 6 * blk;
    const bool ok = std::fread(coeffs, 8, count, f) == count;
    std::fclose(f);
    if (!ok) throw InputErr(std::string("table file truncated: ") + path);
  });
}

int dp_tanh_table(double* coef) {
  // Quadratic tanh table on [0, 8], h = 2^-10 (tanh_table.hpp:14-38, tanh_table.cpp:5-21).
  const double H = 0x1.0p-10, INV_H = 0x1.0p10;
  const int n = 8 * 1024;
  for (int k = 0; k <= n; ++k) {
    const double f = std::tanh(k * H);
    coef[3 * k] = f;
    coef[3 * k + 1] = 1.0 - f * f;
  }
  for (int k = 0; k < n; ++k)
    coef[3 * k + 2] = (coef[3 * (k + 1)] - coef[3 * k] - coef[3 * k + 1] * H) * (INV_H * INV_H);
  coef[3 * n + 2] = 0.0;
  return DP_OK;
}

} // extern "C"
