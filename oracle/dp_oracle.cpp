// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked or called by the product path.
//
// CPU restatement of the reference's per-step DP evaluation (the hot path of SURVEY.md §8), used
// by tests/ (parity checker), __graft_entry__.smoke() and bench.py's cpu_baseline leg. It takes
// the same dp_model_desc / dp_table_desc inputs as the GPU library and follows the reference's
// operation order so that, compiled without FMA contraction, it is bitwise equal to the
// reference (pinned by tests/test_oracle.py against oracle/_ref and tests/golden/).
//
// Restated from (all paths under /root/reference/proj):
//   Cell::refresh / plane_spacing / frac   src/geom.cpp:7-38, include/dpmd/geom.hpp:39-43
//   displacement                           include/dpmd/geom.hpp:61-69
//   scan_images / brute / cells / sort     src/neighbor.cpp:10-158
//   switch_weight(+deriv)                  include/dpmd/switch_fn.hpp:11-25
//   build_environment_matrix               src/env_mat.cpp:10-74
//   locate / eval_table(_value)            src/table.cpp:20-75
//   fused_contract / fused_atom_energy     src/fused.cpp:13-37, 182-243
//   descriptor_from_t / dt_from_dd         include/dpmd/contract.hpp:9-38
//   fitting_forward / fitting_backward     src/model.cpp:151-203
//   scatter_pair_grads                     src/exact.cpp:22-38
//   compute_energy_forces_virial_tabulated src/fused.cpp:245-288
//   run_md                                 src/md.cpp:151-231
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dp_b200.h"

namespace {

struct InErr : std::runtime_error {
  explicit InErr(const std::string& m) : std::runtime_error(m) {}
};
struct NuErr : std::runtime_error {
  explicit NuErr(const std::string& m) : std::runtime_error(m) {}
};

std::string g_err;

template <class F>
int run(F&& f) {
  try {
    f();
    return 0;
  } catch (const InErr& e) {
    g_err = e.what();
    return 2;
  } catch (const NuErr& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct Box {
  double h[9], hinv[9], vol;
  bool per[3];
  void init(const double* hh, const uint8_t* pbc) {
    for (int k = 0; k < 9; ++k) h[k] = hh[k];
    for (int k = 0; k < 3; ++k) per[k] = pbc[k] != 0;
    const double* a = h;
    const double* b = h + 3;
    const double* c = h + 6;
    const double bc[3] = {b[1] * c[2] - b[2] * c[1], b[2] * c[0] - b[0] * c[2],
                          b[0] * c[1] - b[1] * c[0]};
    vol = a[0] * bc[0] + a[1] * bc[1] + a[2] * bc[2];
    if (!(std::fabs(vol) > 1e-12)) throw InErr("cell is singular or has near-zero volume");
    const double ca[3] = {c[1] * a[2] - c[2] * a[1], c[2] * a[0] - c[0] * a[2],
                          c[0] * a[1] - c[1] * a[0]};
    const double ab[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2],
                          a[0] * b[1] - a[1] * b[0]};
    for (int x = 0; x < 3; ++x) {
      hinv[3 * x + 0] = bc[x] / vol;
      hinv[3 * x + 1] = ca[x] / vol;
      hinv[3 * x + 2] = ab[x] / vol;
    }
    if (vol < 0.0) vol = -vol;
  }
  double spacing(int k) const {
    const double* u = h + 3 * ((k + 1) % 3);
    const double* v = h + 3 * ((k + 2) % 3);
    const double cr[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2],
                          u[0] * v[1] - u[1] * v[0]};
    return vol / std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  }
  void frac(const double* r, double* f) const {
    for (int k = 0; k < 3; ++k) f[k] = r[0] * hinv[k] + r[1] * hinv[3 + k] + r[2] * hinv[6 + k];
  }
  // d = (r_j + s.h) - r_i with the reference's left-to-right order.
  void disp(const double* ri, const double* rj, const int* s, double* d) const {
    for (int x = 0; x < 3; ++x) {
      const double img = rj[x] + s[0] * h[x] + s[1] * h[3 + x] + s[2] * h[6 + x];
      d[x] = img - ri[x];
    }
  }
};

struct Entry {
  int j, s[3];
};

bool entry_less(const Entry& a, const Entry& b) {
  if (a.j != b.j) return a.j < b.j;
  if (a.s[0] != b.s[0]) return a.s[0] < b.s[0];
  if (a.s[1] != b.s[1]) return a.s[1] < b.s[1];
  return a.s[2] < b.s[2];
}

using Lists = std::vector<std::vector<Entry>>;

// Direct pair scan over the image range of every (i <= j) pair; each accepted image is inserted
// into both rows from one distance evaluation.
void nlist_brute(const Box& bx, int n, const double* pos, double cutoff, Lists& out) {
  out.assign(n, {});
  std::vector<double> fr(3 * n);
  for (int i = 0; i < n; ++i) bx.frac(pos + 3 * i, &fr[3 * i]);
  double margin[3];
  for (int k = 0; k < 3; ++k) margin[k] = cutoff / bx.spacing(k);
  const double c2 = cutoff * cutoff;
  for (int i = 0; i < n; ++i) {
    for (int j = i; j < n; ++j) {
      int lo[3], hi[3];
      for (int k = 0; k < 3; ++k) {
        if (bx.per[k]) {
          const double df = fr[3 * j + k] - fr[3 * i + k];
          lo[k] = static_cast<int>(std::ceil(-df - margin[k] - 1e-12));
          hi[k] = static_cast<int>(std::floor(-df + margin[k] + 1e-12));
        } else {
          lo[k] = hi[k] = 0;
        }
      }
      int s[3];
      for (s[0] = lo[0]; s[0] <= hi[0]; ++s[0])
        for (s[1] = lo[1]; s[1] <= hi[1]; ++s[1])
          for (s[2] = lo[2]; s[2] <= hi[2]; ++s[2]) {
            if (i == j && s[0] == 0 && s[1] == 0 && s[2] == 0) continue;
            double d[3];
            bx.disp(pos + 3 * i, pos + 3 * j, s, d);
            if (d[0] * d[0] + d[1] * d[1] + d[2] * d[2] <= c2) {
              out[i].push_back({j, {s[0], s[1], s[2]}});
              if (j != i) out[j].push_back({i, {-s[0], -s[1], -s[2]}});
            }
          }
    }
  }
  for (auto& v : out) std::sort(v.begin(), v.end(), entry_less);
}

// Linked-cell search (>= 3 bins on every periodic axis): half walk q > i over the 27
// neighbouring bins, shift = wrap[q] + bin wrap - wrap[i].
void nlist_cells(const Box& bx, int n, const double* pos, double cutoff, const int* nb,
                 Lists& out) {
  out.assign(n, {});
  std::vector<int> wrap(3 * n), bin(n), nxt(n, -1), head(nb[0] * nb[1] * nb[2], -1);
  for (int i = 0; i < n; ++i) {
    double f[3];
    bx.frac(pos + 3 * i, f);
    int b[3];
    for (int k = 0; k < 3; ++k) {
      const double fl = std::floor(f[k]);
      wrap[3 * i + k] = -static_cast<int>(fl);
      int bk = static_cast<int>((f[k] - fl) * nb[k]);
      b[k] = std::min(std::max(bk, 0), nb[k] - 1);
    }
    bin[i] = (b[0] * nb[1] + b[1]) * nb[2] + b[2];
    nxt[i] = head[bin[i]];
    head[bin[i]] = i;
  }
  const double c2 = cutoff * cutoff;
  for (int i = 0; i < n; ++i) {
    const int bi[3] = {bin[i] / (nb[1] * nb[2]), (bin[i] / nb[2]) % nb[1], bin[i] % nb[2]};
    for (int o = 0; o < 27; ++o) {
      const int db[3] = {o / 9 - 1, (o / 3) % 3 - 1, o % 3 - 1};
      int bq[3], wq[3];
      for (int k = 0; k < 3; ++k) {
        int t = bi[k] + db[k];
        wq[k] = 0;
        if (t < 0) {
          t += nb[k];
          wq[k] = -1;
        } else if (t >= nb[k]) {
          t -= nb[k];
          wq[k] = 1;
        }
        bq[k] = t;
      }
      for (int q = head[(bq[0] * nb[1] + bq[1]) * nb[2] + bq[2]]; q >= 0; q = nxt[q]) {
        if (q <= i) continue;
        int s[3];
        for (int k = 0; k < 3; ++k) s[k] = wrap[3 * q + k] + wq[k] - wrap[3 * i + k];
        double d[3];
        bx.disp(pos + 3 * i, pos + 3 * q, s, d);
        if (d[0] * d[0] + d[1] * d[1] + d[2] * d[2] <= c2) {
          out[i].push_back({q, {s[0], s[1], s[2]}});
          out[q].push_back({i, {-s[0], -s[1], -s[2]}});
        }
      }
    }
  }
  for (auto& v : out) std::sort(v.begin(), v.end(), entry_less);
}

void nlist(const Box& bx, int n, const double* pos, double cutoff, Lists& out) {
  if (cutoff <= 0.0) throw InErr("neighbor cutoff must be positive");
  int nb[3];
  bool cells = n > 0;
  for (int k = 0; k < 3 && cells; ++k) {
    if (!bx.per[k]) {
      cells = false;
      break;
    }
    nb[k] = static_cast<int>(std::floor(bx.spacing(k) / cutoff));
    if (nb[k] < 3) cells = false;
  }
  if (cells)
    nlist_cells(bx, n, pos, cutoff, nb, out);
  else
    nlist_brute(bx, n, pos, cutoff, out);
}

// ---- model views ----
struct Net {
  const dp_fitting_desc* f;
};

struct Model {
  const dp_model_desc* md;
  const dp_table_desc* td;
  int M, mlt, stride;
};

double sw(double r, double rs, double rc) {
  if (r >= rc) return 0.0;
  if (r <= rs) return 1.0;
  const double u = (r - rs) / (rc - rs);
  const double uu = u * u;
  return std::max(0.0, uu * u * (-6.0 * uu + 15.0 * u - 10.0) + 1.0);
}

double sw_d(double r, double rs, double rc) {
  if (r >= rc || r <= rs) return 0.0;
  const double inv = 1.0 / (rc - rs);
  const double u = (r - rs) * inv;
  const double um1 = u - 1.0;
  return -30.0 * u * u * um1 * um1 * inv;
}

// Interval lookup with the reference's nudging; returns interval, local u, extrapolation flag.
std::size_t locate(const dp_table_desc* t, double x, double& u, bool& ext) {
  if (!(x >= t->x0)) throw InErr("table input below domain start");
  long th = static_cast<long>(std::floor((x - t->x0) / t->h));
  while (t->x0 + static_cast<double>(th + 1) * t->h <= x) ++th;
  while (th > 0 && t->x0 + static_cast<double>(th) * t->h > x) --th;
  ext = false;
  if (th >= static_cast<long>(t->n)) {
    th = static_cast<long>(t->n) - 1;
    ext = x > t->x0 + t->h * static_cast<double>(t->n);
  }
  u = x - (t->x0 + static_cast<double>(th) * t->h);
  return static_cast<std::size_t>(th);
}

void row_eval(const Model& m, int ty, double x, double* row, double* row1, bool& ext) {
  const dp_table_desc* t = m.td;
  double u;
  const std::size_t th = locate(t, x, u, ext);
  const double* iv = t->coeffs[ty] + th * static_cast<std::size_t>(m.stride);
  const int B = t->block;
  for (int p = 0; p < m.M; ++p) {
    const double* c = iv + static_cast<std::size_t>(p / B) * 6 * B + (p % B);
    const double a0 = c[0], a1 = c[B], a2 = c[2 * B], a3 = c[3 * B], a4 = c[4 * B], a5 = c[5 * B];
    row[p] = ((((a5 * u + a4) * u + a3) * u + a2) * u + a1) * u + a0;
    if (row1) row1[p] = (((5.0 * a5 * u + 4.0 * a4) * u + 3.0 * a3) * u + 2.0 * a2) * u + a1;
  }
}

struct Slot {
  double s, r4[4], d[3], dv[12];
  int j;
};

struct PairGrads {
  std::vector<std::size_t> off;
  std::vector<int> cnt, atom;
  std::vector<double> d, g;
};

struct Counts {
  uint64_t fwd = 0, bwd = 0, ext = 0;
};

// One center through env-mat, fused tabulate+contract, fitting and the gradient pass.
double atom_energy(const Model& m, const Box& bx, const double* pos, const int32_t* ty, int i,
                   const std::vector<Entry>& ents, PairGrads& pg, Counts& ct) {
  const dp_model_desc* md = m.md;
  const int nt = md->n_types;
  const int M = m.M, mlt = m.mlt;
  const double rc2 = md->r_cut * md->r_cut;
  // Environment rows, stable-partitioned by neighbour type (sector order).
  std::vector<std::vector<Slot>> sec(nt);
  for (const Entry& e : ents) {
    double d[3];
    bx.disp(pos + 3 * i, pos + 3 * e.j, e.s, d);
    const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (r2 >= rc2) continue;
    if (r2 < 1e-12) throw NuErr("overlapping atoms in neighbor environment");
    const double r = std::sqrt(r2);
    const int t = ty[e.j];
    if (static_cast<int>(sec[t].size()) >= md->max_nbr[t])
      throw NuErr("neighbor slot capacity exceeded for type " + std::to_string(t));
    Slot sl;
    const double w = sw(r, md->r_smooth, md->r_cut);
    const double wd = sw_d(r, md->r_smooth, md->r_cut);
    const double ir = 1.0 / r;
    sl.s = w * ir;
    const double sd = wd * ir - w * ir * ir;
    const double u[3] = {d[0] * ir, d[1] * ir, d[2] * ir};
    sl.r4[0] = sl.s;
    for (int x = 0; x < 3; ++x) sl.r4[1 + x] = sl.s * u[x];
    for (int x = 0; x < 3; ++x) sl.d[x] = d[x];
    for (int x = 0; x < 3; ++x) sl.dv[x] = sd * u[x];
    for (int y = 0; y < 3; ++y)
      for (int x = 0; x < 3; ++x) {
        double v = sd * u[x] * u[y] - sl.s * ir * u[x] * u[y];
        if (x == y) v += sl.s * ir;
        sl.dv[3 * (1 + y) + x] = v;
      }
    sl.j = e.j;
    sec[t].push_back(sl);
  }
  // Forward: T[a][p] += R[a] * row[p] over real slots.
  std::vector<double> T(4 * M, 0.0), row(M), row1(M);
  for (int t = 0; t < nt; ++t)
    for (const Slot& sl : sec[t]) {
      bool ext;
      row_eval(m, t, sl.s, row.data(), nullptr, ext);
      ++ct.fwd;
      if (ext) ++ct.ext;
      for (int a = 0; a < 4; ++a) {
        const double ra = sl.r4[a];
        for (int p = 0; p < M; ++p) T[a * M + p] += ra * row[p];
      }
    }
  // D = T<^T T.
  std::vector<double> D(static_cast<std::size_t>(mlt) * M);
  for (int q = 0; q < mlt; ++q)
    for (int p = 0; p < M; ++p) {
      double acc = 0.0;
      for (int a = 0; a < 4; ++a) acc += T[a * M + q] * T[a * M + p];
      D[static_cast<std::size_t>(q) * M + p] = acc;
    }
  // Fitting forward, keeping tanh outputs per layer.
  const dp_fitting_desc* f = &md->fitting[ty[i]];
  const int L = f->n_layers;
  std::vector<std::vector<double>> tl(L);
  std::vector<double> cur(D), nxt;
  for (int k = 0; k < L; ++k) {
    const int nin = f->widths[k], nout = f->widths[k + 1];
    const double* W = f->w[k];
    const double* b = f->b[k];
    const bool sc = nin == nout;
    tl[k].resize(nout);
    nxt.assign(nout, 0.0);
    for (int v = 0; v < nout; ++v) {
      double z = b[v];
      for (int u = 0; u < nin; ++u) z += cur[u] * W[static_cast<std::size_t>(u) * nout + v];
      const double t = std::tanh(z);
      tl[k][v] = t;
      nxt[v] = (sc ? cur[v] : 0.0) + t;
    }
    cur.swap(nxt);
  }
  double e = f->b_out;
  for (int u = 0; u < f->widths[L]; ++u) e += cur[u] * f->w_out[u];
  // Fitting backward -> dE/dD.
  std::vector<double> dy(f->w_out, f->w_out + f->widths[L]), dz, dx;
  for (int k = L - 1; k >= 0; --k) {
    const int nin = f->widths[k], nout = f->widths[k + 1];
    const double* W = f->w[k];
    const bool sc = nin == nout;
    dz.assign(nout, 0.0);
    for (int v = 0; v < nout; ++v) dz[v] = dy[v] * (1.0 - tl[k][v] * tl[k][v]);
    dx.assign(nin, 0.0);
    for (int u = 0; u < nin; ++u) {
      double acc = sc ? dy[u] : 0.0;
      for (int v = 0; v < nout; ++v) acc += W[static_cast<std::size_t>(u) * nout + v] * dz[v];
      dx[u] = acc;
    }
    dy.swap(dx);
  }
  const std::vector<double>& dD = dy;
  // dT from dD (adjoint of D = T<^T T).
  std::vector<double> dT(4 * M, 0.0);
  for (int a = 0; a < 4; ++a) {
    const double* ta = &T[a * M];
    double* dta = &dT[a * M];
    for (int q = 0; q < mlt; ++q) {
      const double tq = ta[q];
      const double* ddq = &dD[static_cast<std::size_t>(q) * M];
      for (int p = 0; p < M; ++p) dta[p] += ddq[p] * tq;
    }
    for (int p = 0; p < mlt; ++p) {
      const double* ddp = &dD[static_cast<std::size_t>(p) * M];
      double acc = 0.0;
      for (int r = 0; r < M; ++r) acc += ddp[r] * ta[r];
      dta[p] += acc;
    }
  }
  // Gradient pass: rows re-evaluated, chain into the displacement.
  const std::size_t base = pg.off[i];
  int filled = 0;
  for (int t = 0; t < nt; ++t)
    for (const Slot& sl : sec[t]) {
      bool ext;
      row_eval(m, t, sl.s, row.data(), row1.data(), ext);
      ++ct.bwd;
      double drow[4];
      for (int a = 0; a < 4; ++a) {
        double acc = 0.0;
        for (int p = 0; p < M; ++p) acc += dT[a * M + p] * row[p];
        drow[a] = acc;
      }
      double ds = 0.0;
      for (int p = 0; p < M; ++p) {
        double dg = 0.0;
        for (int a = 0; a < 4; ++a) dg += sl.r4[a] * dT[a * M + p];
        ds += dg * row1[p];
      }
      drow[0] += ds;
      const std::size_t at = base + filled;
      for (int x = 0; x < 3; ++x) {
        double acc = 0.0;
        for (int a = 0; a < 4; ++a) acc += drow[a] * sl.dv[3 * a + x];
        pg.g[3 * at + x] = acc;
        pg.d[3 * at + x] = sl.d[x];
      }
      pg.atom[at] = sl.j;
      ++filled;
    }
  pg.cnt[i] = filled;
  return e;
}

void check_model(const dp_model_desc* md, const dp_table_desc* td) {
  if (!md || !td) throw InErr("null model or tables");
  if (td->n_tables != md->n_types) throw InErr("need one table per neighbor type");
  if (td->m != 4 * md->d1) throw InErr("table feature width does not match the model");
}

void check_cfg(int64_t n, const double* pos, const int32_t* ty, int nt) {
  if (n <= 0) throw InErr("configuration has no atoms");
  for (int64_t i = 0; i < n; ++i)
    if (ty[i] < 0 || ty[i] >= nt) throw InErr("atom type id out of range");
  for (int64_t k = 0; k < 3 * n; ++k)
    if (!std::isfinite(pos[k])) throw InErr("non-finite atom position");
}

struct Eval {
  double energy = 0.0;
  std::vector<double> ae, f;
  double vir[9] = {0};
};

void evaluate(const Model& m, const Box& bx, int n, const double* pos, const int32_t* ty,
              const Lists& lists, Eval& out, Counts& ct) {
  PairGrads pg;
  pg.off.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) pg.off[i + 1] = pg.off[i] + lists[i].size();
  pg.cnt.assign(n, 0);
  pg.atom.assign(pg.off[n], -1);
  pg.d.assign(3 * pg.off[n], 0.0);
  pg.g.assign(3 * pg.off[n], 0.0);
  out.ae.assign(n, 0.0);
  out.f.assign(3 * static_cast<std::size_t>(n), 0.0);
  for (int k = 0; k < 9; ++k) out.vir[k] = 0.0;
  for (int i = 0; i < n; ++i) out.ae[i] = atom_energy(m, bx, pos, ty, i, lists[i], pg, ct);
  out.energy = 0.0;
  for (int i = 0; i < n; ++i) out.energy += out.ae[i];
  for (int i = 0; i < n; ++i)
    for (std::size_t k = pg.off[i]; k < pg.off[i] + pg.cnt[i]; ++k) {
      const double* g = &pg.g[3 * k];
      const double* d = &pg.d[3 * k];
      const int j = pg.atom[k];
      for (int x = 0; x < 3; ++x) {
        out.f[3 * i + x] += g[x];
        out.f[3 * j + x] -= g[x];
      }
      for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y) out.vir[3 * x + y] += d[x] * g[y];
    }
}

Model make_model(const dp_model_desc* md, const dp_table_desc* td) {
  check_model(md, td);
  Model m;
  m.md = md;
  m.td = td;
  m.M = 4 * md->d1;
  m.mlt = md->m_lt;
  m.stride = ((td->m + td->block - 1) / td->block) * 6 * td->block;
  return m;
}

Lists g_lists;

} // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

int or_neighbor_list(int64_t n, const double* pos, const double* box, const uint8_t* pbc,
                     double cutoff, int brute, int64_t* total) {
  return run([&] {
    Box bx;
    bx.init(box, pbc);
    if (brute)
      nlist_brute(bx, static_cast<int>(n), pos, cutoff, g_lists);
    else
      nlist(bx, static_cast<int>(n), pos, cutoff, g_lists);
    int64_t tot = 0;
    for (const auto& v : g_lists) tot += static_cast<int64_t>(v.size());
    *total = tot;
  });
}

int or_neighbor_list_get(int64_t* offsets, int32_t* j, int32_t* shift) {
  int64_t at = 0;
  offsets[0] = 0;
  for (std::size_t i = 0; i < g_lists.size(); ++i) {
    for (const Entry& e : g_lists[i]) {
      j[at] = e.j;
      for (int k = 0; k < 3; ++k) shift[3 * at + k] = e.s[k];
      ++at;
    }
    offsets[i + 1] = at;
  }
  return 0;
}

int or_compute(const dp_model_desc* md, const dp_table_desc* td, int64_t n, const double* pos,
               const int32_t* types, const double* box, const uint8_t* pbc, double list_cutoff,
               double* energy, double* forces, double* virial, double* atom_energy,
               uint64_t* counters) {
  return run([&] {
    Model m = make_model(md, td);
    check_cfg(n, pos, types, md->n_types);
    Box bx;
    bx.init(box, pbc);
    Lists lists;
    nlist(bx, static_cast<int>(n), pos, list_cutoff > 0 ? list_cutoff : md->r_cut, lists);
    Eval ev;
    Counts ct;
    evaluate(m, bx, static_cast<int>(n), pos, types, lists, ev, ct);
    *energy = ev.energy;
    std::memcpy(forces, ev.f.data(), 3 * n * sizeof(double));
    std::memcpy(virial, ev.vir, 9 * sizeof(double));
    if (atom_energy) std::memcpy(atom_energy, ev.ae.data(), n * sizeof(double));
    if (counters) {
      counters[0] = ct.fwd;
      counters[1] = ct.bwd;
      counters[2] = ct.ext;
    }
  });
}

// Velocity Verlet (md.cpp:151-231) with a global list at r_cut + buffer. Entries beyond r_cut
// are dropped by the env-mat filter, so this equals the reference's per-worker subset lists.
int or_run_md(const dp_model_desc* md, const dp_table_desc* td, int64_t n, double* pos,
              double* vel, const int32_t* types, const double* box, const uint8_t* pbc,
              const dp_md_config* mc, dp_thermo* thermo, int64_t cap, int64_t* n_thermo,
              dp_md_result* res) {
  return run([&] {
    Model m = make_model(md, td);
    check_cfg(n, pos, types, md->n_types);
    if (!(mc->dt > 0.0)) throw InErr("time step must be positive");
    if (mc->n_steps < 0) throw InErr("step count must be non-negative");
    if (mc->rebuild_every < 1 || mc->thermo_every < 1)
      throw InErr("rebuild and thermo intervals must be at least 1");
    if (!(mc->buffer >= 0.0)) throw InErr("buffer must be non-negative");
    Box bx;
    bx.init(box, pbc);
    const int N = static_cast<int>(n);
    const double cutoff = md->r_cut + mc->buffer;
    const double K_B = 8.617333262e-5;
    const double MVV = 1.0e7 / (6.02214076e23 * 1.602176634e-19);
    const double ACC = 1.0 / MVV;
    const double BAR = 1.602176634e6;
    std::vector<double> mass(N), accf(N);
    for (int i = 0; i < N; ++i) {
      mass[i] = md->masses[types[i]];
      accf[i] = ACC / mass[i];
    }
    std::memset(res, 0, sizeof(*res));
    Counts ct;
    Lists lists;
    std::vector<double> ref(pos, pos + 3 * N);
    nlist(bx, N, pos, cutoff, lists);
    Eval ev;
    evaluate(m, bx, N, pos, types, lists, ev, ct);
    ++res->force_evals;
    int64_t nth = 0;
    auto kinetic = [&] {
      double ke = 0.0;
      for (int i = 0; i < N; ++i) {
        const double v2 = vel[3 * i] * vel[3 * i] + vel[3 * i + 1] * vel[3 * i + 1] +
                          vel[3 * i + 2] * vel[3 * i + 2];
        ke += 0.5 * mass[i] * v2 * MVV;
      }
      return ke;
    };
    auto record = [&](int64_t step) {
      dp_thermo tr;
      tr.step = step;
      tr.ke = kinetic();
      tr.pe = ev.energy;
      tr.temperature = 2.0 * tr.ke / (3.0 * N * K_B);
      const double trv = ev.vir[0] + ev.vir[4] + ev.vir[8];
      tr.pressure = (2.0 * tr.ke + trv) / (3.0 * bx.vol) * BAR;
      if (nth < cap) thermo[nth] = tr;
      ++nth;
    };
    record(0);
    const double half = 0.5 * mc->dt;
    for (int64_t s = 1; s <= mc->n_steps; ++s) {
      for (int i = 0; i < N; ++i)
        for (int x = 0; x < 3; ++x) vel[3 * i + x] += half * ev.f[3 * i + x] * accf[i];
      for (int k = 0; k < 3 * N; ++k) pos[k] += mc->dt * vel[k];
      if (s % mc->rebuild_every == 0) {
        nlist(bx, N, pos, cutoff, lists);
        ref.assign(pos, pos + 3 * N);
      }
      double best2 = 0.0;
      for (int i = 0; i < N; ++i) {
        double d2 = 0.0;
        for (int x = 0; x < 3; ++x) {
          const double d = pos[3 * i + x] - ref[3 * i + x];
          d2 += d * d;
        }
        if (d2 > best2) best2 = d2;
      }
      const double drift = std::sqrt(best2);
      ++res->staleness_checks;
      if (drift > res->max_drift_seen) res->max_drift_seen = drift;
      if (drift > 0.5 * mc->buffer)
        throw NuErr("neighbor list stale: an atom moved " + std::to_string(drift) +
                    " since the last rebuild, more than half the buffer");
      evaluate(m, bx, N, pos, types, lists, ev, ct);
      ++res->force_evals;
      for (int i = 0; i < N; ++i)
        for (int x = 0; x < 3; ++x) vel[3 * i + x] += half * ev.f[3 * i + x] * accf[i];
      if (s % mc->thermo_every == 0) record(s);
    }
    *n_thermo = nth;
    res->counters.rows_forward = ct.fwd;
    res->counters.rows_backward = ct.bwd;
    res->counters.extrapolations = ct.ext;
    res->final_ke = kinetic();
    res->final_pe = ev.energy;
    res->final_total = res->final_ke + res->final_pe;
  });
}

} // extern "C"
