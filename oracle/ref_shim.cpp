// C shim over the UNMODIFIED reference library (/root/reference/proj/src, compiled by
// oracle/Makefile into oracle/_ref/libdpref.so). Test/bench infrastructure only: it is the
// "reference" arm of bench.py and the pin for oracle/dp_oracle.cpp and for the product's
// host-side generators. Nothing on the product path links it.
//
// Entry points follow the reference's public API:
//   gen_model / gen_config            model_io.hpp:39-47
//   testutil::make_test_model / make_random_config   tests/helpers.hpp:21-99
//   build_tables                      table.hpp:46-50
//   build_neighbor_list               neighbor.hpp:31-36
//   compute_energy_forces_virial_tabulated   fused.hpp:70-73
//   compute_energy_forces_virial (exact)     exact.hpp:66-68
//   init_velocities / run_md          md.hpp:41-60
//   partition_domain                  domain.hpp:29
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "dp_b200.h"
#include "dpmd/domain.hpp"
#include "dpmd/error.hpp"
#include "dpmd/exact.hpp"
#include "dpmd/fused.hpp"
#include "dpmd/md.hpp"
#include "dpmd/model_io.hpp"
#include "dpmd/neighbor.hpp"
#include "dpmd/rmse.hpp"
#include "dpmd/table.hpp"
#include "helpers.hpp"

using namespace dpmd;

namespace {

std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InputError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// Flatten a reference model into the dp_b200.h model blob layout.
void model_to_blob(const DPModel& m, double* blob) {
  std::size_t at = 0;
  auto put = [&](const std::vector<double>& v) {
    std::memcpy(blob + at, v.data(), v.size() * sizeof(double));
    at += v.size();
  };
  for (const auto& e : m.embedding) {
    put(e.w0); put(e.b0); put(e.w1); put(e.b1); put(e.w2); put(e.b2);
  }
  for (const auto& f : m.fitting) {
    for (const auto& l : f.hidden) { put(l.w); put(l.b); }
    put(f.w_out);
    blob[at++] = f.b_out;
  }
}

DPModel blob_to_model(const dp_preset& s, const double* blob) {
  DPModel m;
  m.r_cut = s.r_cut;
  m.r_smooth = s.r_smooth;
  m.m_lt = s.m_lt;
  for (int t = 0; t < s.n_types; ++t) {
    m.species.push_back(std::string(1, static_cast<char>('A' + t)));
    m.masses.push_back(s.masses[t]);
    m.max_nbr.push_back(s.max_nbr[t]);
  }
  std::size_t at = 0;
  auto take = [&](std::vector<double>& v, std::size_t n) {
    v.assign(blob + at, blob + at + n);
    at += n;
  };
  const int d1 = s.d1;
  for (int t = 0; t < s.n_types; ++t) {
    EmbeddingNet e;
    e.d1 = d1;
    take(e.w0, d1); take(e.b0, d1);
    take(e.w1, 2 * d1 * d1); take(e.b1, 2 * d1);
    take(e.w2, 8 * d1 * d1); take(e.b2, 4 * d1);
    m.embedding.push_back(std::move(e));
  }
  for (int t = 0; t < s.n_types; ++t) {
    FittingNet f;
    f.input_width = s.m_lt * 4 * d1;
    f.width = s.fit_width;
    int cur = f.input_width;
    for (int k = 0; k < s.fit_hidden; ++k) {
      DenseLayer l;
      l.in = cur;
      l.out = s.fit_width;
      take(l.w, static_cast<std::size_t>(cur) * s.fit_width);
      take(l.b, s.fit_width);
      cur = s.fit_width;
      f.hidden.push_back(std::move(l));
    }
    take(f.w_out, cur);
    f.b_out = blob[at++];
    m.fitting.push_back(std::move(f));
  }
  m.validate();
  return m;
}

std::vector<CompressionTable> tables_from(const dp_preset& s, uint64_t n, double h,
                                          const double* coeffs) {
  std::vector<CompressionTable> tabs(s.n_types);
  for (int t = 0; t < s.n_types; ++t) {
    CompressionTable& tb = tabs[t];
    tb.x0 = 0.0;
    tb.h = h;
    tb.n = n;
    tb.m = 4 * s.d1;
    tb.block = 16;
    const std::size_t len = n * tb.interval_stride();
    tb.coeffs.assign(coeffs + t * len, coeffs + (t + 1) * len);
  }
  return tabs;
}

AtomicConfig make_cfg(int64_t n, const double* pos, const int32_t* types, const double* box,
                      const uint8_t* pbc, int n_types) {
  AtomicConfig cfg;
  std::array<double, 9> hh;
  for (int k = 0; k < 9; ++k) hh[k] = box[k];
  cfg.cell = Cell(hh, {pbc[0] != 0, pbc[1] != 0, pbc[2] != 0});
  cfg.n_atoms = static_cast<int>(n);
  cfg.pos.assign(pos, pos + 3 * n);
  cfg.type.assign(types, types + n);
  for (int t = 0; t < n_types; ++t) cfg.type_names.push_back(std::string(1, 'A' + t));
  return cfg;
}

NeighborList g_list;

void copy_result(const EvalResult& r, int64_t n, double* energy, double* forces, double* virial,
                 double* atom_energy) {
  *energy = r.energy;
  std::memcpy(forces, r.forces.data(), 3 * n * sizeof(double));
  std::memcpy(virial, r.virial.data(), 9 * sizeof(double));
  if (atom_energy) std::memcpy(atom_energy, r.per_atom_energy.data(), n * sizeof(double));
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_gen_model(const char* preset, uint64_t seed, double* blob) {
  return guarded([&] { model_to_blob(gen_model(get_preset(preset), seed), blob); });
}

int ref_gen_test_model(const dp_preset* s, uint64_t seed, double fit_scale, double* blob) {
  return guarded([&] {
    std::vector<int> cap(s->max_nbr, s->max_nbr + s->n_types);
    auto m = testutil::make_test_model(s->n_types, s->d1, s->m_lt, s->fit_width, s->fit_hidden,
                                       cap, s->r_cut, s->r_smooth, seed, fit_scale);
    model_to_blob(m, blob);
  });
}

int ref_build_tables(const dp_preset* s, const double* blob, double h, uint64_t* n_out,
                     double* coeffs) {
  return guarded([&] {
    auto m = blob_to_model(*s, blob);
    auto tabs = build_tables(m, h);
    *n_out = tabs[0].n;
    if (!coeffs) return;
    std::size_t at = 0;
    for (const auto& t : tabs) {
      std::memcpy(coeffs + at, t.coeffs.data(), t.coeffs.size() * sizeof(double));
      at += t.coeffs.size();
    }
  });
}

int ref_gen_config(const char* preset, int nx, int ny, int nz, double jitter, uint64_t seed,
                   double* pos, int32_t* types, double* box) {
  return guarded([&] {
    auto c = gen_config(get_preset(preset), nx, ny, nz, jitter, seed);
    std::memcpy(pos, c.pos.data(), c.pos.size() * sizeof(double));
    for (int i = 0; i < c.n_atoms; ++i) types[i] = c.type[i];
    for (int k = 0; k < 9; ++k) box[k] = c.cell.h[k];
  });
}

int ref_random_config(int n, int n_types, double L, double min_sep, uint64_t seed, double* pos,
                      int32_t* types) {
  return guarded([&] {
    auto c = testutil::make_random_config(n, n_types, L, min_sep, seed);
    std::memcpy(pos, c.pos.data(), c.pos.size() * sizeof(double));
    for (int i = 0; i < c.n_atoms; ++i) types[i] = c.type[i];
  });
}

int ref_init_velocities(const dp_preset* s, int64_t n, const double* pos, const int32_t* types,
                        const double* box, double t_init, uint64_t seed, double* vel) {
  return guarded([&] {
    DPModel m;
    m.species.resize(s->n_types);
    m.masses.assign(s->masses, s->masses + s->n_types);
    const uint8_t pbc[3] = {1, 1, 1};
    auto cfg = make_cfg(n, pos, types, box, pbc, s->n_types);
    auto v = init_velocities(cfg, m, t_init, seed);
    std::memcpy(vel, v.data(), v.size() * sizeof(double));
  });
}

// Builds and keeps the list; *total receives the entry count. Fetch with ref_neighbor_list_get.
int ref_neighbor_list(int64_t n, const double* pos, const int32_t* types, const double* box,
                      const uint8_t* pbc, double cutoff, int brute, int64_t* total) {
  return guarded([&] {
    auto cfg = make_cfg(n, pos, types, box, pbc, 64);
    g_list = brute ? build_neighbor_list_brute(cfg, cutoff) : build_neighbor_list(cfg, cutoff);
    int64_t tot = 0;
    for (const auto& v : g_list.nbr) tot += static_cast<int64_t>(v.size());
    *total = tot;
  });
}

int ref_neighbor_list_get(int64_t* offsets, int32_t* j, int32_t* shift) {
  int64_t at = 0;
  offsets[0] = 0;
  for (std::size_t i = 0; i < g_list.nbr.size(); ++i) {
    for (const auto& e : g_list.nbr[i]) {
      j[at] = e.j;
      for (int k = 0; k < 3; ++k) shift[3 * at + k] = e.shift[k];
      ++at;
    }
    offsets[i + 1] = at;
  }
  return 0;
}

// compute_energy_forces_virial_tabulated with list = build_neighbor_list(cfg, list_cutoff).
// seconds[0] = list build time, seconds[1] = evaluation time (wall clock).
int ref_compute_tabulated(const dp_preset* s, const double* blob, uint64_t n_int, double h,
                          const double* coeffs, int64_t n, const double* pos,
                          const int32_t* types, const double* box, const uint8_t* pbc,
                          double list_cutoff, int n_workers, int repeats, double* energy,
                          double* forces, double* virial, double* atom_energy,
                          uint64_t* counters, double* seconds) {
  return guarded([&] {
    auto m = blob_to_model(*s, blob);
    auto tabs = tables_from(*s, n_int, h, coeffs);
    auto cfg = make_cfg(n, pos, types, box, pbc, s->n_types);
    auto t0 = std::chrono::steady_clock::now();
    auto list = build_neighbor_list(cfg, list_cutoff > 0 ? list_cutoff : m.r_cut);
    auto t1 = std::chrono::steady_clock::now();
    FusedCounters c;
    EvalResult r;
    for (int k = 0; k < (repeats < 1 ? 1 : repeats); ++k) {
      c = FusedCounters{};
      r = compute_energy_forces_virial_tabulated(cfg, m, tabs, list, n_workers, &c);
    }
    auto t2 = std::chrono::steady_clock::now();
    copy_result(r, n, energy, forces, virial, atom_energy);
    if (counters) {
      counters[0] = c.rows_forward;
      counters[1] = c.rows_backward;
      counters[2] = c.extrapolations;
    }
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds[1] = std::chrono::duration<double>(t2 - t1).count() / (repeats < 1 ? 1 : repeats);
    }
  });
}

int ref_compute_exact(const dp_preset* s, const double* blob, int64_t n, const double* pos,
                      const int32_t* types, const double* box, const uint8_t* pbc,
                      double* energy, double* forces, double* virial, double* atom_energy) {
  return guarded([&] {
    auto m = blob_to_model(*s, blob);
    auto cfg = make_cfg(n, pos, types, box, pbc, s->n_types);
    auto list = build_neighbor_list(cfg, m.r_cut);
    auto r = compute_energy_forces_virial(cfg, m, list);
    copy_result(r, n, energy, forces, virial, atom_energy);
  });
}

int ref_run_md(const dp_preset* s, const double* blob, uint64_t n_int, double h,
               const double* coeffs, int64_t n, double* pos, double* vel, const int32_t* types,
               const double* box, const uint8_t* pbc, const dp_md_config* mc, int n_workers,
               dp_thermo* thermo, int64_t thermo_cap, int64_t* n_thermo, dp_md_result* out) {
  return guarded([&] {
    auto m = blob_to_model(*s, blob);
    auto tabs = tables_from(*s, n_int, h, coeffs);
    auto cfg = make_cfg(n, pos, types, box, pbc, s->n_types);
    std::vector<double> v(vel, vel + 3 * n);
    MDConfig c;
    c.n_steps = mc->n_steps;
    c.dt = mc->dt;
    c.buffer = mc->buffer;
    c.rebuild_every = mc->rebuild_every;
    c.thermo_every = mc->thermo_every;
    c.n_workers = n_workers;
    auto res = run_md(cfg, v, m, tabs, c);
    std::memcpy(pos, cfg.pos.data(), 3 * n * sizeof(double));
    std::memcpy(vel, v.data(), 3 * n * sizeof(double));
    int64_t k = 0;
    for (const auto& tr : res.thermo) {
      if (k < thermo_cap) thermo[k] = dp_thermo{tr.step, tr.ke, tr.pe, tr.temperature, tr.pressure};
      ++k;
    }
    *n_thermo = k;
    out->force_evals = res.force_evals;
    out->staleness_checks = res.staleness_checks;
    out->max_drift_seen = res.max_drift_seen;
    out->counters = dp_counters{res.counters.rows_forward, res.counters.rows_backward,
                                res.counters.extrapolations};
    out->final_ke = res.final_ke;
    out->final_pe = res.final_pe;
    out->final_total = res.final_total;
  });
}

// partition_domain: owner[i] = worker id; ghost_mask[w*n + i] = 1 if i is a ghost of w.
int ref_partition_domain(int64_t n, const double* pos, const double* box, const uint8_t* pbc,
                         int n_workers, double margin, int* axis, int32_t* owner,
                         uint8_t* ghost_mask) {
  return guarded([&] {
    std::vector<int32_t> ty(n, 0);
    auto cfg = make_cfg(n, pos, ty.data(), box, pbc, 1);
    auto part = partition_domain(cfg, n_workers, margin);
    *axis = part.axis;
    std::memset(ghost_mask, 0, static_cast<std::size_t>(part.workers.size()) * n);
    for (std::size_t w = 0; w < part.workers.size(); ++w) {
      for (int i : part.workers[w].owned) owner[i] = static_cast<int32_t>(w);
      for (int i : part.workers[w].ghosts) ghost_mask[w * n + i] = 1;
    }
  });
}

// rmse_sweep (rmse.cpp:63-97) over concatenated configurations; loglog_slope (rmse.cpp:99-116).
int ref_rmse_sweep(const dp_preset* s, const double* blob, int n_configs, const int64_t* n_atoms,
                   const double* pos, const int32_t* types, const double* boxes, const uint8_t* pbcs,
                   int n_h, const double* h_list, double* rmse_e, double* rmse_f, double* slope) {
  return guarded([&] {
    auto m = blob_to_model(*s, blob);
    std::vector<AtomicConfig> cfgs;
    int64_t at = 0;
    for (int c = 0; c < n_configs; ++c) {
      cfgs.push_back(make_cfg(n_atoms[c], pos + 3 * at, types + at, boxes + 9 * c, pbcs + 3 * c, s->n_types));
      at += n_atoms[c];
    }
    std::vector<double> hl(h_list, h_list + n_h);
    auto rows = rmse_sweep(m, hl, cfgs, 1);
    for (int k = 0; k < n_h; ++k) {
      rmse_e[k] = rows[k].rmse_e;
      rmse_f[k] = rows[k].rmse_f;
    }
    *slope = loglog_slope(rows);
  });
}

// write_model / read_model (model_io.cpp:226-283).
int ref_write_model(const char* path, const dp_preset* s, const double* blob, const char* preset, uint64_t seed) {
  return guarded([&] { write_model(path, blob_to_model(*s, blob), preset, seed); });
}

int ref_read_model(const char* path, const dp_preset* s, double* blob, uint64_t* seed) {
  return guarded([&] {
    ModelFile mf = read_model(path);
    if (mf.model.n_types() != s->n_types || mf.model.d1() != s->d1) throw InputError("shape mismatch");
    model_to_blob(mf.model, blob);
    *seed = mf.seed;
  });
}

// bench.py --impl reference / cpu_baseline: the reference's MD-step cost on its OWN inputs, built
// entirely by its public API (gen_model model_io.hpp:40, build_tables table.hpp:42, gen_config
// model_io.hpp:45, build_neighbor_list neighbor.hpp:31) -- nothing of the product involved.
// Per step: one compute_energy_forces_virial_tabulated (fused.hpp:70-73) with n_workers threads on
// the list built once at r_c + skin (cell path). list_s = that build, eval_s[k] = step k's
// evaluation (wall clock). Runs `warmup` untimed evaluations, then up to max_steps timed ones,
// stopping early once budget_s seconds of timed work are done (at least min_steps).
int ref_bench_steps(const char* preset, int nx, int ny, int nz, double jitter, uint64_t cfg_seed,
                    uint64_t model_seed, double h, double skin, int n_workers, int warmup,
                    int max_steps, int min_steps, double budget_s, int64_t* n_atoms, double* list_s,
                    double* eval_s, int* n_done, double* energy) {
  return guarded([&] {
    const Preset& p = get_preset(preset);
    auto m = gen_model(p, model_seed);
    auto tabs = build_tables(m, h);
    auto cfg = gen_config(p, nx, ny, nz, jitter, cfg_seed);
    *n_atoms = cfg.n_atoms;
    auto t0 = std::chrono::steady_clock::now();
    auto list = build_neighbor_list(cfg, m.r_cut + skin);
    *list_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    EvalResult r;
    for (int k = 0; k < warmup; ++k) r = compute_energy_forces_virial_tabulated(cfg, m, tabs, list, n_workers);
    double total = 0.0;
    int done = 0;
    while (done < max_steps && (done < min_steps || total < budget_s)) {
      auto a = std::chrono::steady_clock::now();
      r = compute_energy_forces_virial_tabulated(cfg, m, tabs, list, n_workers);
      eval_s[done] = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
      total += eval_s[done++];
    }
    *n_done = done;
    *energy = r.energy;
  });
}

} // extern "C"

