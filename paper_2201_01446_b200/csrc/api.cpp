// C-ABI of dp_b200 (include/dp_b200.h). Every entry point maps exceptions to the reference
// CLI's exit codes (tools/dpmd.cpp:434-443): InputError -> 2, NumericalError -> 1.
#include <cmath>
#include <cstring>
#include <vector>

#include "engine.hpp"

struct dp_handle {
  dpb::Engine eng;
  double skin = 0.0;
};

using dpb::guard_call;
using dpb::InputErr;

extern "C" {

const char* dp_version(void) { return "dp_b200 0.1 (sm_100a, fp64 DMMA)"; }

int dp_create(const dp_model_desc* model, const dp_table_desc* tables, int device, int precision,
              dp_handle** out) {
  if (!out) return DP_INPUT_ERROR;
  *out = nullptr;
  dp_handle* h = new dp_handle();
  const int rc = guard_call(nullptr, [&] { h->eng.create(model, tables, device, precision); });
  if (rc != DP_OK) {
    h->eng.destroy();
    delete h;
    return rc;
  }
  *out = h;
  return DP_OK;
}

int dp_destroy(dp_handle* h) {
  if (!h) return DP_OK;
  h->eng.destroy();
  delete h;
  return DP_OK;
}

const char* dp_last_error(const dp_handle* h) {
  return h ? h->eng.last_error.c_str() : dpb::global_error().c_str();
}

int dp_set_skin(dp_handle* h, double skin) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    if (!(skin >= 0.0)) throw InputErr("skin must be non-negative");
    h->skin = skin;
    h->eng.list_valid = false;
  });
}

int dp_compute(dp_handle* h, int64_t n, const double* pos, const int32_t* types, const double box[9],
               const uint8_t pbc[3], double* energy, double* forces, double* virial,
               double* atom_energy) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    if (!energy || !forces || !virial) throw InputErr("null output array");
    E.set_config(n, pos, types, box, pbc);
    const double cutoff = E.r_cut + h->skin;
    bool rebuild = !E.list_valid || E.list_cutoff != cutoff;
    if (!rebuild && h->skin > 0.0) rebuild = E.max_drift() > 0.5 * h->skin;
    if (h->skin == 0.0) rebuild = true;
    if (rebuild) E.build_list(cutoff);
    E.reset_counters();
    E.evaluate_retry();
    E.fetch_results(energy, forces, virial, atom_energy);
    E.read_counters();
  });
}

int dp_compute_list(dp_handle* h, int64_t n, const double* pos, const int32_t* types, const double box[9],
                    const uint8_t pbc[3], const int64_t* offsets, const int32_t* j, const int32_t* shift,
                    double* energy, double* forces, double* virial, double* atom_energy) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    if (!energy || !forces || !virial) throw InputErr("null output array");
    E.set_config(n, pos, types, box, pbc);
    E.import_list(offsets, j, shift);
    E.reset_counters();
    E.evaluate_retry();
    E.list_valid = false; // the caller's list serves this call only
    E.fetch_results(energy, forces, virial, atom_energy);
    E.read_counters();
  });
}

int dp_set_chunk_size(dp_handle* h, int64_t centres) {
  if (!h) return DP_INPUT_ERROR;
  if (centres < 0) return DP_INPUT_ERROR;
  h->eng.chunk_max = centres;
  h->eng.plan_dirty = true;
  return DP_OK;
}

int dp_set_pipeline(dp_handle* h, int enable) {
  if (!h) return DP_INPUT_ERROR;
  if (h->eng.pipeline != (enable != 0)) h->eng.plan_dirty = true;
  h->eng.pipeline = enable != 0;
  return DP_OK;
}

int dp_set_embedding(dp_handle* h, const dp_embedding_desc* nets) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] { h->eng.set_embedding(nets); });
}

int dp_compute_exact(dp_handle* h, int64_t n, const double* pos, const int32_t* types, const double box[9],
                     const uint8_t pbc[3], double* energy, double* forces, double* virial,
                     double* atom_energy) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    if (!energy || !forces || !virial) throw InputErr("null output array");
    E.set_config(n, pos, types, box, pbc);
    E.build_list(E.r_cut + h->skin);
    E.evaluate_exact();
    E.check_err();
    E.fetch_results(energy, forces, virial, atom_energy);
  });
}

int dp_build_tables_gpu(dp_handle* h, double step, uint64_t* n_intervals, double* x_end, double* coeffs,
                        int install) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error,
                    [&] { h->eng.build_tables_gpu(step, n_intervals, x_end, coeffs, install != 0); });
}

int dp_rmse_sweep(dp_handle* h, int n_configs, const int64_t* n_atoms, const double* pos, const int32_t* types,
                  const double* boxes, const uint8_t* pbcs, int n_h, const double* h_list, double* rmse_e,
                  double* rmse_f) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    if (n_h < 1) throw InputErr("sweep needs at least one step size");   // rmse.cpp:65
    if (n_configs < 0 || (n_configs > 0 && (!n_atoms || !pos || !types || !boxes || !pbcs)))
      throw InputErr("null configuration arrays");
    // reference energies / forces once per configuration (rmse.cpp:67-75)
    std::vector<double> ref_e(n_configs);
    std::vector<std::vector<double>> ref_f(n_configs);
    std::vector<double> vir(9);
    int64_t at = 0;
    for (int c = 0; c < n_configs; ++c) {
      const int64_t na = n_atoms[c];
      ref_f[c].resize(3 * na);
      E.set_config(na, pos + 3 * at, types + at, boxes + 9 * c, pbcs + 3 * c);
      E.build_list(E.r_cut);
      E.evaluate_exact();
      E.check_err();
      E.fetch_results(&ref_e[c], ref_f[c].data(), vir.data(), nullptr);
      at += na;
    }
    std::vector<double> f(0);
    for (int k = 0; k < n_h; ++k) {
      E.build_tables_gpu(h_list[k], nullptr, nullptr, nullptr, true);
      // Accum (rmse.cpp:11-37)
      double sde2 = 0.0, sdf2 = 0.0;
      int64_t ncomp = 0, natoms_last = 0;
      at = 0;
      for (int c = 0; c < n_configs; ++c) {
        const int64_t na = n_atoms[c];
        f.resize(3 * na);
        double e = 0.0;
        E.set_config(na, pos + 3 * at, types + at, boxes + 9 * c, pbcs + 3 * c);
        E.build_list(E.r_cut);
        E.reset_counters();
        E.evaluate_retry();
        E.fetch_results(&e, f.data(), vir.data(), nullptr);
        E.read_counters();
        const double de = ref_e[c] - e;
        sde2 += de * de;
        for (int64_t q = 0; q < 3 * na; ++q) {
          const double df = ref_f[c][q] - f[q];
          sdf2 += df * df;
        }
        ncomp += 3 * na;
        natoms_last = na;
        at += na;
      }
      rmse_e[k] = n_configs ? std::sqrt(sde2 / n_configs) / static_cast<double>(natoms_last) : 0.0;
      rmse_f[k] = n_configs ? std::sqrt(sdf2 / static_cast<double>(ncomp)) : 0.0;
    }
  });
}

int dp_counters_get(const dp_handle* h, dp_counters* out) {
  if (!h || !out) return DP_INPUT_ERROR;
  *out = h->eng.host_counters;
  return DP_OK;
}

int dp_neighbor_list_build(dp_handle* h, int64_t n, const double* pos, const int32_t* types,
                           const double box[9], const uint8_t pbc[3], double cutoff,
                           int64_t* total) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    E.set_config(n, pos, types, box, pbc);
    E.build_list(cutoff);
    E.check_err();
    E.sync_entry_count();
    if (total) *total = E.n_entries;
  });
}

int dp_neighbor_list_get(dp_handle* h, int64_t* offsets, int32_t* j, int32_t* shift) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    if (!h->eng.list_valid) throw InputErr("no neighbour list built");
    h->eng.download_list(offsets, j, shift);
  });
}

int dp_md_begin(dp_handle* h, int64_t n, const double* pos, const double* vel,
                const int32_t* types, const double box[9], const uint8_t pbc[3],
                const dp_md_config* cfg) {
  if (!h || !cfg || !vel) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    if (n < 1) throw InputErr("configuration has no atoms");
    if (E.dist)
      dpb::dist_md_begin(E, n, pos, vel, types, box, pbc, cfg);
    else
      E.set_config(n, pos, types, box, pbc);
    E.md_begin(pos, vel, cfg);
  });
}

int dp_md_step(dp_handle* h, int64_t k) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] { h->eng.md_steps(k); });
}

int dp_md_end(dp_handle* h, double* pos, double* vel, dp_thermo* thermo, int64_t thermo_cap,
              int64_t* n_thermo, dp_md_result* result) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    dpb::Engine& E = h->eng;
    E.md_end(pos, vel);
    const int64_t nr = static_cast<int64_t>(E.thermo.size());
    if (thermo)
      for (int64_t k = 0; k < nr && k < thermo_cap; ++k) thermo[k] = E.thermo[k];
    if (n_thermo) *n_thermo = nr;
    if (result) *result = E.md_res;
  });
}

int dp_md_run(dp_handle* h, int64_t n, double* pos, double* vel, const int32_t* types,
              const double box[9], const uint8_t pbc[3], const dp_md_config* cfg,
              dp_thermo* thermo, int64_t thermo_cap, int64_t* n_thermo, dp_md_result* result) {
  int rc = dp_md_begin(h, n, pos, vel, types, box, pbc, cfg);
  if (rc) return rc;
  rc = dp_md_step(h, cfg->n_steps);
  if (rc) {
    h->eng.md_active = false;
    return rc;
  }
  return dp_md_end(h, pos, vel, thermo, thermo_cap, n_thermo, result);
}

void* dp_stream(dp_handle* h) { return h ? static_cast<void*>(h->eng.stream) : nullptr; }

uint64_t dp_launch_count(const dp_handle* h) { return h ? h->eng.launches : 0; }

int dp_dist_init(dp_handle* h, int rank, int world, const void* nccl_id) {
  if (!h || !nccl_id) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] { dpb::dist_init(h->eng, rank, world, nccl_id); });
}

int dp_set_timing(dp_handle* h, int enable) {
  if (!h) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] {
    double ms[8];
    uint64_t c[8];
    if (h->eng.timing) h->eng.phase_collect(ms, c);
    h->eng.timing = enable != 0;
  });
}

int dp_phase_times(dp_handle* h, double* ms, uint64_t* counts) {
  if (!h || !ms || !counts) return DP_INPUT_ERROR;
  return guard_call(&h->eng.last_error, [&] { h->eng.phase_collect(ms, counts); });
}

} // extern "C"
