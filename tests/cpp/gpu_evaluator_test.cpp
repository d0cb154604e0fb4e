// Drop-in proof from C++ (TEST INFRASTRUCTURE): include/dp_b200_dpmd.hpp compiled against the
// reference's own headers (/root/reference/proj/include) and linked with the unmodified reference
// objects (oracle/_ref/obj, built by oracle/Makefile) plus libdpb200.so. Each case evaluates the
// same reference-built inputs through GpuEvaluator and through the reference operator
// compute_energy_forces_virial_tabulated (fused.hpp:70-73) and compares E, F, virial and E_i
// normwise and the FusedCounters.
//   ./gpu_evaluator_test           -> one "case <name> ..." line per case, exit 0 when all pass
// Built here (where /root/reference exists) into oracle/_ref/; run on the GPU box by
// tests/test_gpu_cpp_adapter.py.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>

#include "dp_b200_dpmd.hpp"
#include "dpmd/model_io.hpp"
#include "dpmd/rng.hpp"
#include "helpers.hpp"

using namespace dpmd;

namespace {

int failures = 0;

double normwise(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 1e-300;
  for (size_t k = 0; k < a.size(); ++k) {
    num = std::max(num, std::fabs(a[k] - b[k]));
    den = std::max(den, std::fabs(b[k]));
  }
  return num / den;
}

void compare(const std::string& name, const EvalResult& g, const EvalResult& r, const FusedCounters& cg,
             const FusedCounters& cr, double tol) {
  const double de = std::fabs(g.energy - r.energy) / std::max(std::fabs(r.energy), 1e-300);
  const double df = normwise(g.forces, r.forces);
  const double dv = normwise(std::vector<double>(g.virial.begin(), g.virial.end()),
                             std::vector<double>(r.virial.begin(), r.virial.end()));
  const double dei = normwise(g.per_atom_energy, r.per_atom_energy);
  const bool cnt = cg.rows_forward == cr.rows_forward && cg.rows_backward == cr.rows_backward &&
                   cg.extrapolations == cr.extrapolations;
  const bool ok = de <= tol && df <= tol && dv <= tol && dei <= tol && cnt;
  std::printf("case %s %s E=%.17g dE=%.2e dF=%.2e dV=%.2e dEi=%.2e rows=%llu/%llu\n", name.c_str(),
              ok ? "ok" : "FAIL", g.energy, de, df, dv, dei, static_cast<unsigned long long>(cg.rows_forward),
              static_cast<unsigned long long>(cr.rows_forward));
  if (!ok) ++failures;
}

template <class Err>
void expect_throw(const std::string& name, const std::function<void()>& f) {
  try {
    f();
  } catch (const Err& e) {
    std::printf("case %s ok (%s)\n", name.c_str(), e.what());
    return;
  } catch (const std::exception& e) {
    std::printf("case %s FAIL wrong exception: %s\n", name.c_str(), e.what());
    ++failures;
    return;
  }
  std::printf("case %s FAIL no exception\n", name.c_str());
  ++failures;
}

// Replace type t's fitting net by one of a different depth and widths (model.cpp:30-47 accepts it).
void reshape_fitting(DPModel& m, int t, const std::vector<int>& widths, std::uint64_t seed) {
  Rng rng(seed);
  FittingNet f;
  f.input_width = m.descriptor_size();
  f.width = widths.back();
  int cur = f.input_width;
  for (size_t k = 0; k < widths.size(); ++k) {
    DenseLayer l;
    l.in = cur;
    l.out = widths[k];
    const double sigma = (k == 0 ? 0.2 : 1.0) / std::sqrt(double(cur));
    l.w.resize(static_cast<size_t>(l.in) * l.out);
    l.b.resize(l.out);
    for (auto& x : l.w) x = sigma * rng.gaussian();
    for (auto& x : l.b) x = 0.1 * rng.gaussian();
    cur = l.out;
    f.hidden.push_back(std::move(l));
  }
  f.w_out.resize(cur);
  for (auto& x : f.w_out) x = rng.gaussian() / std::sqrt(double(cur));
  f.b_out = 0.3;
  m.fitting[t] = std::move(f);
  m.validate();
}

}  // namespace

int main() {
  const double tol = 1e-10;
  {
    // C1: the copper preset (gen_model seed 7, tables h = 0.01, 8x8x8 cells, jitter 0.1, seed 11)
    const Preset& p = get_preset("copper-like");
    DPModel m = gen_model(p, 7);
    auto tabs = build_tables(m, 0.01);
    AtomicConfig cfg = gen_config(p, 8, 8, 8, 0.1, 11);
    FusedCounters cr, cg, cl;
    EvalResult r = compute_energy_forces_virial_tabulated(cfg, m, tabs, build_neighbor_list(cfg, m.r_cut), 1, &cr);
    GpuEvaluator gpu(m, tabs);
    compare("c1_own_list", gpu.compute(cfg, 2.0, &cg), r, cg, cr, tol);
    NeighborList list = build_neighbor_list(cfg, m.r_cut + 2.0);
    compare("c1_reference_list", gpu.compute(cfg, list, &cl), r, cl, cr, tol);
    // an asymmetric list is rejected as InputError
    list.nbr[0].pop_back();
    expect_throw<InputError>("asymmetric_list_input_error", [&] {
      FusedCounters c;
      gpu.compute(cfg, list, &c);
    });
    // overlapping atoms: NumericalError, as env_mat.cpp:33
    AtomicConfig bad = cfg;
    for (int x = 0; x < 3; ++x) bad.pos[3 + x] = bad.pos[x] + 1e-8;
    expect_throw<NumericalError>("overlap_numerical_error", [&] { gpu.compute(bad, 0.0); });
    expect_throw<NumericalError>("overlap_reference_agrees", [&] {
      compute_energy_forces_virial_tabulated(bad, m, tabs, build_neighbor_list(bad, m.r_cut));
    });
  }
  {
    // heterogeneous per-type fitting nets: type 0 din->20->20, type 1 din->16->16->12
    DPModel m = testutil::make_test_model(2, 6, 8, 20, 2, {40, 40}, 6.0, 5.0, 401);
    reshape_fitting(m, 1, {16, 16, 12}, 77);
    auto tabs = build_tables(m, 0.05);
    AtomicConfig cfg = testutil::make_random_config(120, 2, 13.0, 1.7, 5);
    FusedCounters cr, cg;
    EvalResult r = compute_energy_forces_virial_tabulated(cfg, m, tabs, build_neighbor_list(cfg, m.r_cut), 1, &cr);
    GpuEvaluator gpu(m, tabs);
    compare("hetero_fitting_nets", gpu.compute(cfg, 1.0, &cg), r, cg, cr, tol);
    expect_throw<InputError>("hetero_mixed_input_error", [&] { GpuEvaluator mixed(m, tabs, 0, 1); });
  }
  {
    // water preset, two species (O, H), 4x4x4 cells
    const Preset& p = get_preset("water-like");
    DPModel m = gen_model(p, 3);
    auto tabs = build_tables(m, 0.01);
    AtomicConfig cfg = gen_config(p, 4, 4, 4, 0.1, 4);
    FusedCounters cr, cg;
    EvalResult r = compute_energy_forces_virial_tabulated(cfg, m, tabs, build_neighbor_list(cfg, m.r_cut), 4, &cr);
    GpuEvaluator gpu(m, tabs);
    compare("water_two_species", gpu.compute(cfg, 0.0, &cg), r, cg, cr, tol);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
