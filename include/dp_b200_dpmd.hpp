// dp_b200_dpmd.hpp -- reference-side C++ adapter: a GPU twin of the dpmd operator.
//
// Include from code built against the reference's headers (/root/reference/proj/include) and
// link with -L<repo>/paper_2201_01446_b200/lib -ldpb200. It maps the reference's own types onto
// the C-ABI of dp_b200.h:
//   DPModel / FittingNet / DenseLayer  model.hpp:22-58     -> dp_model_desc / dp_fitting_desc
//   CompressionTable                   table.hpp:20-35     -> dp_table_desc
//   AtomicConfig / Cell                geom.hpp:14-54      -> dp_compute arguments
//   NeighborList                       neighbor.hpp:14-23  -> dp_compute_list (caller's list)
//   EvalResult / FusedCounters         exact.hpp:12-17, fused.hpp:10-21
//   InputError / NumericalError        error.hpp:9-17      <- return codes 2 / 1
// Per-type fitting nets may differ in depth and widths (model.cpp:30-47), as in the reference.
// tests/cpp/gpu_evaluator_test.cpp compiles this header against the reference and compares
// GpuEvaluator::compute with compute_energy_forces_virial_tabulated (fused.hpp:70-73).
#pragma once

#include <stdexcept>
#include <vector>

#include "dp_b200.h"
#include "dpmd/error.hpp"
#include "dpmd/exact.hpp"
#include "dpmd/fused.hpp"
#include "dpmd/geom.hpp"
#include "dpmd/model.hpp"
#include "dpmd/neighbor.hpp"
#include "dpmd/table.hpp"

namespace dpmd {

class GpuEvaluator {
 public:
  // precision 0: FP64 (1e-10 parity); 1: mixed (tcgen05 fitting, 1e-5)
  GpuEvaluator(const DPModel& m, const std::vector<CompressionTable>& tabs, int device = 0, int precision = 0) {
    const int nt = m.n_types();
    widths_.resize(nt);
    w_.resize(nt);
    b_.resize(nt);
    fits_.resize(nt);
    for (int t = 0; t < nt; ++t) {
      const FittingNet& f = m.fitting[t];
      widths_[t].push_back(f.input_width);
      for (const auto& l : f.hidden) {
        widths_[t].push_back(l.out);
        w_[t].push_back(l.w.data());
        b_[t].push_back(l.b.data());
      }
    }
    for (int t = 0; t < nt; ++t)
      fits_[t] = dp_fitting_desc{static_cast<int>(m.fitting[t].hidden.size()), widths_[t].data(), w_[t].data(),
                                 b_[t].data(), m.fitting[t].w_out.data(), m.fitting[t].b_out};
    dp_model_desc md{nt, m.r_cut, m.r_smooth, m.d1(), m.m_lt, m.masses.data(), m.max_nbr.data(), fits_.data()};
    for (const auto& t : tabs) c_.push_back(t.coeffs.data());
    if (tabs.empty()) throw InputError("need one table per neighbor type");
    dp_table_desc td{static_cast<int>(tabs.size()), tabs[0].x0, tabs[0].h, tabs[0].n, tabs[0].m, tabs[0].block,
                     c_.data()};
    check(dp_create(&md, &td, device, precision, &h_));
  }
  ~GpuEvaluator() { dp_destroy(h_); }
  GpuEvaluator(const GpuEvaluator&) = delete;
  GpuEvaluator& operator=(const GpuEvaluator&) = delete;

  // compute_energy_forces_virial_tabulated with the GPU's own cell list (cutoff r_cut + skin).
  EvalResult compute(const AtomicConfig& cfg, double skin = 0.0, FusedCounters* ctr = nullptr) {
    check(dp_set_skin(h_, skin));
    EvalResult r = blank(cfg);
    const uint8_t pbc[3] = {cfg.cell.periodic[0], cfg.cell.periodic[1], cfg.cell.periodic[2]};
    check(dp_compute(h_, cfg.n_atoms, cfg.pos.data(), cfg.type.data(), cfg.cell.h.data(), pbc, &r.energy,
                     r.forces.data(), r.virial.data(), r.per_atom_energy.data()));
    add_counters(ctr);
    return r;
  }

  // The reference signature itself: the caller's NeighborList (full, symmetric, any cutoff
  // >= r_cut, as build_neighbor_list returns it).
  EvalResult compute(const AtomicConfig& cfg, const NeighborList& list, FusedCounters* ctr) {
    EvalResult r = blank(cfg);
    std::vector<int64_t> off(cfg.n_atoms + 1, 0);
    for (int i = 0; i < cfg.n_atoms; ++i) off[i + 1] = off[i] + static_cast<int64_t>(list.nbr[i].size());
    std::vector<int32_t> j(off[cfg.n_atoms]), s(3 * off[cfg.n_atoms]);
    for (int i = 0; i < cfg.n_atoms; ++i)
      for (size_t k = 0; k < list.nbr[i].size(); ++k) {
        const NeighborEntry& e = list.nbr[i][k];
        j[off[i] + k] = e.j;
        for (int x = 0; x < 3; ++x) s[3 * (off[i] + k) + x] = e.shift[x];
      }
    const uint8_t pbc[3] = {cfg.cell.periodic[0], cfg.cell.periodic[1], cfg.cell.periodic[2]};
    check(dp_compute_list(h_, cfg.n_atoms, cfg.pos.data(), cfg.type.data(), cfg.cell.h.data(), pbc, off.data(),
                          j.data(), s.data(), &r.energy, r.forces.data(), r.virial.data(),
                          r.per_atom_energy.data()));
    add_counters(ctr);
    return r;
  }

  dp_handle* handle() { return h_; }

 private:
  static EvalResult blank(const AtomicConfig& cfg) {
    EvalResult r;
    r.per_atom_energy.assign(cfg.n_atoms, 0.0);
    r.forces.assign(3 * static_cast<size_t>(cfg.n_atoms), 0.0);
    return r;
  }
  void add_counters(FusedCounters* ctr) {
    if (!ctr) return;
    dp_counters c;
    dp_counters_get(h_, &c);
    ctr->rows_forward += c.rows_forward;
    ctr->rows_backward += c.rows_backward;
    ctr->extrapolations += c.extrapolations;
  }
  void check(int rc) {
    if (rc == DP_OK) return;
    const char* msg = h_ ? dp_last_error(h_) : dp_last_error(nullptr);
    if (rc == DP_INPUT_ERROR) throw InputError(msg);
    if (rc == DP_NUMERICAL_ERROR) throw NumericalError(msg);
    throw std::runtime_error(msg);
  }
  dp_handle* h_ = nullptr;
  std::vector<std::vector<int>> widths_;
  std::vector<std::vector<const double*>> w_, b_;
  std::vector<const double*> c_;
  std::vector<dp_fitting_desc> fits_;
};

}  // namespace dpmd
