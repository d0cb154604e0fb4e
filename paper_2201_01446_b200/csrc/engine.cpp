// Host side of the Engine: model upload, configuration handling, evaluation sequencing and the
// device-resident MD loop. Mirrors the reference orchestration:
//   compute_energy_forces_virial_tabulated   fused.cpp:245-288
//   run_md / rebuild / evaluate              md.cpp:70-134, 151-231
#include <cstring>
#include <mutex>
#include <set>
#include <tuple>

#include "engine.hpp"

namespace dpb {

void smem_optin_raw(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, size_t>> done;
  int dev = 0;
  DPB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({fn, dev, bytes})) return;
  DPB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  done.insert({fn, dev, bytes});
}

std::string& global_error() {
  static thread_local std::string e;
  return e;
}

namespace {

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Fitting widths are padded (zero weights) to a GEMM-friendly size: a multiple of 16 that the
// 80- or 64-column tiles divide (240 stays 240), else a multiple of 64.
int pad_width(int w) {
  const int w16 = round_up(w, 16);
  if (w16 % 80 == 0 || w16 % 64 == 0) return w16;
  return round_up(w, 64);
}

void raise_device_error(int code) {
  switch (code) {
    case DEV_OK: return;
    case DEV_OVERLAP: throw NumErr("overlapping atoms in neighbor environment");
    case DEV_OVERFLOW: throw NumErr("neighbor slot capacity exceeded");
    case DEV_TABLE_LOW: throw InputErr("table input below domain start");
    case DEV_SHIFT_RANGE: throw InputErr("image shift outside +-511 cells (positions too far from the box)");
    case DEV_ROW_CAP: throw NumErr("neighbour row exceeds the kernel capacity");
    case DEV_PBUF: throw NumErr("tabulate group buffer overflow (retry: it grows at the next rebuild)");
    case DEV_TABLE_VERIFY: throw NumErr("table verification failed at a node");
    case DEV_LIST_CAP: throw NumErr("neighbour rows exceed the evaluation chunk's entry capacity");
    case DEV_GCAP: throw NumErr("more real pairs than the pair-gradient buffer holds (12.5 % above the last list build)");
    case DEV_ASYMMETRIC: throw InputErr("neighbour list is not symmetric: an entry (i -> j, s) has no (j -> i, -s)");
    case DEV_STALE: throw NumErr("neighbor list stale: an atom moved more than half the buffer since the last rebuild");
    default: throw CudaErr("unknown device error " + std::to_string(code));
  }
}

} // namespace

void Engine::upload_tables(const dp_table_desc& tdr) {
  const dp_table_desc* td = &tdr;
  // tables -> [type][interval][6][Mp]
  tab_x0 = td->x0;
  tab_h = td->h;
  tab_n = td->n;
  const int B = td->block;
  const int nb = (td->m + B - 1) / B;
  const size_t src_stride = static_cast<size_t>(nb) * 6 * B;
  const size_t dst_stride = static_cast<size_t>(6) * Mp;
  std::vector<double> tbuf(static_cast<size_t>(n_types) * tab_n * dst_stride, 0.0);
  for (int t = 0; t < n_types; ++t)
    for (uint64_t th = 0; th < tab_n; ++th) {
      const double* src = td->coeffs[t] + th * src_stride;
      double* dst = tbuf.data() + (static_cast<size_t>(t) * tab_n + th) * dst_stride;
      for (int p = 0; p < M; ++p)
        for (int m = 0; m < 6; ++m)
          dst[m * Mp + p] = src[static_cast<size_t>(p / B) * 6 * B + m * B + (p % B)];
    }
  tab.ensure(tbuf.size());
  DPB_CUDA(cudaMemcpy(tab.p, tbuf.data(), tbuf.size() * sizeof(double), cudaMemcpyHostToDevice));
  ++tab_ver;
  tab_block = B;
  pbuf_cap = 0;
}

void Engine::create(const dp_model_desc* md, const dp_table_desc* td, int dev, int prec) {
  // td may be NULL: tables are then built on the device (dp_build_tables_gpu) before use
  if (!md) throw InputErr("null model descriptor");
  if (md->n_types < 1 || md->n_types > 63) throw InputErr("model needs 1..63 species");
  if (!(md->r_cut > 0.0) || !(md->r_smooth >= 0.0) || !(md->r_smooth < md->r_cut))
    throw InputErr("model cutoffs must satisfy 0 <= r_smooth < r_cut");
  if (md->d1 < 1) throw InputErr("embedding width must be positive");
  if (md->m_lt < 1 || md->m_lt > 4 * md->d1) throw InputErr("m_lt must lie in [1, 4*d1]");
  if (td && td->n_tables != md->n_types) throw InputErr("need one table per neighbor type");
  if (td && td->m != 4 * md->d1) throw InputErr("table feature width does not match 4*d1");
  if (td && (td->block < 1 || td->n < 1 || !(td->h > 0.0))) throw InputErr("table header is inconsistent");
  if (prec != 0 && prec != 1) throw InputErr("precision must be 0 (fp64) or 1 (mixed)");
  precision = prec;
  device = dev;
  DPB_CUDA(cudaSetDevice(dev));
  DPB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  DPB_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&ev_join, &ev_fwd[0], &ev_fwd[1], &ev_kd, &ev_halo})
    DPB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  DPB_CUDA(cudaStreamCreateWithFlags(&st_comm, cudaStreamNonBlocking));
  n_types = md->n_types;
  r_cut = md->r_cut;
  r_smooth = md->r_smooth;
  d1 = md->d1;
  M = 4 * d1;
  Mp = round_up(M, 32);
  if (Mp > 256) throw InputErr("feature width 4*d1 must be at most 256");
  mlt = md->m_lt;
  K0 = mlt * M;
  K0p = round_up(K0, 64);
  masses.assign(md->masses, md->masses + n_types);
  max_nbr.assign(md->max_nbr, md->max_nbr + n_types);
  for (int t = 0; t < n_types; ++t) {
    if (max_nbr[t] <= 0) throw InputErr("model max_nbr entries must be positive");
    if (!(masses[t] > 0.0)) throw InputErr("model masses must be positive");
  }
  // fitting structure, per centre type
  tlayers.assign(n_types, {});
  fit_off.assign(n_types + 1, 0);
  widthp_max = 16;
  max_layers = 0;
  for (int t = 0; t < n_types; ++t) {
    const dp_fitting_desc& f = md->fitting[t];
    if (f.n_layers < 1) throw InputErr("fitting net needs at least one hidden layer");
    if (!f.widths || !f.w || !f.b || !f.w_out) throw InputErr("null fitting net array");
    if (f.widths[0] != K0) throw InputErr("fitting input width does not match descriptor");
    std::vector<FitLayer>& ls = tlayers[t];
    ls.resize(f.n_layers);
    for (int k = 0; k < f.n_layers; ++k) {
      FitLayer& fl = ls[k];
      fl.in = f.widths[k];
      fl.out = f.widths[k + 1];
      if (fl.out <= 0) throw InputErr("fitting layer widths are inconsistent");
      fl.inp = k == 0 ? K0p : pad_width(fl.in);
      fl.outp = pad_width(fl.out);
      fl.shortcut = fl.in == fl.out;
      widthp_max = std::max(widthp_max, fl.outp);
    }
    fit_off[t + 1] = fit_off[t] + f.n_layers;
    max_layers = std::max(max_layers, f.n_layers);
  }
  layers = tlayers[0];
  uniform_fit = true;
  for (int t = 1; t < n_types; ++t) {
    if (tlayers[t].size() != layers.size()) uniform_fit = false;
    else
      for (size_t k = 0; k < layers.size(); ++k)
        if (tlayers[t][k].out != layers[k].out) uniform_fit = false;
  }
  if (td) upload_tables(*td);
  // fitting weights, zero padded
  const int nfit = fit_off[n_types];
  fit_wt.resize(nfit);
  fit_w.resize(nfit);
  fit_b.resize(nfit);
  fit_wout.resize(n_types);
  b_out.resize(n_types);
  for (int t = 0; t < n_types; ++t) {
    const dp_fitting_desc& f = md->fitting[t];
    const std::vector<FitLayer>& ls = tlayers[t];
    const int L = static_cast<int>(ls.size());
    for (int k = 0; k < L; ++k) {
      const FitLayer& fl = ls[k];
      std::vector<double> w(static_cast<size_t>(fl.inp) * fl.outp, 0.0), wt(w.size(), 0.0),
          b(fl.outp, 0.0);
      for (int u = 0; u < fl.in; ++u)
        for (int v = 0; v < fl.out; ++v) {
          const double x = f.w[k][static_cast<size_t>(u) * fl.out + v];
          w[static_cast<size_t>(u) * fl.outp + v] = x;
          wt[static_cast<size_t>(v) * fl.inp + u] = x;
        }
      for (int v = 0; v < fl.out; ++v) b[v] = f.b[k][v];
      DevBuf<double>& dw = fit_w[fit_off[t] + k];
      DevBuf<double>& dwt = fit_wt[fit_off[t] + k];
      DevBuf<double>& db = fit_b[fit_off[t] + k];
      dw.ensure(w.size());
      dwt.ensure(wt.size());
      db.ensure(b.size());
      DPB_CUDA(cudaMemcpy(dw.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
      DPB_CUDA(cudaMemcpy(dwt.p, wt.data(), wt.size() * 8, cudaMemcpyHostToDevice));
      DPB_CUDA(cudaMemcpy(db.p, b.data(), b.size() * 8, cudaMemcpyHostToDevice));
    }
    const int last = ls[L - 1].out;
    std::vector<double> wo(ls[L - 1].outp, 0.0);
    for (int v = 0; v < last; ++v) wo[v] = f.w_out[v];
    fit_wout[t].ensure(wo.size());
    DPB_CUDA(cudaMemcpy(fit_wout[t].p, wo.data(), wo.size() * 8, cudaMemcpyHostToDevice));
    b_out[t] = f.b_out;
  }
  if (precision == 1) prepare_mixed();
  d_max_nbr.ensure(n_types);
  DPB_CUDA(cudaMemcpy(d_max_nbr.p, max_nbr.data(), n_types * sizeof(int), cudaMemcpyHostToDevice));
  // Buffers that may grow inside the MD loop are stream-ordered: growing them must not
  // synchronise the device (a cudaFree would drain the whole queued trajectory). Keep freed
  // pool memory cached so regrowth is cheap.
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    Pbuf.ord = stream;
  }
  err.ensure(1);
  counters.ensure(3);
  exact_ctr.ensure(3);
  red.ensure(256 * 10 + 64);
  DPB_CUDA(cudaMemset(err.p, 0, sizeof(int)));
  DPB_CUDA(cudaMemset(counters.p, 0, 3 * sizeof(unsigned long long)));
  DPB_CUDA(cudaMemset(red.p, 0, 64 * sizeof(double)));
}

void Engine::destroy() {
  if (stream) cudaStreamSynchronize(stream);
  auto rel = [](auto& v) {
    for (auto& b : v) b.release();
  };
  tab.release(); tab32.release(); rel(fit_wt); rel(fit_w); rel(fit_b); rel(fit_wout);
  d_max_nbr.release(); tanh_tab.release(); pos4.release(); pos3.release(); vel3.release();
  types.release(); center.release(); slot_of.release(); atom_of.release(); row_off.release(); keys.release();
  rev.release(); ridx.release(); inner_cnt.release(); bin_of.release(); bin_start.release(); bin_atoms.release(); bin_fill.release();
  frac.release(); ref_pos.release(); row_len.release(); nl_len.release(); scan_tmp.release();
  rec.release(); egrp.release(); gbin.release(); realoff.release(); rbase.release(); sscr.release(); xbin.release(); xrc.release(); n_grp.release(); goff.release(); Pbuf.release(); pbuf_cap = 0; n_real.release(); T.release(); D.release(); dD.release(); rel(act_t);
  rel(act_y); dz.release(); dy.release(); dz2.release(); dy2.release(); e_slot.release();
  e_atom.release(); g.release(); vpart.release(); forces.release();
  red.release(); counters.release(); err.release(); acc_fac.release();
  for (auto& p : phase_ev) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ev_pool) cudaEventDestroy(e);
  phase_ev.clear();
  ev_pool.clear();
  scratch.mass_atom.release();
  scratch.ke.release();
  scratch.rec.release();
  if (dist) dist_destroy(*this);
  for (auto* v : {&tc_wf, &tc_wb, &tc_bias, &tc_wout, &tc_t})
    for (auto& b : *v) b.release();
  tc_tanh.release(); tc_d2.release(); tc_y2a.release(); tc_y2b.release(); tc_dz2a.release();
  tc_dz2b.release(); tc_dya.release(); tc_dyb.release();
  dTbuf.release(); fb_list.release(); emb_w.release(); emb_ptrs.release(); exact_ctr.release();
  for (cudaStream_t* s : {&st2, &st_comm})
    if (*s) {
      cudaStreamSynchronize(*s);
      cudaStreamDestroy(*s);
      *s = nullptr;
    }
  if (stream) cudaStreamDestroy(stream);
  stream = nullptr;
  for (cudaEvent_t* e : {&ev_join, &ev_fwd[0], &ev_fwd[1], &ev_kd, &ev_halo})
    if (*e) {
      cudaEventDestroy(*e);
      *e = nullptr;
    }
  gtot.release();
  scan_tmp2.release();
  if (h_gtotal) {
    cudaFreeHost(h_gtotal);
    h_gtotal = nullptr;
  }
}

void Engine::set_config(int64_t nn, const double* pos, const int32_t* ty, const double* box,
                        const uint8_t* pbc, const uint8_t* cmask) {
  // validate_config (geom.cpp:40-56) and Cell::refresh (geom.cpp:7-29)
  if (nn <= 0) throw InputErr("configuration has no atoms");
  if (!pos || !ty || !box || !pbc) throw InputErr("null configuration array");
  for (int64_t i = 0; i < nn; ++i)
    if (ty[i] < 0 || ty[i] >= n_types) throw InputErr("atom type id out of range");
  for (int64_t k = 0; k < 3 * nn; ++k)
    if (!std::isfinite(pos[k])) throw InputErr("non-finite atom position");
  DevCell c{};
  for (int k = 0; k < 9; ++k) c.h[k] = box[k];
  for (int k = 0; k < 3; ++k) c.per[k] = pbc[k] ? 1 : 0;
  const double* a = c.h;
  const double* b = c.h + 3;
  const double* cc = c.h + 6;
  const double bxc[3] = {b[1] * cc[2] - b[2] * cc[1], b[2] * cc[0] - b[0] * cc[2], b[0] * cc[1] - b[1] * cc[0]};
  double vol = a[0] * bxc[0] + a[1] * bxc[1] + a[2] * bxc[2];
  if (!(std::fabs(vol) > 1e-12)) throw InputErr("cell is singular or has near-zero volume");
  const double cxa[3] = {cc[1] * a[2] - cc[2] * a[1], cc[2] * a[0] - cc[0] * a[2], cc[0] * a[1] - cc[1] * a[0]};
  const double axb[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
  for (int x = 0; x < 3; ++x) {
    c.hinv[3 * x + 0] = bxc[x] / vol;
    c.hinv[3 * x + 1] = cxa[x] / vol;
    c.hinv[3 * x + 2] = axb[x] / vol;
  }
  c.vol = vol < 0.0 ? -vol : vol;
  bool same = nn == n && std::memcmp(c.h, cell.h, sizeof(c.h)) == 0 &&
              std::memcmp(c.per, cell.per, sizeof(c.per)) == 0 &&
              static_cast<int64_t>(h_types.size()) == nn &&
              std::memcmp(h_types.data(), ty, nn * sizeof(int32_t)) == 0 &&
              static_cast<int64_t>(h_center.size()) == nn &&
              (cmask ? std::memcmp(h_center.data(), cmask, nn) == 0
                     : std::all_of(h_center.begin(), h_center.end(), [](uint8_t v) { return v != 0; }));
  cell = c;
  if (!same) {
    n = nn;
    list_valid = false;
    pbuf_cap = 0; // resize the group buffer from the next evaluation's exact total
    plan_dirty = true;
    row_cap = 0;  // and the row capacity from the next (synchronous) list build
    h_types.assign(ty, ty + nn);
    types.ensure(n);
    DPB_CUDA(cudaMemcpyAsync(types.p, ty, n * sizeof(int32_t), cudaMemcpyHostToDevice, stream));
    if (cmask)
      h_center.assign(cmask, cmask + nn);
    else
      h_center.assign(nn, 1);
    n_centers = 0;
    for (int64_t i = 0; i < n; ++i) n_centers += h_center[i] != 0;
    center.ensure(n);
    DPB_CUDA(cudaMemcpyAsync(center.p, h_center.data(), n, cudaMemcpyHostToDevice, stream));
    // slots: atoms grouped by centre type, each segment padded to the GEMM tile (64 rows)
    seg_count.assign(n_types, 0);
    for (int64_t i = 0; i < n; ++i)
      if (h_center[i]) ++seg_count[ty[i]];
    seg_start.assign(n_types, 0);
    seg_rows.assign(n_types, 0);
    int64_t at = 0;
    for (int t = 0; t < n_types; ++t) {
      seg_start[t] = static_cast<int>(at);
      seg_rows[t] = round_up(seg_count[t], 128);
      at += seg_rows[t];
    }
    n_slots = at;
    std::vector<int32_t> so(n), ao(n_slots, -1);
    std::vector<int> fill(n_types, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (!h_center[i]) {
        so[i] = -1;
        continue;
      }
      const int t = ty[i];
      const int s = seg_start[t] + fill[t]++;
      so[i] = s;
      ao[s] = static_cast<int32_t>(i);
    }
    slot_of.ensure(n);
    atom_of.ensure(n_slots);
    DPB_CUDA(cudaMemcpyAsync(slot_of.p, so.data(), n * 4, cudaMemcpyHostToDevice, stream));
    DPB_CUDA(cudaMemcpyAsync(atom_of.p, ao.data(), n_slots * 4, cudaMemcpyHostToDevice, stream));
    ensure_step_buffers();
    DPB_CUDA(cudaStreamSynchronize(stream));
  }
  upload_positions(pos);
}

// Chunk plan (see engine.hpp). Single centre type: chunks of consecutive slots (a multiple of
// 128 rows: GEMM and P2 tiles), two chunks at least once the system is large enough for the
// two-stream overlap (FP64), at most DPB_CHUNK centres each (default 131,072: two buffer sets of
// ~12 GB). Several centre types: one chunk holding every segment.
void Engine::plan_chunks() {
  int64_t cmax = 131072;
  if (const char* v = std::getenv("DPB_CHUNK")) cmax = std::atoll(v);
  if (chunk_max > 0) cmax = chunk_max;
  cmax = std::max<int64_t>(128, cmax / 128 * 128);
  int nk = 1;
  const int64_t nc = n_centers;
  if (n_types == 1 && !force_single_chunk && nc > 0) {
    const bool overlap = pipeline && precision == 0 && Mp <= 128 && nc >= 8192;
    nk = static_cast<int>((nc + cmax - 1) / cmax);
    if (overlap) nk = std::max(nk, 2);
    nk = std::max(nk, 1);
    if (nk > MAX_CHUNKS) throw InputErr("too many evaluation chunks (raise DPB_CHUNK)");
  }
  n_chunks = nk;
  ck_sets = nk > 1 ? 2 : 1;
  ck_a.assign(nk + 1, 0);
  ck_s.assign(nk + 1, 0);
  ck_rows.assign(nk, 0);
  if (nk == 1) {
    ck_a[1] = n;
    ck_s[1] = n_slots;
    ck_rows[0] = n_slots;
  } else {
    // slot boundaries every cs centres; atom boundary = index of the first centre of the chunk
    // (decomposed runs: chunks span first..last centre; the rows of the ghosts outside every
    // chunk are marked non-real once per list build, mark_ghost_rows)
    // centre count before chunk q: equal chunks of cs (a multiple of 128). Uneven plans (a small
    // first and last chunk to shorten the pipeline's head and tail) measured 0.2-0.4 ms slower
    // at C2.
    std::vector<int64_t> start(nk + 1, nc);
    const int64_t cs = round_up((nc + nk - 1) / nk, 128);
    for (int q = 0; q < nk; ++q) start[q] = std::min<int64_t>(static_cast<int64_t>(q) * cs, nc);
    int64_t c = 0, last = 0;
    int k = 0;
    for (int64_t i = 0; i < n; ++i)
      if (h_center[i]) {
        while (k < nk && c == start[k]) ck_a[k++] = i;
        ++c;
        last = i;
      }
    for (; k < nk; ++k) ck_a[k] = last + 1; // (cannot happen: the chunks cover nc)
    ck_a[nk] = last + 1;
    for (int q = 0; q <= nk; ++q) ck_s[q] = start[q];
    for (int q = 0; q < nk; ++q) ck_rows[q] = (q == nk - 1 ? seg_rows[0] : ck_s[q + 1]) - ck_s[q];
  }
  ck_ghost.assign(nk, 1);
  ck_order.resize(nk);
  for (int q = 0; q < nk; ++q) ck_order[q] = q;
  ck_cap_a = ck_cap_s = 0;
  for (int q = 0; q < nk; ++q) {
    ck_cap_a = std::max(ck_cap_a, ck_a[q + 1] - ck_a[q]);
    ck_cap_s = std::max(ck_cap_s, ck_rows[q]);
  }
  if (nk == 1) ck_cap_s = n_slots;
  plan_dirty = false;
}

// Per-set buffers for the current plan; grows only (ensure) and zeroes what the GEMMs read as
// padding (D columns K0..K0p). Pbuf is re-sized from the next evaluation.
void Engine::apply_plan() {
  plan_chunks();
  if (h_gtotal) std::memset(h_gtotal, 0, MAX_CHUNKS * sizeof(int64_t)); // totals of the old plan
  ensure_step_buffers();
  ensure_entry_step_buffers();
  pbuf_cap = 0;
}

void Engine::ensure_step_buffers() {
  if (plan_dirty) plan_chunks();
  const int L = max_layers;
  const size_t sa = static_cast<size_t>(ck_sets) * ck_cap_a, ss = static_cast<size_t>(ck_sets) * ck_cap_s;
  T.ensure(sa * 4 * Mp);
  dTbuf.ensure(sa * 4 * Mp);
  const size_t dsz = ss * K0p;
  dD.ensure(dsz);
  if (precision == 1) {
    // mixed: the tabulate kernel writes D directly as the split FP32 operand of the tcgen05 GEMM
    ensure_mixed_buffers();
  } else {
    const size_t had = D.n;
    D.ensure(dsz);
    if (D.n != had) DPB_CUDA(cudaMemsetAsync(D.p, 0, D.n * sizeof(double), stream));
    act_t.resize(L);
    act_y.resize(L);
    const size_t asz = ss * widthp_max;
    for (int k = 0; k < L; ++k) {
      act_t[k].ensure(asz);
      act_y[k].ensure(asz);
    }
    dz.ensure(asz); dy.ensure(asz); dz2.ensure(asz); dy2.ensure(asz);
  }
  e_slot.ensure(n_slots);
  e_atom.ensure(n);

  vpart.ensure(9 * n);
  forces.ensure(3 * n);
  n_real.ensure(n);
  n_grp.ensure(n + 1);
  goff.ensure(n + 1);
  realoff.ensure(n + 1);
  rbase.ensure(MAX_CHUNKS + 1);
  pos4.ensure(n);
  pos3.ensure(3 * n);
}

// Chunk-local entry arrays: a chunk's rows hold at most (atoms in the chunk) x row_cap entries
// (row lengths are checked against row_cap on the device at every rebuild).
void Engine::ensure_entry_step_buffers() {
  if (e_cap == 0) return;
  if (n_chunks == 1) {
    ck_cap_e = e_cap;
  } else if (list_valid) {
    // exact entry count of every chunk from the list's offsets at the chunk boundaries (the list
    // and the plan only change together with this call): the per-real records of a 13.5 M-atom
    // system then take 64 B x the chunk's entries, not x its atoms x the row capacity
    std::vector<int64_t> b(n_chunks + 1);
    for (int k = 0; k <= n_chunks; ++k)
      DPB_CUDA(cudaMemcpyAsync(&b[k], row_off.p + ck_a[k], sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
    DPB_CUDA(cudaStreamSynchronize(stream));
    int64_t mx = 0;
    for (int k = 0; k < n_chunks; ++k) mx = std::max(mx, b[k + 1] - b[k]);
    // + 1/16: rebuilds inside an MD run change the counts slightly; growing these buffers would
    // reallocate ~1 GB (a device-wide stall) at the first rebuild
    ck_cap_e = std::min<int64_t>(e_cap, mx + mx / 16 + 1024);
  } else {
    ck_cap_e = std::min<int64_t>(e_cap, ck_cap_a * std::max(row_cap, 1));
  }
  const size_t se = static_cast<size_t>(ck_sets) * ck_cap_e;
  egrp.ensure(se + 1);
  gbin.ensure(se + 1);
  sscr.ensure(se + 1);
  rec.ensure(8 * se + 8);
}

void Engine::upload_positions(const double* pos) {
  DPB_CUDA(cudaMemcpyAsync(pos3.p, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, stream));
  launch_pos4(*this);
}

void Engine::build_list(double cutoff) {
  phase_begin(0);
  launch_nlist(cutoff);
  phase_end();
}

void Engine::evaluate() {
  if (!list_valid) throw InputErr("no neighbour list");
  if (tab_n == 0) throw InputErr("no compression tables: pass them to dp_create or build them with dp_build_tables_gpu");
  if (plan_dirty) apply_plan();
  if (n_chunks > 1) {
    evaluate_chunked();
    return;
  }
  use_chunk(0);
  if (halo_pending) {
    DPB_CUDA(cudaStreamWaitEvent(stream, ev_halo, 0));
    halo_pending = false;
  }
  phase_begin(1);
  launch_tab_fwd();
  phase_begin(2);
  if (precision == 1)
    launch_fitting_mixed();
  else
    launch_fitting();
  phase_begin(3);
  launch_tab_bwd();
  phase_begin(4);
  launch_forces();
  phase_end();
}

// Chunks k = 0..n_chunks-1 on two streams (FP64: chunk k on stream k % 2 with buffer set
// k % 2), each one stage behind the previous one: the latency-bound tabulate kernels of one
// chunk run beside the tensor-pipe GEMMs of the other (C2, two chunks: 5.40 -> 5.30 ms/step;
// stream priorities or a three-stream split by kernel class were slower). Mixed mode and
// dp_set_pipeline(0) run the chunks in order on one stream (the tcgen05 GEMMs lose more to
// half-size grids than the overlap gains).
bool Engine::pipeline_ok() const { return pipeline && precision == 0 && Mp <= 128 && n_chunks > 1; }

void Engine::evaluate_chunked() {
  const bool two = pipeline_ok();
  cudaStream_t last = stream;
  DPB_CUDA(cudaMemsetAsync(rbase.p, 0, sizeof(int64_t), stream)); // pair-gradient base of chunk 0
  for (int q = 0; q < n_chunks; ++q) {
    const int k = ck_order[q]; // interior chunks first (decomposed runs)
    use_chunk(k, q & 1);
    cudaStream_t st = two && (q & 1) ? st2 : stream;
    if (two && q >= 1) DPB_CUDA(cudaStreamWaitEvent(st, ev_fwd[(q - 1) & 1], 0));
    if (halo_pending && ck_ghost[k]) DPB_CUDA(cudaStreamWaitEvent(st, ev_halo, 0)); // ghost positions
    phase_begin(1);
    tab_fwd_range(k, q, ck_a[k], ck_a[k + 1], st);
    if (two) DPB_CUDA(cudaEventRecord(ev_fwd[q & 1], st));
    if (pbuf_cap == 0) {
      // first evaluation of this system/plan: size the group buffer from chunk 0's exact total
      DPB_CUDA(cudaStreamSynchronize(st));
      grow_pbuf();
    }
    phase_begin(2);
    if (precision == 1)
      fitting_rows_mixed(ck_s[k], ck_rows[k], st);
    else
      fitting_rows(ck_s[k], ck_rows[k], st);
    phase_begin(3);
    tab_bwd_range(k, ck_a[k], ck_a[k + 1], st);
    last = st;
  }
  phase_end();
  if (two) {
    DPB_CUDA(cudaEventRecord(ev_join, st2));
    DPB_CUDA(cudaStreamWaitEvent(stream, ev_join, 0));
  }
  (void)last;
  if (halo_pending) {
    DPB_CUDA(cudaStreamWaitEvent(stream, ev_halo, 0)); // the force kernel reads ghost positions
    halo_pending = false;
  }
  phase_begin(4);
  finish_energy();
  launch_forces();
  phase_end();
}

// A single evaluation with a group buffer sized from the previous call: if this configuration
// has more (centre, interval) groups than the slack covers, grow and evaluate once more.
void Engine::evaluate_retry() {
  evaluate();
  int code = 0;
  DPB_CUDA(cudaMemcpyAsync(&code, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  if (code == DEV_PBUF) {
    DPB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
    DPB_CUDA(cudaDeviceSynchronize());
    grow_pbuf();
    reset_counters();
    evaluate();
  }
  check_err();
}

void Engine::phase_begin(int ph) {
  if (!timing) return;
  phase_end();
  cudaEvent_t a, b;
  if (ev_pool.size() >= 2) {
    a = ev_pool.back();
    ev_pool.pop_back();
    b = ev_pool.back();
    ev_pool.pop_back();
  } else {
    DPB_CUDA(cudaEventCreate(&a));
    DPB_CUDA(cudaEventCreate(&b));
  }
  DPB_CUDA(cudaEventRecord(a, stream));
  phase_ev.push_back({ph, a, b});
  open_phase = static_cast<int>(phase_ev.size()) - 1;
}

void Engine::phase_end() {
  if (!timing || open_phase < 0) return;
  DPB_CUDA(cudaEventRecord(phase_ev[open_phase].b, stream));
  open_phase = -1;
}

void Engine::phase_collect(double* ms, uint64_t* counts) {
  phase_end();
  DPB_CUDA(cudaStreamSynchronize(stream));
  for (int k = 0; k < 8; ++k) {
    ms[k] = 0.0;
    counts[k] = 0;
  }
  for (auto& p : phase_ev) {
    float t = 0.f;
    DPB_CUDA(cudaEventElapsedTime(&t, p.a, p.b));
    if (p.phase >= 0 && p.phase < 8) {
      ms[p.phase] += t;
      ++counts[p.phase];
    }
    ev_pool.push_back(p.a);
    ev_pool.push_back(p.b);
  }
  phase_ev.clear();
}

void Engine::check_err() {
  // decomposed runs: every rank raises the same error together (a rank that threw alone would
  // leave its peers blocked in the next collective)
  if (dist) dist_agree_err(*this);
  int code = 0;
  DPB_CUDA(cudaMemcpyAsync(&code, err.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  DPB_CUDA(cudaGetLastError());
  if (code) {
    DPB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), stream));
    list_valid = false;
    raise_device_error(code);
  }
}

void Engine::reset_counters() {
  DPB_CUDA(cudaMemsetAsync(counters.p, 0, 3 * sizeof(unsigned long long), stream));
}

void Engine::read_counters() {
  unsigned long long c[3];
  DPB_CUDA(cudaMemcpyAsync(c, counters.p, sizeof(c), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  host_counters.rows_forward = c[0];
  host_counters.rows_backward = c[1];
  host_counters.extrapolations = c[2];
}

void Engine::fetch_results(double* energy, double* f, double* virial, double* atom_energy) {
  double r[10];
  DPB_CUDA(cudaMemcpyAsync(r, red.p, sizeof(r), cudaMemcpyDeviceToHost, stream));
  if (f) DPB_CUDA(cudaMemcpyAsync(f, forces.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, stream));
  if (atom_energy)
    DPB_CUDA(cudaMemcpyAsync(atom_energy, e_atom.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  if (energy) *energy = r[0];
  if (virial)
    for (int k = 0; k < 9; ++k) virial[k] = r[1 + k];
}

double Engine::max_drift() { return host_max_drift(*this); }

// ---------------------------------------------------------------- MD (md.cpp:151-231)

void Engine::md_upload_atoms(const double* vel_local) {
  MdScratch& S = scratch;
  std::vector<double> m(n), af(n);
  for (int64_t i = 0; i < n; ++i) {
    m[i] = masses[h_types[i]];
    af[i] = units::EVA_PER_MASS_TO_ACC / m[i];
  }
  S.mass_atom.ensure(n);
  S.ke.ensure(n);
  acc_fac.ensure(n);
  vel3.ensure(3 * n);
  DPB_CUDA(cudaMemcpyAsync(S.mass_atom.p, m.data(), n * 8, cudaMemcpyHostToDevice, stream));
  DPB_CUDA(cudaMemcpyAsync(acc_fac.p, af.data(), n * 8, cudaMemcpyHostToDevice, stream));
  DPB_CUDA(cudaMemcpyAsync(vel3.p, vel_local, 3 * n * 8, cudaMemcpyHostToDevice, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
}

void Engine::md_begin(const double* pos, const double* vel, const dp_md_config* cfg) {
  (void)pos;
  if (!(cfg->dt > 0.0)) throw InputErr("time step must be positive");
  if (cfg->n_steps < 0) throw InputErr("step count must be non-negative");
  if (cfg->rebuild_every < 1 || cfg->thermo_every < 1)
    throw InputErr("rebuild and thermo intervals must be at least 1");
  if (!(cfg->buffer >= 0.0)) throw InputErr("buffer must be non-negative");
  md = *cfg;
  MdScratch& S = scratch;
  if (!dist) {
    md_upload_atoms(vel);
    build_list(r_cut + md.buffer);
  }
  const int64_t n_rec = cfg->n_steps / cfg->thermo_every + 1;
  S.rec.ensure(n_rec + 1);
  S.n_rec = 0;
  md_res = dp_md_result{};
  DPB_CUDA(cudaMemsetAsync(red.p + 11, 0, sizeof(double), stream)); // max drift seen
  reset_counters();
  evaluate();
  md_res.force_evals = 1;
  launch_thermo(*this, 0, S.rec.p + S.n_rec++, S.mass_atom.p, S.ke.p);
  md_step = 0;
  md_active = true;
  check_err();
  // The group count grows while a lattice start thermalises; Pbuf then regrows inside the loop.
  // Pre-warm the stream-ordered pool (kept, release threshold = max) so that regrowth is a
  // sub-allocation instead of a physical allocation stalling the host for tens of ms.
  if (std::getenv("DPB_TRACE")) {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    std::fprintf(stderr, "[dpb] md_begin: n %lld, entries cap %lld, chunks %d (set: %lld atoms, %lld slots, %lld entries), "
                 "device memory used %.1f of %.1f GB\n", static_cast<long long>(n), static_cast<long long>(e_cap),
                 n_chunks, static_cast<long long>(ck_cap_a), static_cast<long long>(ck_cap_s),
                 static_cast<long long>(ck_cap_e), (tot - fr) / 1e9, tot / 1e9);
  }
  if (Pbuf.n && Pbuf.n * sizeof(double) < (size_t(1) << 29)) { // large systems: no pool reserve
    void* tmp = nullptr;
    if (cudaMallocAsync(&tmp, Pbuf.n * sizeof(double) * 3, stream) == cudaSuccess) cudaFreeAsync(tmp, stream);
    else cudaGetLastError();
  }
}

void Engine::md_steps(int64_t k) {
  if (!md_active) throw InputErr("no MD run in progress");
  if (k < 0 || md_step + k > md.n_steps)
    throw InputErr("MD step count exceeds the configured n_steps of this run");
  MdScratch& S = scratch;
  const double half = 0.5 * md.dt;
  for (int64_t it = 0; it < k; ++it) {
    const int64_t s = ++md_step;
    phase_begin(5);
    launch_kick_drift(*this, half, md.dt);
    phase_end();
    if (s % md.rebuild_every == 0) {
      if (dist)
        dist_rebuild(*this);
      else
        // synchronous sizing (one read-back every rebuild_every steps): the list capacity always
        // fits the new list, so no kernel ever indexes past it
        build_list(r_cut + md.buffer);
    } else if (dist) {
      phase_begin(6);
      dist_halo_forward(*this);
      phase_end();
    }
    phase_begin(5);
    launch_stale_check(*this, 0.5 * md.buffer);
    phase_end();
    ++md_res.staleness_checks;
    evaluate();
    ++md_res.force_evals;
    phase_begin(5);
    launch_kick(*this, half);
    if (s % md.thermo_every == 0) launch_thermo(*this, s, S.rec.p + S.n_rec++, S.mass_atom.p, S.ke.p);
    phase_end();
  }
}

void Engine::md_record(int64_t, bool) {}

void Engine::md_end(double* pos, double* vel) {
  MdScratch& S = scratch;
  md_active = false;
  check_err();
  thermo.resize(S.n_rec);
  if (S.n_rec)
    DPB_CUDA(cudaMemcpyAsync(thermo.data(), S.rec.p, S.n_rec * sizeof(dp_thermo), cudaMemcpyDeviceToHost, stream));
  if (dist) {
    dist_md_end(*this, pos, vel);
  } else {
    if (pos) DPB_CUDA(cudaMemcpyAsync(pos, pos3.p, 3 * n * 8, cudaMemcpyDeviceToHost, stream));
    if (vel) DPB_CUDA(cudaMemcpyAsync(vel, vel3.p, 3 * n * 8, cudaMemcpyDeviceToHost, stream));
  }
  // final KE/PE (md.cpp:227-229)
  DevBuf<dp_thermo> fin;
  fin.ensure(1);
  launch_thermo(*this, md_step, fin.p, S.mass_atom.p, S.ke.p);
  dp_thermo ft;
  DPB_CUDA(cudaMemcpyAsync(&ft, fin.p, sizeof(ft), cudaMemcpyDeviceToHost, stream));
  double seen = 0.0;
  DPB_CUDA(cudaMemcpyAsync(&seen, red.p + 11, sizeof(double), cudaMemcpyDeviceToHost, stream));
  DPB_CUDA(cudaStreamSynchronize(stream));
  fin.release();
  read_counters();
  md_res.max_drift_seen = seen;
  md_res.counters = host_counters;
  md_res.final_ke = ft.ke;
  md_res.final_pe = ft.pe;
  md_res.final_total = ft.ke + ft.pe;
}

} // namespace dpb
