// Engine: device-resident state of one dp_handle and the launchers of every kernel.
// HBM layout:
//   pos4[n]            double4 (x, y, z, 0): one 32-byte sector per neighbour gather
//   types[n]           int32
//   row_off[n+1]       int64 CSR offsets of the neighbour rows (list cutoff = r_cut + skin)
//   keys[E]            uint64 packed (type_j, j, shift) -- rows sorted = type-sectored canonical
//   rev[E]             uint16 position of the reverse entry (j -> i, -s) inside row j
//   ridx[E]            int16 per step: rank of a real entry among its row's reals (list order), -1
//   realoff[n+1]       int64 per step: first compact pair-gradient slot of each centre
//   rec[Ec][8]         chunk-local per-real records (R0..R3, u, d) in list-rank order
//   T[n][4][Mp]        contraction T = sum_k R_k (x) G(s_k)
//   D/dD[slots][K0p]   descriptor rows (fitting input / its gradient), slot = type-sorted atom
//   act[...]           fitting activations (t_k, y_k) and adjoints (dz_k, dy_k) per layer
//   g[G]               double3 pair gradient dE_i/dd_ij of real pair k of centre i at realoff[i] + k
//   vpart[n][9]        per-centre virial partials, reduced in a fixed order
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "dp_b200.h"

namespace dpb {

struct Dist; // dist.cpp: slab decomposition + NCCL halo exchange

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t ord = nullptr; // set: stream-ordered (cudaMallocAsync / cudaFreeAsync) buffer
  void ensure(size_t count) {
    if (count <= n) return;
    static const bool trace = std::getenv("DPB_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    release();
    size_t want = count + std::min<size_t>(count / 8, size_t(1) << 22) + 64; // growth slack, capped
    auto alloc = [&] {
      return ord ? cudaMallocAsync(reinterpret_cast<void**>(&p), want * sizeof(T), ord)
                 : cudaMalloc(&p, want * sizeof(T));
    };
    cudaError_t e = alloc();
    if (e == cudaErrorMemoryAllocation) {
      // memory parked in the stream-ordered pool (release threshold = max) is not available to
      // cudaMalloc: hand it back and retry once
      cudaGetLastError();
      cudaDeviceSynchronize();
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0);
      e = alloc();
    }
    DPB_CUDA(e);
    n = want;
    if (trace)
      std::fprintf(stderr, "[dpb] %salloc %zu B: %.2f ms\n", ord ? "stream-ordered " : "", want * sizeof(T),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  void release() {
    if (p) {
      if (ord)
        cudaFreeAsync(p, ord);
      else
        cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
};

struct FitLayer {
  int in = 0, out = 0;   // real widths
  int inp = 0, outp = 0; // padded widths
  bool shortcut = false;
};

// Device pointers of one embedding net (model.hpp:14-20) inside Engine::emb_w.
struct EmbPtrs {
  const double *w0, *b0, *w1, *b1, *w2, *b2;
};

struct Engine {
  // ---- model (immutable after create) ----
  int precision = 0;
  int device = 0;
  int n_types = 0;
  double r_cut = 0, r_smooth = 0;
  int d1 = 0, M = 0, Mp = 0, mlt = 0, K0 = 0, K0p = 0;
  std::vector<double> masses;
  std::vector<int> max_nbr;
  // fitting nets per centre type (model.cpp:30-47 validates each net on its own, so depth and
  // widths may differ between types); fit_*[fit_off[t] + k] hold type t's layer k
  std::vector<std::vector<FitLayer>> tlayers;
  std::vector<int> fit_off;
  int max_layers = 0;
  bool uniform_fit = true;
  std::vector<FitLayer> layers; // type 0's layers (= every type's when uniform_fit)
  int widthp_max = 0;
  // tables, device layout [type][interval][6][Mp]
  double tab_x0 = 0, tab_h = 0;
  uint64_t tab_n = 0;
  int tab_block = 16;
  DevBuf<double> tab;
  // embedding nets (exact path, GPU table build), optional: dp_set_embedding
  bool has_embedding = false;
  DevBuf<double> emb_w;
  DevBuf<EmbPtrs> emb_ptrs;
  std::vector<EmbPtrs> emb_ptrs_host;
  DevBuf<unsigned long long> exact_ctr;
  DevBuf<double> dTbuf;  // [n][4][Mp] adjoint of T (tabulate backward)
  DevBuf<int> fb_list;   // atom blocks left to the per-warp projection kernel (+ count)
  DevBuf<float> tab32; // mixed mode: FP32 copy of tab for the forward contraction
  uint64_t tab_ver = 0, tab32_ver = ~0ull; // tab32 is refreshed when tab changes
  void ensure_tab32();
  // fitting weights per type and layer: wt = W^T [outp][inp], w = W [inp][outp]
  std::vector<DevBuf<double>> fit_wt, fit_w, fit_b;
  std::vector<DevBuf<double>> fit_wout;
  std::vector<double> b_out;
  DevBuf<int> d_max_nbr;
  DevBuf<double> tanh_tab;

  // ---- configuration ----
  int64_t n = 0;
  DevCell cell{};
  DevBuf<double4> pos4;
  DevBuf<double> pos3; // AoS host layout mirror (MD state)
  DevBuf<double> vel3;
  DevBuf<int32_t> types;
  std::vector<int32_t> h_types;
  std::vector<uint8_t> h_center;  // 1 = centre evaluated here (owned), 0 = ghost (halo only)
  DevBuf<uint8_t> center;
  int64_t n_centers = 0;
  std::vector<int> seg_start, seg_count, seg_rows; // slots per centre type (padded to 64)
  int64_t n_slots = 0;
  DevBuf<int32_t> slot_of; // atom -> slot
  DevBuf<int32_t> atom_of; // slot -> atom (-1 for padding)

  // ---- neighbour list ----
  double list_cutoff = 0;
  bool list_valid = false;
  int64_t n_entries = 0; // -1 after an asynchronous rebuild (see sync_entry_count)
  int max_row = 0;
  int64_t e_cap = 0;      // per-entry buffer capacity (SoA stride of the step buffers)
  int row_cap = 0;        // row length capacity (power of two)
  DevBuf<int64_t> row_off;
  DevBuf<uint64_t> keys;
  DevBuf<uint16_t> rev; // position of the reverse entry inside row j (rows <= 8192 entries)
  DevBuf<int16_t> ridx; // per step: list-order rank of a real entry within its row, -1 otherwise
  DevBuf<unsigned long long> inner_cnt; // list build: entries inside r_cut (pair-gradient capacity)
  int64_t g_cap = 0;    // compact pair-gradient capacity (pairs)
  void set_gcap(int64_t need, int64_t want);
  DevBuf<int32_t> bin_of, bin_start, bin_atoms, bin_fill;
  DevBuf<double> frac;
  DevBuf<double> ref_pos;
  DevBuf<int> row_len;
  DevBuf<int64_t> nl_len;
  DevBuf<unsigned char> scan_tmp;

  // ---- chunked evaluation ----
  // Centres are evaluated in chunks of consecutive slots (single centre type; one chunk for
  // several types). Every per-centre step buffer (T, dT, D, dD, activations) and the per-entry
  // step arrays (rec, sscr, gbin, egrp) exist twice (two buffer sets, chunk k uses set k % 2)
  // and are sized for one chunk, so the step working set no longer grows with the system
  // (13.5 M atoms would need ~1 TB unchunked). Kernels keep global atom / slot indices: the
  // window pointers wa()/ws() are based so that index a0 (s0) of the current chunk lands at
  // the start of its buffer set; entry arrays are indexed e - row_off[i0] on the device.
  int n_chunks = 1;
  bool plan_dirty = true;
  bool force_single_chunk = false; // exact path: whole system in one chunk
  int64_t chunk_max = 0;           // dp_set_chunk_size (0: DPB_CHUNK or the default)
  std::vector<int64_t> ck_a, ck_s, ck_rows; // atom / slot boundaries [n_chunks + 1], GEMM rows
  int64_t ck_cap_a = 0, ck_cap_s = 0, ck_cap_e = 0; // capacities of one buffer set
  int ck_sets = 1;
  int cur_set = 0;
  int64_t cur_a0 = 0, cur_s0 = 0;
  cudaEvent_t ev_fwd[2] = {nullptr, nullptr};
  // domain decomposition: chunks whose centres have ghost neighbours (device-classified at each
  // rebuild) are evaluated last, so the forward halo (NCCL on st_comm) overlaps the interior
  // chunks; the reverse halo of the ghost force partials overlaps the owned-atom force kernel
  std::vector<uint8_t> ck_ghost; // [n_chunks] 1 = some centre of the chunk has a ghost neighbour
  std::vector<int> ck_order;     // evaluation order: interior chunks first
  cudaStream_t st_comm = nullptr;
  cudaEvent_t ev_kd = nullptr, ev_halo = nullptr;
  bool halo_overlap = std::getenv("DPB_NO_HALO_OVERLAP") == nullptr;
  bool halo_pending = false; // forward halo in flight on st_comm (ev_halo marks its end)
  void classify_chunks();
  void plan_chunks();
  void apply_plan();
  void ensure_entry_step_buffers();
  void use_chunk(int k, int set = 0) {
    cur_set = ck_sets > 1 ? set : 0;
    cur_a0 = ck_a[k];
    cur_s0 = ck_s[k];
  }
  template <class T>
  T* wa(const DevBuf<T>& b, int64_t stride) const {
    return b.p + (static_cast<int64_t>(cur_set) * ck_cap_a - cur_a0) * stride;
  }
  template <class T>
  T* ws(const DevBuf<T>& b, int64_t stride) const {
    return b.p + (static_cast<int64_t>(cur_set) * ck_cap_s - cur_s0) * stride;
  }
  template <class T>
  T* we(const DevBuf<T>& b, int64_t per_entry = 1) const {
    return b.p + static_cast<int64_t>(cur_set) * ck_cap_e * per_entry;
  }
  void evaluate_chunked();

  // ---- per-step buffers ----
  DevBuf<uint64_t> sscr;        // [sets][Ec] sort scratch of k_tab_fwd (wide bin ranges)
  DevBuf<double> rec;           // [sets][Ec][8] per-real records R0..R3, u, d0..d2 (list-rank order)
  DevBuf<int32_t> egrp, gbin;   // [sets][Ec] group of real k; the centre's group bins (ascending)
  DevBuf<int64_t> realoff;      // [n+1] first compact pair-gradient slot of each centre
  DevBuf<int64_t> rbase;        // [MAX_CHUNKS+1] pair-gradient base of each chunk (evaluation order)
  DevBuf<int32_t> xbin;         // exact path: [E] neighbour type of a real entry, -1 otherwise
  DevBuf<double> xrc;           // exact path: [4][E] R0..R3 per entry
  DevBuf<int32_t> n_grp;        // [n+1]
  DevBuf<int64_t> goff;         // [n+1]
  DevBuf<double> Pbuf;          // [groups][24]
  int64_t pbuf_cap = 0;
  int64_t* h_gtotal = nullptr;  // pinned: total groups per chunk of the last evaluation
  static constexpr int MAX_CHUNKS = 4096;
  DevBuf<int64_t> gtot;
  DevBuf<unsigned char> scan_tmp2; // scan scratch of buffer set 1
  cudaStream_t st2 = nullptr; // odd chunks of a two-stream evaluation
  cudaEvent_t ev_join = nullptr; // end of the second stream's chunks
  bool pipeline = std::getenv("DPB_NO_PIPELINE") == nullptr;
  void grow_pbuf();
  DevBuf<int32_t> n_real;
  DevBuf<double> T;
  DevBuf<double> D, dD;
  std::vector<DevBuf<double>> act_t, act_y; // per layer [slots][outp]
  DevBuf<double> dz, dy, dz2, dy2;
  DevBuf<double> e_slot, e_atom;
  DevBuf<double> g;

  DevBuf<double> vpart;
  DevBuf<double> forces;
  DevBuf<double> red; // reduction scratch: energy, virial[9], drift...
  DevBuf<unsigned long long> counters; // rows_forward, rows_backward, extrapolations
  DevBuf<int> err;

  cudaStream_t stream = nullptr;
  uint64_t launches = 0;
  // optional per-phase CUDA-event timing (bench.py roofline): 0 nlist, 1 tab_fwd, 2 fitting,
  // 3 tab_bwd, 4 forces+reductions, 5 integrator
  bool timing = false;
  struct PhaseEv {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<PhaseEv> phase_ev;
  std::vector<cudaEvent_t> ev_pool;
  int open_phase = -1;
  void phase_begin(int ph);
  void phase_end();
  void phase_collect(double* ms, uint64_t* counts);
  std::string last_error;
  dp_counters host_counters{};

  // ---- MD state ----
  dp_md_config md{};
  bool md_active = false;
  int64_t md_step = 0;
  std::vector<dp_thermo> thermo;
  dp_md_result md_res{};
  DevBuf<double> acc_fac;
  struct MdScratch {
    DevBuf<double> mass_atom, ke;
    DevBuf<dp_thermo> rec;
    int64_t n_rec = 0;
  } scratch;

  Dist* dist = nullptr; // non-null when this handle is one rank of a domain-decomposed run
  // decomposed runs: local index -> global id and global id -> local index (-1), so the list rows
  // are in the single-GPU (global id) order; null on one GPU
  const int32_t* gid_of = nullptr;
  const int32_t* local_of = nullptr;
  void md_upload_atoms(const double* vel_local);

  // lifecycle
  void create(const dp_model_desc* md, const dp_table_desc* td, int device, int precision);
  void destroy();
  // configuration upload (host AoS positions); resets the list when n/types/box change
  void set_config(int64_t n, const double* pos, const int32_t* types, const double* box,
                  const uint8_t* pbc, const uint8_t* center_mask = nullptr);
  void upload_positions(const double* pos);
  // neighbour list at `cutoff`, device resident
  void build_list(double cutoff);
  void sync_entry_count();
  void finish_list(double cutoff);
  void import_list(const int64_t* offsets, const int32_t* j, const int32_t* shift);
  void download_list(int64_t* offsets, int32_t* j, int32_t* shift);
  // one evaluation on the current positions/list; results stay on device
  void evaluate();
  void fetch_results(double* energy, double* forces, double* virial, double* atom_energy);
  double max_drift(); // device reduction, synchronizes
  void check_err();   // synchronizes and raises on device error
  void reset_counters();
  void read_counters();
  // kernels (defined in the .cu files)
  void launch_nlist(double cutoff);
  void launch_tab_fwd();
  void tab_fwd_range(int k, int q, int64_t i0, int64_t i1, cudaStream_t st);
  bool virial_in_forces = false; // exact path: the force kernel forms the virial (no records)
  void zero_ghost_vpart();
  void tab_bwd_range(int c, int64_t i0, int64_t i1, cudaStream_t st);
  void size_pbuf_if_needed();
  void fitting_rows(int64_t r0, int64_t rows, cudaStream_t st); // FP64, single centre type
  void fitting_type_rows(int t, int64_t r0, int64_t rows, cudaStream_t st);
  void fitting_type_rows_mixed(int t, int64_t r0, int64_t rows, cudaStream_t st);
  void finish_energy();
  void fitting_rows_mixed(int64_t r0, int64_t rows, cudaStream_t st);
  void evaluate_retry();
  bool pipeline_ok() const;
  void launch_fitting();
  void launch_fitting_mixed();
  void set_embedding(const dp_embedding_desc* nets);
  void upload_tables(const dp_table_desc& td);
  void evaluate_exact();
  void launch_env_exact();
  void build_tables_gpu(double step, uint64_t* n_out, double* x_end_out, double* coeffs_out, bool install);
  void ensure_mixed_buffers();
  void prepare_mixed();
  // mixed precision (tcgen05 3xTF32) buffers
  std::vector<DevBuf<float>> tc_wf, tc_wb, tc_bias, tc_wout, tc_t;
  DevBuf<double> tc_tanh;
  DevBuf<float> tc_d2, tc_y2a, tc_y2b, tc_dz2a, tc_dz2b, tc_dya, tc_dyb;

  void launch_tab_bwd();
  void launch_forces();
  // MD
  void md_begin(const double* pos, const double* vel, const dp_md_config* cfg);
  void md_steps(int64_t k);
  void md_record(int64_t step, bool sync_read);
  void md_end(double* pos, double* vel);
  void ensure_step_buffers();
};

// Small launch helpers.
inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// fitting.cu
void scatter_energy(Engine& E);

// force.cu
void launch_pos4(Engine& E);
void launch_kick_drift(Engine& E, double half, double dt);
void launch_kick(Engine& E, double half);
void launch_stale_check(Engine& E, double half_buffer);
double host_max_drift(Engine& E);
void launch_thermo(Engine& E, int64_t step, dp_thermo* dst, double* mass_atom, double* ke_scratch);

// dist.cpp
void dist_init(Engine& E, int rank, int world, const void* uid);
void dist_destroy(Engine& E);
void dist_md_begin(Engine& E, int64_t N, const double* pos, const double* vel, const int32_t* types,
                   const double* box, const uint8_t* pbc, const dp_md_config* cfg);
void dist_rebuild(Engine& E);
void dist_halo_forward(Engine& E);
void dist_exchange_g(Engine& E, const int32_t** rslot, const double** grecv, const int32_t** inner,
                     int64_t* n_inner, const int32_t** bound, int64_t* n_bound);
void dist_allreduce_sum(Engine& E, double* dev, int count);
void dist_agree_err(Engine& E); // err := max over ranks
int64_t dist_n_total(const Engine& E);
void dist_md_end(Engine& E, double* gpos, double* gvel);

} // namespace dpb
