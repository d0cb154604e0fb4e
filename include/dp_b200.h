/*
 * dp_b200.h — C-ABI of the B200-native Deep Potential force evaluation.
 *
 * Drop-in boundary for the reference's hot path:
 *   compute_energy_forces_virial_tabulated   /root/reference/proj/include/dpmd/fused.hpp:70-73
 *   build_neighbor_list                      /root/reference/proj/include/dpmd/neighbor.hpp:31-36
 *   run_md (+ MDConfig/ThermoRecord/MDResult) /root/reference/proj/include/dpmd/md.hpp:14-60
 *   FusedCounters                            /root/reference/proj/include/dpmd/fused.hpp:10-21
 * plus the host-side fixture generators the reference's tests and CLI use to make inputs
 * (gen_model/gen_config model_io.hpp:39-47, build_tables table.hpp:46-50, init_velocities
 * md.hpp:41-44, testutil::make_test_model/make_random_config tests/helpers.hpp:21-99).
 *
 * Conventions (same as the reference):
 *   - positions: 3n doubles, Angstrom, cartesian, raw (unwrapped);
 *   - box: 9 doubles, ROWS are the cell vectors (geom.hpp:14-16);
 *   - virial[3x+y] = sum over pairs of d_x * dE/dd_y (exact.cpp:22-38);
 *   - forces: 3n doubles, eV/A.
 * Return codes mirror the reference CLI (tools/dpmd.cpp:434-443):
 *   0 ok, 1 NumericalError class, 2 InputError class, 3 CUDA/runtime failure.
 * Threading: one dp_handle per host thread; every device buffer is owned by its handle.
 * No torch types cross this boundary; the library has no CPU fallback for the compute path.
 */
#ifndef DP_B200_H
#define DP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_OK 0
#define DP_NUMERICAL_ERROR 1
#define DP_INPUT_ERROR 2
#define DP_RUNTIME_ERROR 3

/* Fitting net of one center type (model.hpp:22-36). Layer k maps widths[k] -> widths[k+1],
 * weights row-major in x out; identity shortcut when in == out. Each type's net has its own
 * n_layers and widths (model.cpp:30-47 validates the nets one by one). */
typedef struct {
  int n_layers;
  const int* widths;        /* n_layers + 1 */
  const double* const* w;   /* n_layers pointers, widths[k]*widths[k+1] */
  const double* const* b;   /* n_layers pointers, widths[k+1] */
  const double* w_out;      /* widths[n_layers] */
  double b_out;
} dp_fitting_desc;

/* DPModel (model.hpp:38-58) as seen by the tabulated path: the embedding nets are replaced
 * by the compression tables, so only cutoffs, capacities, m_lt and fitting nets remain. */
typedef struct {
  int n_types;
  double r_cut;
  double r_smooth;
  int d1;                          /* feature width M = 4*d1 */
  int m_lt;
  const double* masses;            /* n_types, g/mol */
  const int* max_nbr;              /* n_types slot capacity per neighbor type */
  const dp_fitting_desc* fitting;  /* n_types, one per center type */
} dp_model_desc;

/* CompressionTable (table.hpp:20-35); header fields are those of the DPTB file
 * (table_io.hpp:10-21). Coefficient layout per interval: [block][k=0..5][f<B]. */
typedef struct {
  int n_tables;                /* == n_types, one per neighbor type */
  double x0;
  double h;
  uint64_t n;                  /* intervals */
  int m;                       /* features, == 4*d1 */
  int block;                   /* B */
  const double* const* coeffs; /* n_tables pointers, n * ceil(m/B) * 6 * B doubles */
} dp_table_desc;

typedef struct {
  uint64_t rows_forward;
  uint64_t rows_backward;
  uint64_t extrapolations;
} dp_counters;

/* MDConfig (md.hpp:14-21). n_workers has no meaning on the GPU and is ignored. */
typedef struct {
  int64_t n_steps;
  double dt;
  double buffer;
  int rebuild_every;
  int thermo_every;
} dp_md_config;

/* ThermoRecord (md.hpp:23-29). */
typedef struct {
  int64_t step;
  double ke, pe, temperature, pressure;
} dp_thermo;

/* MDResult (md.hpp:31-39), thermo records returned separately. */
typedef struct {
  uint64_t force_evals;
  uint64_t staleness_checks;
  double max_drift_seen;
  dp_counters counters;
  double final_ke, final_pe, final_total;
} dp_md_result;

typedef struct dp_handle dp_handle;

/* ---- evaluation handle -------------------------------------------------------------------- */

/* precision: 0 = FP64 (parity mode, 1e-10); 1 = mixed (1e-5): FP32 coefficient contraction in
 * the tabulation, tcgen05 3xTF32 fitting GEMMs with FP64 accumulation of short K chains in the
 * forward layers, the reference's tanh table. Fitting nets may differ in depth and widths per
 * centre type (model.cpp:30-47) in FP64 mode; mixed mode needs one shape for all types. */
int dp_create(const dp_model_desc* model, const dp_table_desc* tables, int device, int precision,
              dp_handle** out);
int dp_destroy(dp_handle* h);
const char* dp_last_error(const dp_handle* h);
const char* dp_version(void);

/* ---- exact (untabulated) path, GPU table build, rmse tooling ---- */

/* EmbeddingNet (model.hpp:14-20) of one neighbour type: 1 -> d1 -> 2 d1 -> 4 d1, row-major
 * w1[d1][2 d1], w2[2 d1][4 d1]. */
typedef struct {
  int d1;
  const double *w0, *b0, *w1, *b1, *w2, *b2;
} dp_embedding_desc;

/* Attach the embedding nets (n_types of them, indexed by neighbour type) to a handle; needed by
 * dp_compute_exact and dp_build_tables_gpu. dp_create accepts tables == NULL when the tables
 * are to be built on the device. */
int dp_set_embedding(dp_handle* h, const dp_embedding_desc* nets);

/* compute_energy_forces_virial (exact.cpp:155-173): the full embedding net per neighbour, on the
 * GPU. Same arguments and outputs as dp_compute; the list cutoff is r_cut (+ skin). */
int dp_compute_exact(dp_handle* h, int64_t n, const double* pos, const int32_t* types, const double box[9],
                     const uint8_t pbc[3], double* energy, double* forces, double* virial,
                     double* atom_energy);

/* build_tables (table.cpp:77-162) on the GPU from the attached embedding nets: domain
 * [0, table_domain_end(model, 0.5)], step h. First call with coeffs == NULL returns n_intervals
 * and x_end; coeffs (n_types * n * ceil(4 d1 / 16) * 6 * 16 doubles, block B = 16) is filled on
 * the second call. install != 0 makes these the handle's tables. A table that does not
 * reproduce the net at a node within 1e-10 returns DP_NUMERICAL_ERROR (table.cpp:133-147). */
int dp_build_tables_gpu(dp_handle* h, double step, uint64_t* n_intervals, double* x_end, double* coeffs,
                        int install);

/* rmse_sweep (rmse.cpp:63-97): for every step in h_list, build + install tables on the GPU and
 * compare the tabulated path with the exact path on every configuration (lists at r_cut).
 * Configurations are concatenated: n_atoms[c] atoms each, pos/types/box/pbc back to back.
 * Outputs rmse_e (eV/atom) and rmse_f (eV/A) per step. The handle keeps the last tables. */
int dp_rmse_sweep(dp_handle* h, int n_configs, const int64_t* n_atoms, const double* pos, const int32_t* types,
                  const double* boxes, const uint8_t* pbcs, int n_h, const double* h_list, double* rmse_e,
                  double* rmse_f);

/* Neighbor-list skin for dp_compute: lists are built at r_cut + skin and reused while every atom
 * stayed within skin/2 of its build position (same staleness rule as run_md, md.cpp:211-217).
 * skin = 0 (default) rebuilds on every call, i.e. list = build_neighbor_list(cfg, r_cut). */
int dp_set_skin(dp_handle* h, double skin);

/* compute_energy_forces_virial_tabulated (fused.cpp:245-288) on the GPU. Host buffers in and out.
 * atom_energy may be NULL. Counters of the last call are available from dp_counters_get. */
int dp_compute(dp_handle* h, int64_t n, const double* pos, const int32_t* types,
               const double box[9], const uint8_t pbc[3], double* energy, double* forces,
               double* virial, double* atom_energy);
int dp_counters_get(const dp_handle* h, dp_counters* out);

/* The same operator on the CALLER's neighbour list, exactly the reference signature
 * compute_energy_forces_virial_tabulated(cfg, model, tables, list) (fused.hpp:70-73): list =
 * NeighborList (neighbor.hpp:14-23) flattened to offsets[n+1], j[offsets[n]], shift[3*offsets[n]].
 * The list must be full and symmetric (every (i -> j, s) has its (j -> i, -s), as
 * build_neighbor_list returns it) at any cutoff >= r_cut; entries beyond r_cut are filtered
 * exactly as env_mat.cpp:32 does. Returns 2 (InputError) for an asymmetric or malformed list. */
int dp_compute_list(dp_handle* h, int64_t n, const double* pos, const int32_t* types,
                    const double box[9], const uint8_t pbc[3], const int64_t* offsets,
                    const int32_t* j, const int32_t* shift, double* energy, double* forces,
                    double* virial, double* atom_energy);

/* build_neighbor_list (neighbor.cpp:162-179) on the GPU, canonical order (ascending j, then
 * shift lexicographic). Two calls: dp_neighbor_list_build returns the total entry count, then
 * dp_neighbor_list_get copies offsets[n+1], j[total] and shift[3*total] to host. */
int dp_neighbor_list_build(dp_handle* h, int64_t n, const double* pos, const int32_t* types,
                           const double box[9], const uint8_t pbc[3], double cutoff,
                           int64_t* total);
int dp_neighbor_list_get(dp_handle* h, int64_t* offsets, int32_t* j, int32_t* shift);

/* run_md (md.cpp:151-231) fully device resident. pos/vel are updated in place. thermo receives
 * up to thermo_cap records (n_steps/thermo_every + 1 are produced); *n_thermo is the count. */
int dp_md_run(dp_handle* h, int64_t n, double* pos, double* vel, const int32_t* types,
              const double box[9], const uint8_t pbc[3], const dp_md_config* cfg,
              dp_thermo* thermo, int64_t thermo_cap, int64_t* n_thermo, dp_md_result* result);

/* Split form of dp_md_run for benchmarking with device-resident state: begin uploads and
 * evaluates step 0, step advances k Verlet steps asynchronously on the handle's stream (the host
 * waits once per list rebuild, to size the new list), end synchronizes and copies state back.
 * Stepping past cfg->n_steps is an InputError. */
int dp_md_begin(dp_handle* h, int64_t n, const double* pos, const double* vel,
                const int32_t* types, const double box[9], const uint8_t pbc[3],
                const dp_md_config* cfg);
int dp_md_step(dp_handle* h, int64_t k);
int dp_md_end(dp_handle* h, double* pos, double* vel, dp_thermo* thermo, int64_t thermo_cap,
              int64_t* n_thermo, dp_md_result* result);

/* ---- multi-GPU: one process (one handle) per GPU, spatial domain decomposition ----------------
 * Slab partition with partition_domain semantics (domain.cpp:21-82); ghost positions go to
 * neighbours and the pair gradients of ghost-adjacent pairs come back through NCCL send/recv
 * every step, so forces, positions and velocities are bitwise independent of the number of GPUs
 * (thermo sums are reduced across ranks and agree to rounding). Rank 0 creates
 * the NCCL id with dp_nccl_unique_id (128 bytes) and shares it (e.g. torch.distributed); every rank
 * then calls dp_dist_init on its handle. After that dp_md_begin takes the GLOBAL initial state on
 * every rank and dp_md_end returns the global final state on every rank; thermo records hold
 * global sums. */
int dp_nccl_unique_id(void* out, int len);
/* partition_domain (domain.cpp:21-82) on the host: owner[n], ghost_mask[n_workers * n]. */
int dp_partition_domain(int64_t n, const double* pos, const double* box, const uint8_t* pbc,
                        int n_workers, double margin, int32_t* owner, uint8_t* ghost_mask);
/* Host plan of one rank: local atoms (ascending global id), centre mask, per-peer send/recv
 * global ids (offsets n_workers+1). All arrays sized n. For tests without GPUs. */
int dp_dist_plan(int64_t n, const double* pos, const double* box, const uint8_t* pbc, int n_workers,
                 int rank, double margin, int64_t* n_local, int64_t* lgid, uint8_t* center,
                 int64_t* send_off, int64_t* send_gid, int64_t* recv_off, int64_t* recv_gid);
int dp_dist_init(dp_handle* h, int rank, int world, const void* nccl_id);

/* Two-stream pipelined evaluation (FP64, one centre type; on by default). Phase times are only
 * per-kernel-group meaningful with it off, which is how bench.py measures its roofline. */
int dp_set_pipeline(dp_handle* h, int enable);

/* Largest number of centres evaluated per chunk (a multiple of 128; 0 = default 131,072 or the
 * DPB_CHUNK environment variable). The per-step working set (descriptors, activations, per-real
 * records) is sized for two chunks; the whole-system state is 12 bytes per neighbour-list entry
 * plus 24 bytes per real pair, so the paper's 13.5 M-atom copper system fits one B200 (157 GB).
 * Results are bitwise independent of the chunk size. One centre type only (systems with several
 * centre types are evaluated as one chunk). */
int dp_set_chunk_size(dp_handle* h, int64_t centres);

/* cudaStream_t of the handle (for CUDA-event timing on the launching stream). */
void* dp_stream(dp_handle* h);
/* Number of kernels this handle has launched since creation. */
uint64_t dp_launch_count(const dp_handle* h);
/* Per-phase CUDA-event timing on the handle's stream (off by default). dp_phase_times
 * synchronizes and returns accumulated milliseconds and interval counts for the phases
 * 0 neighbour list, 1 env-mat + tabulate forward, 2 fitting net (DMMA GEMMs), 3 tabulate
 * backward, 4 force gather + reductions, 5 integrator, 6 halo exchange; then resets them. */
int dp_set_timing(dp_handle* h, int enable);
int dp_phase_times(dp_handle* h, double* ms /* 8 */, uint64_t* counts /* 8 */);

/* ---- host-side fixture generators (CPU, deterministic, bit-identical to the reference) ---- */

/* Model flat layout ("model blob"), per type t in order:
 *   embedding: w0[d1] b0[d1] w1[d1*2d1] b1[2d1] w2[2d1*4d1] b2[4d1]
 * then per type t: fitting layers k: w[in*out] b[out], then w_out[width], b_out[1].
 * dp_model_blob_size gives the length for the shape below. */
typedef struct {
  int n_types;
  double r_cut, r_smooth;
  int d1, m_lt;
  int fit_width, fit_hidden;
  double masses[8];
  int max_nbr[8];
  double lattice_a;
  int site_pattern[8];
  int n_sites;
} dp_preset;

int dp_preset_get(const char* name, dp_preset* out);                     /* model_io.cpp:16-61 */
int64_t dp_model_blob_size(const dp_preset* shape);
int dp_gen_model(const char* preset, uint64_t seed, double* blob);      /* model_io.cpp:129-188 */
int dp_gen_test_model(const dp_preset* shape, uint64_t seed, double fit_scale,
                      double* blob);                                     /* helpers.hpp:21-72 */
/* Table build from a model blob (table.cpp:77-162): n_intervals first (coeffs NULL) then fill. */
int dp_build_tables(const dp_preset* shape, const double* blob, double h, uint64_t* n_intervals,
                    double* x_end, double* coeffs);
int dp_gen_config(const char* preset, int nx, int ny, int nz, double jitter, uint64_t seed,
                  double* pos, int32_t* types, double box[9]);           /* model_io.cpp:190-224 */
int dp_gen_random_config(int n, int n_types, double box_len, double min_sep, uint64_t seed,
                         double* pos, int32_t* types);                  /* helpers.hpp:75-99 */
int dp_init_velocities(int64_t n, const int32_t* types, const double* masses, double t_init,
                       uint64_t seed, double* vel);                     /* md.cpp:14-55 */
uint64_t dp_mix_seed(uint64_t seed, uint64_t k);                        /* rng.hpp:44-49 */

/* DPTB container (table_io.cpp:32-89). */
int dp_write_tables(const char* path, const dp_table_desc* tables);
int dp_read_tables_header(const char* path, int* n_tables, int* m, int* block, uint64_t* n,
                          double* x0, double* h);
int dp_read_tables(const char* path, double* coeffs /* n_tables * n * stride */);

/* JSON model files, write_model / read_model (model_io.cpp:226-283). species_csv: comma-separated
 * species names (NULL: "A", "B", ...). The reader fills the shape first; call it again with a blob
 * of dp_model_blob_size(shape) doubles to get the weights. Non-uniform fitting widths are
 * rejected (the blob layout has one width). Errors: DP_INPUT_ERROR as the reference's InputError. */
int dp_write_model_json(const char* path, const dp_preset* shape, const double* blob, const char* species_csv,
                        const char* preset, uint64_t seed);
int dp_read_model_json(const char* path, dp_preset* shape, double* blob, int64_t blob_cap, char* species_csv,
                       int species_cap, char* preset, int preset_cap, uint64_t* seed);

/* TanhTable (tanh_table.cpp:5-21) coefficients, 3 * 8193 doubles; mixed-precision mode only. */
int dp_tanh_table(double* coef);

#ifdef __cplusplus
}
#endif

#endif /* DP_B200_H */
