// Fitting net forward + backward on the FP64 tensor pipe.
//
// Reference: fitting_forward model.cpp:151-180 (z = b + x W, t = tanh z, y = [in==out] x + t,
// E = b_out + y . w_out) and fitting_backward model.cpp:182-203 (dz = dy (1 - t^2),
// dx = [in==out] dy + W dz). The reference walks one centre at a time as GEMVs; here all
// centres of one type form the M dimension of dense GEMMs:
//   forward layer k   Y_k = X_k W_k        [slots x in] . [in x out]     epilogue: +b, tanh, shortcut
//   readout           E = Y_L w_out + b_out, dZ_L = w_out (1 - T_L^2)
//   backward layer k  dY_{k-1} = dZ_k W_k^T (+ dY_k)                      epilogue: * (1 - T_{k-1}^2)
//   layer 0           dD = dZ_0 W_0^T
// FP64 has no tcgen05 kind, so the MMA is the FP64 tensor instruction (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4), measured at 37.1 TFLOP/s on this B200 (profiles/r01_fp64_peak_microbench.log).
// Tiles: CTA 64x64, BK 16, 4 warps of 32x32 (4x4 DMMA tiles), 3-stage cp.async pipeline; both
// operands K-contiguous in shared memory with a 20-double row pitch (bank-conflict free).
#include <cstdlib>
#include <map>
#include <mutex>

#include "engine.hpp"

namespace dpb {

namespace {

constexpr int BK = 16, PITCH = BK + 4;

enum Epi : int { EPI_FWD = 0, EPI_BWD = 1 };

struct GemmArgs {
  const double* A;  // [M][lda], K-contiguous
  const double* Bt; // [N][ldb], K-contiguous
  int lda, ldb, K;
  // forward epilogue
  const double* bias; // [N]
  const double* xin;  // shortcut source [M][ldx] or null
  double* tout;       // tanh output [M][ldc]
  double* yout;       // layer output [M][ldc]
  // backward epilogue
  const double* dyin; // shortcut adjoint [M][ldc] or null
  const double* tprev;// tanh output of the previous layer [M][ldc] or null
  double* dyout;      // [M][ldc]
  double* dzout;      // [M][ldc] or null
  int ldc, ldx, ldd; // ldd: pitch of tprev / dzout
  int ldy;            // pitch of dyin (0: one row for all rows, the readout's dY_L = w_out)
  int ntn, ntm;       // column / row tiles
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// BN = 64 (4 DMMA column tiles per warp) or 80 (5): 240-wide layers tile exactly with 80.
// BM = 64 (warp rows 32: 4 DMMA row tiles) or 32 (2): the smaller tile is chosen when it fills
// the waves of resident CTAs better (run_gemm); every output element accumulates its K terms in
// the same order for either tile, so the choice never changes a result bit.
template <int EPI, int BM, int BN, int STAGES>
__device__ __forceinline__ void gemm_body(const GemmArgs& g) {
  constexpr int NT = BN / 16; // 8-wide column tiles per warp (2 warps across BN)
  constexpr int MT = BM / 16; // 8-high row tiles per warp (2 warps across BM)
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                                // [STAGES][BM][PITCH]
  double* Bs = sm + STAGES * BM * PITCH;          // [STAGES][BN][PITCH]
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int gid = lane >> 2, tig = lane & 3;
  const int KT = g.K / BK;
  // persistent over tiles when the grid is capped (g.ntn column tiles x g.ntm row tiles): fewer
  // resident CTAs per SM leave room for the other stream's tabulate kernels on the same SMs
  for (int tile = blockIdx.x; tile < g.ntn * g.ntm; tile += gridDim.x) {
  const int m0 = (tile / g.ntn) * BM, n0 = (tile % g.ntn) * BN;
  const double* A = g.A + static_cast<size_t>(m0) * g.lda;
  const double* B = g.Bt + static_cast<size_t>(n0) * g.ldb;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * BM * PITCH;
    double* bs = Bs + stage * BN * PITCH;
#pragma unroll
    for (int c = 0; c < BM / 16; ++c) {
      const int idx = tid + c * 128; // BM*8 chunks of 2 doubles for the A tile
      const int row = idx >> 3, col = (idx & 7) * 2;
      cp_async16(as + row * PITCH + col, A + static_cast<size_t>(row) * g.lda + k0 + col);
    }
#pragma unroll
    for (int c = 0; c < BN / 16; ++c) {
      const int idx = tid + c * 128; // BN*8 chunks for the B tile
      const int row = idx >> 3, col = (idx & 7) * 2;
      cp_async16(bs + row * PITCH + col, B + static_cast<size_t>(row) * g.ldb + k0 + col);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) load_stage(nk % STAGES, nk);
    cp_commit();
    const double* as = As + (kt % STAGES) * BM * PITCH + (wm * (BM / 2) + gid) * PITCH + tig;
    const double* bs = Bs + (kt % STAGES) * BN * PITCH + (wn * (BN / 2) + gid) * PITCH + tig;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = as[i * 8 * PITCH + kk * 4];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[j * 8 * PITCH + kk * 4];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_wait<0>();

  // Epilogue: thread holds rows (m0 + wm*BM/2 + i*8 + gid), cols (n0 + wn*BN/2 + j*8 + 2*tig + {0,1}).
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int row = m0 + wm * (BM / 2) + i * 8 + gid;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int col = n0 + wn * (BN / 2) + j * 8 + 2 * tig;
      const size_t o = static_cast<size_t>(row) * g.ldc + col;
      if (EPI == EPI_FWD) {
        const double2 b = *reinterpret_cast<const double2*>(g.bias + col);
        const double t0 = tanh_fp64(acc[i][j][0] + b.x);
        const double t1 = tanh_fp64(acc[i][j][1] + b.y);
        double2 y = make_double2(t0, t1);
        if (g.xin) {
          const double2 x = *reinterpret_cast<const double2*>(g.xin + static_cast<size_t>(row) * g.ldx + col);
          y.x = x.x + t0;
          y.y = x.y + t1;
        }
        *reinterpret_cast<double2*>(g.tout + o) = make_double2(t0, t1);
        *reinterpret_cast<double2*>(g.yout + o) = y;
      } else {
        double v0 = acc[i][j][0], v1 = acc[i][j][1];
        if (g.dyin) {
          const double2 d = *reinterpret_cast<const double2*>(g.dyin + static_cast<size_t>(row) * g.ldy + col);
          v0 = d.x + v0;
          v1 = d.y + v1;
        }
        *reinterpret_cast<double2*>(g.dyout + o) = make_double2(v0, v1);
        if (g.dzout) {
          const size_t od = static_cast<size_t>(row) * g.ldd + col;
          const double2 t = *reinterpret_cast<const double2*>(g.tprev + od);
          *reinterpret_cast<double2*>(g.dzout + od) =
              make_double2(v0 * (1.0 - t.x * t.x), v1 * (1.0 - t.y * t.y));
        }
      }
    }
  }
  __syncthreads(); // the next tile's prologue overwrites the stage buffers
  }
}

template <int EPI, int BM, int BN, int STAGES>
__global__ void __launch_bounds__(128) k_gemm(GemmArgs g) {
  gemm_body<EPI, BM, BN, STAGES>(g);
}

// Short-K (240-wide hidden) layers capped at 128 registers: 4 CTAs (16 warps) per SM instead of 3
// (C2 fitting phase 2.74 -> see DESIGN.md §3)
template <int EPI, int BM, int BN, int STAGES>
__global__ void __launch_bounds__(128, 4) k_gemm4(GemmArgs g) {
  gemm_body<EPI, BM, BN, STAGES>(g);
}

// 32 x 48 tiles of the short-K layers: 6 CTAs (24 warps) per SM; chosen when they fill the
// waves better than 32 x 80 (16k-row chunks: 2,500 tiles on 888 slots, 94 %, vs 1,500 on 592, 84 %)
template <int EPI, int BM, int BN, int STAGES>
__global__ void __launch_bounds__(128, 6) k_gemm6(GemmArgs g) {
  gemm_body<EPI, BM, BN, STAGES>(g);
}

// Readout: E = b_out + y . w_out (warp per row); dZ_L = w_out (1 - t^2). dY_L = w_out is the
// same row for every centre: the first backward GEMM reads it from w_out itself (ldy = 0).
__global__ void k_readout(int rows, int ld, int width, const double* __restrict__ y,
                          const double* __restrict__ t, const double* __restrict__ wout,
                          double bout, double* __restrict__ e, double* __restrict__ dz) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const double* yr = y + static_cast<size_t>(r) * ld;
  const double* tr = t + static_cast<size_t>(r) * ld;
  double acc = 0.0;
  for (int c = lane; c < ld; c += 32) {
    const double w = c < width ? wout[c] : 0.0;
    acc += yr[c] * w;
    const double tt = tr[c];
    dz[static_cast<size_t>(r) * ld + c] = w * (1.0 - tt * tt);
  }
  acc = warp_sum(acc);
  if (lane == 0) e[r] = bout + acc;
}

__global__ void k_scatter_energy(int64_t slots, const int32_t* __restrict__ atom_of,
                                 const double* __restrict__ e_slot, double* __restrict__ e_atom) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= slots) return;
  const int a = atom_of[s];
  if (a >= 0) e_atom[a] = e_slot[s];
}

// Resident CTAs per SM of a kernel at its dynamic shared memory (cached per kernel and size).
int ctas_per_sm(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, size_t>, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({kern, bytes});
  if (it != cache.end()) return it->second;
  int n = 0;
  DPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, 128, bytes));
  cache[{kern, bytes}] = std::max(n, 1);
  return std::max(n, 1);
}

int sm_count_fit() {
  int dev = 0, s = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
  return s > 0 ? s : 148;
}

template <int EPI, int BM, int BN, int STAGES>
struct GemmKernel {
  static constexpr size_t bytes = static_cast<size_t>(STAGES) * (BM + BN) * PITCH * sizeof(double);
  static constexpr bool four = BN == 80 && STAGES == 2;
  static constexpr bool six = BN == 48;
  static auto kern() {
    if constexpr (six) return k_gemm6<EPI, BM, BN, STAGES>;
    else if constexpr (four) return k_gemm4<EPI, BM, BN, STAGES>;
    else return k_gemm<EPI, BM, BN, STAGES>;
  }
  // fraction of the resident-CTA slots the tiles fill over the waves they need
  static double wave_eff(int rows, int N) {
    const int tiles = (N / BN) * (rows / BM);
    const int slots = ctas_per_sm(reinterpret_cast<const void*>(kern()), bytes) * sm_count_fit();
    const int waves = (tiles + slots - 1) / slots;
    return static_cast<double>(tiles) / (static_cast<double>(waves) * slots);
  }
  static void launch(const GemmArgs& a, int rows, int N, cudaStream_t st) {
    auto k = kern();
    smem_optin(k, bytes);
    GemmArgs g = a;
    g.ntn = N / BN;
    g.ntm = rows / BM;
    k<<<g.ntn * g.ntm, 128, bytes, st>>>(g);
    DPB_CUDA(cudaGetLastError());
  }
};

// 64- or 32-row tiles, whichever fills the waves better (ties: 64, the higher per-tile rate)
template <int EPI, int BN, int STAGES>
void launch_gemm(const GemmArgs& a, int rows, int N, cudaStream_t st) {
  using K64 = GemmKernel<EPI, 64, BN, STAGES>;
  using K32 = GemmKernel<EPI, 32, BN, STAGES>;
  // long K (the layer-0 forward): the 64-row tile wins in the running step even where its wave
  // fill is worse (C2: 0.845 vs 0.921; 4.207 vs 4.234 ms/step with two chunks, 4.205 vs 4.233
  // with one), although ncu's cold, serialised launch of it is slower (586 vs 559 us)
  const double tol = a.K > 256 ? 0.10 : 0.05;
  if (rows % 64 == 0 && K64::wave_eff(rows, N) >= K32::wave_eff(rows, N) - tol)
    K64::launch(a, rows, N, st);
  else
    K32::launch(a, rows, N, st);
}

// N is a multiple of 80 or 64 (widths are padded by pad_width()).
// Short K (hidden layers): 2 stages -> 4 CTAs/SM to hide the epilogue's global latency.
void run_gemm(int epi, const GemmArgs& a, int rows, int N, cudaStream_t st) {
  const bool b80 = N % 80 == 0;
  const bool s2 = a.K <= 256;
  if (s2 && b80 && N % 48 == 0) {
    // short K: 32 x 48 or 32 x 80 (or 64 x 80) tiles by wave fill
    if (epi == EPI_FWD) {
      using K48 = GemmKernel<EPI_FWD, 32, 48, 2>;
      if (K48::wave_eff(rows, N) > std::max(GemmKernel<EPI_FWD, 32, 80, 2>::wave_eff(rows, N),
                                            GemmKernel<EPI_FWD, 64, 80, 2>::wave_eff(rows, N)) + 0.02) {
        K48::launch(a, rows, N, st);
        return;
      }
    } else {
      using K48 = GemmKernel<EPI_BWD, 32, 48, 2>;
      if (K48::wave_eff(rows, N) > std::max(GemmKernel<EPI_BWD, 32, 80, 2>::wave_eff(rows, N),
                                            GemmKernel<EPI_BWD, 64, 80, 2>::wave_eff(rows, N)) + 0.02) {
        K48::launch(a, rows, N, st);
        return;
      }
    }
  }
  if (epi == EPI_FWD) {
    if (b80) s2 ? launch_gemm<EPI_FWD, 80, 2>(a, rows, N, st) : launch_gemm<EPI_FWD, 80, 3>(a, rows, N, st);
    else s2 ? launch_gemm<EPI_FWD, 64, 2>(a, rows, N, st) : launch_gemm<EPI_FWD, 64, 3>(a, rows, N, st);
  } else {
    if (b80) s2 ? launch_gemm<EPI_BWD, 80, 2>(a, rows, N, st) : launch_gemm<EPI_BWD, 80, 3>(a, rows, N, st);
    else s2 ? launch_gemm<EPI_BWD, 64, 2>(a, rows, N, st) : launch_gemm<EPI_BWD, 64, 3>(a, rows, N, st);
  }
}

} // namespace

void scatter_energy(Engine& E) {
  k_scatter_energy<<<ceil_div(E.n_slots, 256), 256, 0, E.stream>>>(E.n_slots, E.atom_of.p, E.e_slot.p, E.e_atom.p);
  ++E.launches;
}

void Engine::fitting_type_rows(int t, int64_t r0_, int64_t rows_, cudaStream_t st) {
  const std::vector<FitLayer>& layers = tlayers[t]; // this centre type's net (model.cpp:151-203)
  const int L = static_cast<int>(layers.size());
  const int fo = fit_off[t];
  const int wpm = widthp_max;
  const int rows = static_cast<int>(rows_);
  const size_t r0 = static_cast<size_t>(r0_);
  // forward
  const double* x = ws(D, K0p) + r0 * K0p; // chunk windows (engine.hpp)
  int ldx = K0p;
  for (int k = 0; k < L; ++k) {
    const FitLayer& fl = layers[k];
    GemmArgs a{};
    a.A = x;
    a.lda = ldx;
    a.Bt = fit_wt[fo + k].p;
    a.ldb = fl.inp;
    a.K = fl.inp;
    a.bias = fit_b[fo + k].p;
    a.xin = fl.shortcut ? x : nullptr;
    a.ldx = ldx;
    a.tout = ws(act_t[k], wpm) + r0 * wpm;
    a.yout = ws(act_y[k], wpm) + r0 * wpm;
    a.ldc = wpm;
    run_gemm(EPI_FWD, a, rows, fl.outp, st);
    ++launches;
    x = a.yout;
    ldx = wpm;
  }
  // readout
  const FitLayer& last = layers[L - 1];
  double* dzc = ws(dz, wpm) + r0 * wpm;
  double* dyc = ws(dy, wpm) + r0 * wpm;
  double* dzn = ws(dz2, wpm) + r0 * wpm;
  double* dyn = ws(dy2, wpm) + r0 * wpm;
  k_readout<<<ceil_div(rows, 4), 128, 0, st>>>(rows, wpm, last.out, ws(act_y[L - 1], wpm) + r0 * wpm,
                                                   ws(act_t[L - 1], wpm) + r0 * wpm, fit_wout[t].p,
                                                   b_out[t], e_slot.p + r0, dzc);
  ++launches;
  // backward
  for (int k = L - 1; k >= 0; --k) {
    const FitLayer& fl = layers[k];
    GemmArgs a{};
    a.A = dzc;
    a.lda = wpm;
    a.Bt = fit_w[fo + k].p; // W [inp][outp]: K = outp contiguous
    a.ldb = fl.outp;
    a.K = fl.outp;
    a.dyin = fl.shortcut ? (k == L - 1 ? fit_wout[t].p : dyc) : nullptr;
    a.ldy = k == L - 1 ? 0 : wpm;
    a.ldd = wpm;
    if (k > 0) {
      a.tprev = ws(act_t[k - 1], wpm) + r0 * wpm;
      a.dyout = dyn;
      a.dzout = dzn;
      a.ldc = wpm;
    } else {
      a.tprev = nullptr;
      a.dyout = ws(dD, K0p) + r0 * K0p;
      a.dzout = nullptr;
      a.ldc = K0p;
    }
    run_gemm(EPI_BWD, a, rows, fl.inp, st);
    ++launches;
    std::swap(dzc, dzn);
    std::swap(dyc, dyn);
  }
}

void Engine::fitting_rows(int64_t r0, int64_t rows, cudaStream_t st) { fitting_type_rows(0, r0, rows, st); }

void Engine::launch_fitting() {
  for (int t = 0; t < n_types; ++t)
    if (seg_rows[t] > 0) fitting_type_rows(t, seg_start[t], seg_rows[t], stream);
  finish_energy();
}

void Engine::finish_energy() {
  if (n_centers < n) DPB_CUDA(cudaMemsetAsync(e_atom.p, 0, n * sizeof(double), stream));
  scatter_energy(*this);
}

} // namespace dpb
