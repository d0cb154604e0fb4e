// Mixed-precision fitting net on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Same algebra as fitting.cu (model.cpp:151-203), but each GEMM runs on tcgen05 with FP32
// accumulation in TMEM and FP32-level accuracy from the 3xTF32 split: every FP32 operand x is
// written as x_hi = tf32(x), x_lo = tf32(x - x_hi) and A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi,
// realised as ONE GEMM over a K-concatenated operand pair [A_hi|A_hi|A_lo] . [B_hi|B_lo|B_hi]^T.
// The activation is the reference's quadratic tanh table (tanh_table.cpp:5-21, mixed mode only).
//
// Kernel: CTA 128 x BN tile (UMMA M=128, N=BN <= 256), warp-specialized: warp 0 issues TMA tile
// loads (128-byte K atoms, SWIZZLE_128B canonical K-major layout), warp 1 issues tcgen05.mma from
// one thread, warps 2-5 drain the TMEM accumulator (tcgen05.ld 32x32b) and run the fused epilogue.
// 4-stage smem ring with full/empty mbarriers; tcgen05.commit releases stages.
#include <cuda.h>

#include <mutex>

#include "engine.hpp"
#include "tc_common.cuh"

namespace dpb {

namespace {

constexpr int TBM = 128, TBKB = 128, TST = 4; // one 128-byte swizzle atom of K per stage

enum TEpi : int { T_FWD = 0, T_BWD = 1 };

struct TArgs {
  int K3bytes;          // 3*K*4
  // forward
  const float* bias;    // [N]
  const float* xin;     // shortcut source [M][ldx] or null
  float* tout;          // [M][ldc] tanh'(z) = 1 - t^2 (evaluated in FP64: no cancellation near |t| = 1)
  float* yout;          // [M][ldc]
  float* y3;            // [M][3*ldc] split of y for the next layer (or null)
  // backward
  const float* dyin;    // [M][ldc] or null
  const float* tprev;   // [M][ldc] or null
  float* dyout;         // [M][ldc] or null
  float* dz3;           // [M][3*ld3] split of dz for the next GEMM (or null)
  double* dD;           // [M][ldD] final layer-0 adjoint (FP64) or null
  int ldc, ldx, ld3, ldD;
  const double* tanh_c; // [8193][3]
};

__device__ __forceinline__ float tf32r(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void split_store(float* base, int K, int col, float x) {
  const float hi = tf32r(x);
  const float lo = tf32r(x - hi);
  base[col] = hi;
  base[K + col] = hi;
  base[2 * K + col] = lo;
}

// TanhTable::operator() (tanh_table.hpp:18-30).
__device__ __forceinline__ double tanh_tab(const double* c, double x) {
  const double ax = fabs(x);
  double t;
  if (ax > 8.0) {
    t = 1.0;
  } else {
    const int k = static_cast<int>(ax * 1024.0);
    const double u = ax - k * (1.0 / 1024.0);
    const double* q = c + 3 * k;
    t = q[0] + u * (q[1] + u * q[2]);
  }
  return signbit(x) ? -t : t;
}

template <int EPI, int BN>
__global__ void __launch_bounds__(192, 1) k_tc_gemm(const __grid_constant__ CUtensorMap ta,
                                                   const __grid_constant__ CUtensorMap tb, TArgs g) {
  using namespace tc;
  constexpr int A_ST = TBM * TBKB, B_ST = BN * TBKB;
  constexpr int TCOLS = BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // SWIZZLE_128B tiles need 1024-byte aligned bases
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* sa = smem;
  unsigned char* sb = smem + TST * A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + TST * B_ST);
  uint64_t* empty = full + TST;
  uint64_t* accf = empty + TST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TBM, n0 = blockIdx.y * BN;
  const int KT = (g.K3bytes + TBKB - 1) / TBKB; // TMA zero-fills the tail of the last block
  if (warp == 0) {
    tmem_alloc<TCOLS>(tslot);
    if (lane == 0) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
    }
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < TST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0) {
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % TST;
      if (kt >= TST) mbar_wait(empty + s, ((kt / TST) - 1) & 1);
      mbar_expect_tx(full + s, A_ST + B_ST);
      tma_load_2d(sa + s * A_ST, &ta, kt * TBKB, m0, full + s);
      tma_load_2d(sb + s * B_ST, &tb, kt * TBKB, n0, full + s);
    }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = make_idesc(TBM, BN, 2, 1);
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % TST;
      mbar_wait(full + s, (kt / TST) & 1);
      fence_after();
      const uint32_t a0 = smem_u32(sa + s * A_ST), b0 = smem_u32(sb + s * B_ST);
#pragma unroll
      for (int k = 0; k < TBKB / 32; ++k) {
        mma_tf32(tmem, make_desc_sw128(a0 + k * 32), make_desc_sw128(b0 + k * 32), idesc, (kt | k) ? 1u : 0u);
      }
      commit(empty + s);
    }
    commit(accf);
  } else if (warp >= 2) {
    mbar_wait(accf, 0);
    fence_after();
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c0, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int col = n0 + c0 + j;
        const float acc = __uint_as_float(v[j]);
        const size_t o = static_cast<size_t>(row) * g.ldc + col;
        if (EPI == T_FWD) {
          const double td = tanh_tab(g.tanh_c, static_cast<double>(acc) + g.bias[col]);
          const float y = (g.xin ? g.xin[static_cast<size_t>(row) * g.ldx + col] : 0.0f) + static_cast<float>(td);
          g.tout[o] = static_cast<float>((1.0 - td) * (1.0 + td));
          g.yout[o] = y;
          if (g.y3) split_store(g.y3 + static_cast<size_t>(row) * 3 * g.ld3, g.ld3, col, y);
        } else {
          const float vv = acc + (g.dyin ? g.dyin[o] : 0.0f);
          if (g.dD) {
            g.dD[static_cast<size_t>(row) * g.ldD + col] = static_cast<double>(vv);
          } else {
            g.dyout[o] = vv;
            split_store(g.dz3 + static_cast<size_t>(row) * 3 * g.ld3, g.ld3, col, vv * g.tprev[o]);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<TCOLS>(tmem);
}

// FP64 D rows -> 3xTF32 split [hi|hi|lo] along K.
__global__ void k_split_d(int64_t rows, int K, const double* __restrict__ D, float* __restrict__ X3) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * K) return;
  const int64_t r = idx / K;
  const int c = static_cast<int>(idx % K);
  split_store(X3 + r * 3 * K, K, c, static_cast<float>(D[idx]));
}

// Readout: E = b_out + y . w_out; dz_L = w_out (1 - t^2) (split), dy_L = w_out.
__global__ void k_readout_tc(int rows, int ld, int width, const float* __restrict__ y,
                             const float* __restrict__ t, const float* __restrict__ wout, double bout,
                             double* __restrict__ e, float* __restrict__ dz3, float* __restrict__ dy) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  double acc = 0.0;
  for (int c = lane; c < ld; c += 32) {
    const float w = c < width ? wout[c] : 0.0f;
    acc += static_cast<double>(y[static_cast<size_t>(r) * ld + c]) * w;
    split_store(dz3 + static_cast<size_t>(r) * 3 * ld, ld, c, w * t[static_cast<size_t>(r) * ld + c]);
    dy[static_cast<size_t>(r) * ld + c] = w;
  }
  acc = warp_sum(acc);
  if (lane == 0) e[r] = bout + acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw CudaErr("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// Byte-level 2-D map over [rows][row_bytes] with 128-byte x box_rows boxes, 128B swizzle.
CUtensorMap byte_map(const void* ptr, uint64_t rows, uint64_t row_bytes, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box,
                               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaErr("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

template <int EPI, int BN>
void launch_tc(const float* A3, const float* B3, int rows, int N, int K, TArgs g, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(TST) * (TBM + BN) * TBKB + 8 * (2 * TST + 1) + 16 + 1024;
  static bool init = false;
  if (!init) {
    DPB_CUDA(cudaFuncSetAttribute(k_tc_gemm<EPI, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    init = true;
  }
  g.K3bytes = 3 * K * 4;
  const CUtensorMap ta = byte_map(A3, rows, static_cast<uint64_t>(3) * K * 4, TBM);
  const CUtensorMap tb = byte_map(B3, N, static_cast<uint64_t>(3) * K * 4, BN);
  k_tc_gemm<EPI, BN><<<dim3(rows / TBM, N / BN), 192, smem, st>>>(ta, tb, g);
  DPB_CUDA(cudaGetLastError());
}

void run_tc(int epi, const float* A3, const float* B3, int rows, int N, int K, const TArgs& g, cudaStream_t st) {
  if (N % 240 == 0 && N <= 240) {
    if (epi == T_FWD) launch_tc<T_FWD, 240>(A3, B3, rows, N, K, g, st);
    else launch_tc<T_BWD, 240>(A3, B3, rows, N, K, g, st);
  } else if (N % 256 == 0) {
    if (epi == T_FWD) launch_tc<T_FWD, 256>(A3, B3, rows, N, K, g, st);
    else launch_tc<T_BWD, 256>(A3, B3, rows, N, K, g, st);
  } else if (N % 128 == 0) {
    if (epi == T_FWD) launch_tc<T_FWD, 128>(A3, B3, rows, N, K, g, st);
    else launch_tc<T_BWD, 128>(A3, B3, rows, N, K, g, st);
  } else if (N % 64 == 0) {
    if (epi == T_FWD) launch_tc<T_FWD, 64>(A3, B3, rows, N, K, g, st);
    else launch_tc<T_BWD, 64>(A3, B3, rows, N, K, g, st);
  } else if (N % 16 == 0 && N <= 256) {
    // single tile of N columns: round the tile to the next supported size is not allowed (the
    // map would read past the operand), so widths are padded to 64 by the engine in mixed mode
    throw InputErr("mixed precision needs fitting widths padded to 64");
  } else {
    throw InputErr("unsupported fitting width for the tensor-core path");
  }
}

} // namespace

void Engine::prepare_mixed() {
  for (size_t k = 1; k < layers.size(); ++k)
    if (layers[k].outp != widthp_max || layers[k].inp != widthp_max)
      throw InputErr("mixed precision needs equal hidden widths");
  // weights: forward B = W^T rows [out][in] -> [hi|lo|hi] along in; backward B = W rows [in][out]
  const int L = static_cast<int>(layers.size());
  tc_wf.resize(n_types * L);
  tc_wb.resize(n_types * L);
  tc_bias.resize(n_types * L);
  tc_wout.resize(n_types);
  std::vector<double> hw;
  auto split3 = [](std::vector<float>& dst, const std::vector<double>& src, int rows, int K) {
    dst.assign(static_cast<size_t>(rows) * 3 * K, 0.f);
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < K; ++c) {
        const float x = static_cast<float>(src[static_cast<size_t>(r) * K + c]);
        uint32_t xb;
        std::memcpy(&xb, &x, 4);
        // host tf32 round-to-nearest-away (cvt.rna): add half an ulp of tf32 and truncate
        auto rna = [](float v) {
          uint32_t b;
          std::memcpy(&b, &v, 4);
          b = (b + 0x1000u) & 0xFFFFE000u;
          float o;
          std::memcpy(&o, &b, 4);
          return o;
        };
        const float hi = rna(x);
        const float lo = rna(x - hi);
        float* d = dst.data() + static_cast<size_t>(r) * 3 * K;
        d[c] = hi;
        d[K + c] = lo;
        d[2 * K + c] = hi;
        (void)xb;
      }
  };
  for (int t = 0; t < n_types; ++t)
    for (int k = 0; k < L; ++k) {
      const FitLayer& fl = layers[k];
      std::vector<double> w(static_cast<size_t>(fl.inp) * fl.outp), wt(w.size()), b(fl.outp);
      DPB_CUDA(cudaMemcpy(w.data(), fit_w[t * L + k].p, w.size() * 8, cudaMemcpyDeviceToHost));
      DPB_CUDA(cudaMemcpy(wt.data(), fit_wt[t * L + k].p, wt.size() * 8, cudaMemcpyDeviceToHost));
      DPB_CUDA(cudaMemcpy(b.data(), fit_b[t * L + k].p, b.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<float> f;
      split3(f, wt, fl.outp, fl.inp);
      tc_wf[t * L + k].ensure(f.size());
      DPB_CUDA(cudaMemcpy(tc_wf[t * L + k].p, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
      split3(f, w, fl.inp, fl.outp);
      tc_wb[t * L + k].ensure(f.size());
      DPB_CUDA(cudaMemcpy(tc_wb[t * L + k].p, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
      std::vector<float> bf(b.begin(), b.end());
      tc_bias[t * L + k].ensure(bf.size());
      DPB_CUDA(cudaMemcpy(tc_bias[t * L + k].p, bf.data(), bf.size() * 4, cudaMemcpyHostToDevice));
    }
  for (int t = 0; t < n_types; ++t) {
    const FitLayer& last = layers[L - 1];
    std::vector<double> wo(last.outp);
    DPB_CUDA(cudaMemcpy(wo.data(), fit_wout[t].p, wo.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<float> wf(wo.begin(), wo.end());
    tc_wout[t].ensure(wf.size());
    DPB_CUDA(cudaMemcpy(tc_wout[t].p, wf.data(), wf.size() * 4, cudaMemcpyHostToDevice));
  }
  std::vector<double> tt(3 * 8193);
  dp_tanh_table(tt.data());
  tc_tanh.ensure(tt.size());
  DPB_CUDA(cudaMemcpy(tc_tanh.p, tt.data(), tt.size() * 8, cudaMemcpyHostToDevice));
}

void Engine::launch_fitting_mixed() {
  const int L = static_cast<int>(layers.size());
  const int wpm = widthp_max;
  const size_t kmax = static_cast<size_t>(std::max(K0p, wpm));
  tc_a3.ensure(static_cast<size_t>(n_slots) * 3 * kmax);
  tc_dz3.ensure(static_cast<size_t>(n_slots) * 3 * wpm);
  tc_dz3b.ensure(static_cast<size_t>(n_slots) * 3 * wpm);
  tc_t.resize(L);
  tc_y.resize(L);
  for (int k = 0; k < L; ++k) {
    tc_t[k].ensure(static_cast<size_t>(n_slots) * wpm);
    tc_y[k].ensure(static_cast<size_t>(n_slots) * wpm);
  }
  tc_y3a.ensure(static_cast<size_t>(n_slots) * 3 * wpm);
  tc_y3b.ensure(static_cast<size_t>(n_slots) * 3 * wpm);
  tc_dy.ensure(static_cast<size_t>(n_slots) * wpm);
  tc_dy2.ensure(static_cast<size_t>(n_slots) * wpm);
  // the layer-0 input: D rows (FP64) -> split3
  {
    const int64_t tot = n_slots * static_cast<int64_t>(K0p);
    k_split_d<<<ceil_div(tot, 256), 256, 0, stream>>>(n_slots, K0p, D.p, tc_a3.p);
    ++launches;
  }
  for (int t = 0; t < n_types; ++t) {
    const int rows = seg_rows[t];
    if (rows == 0) continue;
    const size_t r0 = static_cast<size_t>(seg_start[t]);
    // forward: layer 0 reads the split D from a3, layer k > 0 the split y_{k-1} (ping-pong)
    const float* xin_prev = nullptr;
    const float* A3 = tc_a3.p + r0 * 3 * static_cast<size_t>(K0p);
    int ldk = K0p;
    for (int k = 0; k < L; ++k) {
      const FitLayer& fl = layers[k];
      TArgs g{};
      g.bias = tc_bias[t * L + k].p;
      g.xin = fl.shortcut ? xin_prev : nullptr;
      g.ldx = wpm;
      g.tout = tc_t[k].p + r0 * wpm;
      g.yout = tc_y[k].p + r0 * wpm;
      g.ldc = wpm;
      float* y3 = (k & 1 ? tc_y3b.p : tc_y3a.p) + r0 * 3 * static_cast<size_t>(wpm);
      g.y3 = k + 1 < L ? y3 : nullptr;
      g.ld3 = wpm;
      g.tanh_c = tc_tanh.p;
      run_tc(T_FWD, A3, tc_wf[t * L + k].p, rows, fl.outp, ldk, g, stream);
      ++launches;
      xin_prev = g.yout;
      A3 = y3;
      ldk = fl.outp;
    }
    // readout
    const FitLayer& last = layers[L - 1];
    float* dz3c = tc_dz3.p + r0 * 3 * wpm;
    float* dz3n = tc_dz3b.p + r0 * 3 * wpm;
    float* dyc = tc_dy.p + r0 * wpm;
    float* dyn = tc_dy2.p + r0 * wpm;
    k_readout_tc<<<ceil_div(rows, 4), 128, 0, stream>>>(rows, wpm, last.out, tc_y[L - 1].p + r0 * wpm,
                                                        tc_t[L - 1].p + r0 * wpm, tc_wout[t].p, b_out[t],
                                                        e_slot.p + r0, dz3c, dyc);
    ++launches;
    for (int k = L - 1; k >= 0; --k) {
      const FitLayer& fl = layers[k];
      TArgs g{};
      g.dyin = fl.shortcut ? dyc : nullptr;
      g.ldc = wpm;
      g.tanh_c = tc_tanh.p;
      if (k > 0) {
        g.tprev = tc_t[k - 1].p + r0 * wpm;
        g.dyout = dyn;
        g.dz3 = dz3n;
        g.ld3 = wpm;
      } else {
        g.dD = dD.p + r0 * K0p;
        g.ldD = K0p;
      }
      run_tc(T_BWD, dz3c, tc_wb[t * L + k].p, rows, fl.inp, fl.outp, g, stream);
      ++launches;
      std::swap(dz3c, dz3n);
      std::swap(dyc, dyn);
    }
  }
  if (n_centers < n) DPB_CUDA(cudaMemsetAsync(e_atom.p, 0, n * sizeof(double), stream));
  scatter_energy(*this);
}

} // namespace dpb
