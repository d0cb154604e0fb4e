// Mixed-precision fitting net on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
// Same algebra as fitting.cu (model.cpp:151-203), but each GEMM runs on tcgen05 with FP32-level
// operands from the 3xTF32 split: every FP32 operand x is written as x_hi = tf32(x),
// x_lo = tf32(x - x_hi) and A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi, realised as ONE K-concatenated
// accumulation over [A_hi|A_hi|A_lo] . [B_hi|B_lo|B_hi]^T. The activation is the reference's
// quadratic tanh table (tanh_table.cpp:5-21, mixed mode only).
//
// Kernels:
//   k_tc_fwd64  forward layers: 128 x 80 tiles; short TMEM chains (1 K block of each segment)
//               drained into FP64 registers by 8 epilogue warps while the next chain runs on the
//               other TMEM buffer -- the tensor core's FP32 accumulation over the whole 6144-term
//               first layer biased small total energies by 1e-4 (water preset), this keeps every
//               preset within 1e-5 (tests/test_gpu_mixed.py);
//   k_tc_gemm   backward layers: CTA 128 x BN (UMMA M=128, N=BN <= 256), warp-specialized: warp 0
//               issues TMA tile loads (128-byte K atoms, SWIZZLE_128B canonical K-major layout),
//               warp 1 issues tcgen05.mma from one thread, warps 2-5 drain the TMEM accumulator
//               (tcgen05.ld 32x32b) and run the fused epilogue; smem ring with full/empty
//               mbarriers; tcgen05.commit releases stages.
#include <cuda.h>

#include <mutex>

#include "engine.hpp"
#include "tc_common.cuh"

namespace dpb {

namespace {

constexpr int TBM = 128, TBKB = 128, TST = 2; // one 128-byte swizzle atom of K per stage; 2 CTAs/SM
constexpr int CW = 16;                          // epilogue column chunk
constexpr int SP = CW + 4;                      // staging row pitch in floats (conflict-free v4 access)
constexpr int SPD = CW + 2;                     // staging row pitch in doubles
constexpr int STAGE_IN = 2 * TBM * SP * 4;      // two input arrays
constexpr int STAGE_OUT = 3 * TBM * SP * 4;     // three output arrays (one buffer)
constexpr int STAGE_BYTES = STAGE_IN + 2 * STAGE_OUT;

enum TEpi : int { T_FWD = 0, T_BWD = 1 };

// Operands are stored as [hi | lo] halves of kseg floats each (kseg a multiple of 32 so every
// 128-byte TMA box lies inside one half); the 3xTF32 product A.B ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi
// is three K segments of ONE accumulation chain, selected by the TMA x coordinate.
struct TArgs {
  int kseg;             // floats per half of an A / B row
  // forward
  const float* bias;    // [N]
  const float* xin2;    // shortcut source y_{k-1} as [M][2*ldx] (hi|lo) or null
  int ldx;
  float* tout;          // [M][ldc] tanh'(z) = (1 - t)(1 + t), t from the FP64 table (no cancellation)
  float* y2;            // [M][2*ld2] (hi|lo) split of y for the next layer / readout
  // backward
  const float* dyin;    // [M][ldc] shortcut adjoint or null
  const float* dyvec;   // [N] row-independent shortcut adjoint (readout's dy = w_out) or null
  const float* tprev;   // [M][ldc] tanh' of the previous layer (null for layer 0)
  float* dyout;         // [M][ldc]
  float* dz2;           // [M][2*ld2] (hi|lo) split of dz for the next GEMM
  double* dD;           // [M][ldD] layer-0 adjoint (FP64) or null
  int ldc, ld2, ldD;
  const double* tanh_c; // [8193][3]
};

__device__ __forceinline__ float tf32r(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
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

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// Coalesced [128 x CW] float tile copies between global (row pitch ld floats) and staging.
__device__ __forceinline__ void tile_in(float* s, const float* g, size_t ld, int et) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int idx = et + 128 * j, r = idx >> 2, c4 = idx & 3;
    *reinterpret_cast<float4*>(s + r * SP + 4 * c4) =
        __ldg(reinterpret_cast<const float4*>(g + r * ld + 4 * c4));
  }
}
__device__ __forceinline__ void tile_out(float* g, const float* s, size_t ld, int et) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int idx = et + 128 * j, r = idx >> 2, c4 = idx & 3;
    *reinterpret_cast<float4*>(g + r * ld + 4 * c4) = *reinterpret_cast<const float4*>(s + r * SP + 4 * c4);
  }
}

template <int EPI, int BN>
__global__ void __launch_bounds__(192, 2) k_tc_gemm(const __grid_constant__ CUtensorMap ta,
                                                   const __grid_constant__ CUtensorMap tb, TArgs g) {
  using namespace tc;
  constexpr int A_ST = TBM * TBKB, B_ST = BN * TBKB;
  constexpr int PIPE = TST * (A_ST + B_ST);
  constexpr int BODY = PIPE > STAGE_BYTES ? PIPE : STAGE_BYTES;
  constexpr int TCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // SWIZZLE_128B tiles need 1024-byte aligned bases
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* sa = smem;
  unsigned char* sb = smem + TST * A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BODY);
  uint64_t* empty = full + TST;
  uint64_t* accf = empty + TST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TBM, n0 = blockIdx.y * BN;
  const int KB = g.kseg / 32;   // 128-byte blocks per half
  const int KT = 3 * KB;
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
    const int half = g.kseg * 4;
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % TST;
      const int seg = kt / KB, kb = kt - seg * KB;
      if (kt >= TST) mbar_wait(empty + s, ((kt / TST) - 1) & 1);
      mbar_expect_tx(full + s, A_ST + B_ST);
      tma_load_2d(sa + s * A_ST, &ta, (seg == 2 ? half : 0) + kb * TBKB, m0, full + s);
      tma_load_2d(sb + s * B_ST, &tb, (seg == 1 ? half : 0) + kb * TBKB, n0, full + s);
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
    // the operand ring is drained: reuse it as epilogue staging
    float* sin0 = reinterpret_cast<float*>(smem);
    float* sin1 = sin0 + TBM * SP;
    float* sout = sin0 + 2 * TBM * SP;
    const int q = warp & 3;
    const int et = threadIdx.x - 64;         // 0..127 epilogue thread
    const int r = q * 32 + lane;             // tile row owned after tcgen05.ld (TMEM lane)
    const size_t row0 = static_cast<size_t>(m0);
    for (int c0 = 0, ci = 0; c0 < BN; c0 += CW, ++ci) {
      const int col0 = n0 + c0;
      float* so = sout + (ci & 1) * 3 * TBM * SP;
      // stage the inputs of this chunk (coalesced)
      bool staged = false;
      if (g.dyin) {
        tile_in(sin0, g.dyin + row0 * g.ldc + col0, g.ldc, et);
        staged = true;
      }
      if (g.tprev) {
        tile_in(sin1, g.tprev + row0 * g.ldc + col0, g.ldc, et);
        staged = true;
      }
      uint32_t v[CW];
      tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + c0, v);
      tmem_wait_ld();
      if (staged) epi_bar();
      if (g.dD) {
        double* sd = reinterpret_cast<double*>(so);
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          float vv = __uint_as_float(v[j]);
          if (g.dyin) vv += sin0[r * SP + j];
          else if (g.dyvec) vv += g.dyvec[col0 + j];
          sd[r * SPD + j] = static_cast<double>(vv);
        }
        epi_bar();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int idx = et + 128 * jj, rr = idx >> 3, c2 = idx & 7;
          *reinterpret_cast<double2*>(g.dD + (row0 + rr) * g.ldD + col0 + 2 * c2) =
              *reinterpret_cast<const double2*>(sd + rr * SPD + 2 * c2);
        }
      } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          float vv = __uint_as_float(v[j]);
          if (g.dyin) vv += sin0[r * SP + j];
          else if (g.dyvec) vv += g.dyvec[col0 + j];
          const float dz = vv * sin1[r * SP + j];
          const float hi = tf32r(dz);
          so[r * SP + j] = vv;
          so[TBM * SP + r * SP + j] = hi;
          so[2 * TBM * SP + r * SP + j] = tf32r(dz - hi);
        }
        epi_bar();
        tile_out(g.dyout + row0 * g.ldc + col0, so, g.ldc, et);
        const size_t ld = 2 * static_cast<size_t>(g.ld2);
        tile_out(g.dz2 + row0 * ld + col0, so + TBM * SP, ld, et);
        tile_out(g.dz2 + row0 * ld + g.ld2 + col0, so + 2 * TBM * SP, ld, et);
      }
      // the next chunk overwrites sin0/sin1: every thread must be done reading them
      if (staged) epi_bar();
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<TCOLS>(tmem);
}

// Forward layer with FP64 accumulation of short tcgen05 chains (mixed mode). The tensor core's
// FP32 accumulation loses low-order bits at every add; over the 3 x 2048-term first layer (a
// cancelling sum, |z| ~ sum|D W| / 45) that bias reached 1e-4 on small total energies (water
// preset). Here the MMA warp accumulates only F64_CH 128-byte K blocks of each of the three
// 3xTF32 segments (3 x 64 K terms) per chain, alternating between two TMEM accumulators; eight
// epilogue warps (two per TMEM lane quarter, half the columns each) drain each finished chain
// into FP64 registers while the next one runs, so the FP32 error is bounded per chain and the K
// reduction itself is FP64. Tile 128 x BN (BN <= 128), one CTA per SM.
constexpr int F64_ST = 8; // 8 x 26 KB stages: one N=80 stage is only ~90 ns of MMA work
constexpr int F64_CH = 1; // K blocks per segment per chain: water E 3.1e-6 and 3.26 ms/step at C2
                          // (2 blocks: 5.3e-6 and 3.31 ms; FP32 hidden layers: 1.1e-5, over 1e-5)
constexpr int F64_THREADS = 320; // TMA warp, MMA warp, 8 epilogue warps

template <int BN>
constexpr int f64_zpitch() { return BN + 2; }

template <int BN>
constexpr size_t f64_smem_body() {
  constexpr size_t pipe = static_cast<size_t>(F64_ST) * (TBM + BN) * TBKB;
  constexpr size_t epi = static_cast<size_t>(STAGE_BYTES) + static_cast<size_t>(TBM) * f64_zpitch<BN>() * 8;
  return pipe > epi ? pipe : epi;
}

__device__ __forceinline__ void epi2_bar() { asm volatile("bar.sync 2, 256;\n" ::: "memory"); }

template <int BN>
__global__ void __launch_bounds__(F64_THREADS, 1) k_tc_fwd64(const __grid_constant__ CUtensorMap ta,
                                                            const __grid_constant__ CUtensorMap tb, TArgs g) {
  using namespace tc;
  static_assert(BN % 16 == 0 && BN <= 128, "one 128-column TMEM buffer per chain");
  constexpr int A_ST = TBM * TBKB, B_ST = BN * TBKB;
  constexpr size_t BODY = f64_smem_body<BN>();
  constexpr int ZP = f64_zpitch<BN>();
  constexpr int HB = BN / 2; // columns per epilogue warp
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* sa = smem;
  unsigned char* sb = smem + F64_ST * A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BODY);
  uint64_t* empty = full + F64_ST;
  uint64_t* accf = empty + F64_ST; // [2] chain finished (MMA -> epilogue)
  uint64_t* acce = accf + 2;       // [2] chain drained (epilogue -> MMA), 256 arrivals
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acce + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * BN; // column tiles of a row tile adjacent: A shared in L2
  const int KB = g.kseg / 32;                  // 128-byte K blocks per half
  const int NC = (KB + F64_CH - 1) / F64_CH;   // chains
  if (warp == 0) {
    tmem_alloc<256>(tslot);
    if (lane == 0) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
    }
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < F64_ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf + b, 1);
      mbar_init(acce + b, 256);
    }
    fence_barrier_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  // k-block order: chain c, segment seg, block kb in [c*CH, min(KB, c*CH + CH))
  if (warp == 0 && lane == 0) {
    const int half = g.kseg * 4;
    int kt = 0;
    for (int c = 0; c < NC; ++c)
      for (int seg = 0; seg < 3; ++seg)
        for (int kb = c * F64_CH; kb < min(KB, c * F64_CH + F64_CH); ++kb, ++kt) {
          const int s = kt % F64_ST;
          if (kt >= F64_ST) mbar_wait(empty + s, ((kt / F64_ST) - 1) & 1);
          mbar_expect_tx(full + s, A_ST + B_ST);
          tma_load_2d(sa + s * A_ST, &ta, (seg == 2 ? half : 0) + kb * TBKB, m0, full + s);
          tma_load_2d(sb + s * B_ST, &tb, (seg == 1 ? half : 0) + kb * TBKB, n0, full + s);
        }
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = make_idesc(TBM, BN, 2, 1);
    int kt = 0;
    for (int c = 0; c < NC; ++c) {
      const int b = c & 1;
      if (c >= 2) mbar_wait(acce + b, ((c >> 1) - 1) & 1);
      fence_after();
      const uint32_t td = tmem + static_cast<uint32_t>(b * 128);
      bool first = true;
      for (int seg = 0; seg < 3; ++seg)
        for (int kb = c * F64_CH; kb < min(KB, c * F64_CH + F64_CH); ++kb, ++kt) {
          const int s = kt % F64_ST;
          mbar_wait(full + s, (kt / F64_ST) & 1);
          fence_after();
          const uint32_t a0 = smem_u32(sa + s * A_ST), b0 = smem_u32(sb + s * B_ST);
#pragma unroll
          for (int k = 0; k < TBKB / 32; ++k) {
            mma_tf32(td, make_desc_sw128(a0 + k * 32), make_desc_sw128(b0 + k * 32), idesc, first ? 0u : 1u);
            first = false;
          }
          commit(empty + s);
        }
      commit(accf + b);
    }
  } else if (warp >= 2) {
    const int q = warp & 3;             // TMEM lane quarter
    const int hh = (warp - 2) >> 2;     // column half
    const int r = q * 32 + lane;        // tile row
    double acc[HB];
#pragma unroll
    for (int j = 0; j < HB; ++j) acc[j] = 0.0;
    for (int c = 0; c < NC; ++c) {
      const int b = c & 1;
      mbar_wait(accf + b, (c >> 1) & 1);
      fence_after();
      const uint32_t ta0 =
          tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * 128 + hh * HB);
      uint32_t v[HB];
#pragma unroll
      for (int j0 = 0; j0 + 16 <= HB; j0 += 16) tmem_ld16(ta0 + j0, v + j0);
      if constexpr (HB % 16 == 8) tmem_ld8(ta0 + (HB - 8), v + (HB - 8));
      tmem_wait_ld();
      fence_before();
      mbar_arrive(acce + b);
#pragma unroll
      for (int j = 0; j < HB; ++j) acc[j] += static_cast<double>(__uint_as_float(v[j]));
    }
    // every chain is drained (the operand ring is free): z rows to shared memory, then the layer
    // epilogue of k_tc_gemm (bias, tanh table, shortcut, hi|lo split) in 16-column chunks by the
    // first four epilogue warps
    double* zs = reinterpret_cast<double*>(smem + STAGE_BYTES);
#pragma unroll
    for (int j = 0; j < HB; ++j) zs[r * ZP + hh * HB + j] = acc[j];
    epi2_bar();
    if (hh == 0) {
      const int et = threadIdx.x - 64;
      float* sin0 = reinterpret_cast<float*>(smem);
      float* sin1 = sin0 + TBM * SP;
      float* sout = sin0 + 2 * TBM * SP;
      const size_t row0 = static_cast<size_t>(m0);
      for (int c0 = 0, ci = 0; c0 < BN; c0 += CW, ++ci) {
        const int col0 = n0 + c0;
        float* so = sout + (ci & 1) * 3 * TBM * SP;
        if (g.xin2) {
          const size_t ld = 2 * static_cast<size_t>(g.ldx);
          tile_in(sin0, g.xin2 + row0 * ld + col0, ld, et);
          tile_in(sin1, g.xin2 + row0 * ld + g.ldx + col0, ld, et);
          epi_bar();
        }
        double z[CW], c0v[CW], c1v[CW], c2v[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          z[j] = zs[r * ZP + c0 + j] + static_cast<double>(__ldg(g.bias + col0 + j));
          const int k = min(static_cast<int>(fabs(z[j]) * 1024.0), 8191);
          const double* qq = g.tanh_c + 3 * k;
          c0v[j] = __ldg(qq);
          c1v[j] = __ldg(qq + 1);
          c2v[j] = __ldg(qq + 2);
        }
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          // TanhTable::operator() (tanh_table.hpp:18-30)
          const double ax = fabs(z[j]);
          const int k = min(static_cast<int>(ax * 1024.0), 8191);
          const double u = ax - k * (1.0 / 1024.0);
          double td = ax > 8.0 ? 1.0 : c0v[j] + u * (c1v[j] + u * c2v[j]);
          td = signbit(z[j]) ? -td : td;
          double y = td;
          if (g.xin2) y += static_cast<double>(sin0[r * SP + j]) + static_cast<double>(sin1[r * SP + j]);
          const float yf = static_cast<float>(y);
          const float hi = tf32r(yf);
          so[r * SP + j] = static_cast<float>((1.0 - td) * (1.0 + td));
          so[TBM * SP + r * SP + j] = hi;
          so[2 * TBM * SP + r * SP + j] = tf32r(yf - hi);
        }
        epi_bar();
        tile_out(g.tout + row0 * g.ldc + col0, so, g.ldc, et);
        if (g.y2) {
          const size_t ld = 2 * static_cast<size_t>(g.ld2);
          tile_out(g.y2 + row0 * ld + col0, so + TBM * SP, ld, et);
          tile_out(g.y2 + row0 * ld + g.ld2 + col0, so + 2 * TBM * SP, ld, et);
        }
        if (g.xin2) epi_bar();
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

// Readout: E = b_out + y . w_out (y = hi + lo); dz_L = w_out tanh'(z_L) split (hi|lo).
__global__ void k_readout_tc(int rows, int ld, int ld2, int width, const float* __restrict__ y2,
                             const float* __restrict__ t, const float* __restrict__ wout, double bout,
                             double* __restrict__ e, float* __restrict__ dz2) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* yr = y2 + static_cast<size_t>(r) * 2 * ld2;
  float* dr = dz2 + static_cast<size_t>(r) * 2 * ld2;
  double acc = 0.0;
  for (int c = lane; c < ld; c += 32) {
    const float w = c < width ? wout[c] : 0.0f;
    acc += (static_cast<double>(yr[c]) + static_cast<double>(yr[ld2 + c])) * w;
    const float dz = w * t[static_cast<size_t>(r) * ld + c];
    const float hi = tf32r(dz);
    dr[c] = hi;
    dr[ld2 + c] = tf32r(dz - hi);
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

template <int BN>
void launch_tc_fwd64(const float* A2, const float* B2, int rows, int N, TArgs g, cudaStream_t st) {
  const size_t smem = f64_smem_body<BN>() + 8 * (2 * F64_ST + 4) + 16 + 1024;
  smem_optin(k_tc_fwd64<BN>, smem);
  const uint64_t row_bytes = static_cast<uint64_t>(2) * g.kseg * 4;
  const CUtensorMap ta = byte_map(A2, rows, row_bytes, TBM);
  const CUtensorMap tb = byte_map(B2, N, row_bytes, BN);
  k_tc_fwd64<BN><<<dim3(N / BN, rows / TBM), F64_THREADS, smem, st>>>(ta, tb, g);
  DPB_CUDA(cudaGetLastError());
}

template <int EPI, int BN>
void launch_tc(const float* A2, const float* B2, int rows, int N, TArgs g, cudaStream_t st) {
  constexpr int PIPE = TST * (TBM + BN) * TBKB;
  const size_t smem = static_cast<size_t>(PIPE > STAGE_BYTES ? PIPE : STAGE_BYTES) + 8 * (2 * TST + 1) + 16 + 1024;
  smem_optin(k_tc_gemm<EPI, BN>, smem);
  const uint64_t row_bytes = static_cast<uint64_t>(2) * g.kseg * 4;
  const CUtensorMap ta = byte_map(A2, rows, row_bytes, TBM);
  const CUtensorMap tb = byte_map(B2, N, row_bytes, BN);
  k_tc_gemm<EPI, BN><<<dim3(rows / TBM, N / BN), 192, smem, st>>>(ta, tb, g);
  DPB_CUDA(cudaGetLastError());
}

template <int EPI>
void run_tc_epi(const float* A2, const float* B2, int rows, int N, const TArgs& g, cudaStream_t st) {
  if (N % 240 == 0 && N <= 240) launch_tc<EPI, 240>(A2, B2, rows, N, g, st);
  else if (N % 256 == 0) launch_tc<EPI, 256>(A2, B2, rows, N, g, st);
  else if (N % 160 == 0 && N <= 160) launch_tc<EPI, 160>(A2, B2, rows, N, g, st);
  else if (N % 128 == 0) launch_tc<EPI, 128>(A2, B2, rows, N, g, st);
  else if (N % 80 == 0) launch_tc<EPI, 80>(A2, B2, rows, N, g, st);
  else if (N % 64 == 0) launch_tc<EPI, 64>(A2, B2, rows, N, g, st);
  else throw InputErr("unsupported fitting width for the tensor-core path");
}

// Forward layer with FP64 K accumulation (k_tc_fwd64), column tiles of 80 / 64 / 128.
void run_tc_fwd64(const float* A2, const float* B2, int rows, int N, const TArgs& g, cudaStream_t st) {
  if (N % 80 == 0) launch_tc_fwd64<80>(A2, B2, rows, N, g, st);
  else if (N % 128 == 0) launch_tc_fwd64<128>(A2, B2, rows, N, g, st);
  else if (N % 64 == 0) launch_tc_fwd64<64>(A2, B2, rows, N, g, st);
  else throw InputErr("unsupported fitting width for the tensor-core path");
}

void run_tc(int epi, const float* A2, const float* B2, int rows, int N, const TArgs& g, cudaStream_t st) {
  if (epi != T_BWD) throw CudaErr("forward layers run on k_tc_fwd64");
  run_tc_epi<T_BWD>(A2, B2, rows, N, g, st);
}

} // namespace

namespace {
int seg32(int k) { return (k + 31) / 32 * 32; }

// host tf32 round-to-nearest-away (matches cvt.rna): add half a tf32 ulp and truncate
float rna_tf32(float v) {
  uint32_t b;
  std::memcpy(&b, &v, 4);
  b = (b + 0x1000u) & 0xFFFFE000u;
  float o;
  std::memcpy(&o, &b, 4);
  return o;
}

// rows x K (row-major FP64) -> rows x [hi(kseg) | lo(kseg)] FP32, zero padded
void split2(std::vector<float>& dst, const std::vector<double>& src, int rows, int K, int kseg) {
  dst.assign(static_cast<size_t>(rows) * 2 * kseg, 0.f);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < K; ++c) {
      const float x = static_cast<float>(src[static_cast<size_t>(r) * K + c]);
      const float hi = rna_tf32(x);
      float* d = dst.data() + static_cast<size_t>(r) * 2 * kseg;
      d[c] = hi;
      d[kseg + c] = rna_tf32(x - hi);
    }
}

void ensure_zeroed(DevBuf<float>& b, size_t count, cudaStream_t st) {
  if (count <= b.n) return;
  b.ensure(count);
  DPB_CUDA(cudaMemsetAsync(b.p, 0, b.n * sizeof(float), st));
}
} // namespace

void Engine::prepare_mixed() {
  if (!uniform_fit) throw InputErr("mixed precision needs the same fitting-net shape for every centre type");
  for (size_t k = 1; k < layers.size(); ++k)
    if (layers[k].outp != widthp_max || layers[k].inp != widthp_max)
      throw InputErr("mixed precision needs equal hidden widths");
  if (K0p % 32 != 0) throw InputErr("mixed precision needs a descriptor width that is a multiple of 32");
  // forward B = W^T rows [out][in] split along in; backward B = W rows [in][out] split along out
  const int L = static_cast<int>(layers.size());
  tc_wf.resize(n_types * L);
  tc_wb.resize(n_types * L);
  tc_bias.resize(n_types * L);
  tc_wout.resize(n_types);
  for (int t = 0; t < n_types; ++t)
    for (int k = 0; k < L; ++k) {
      const FitLayer& fl = layers[k];
      std::vector<double> w(static_cast<size_t>(fl.inp) * fl.outp), wt(w.size()), b(fl.outp);
      DPB_CUDA(cudaMemcpy(w.data(), fit_w[t * L + k].p, w.size() * 8, cudaMemcpyDeviceToHost));
      DPB_CUDA(cudaMemcpy(wt.data(), fit_wt[t * L + k].p, wt.size() * 8, cudaMemcpyDeviceToHost));
      DPB_CUDA(cudaMemcpy(b.data(), fit_b[t * L + k].p, b.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<float> f;
      split2(f, wt, fl.outp, fl.inp, seg32(fl.inp));
      tc_wf[t * L + k].ensure(f.size());
      DPB_CUDA(cudaMemcpy(tc_wf[t * L + k].p, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
      split2(f, w, fl.inp, fl.outp, seg32(fl.outp));
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

// Mixed-mode buffers. Pad columns of the split operands must stay zero: they are cleared once
// at allocation and never written (the epilogues write only the real N columns).
void Engine::ensure_mixed_buffers() {
  const int L = static_cast<int>(layers.size());
  const int wpm = widthp_max, s2 = seg32(wpm);
  const size_t ss = static_cast<size_t>(ck_sets) * ck_cap_s; // rows of the chunk buffer sets
  ensure_zeroed(tc_d2, ss * 2 * K0p, stream);
  ensure_zeroed(tc_y2a, ss * 2 * s2, stream);
  ensure_zeroed(tc_y2b, ss * 2 * s2, stream);
  ensure_zeroed(tc_dz2a, ss * 2 * s2, stream);
  ensure_zeroed(tc_dz2b, ss * 2 * s2, stream);
  tc_t.resize(L);
  for (int k = 0; k < L; ++k) tc_t[k].ensure(ss * wpm);
  tc_dya.ensure(ss * wpm);
  tc_dyb.ensure(ss * wpm);
}

void Engine::fitting_type_rows_mixed(int t, int64_t r0_, int64_t rows_, cudaStream_t st) {
  const int L = static_cast<int>(layers.size());
  const int wpm = widthp_max, s2 = seg32(wpm);
  const int rows = static_cast<int>(rows_);
  const size_t r0 = static_cast<size_t>(r0_);
  // forward: layer 0 reads the split D (written by the tabulate kernel), layer k > 0 the split
  // y_{k-1} (ping-pong), which is also the shortcut source
  const float* A2 = ws(tc_d2, 2 * K0p) + r0 * 2 * K0p; // chunk windows (engine.hpp)
  const float* yprev = nullptr;
  for (int k = 0; k < L; ++k) {
    const FitLayer& fl = layers[k];
    TArgs g{};
    g.kseg = k == 0 ? K0p : s2;
    g.bias = tc_bias[t * L + k].p;
    g.xin2 = fl.shortcut ? yprev : nullptr;
    g.ldx = s2;
    g.tout = ws(tc_t[k], wpm) + r0 * wpm;
    g.ldc = wpm;
    float* y2 = ws(k & 1 ? tc_y2b : tc_y2a, 2 * s2) + r0 * 2 * s2;
    g.y2 = y2;
    g.ld2 = s2;
    g.tanh_c = tc_tanh.p;
    // FP64 K accumulation (k_tc_fwd64) for the forward layers: the energy path
    run_tc_fwd64(A2, tc_wf[t * L + k].p, rows, fl.outp, g, st);
    ++launches;
    yprev = y2;
    A2 = y2;
  }
  // readout
  const FitLayer& last = layers[L - 1];
  float* dzc = ws(tc_dz2a, 2 * s2) + r0 * 2 * s2;
  float* dzn = ws(tc_dz2b, 2 * s2) + r0 * 2 * s2;
  float* dyc = ws(tc_dya, wpm) + r0 * wpm;
  float* dyn = ws(tc_dyb, wpm) + r0 * wpm;
  k_readout_tc<<<ceil_div(rows, 4), 128, 0, st>>>(rows, wpm, s2, last.out, yprev, ws(tc_t[L - 1], wpm) + r0 * wpm,
                                                      tc_wout[t].p, b_out[t], e_slot.p + r0, dzc);
  ++launches;
  const float* dy_mat = nullptr;     // dy of the layer above (matrix), null at the top
  const float* dy_vec = tc_wout[t].p; // dy_L = w_out for every row
  for (int k = L - 1; k >= 0; --k) {
    const FitLayer& fl = layers[k];
    TArgs g{};
    g.kseg = s2;
    g.ldc = wpm;
    g.ld2 = s2;
    if (fl.shortcut) {
      g.dyin = dy_mat;
      g.dyvec = dy_mat ? nullptr : dy_vec;
    }
    if (k > 0) {
      g.tprev = ws(tc_t[k - 1], wpm) + r0 * wpm;
      g.dyout = dyn;
      g.dz2 = dzn;
    } else {
      g.dD = ws(dD, K0p) + r0 * K0p;
      g.ldD = K0p;
    }
    run_tc(T_BWD, dzc, tc_wb[t * L + k].p, rows, fl.inp, g, st);
    ++launches;
    std::swap(dzc, dzn);
    std::swap(dyc, dyn);
    dy_mat = dyc;
  }
}

void Engine::fitting_rows_mixed(int64_t r0, int64_t rows, cudaStream_t st) { fitting_type_rows_mixed(0, r0, rows, st); }

void Engine::launch_fitting_mixed() {
  for (int t = 0; t < n_types; ++t)
    if (seg_rows[t] > 0) fitting_type_rows_mixed(t, seg_start[t], seg_rows[t], stream);
  finish_energy();
}

} // namespace dpb
