// Warp-specialized tcgen05 GEMM with TMA + mbarrier pipeline: C[M x N] = A[M x K] . B[N x K]^T.
// Byte-generic: KIND 0 = tf32 (4-byte elements), KIND 1 = s8 (1-byte, int32 accumulate).
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc_common.cuh"
using namespace dpb::tc;

#ifndef STAGES
#define STAGES 4
#endif
#ifndef MINB
#define MINB 1
#endif
constexpr int BM = 128, BN = 240, BKB = 128, ST = STAGES; // BKB: K bytes per stage = one 128B swizzle atom
constexpr int A_ST = BM * BKB, B_ST = BN * BKB;

template <int KIND>
__global__ void __launch_bounds__(192, MINB) k_gemm2(const __grid_constant__ CUtensorMap ta,
                                                 const __grid_constant__ CUtensorMap tb, void* C, int M, int N,
                                                 int Kbytes) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;
  unsigned char* sb = smem + ST * A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + ST * B_ST);
  uint64_t* empty = full + ST;
  uint64_t* accf = empty + ST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM;
  const int KT = Kbytes / BKB;
  if (warp == 0) {
    tmem_alloc<256>(tslot);
    if (lane == 0) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tb);
    }
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < ST; ++s) {
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
    // producer
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % ST;
      if (kt >= ST) mbar_wait(empty + s, ((kt / ST) - 1) & 1);
      mbar_expect_tx(full + s, A_ST + B_ST);
      tma_load_2d(sa + s * A_ST, &ta, kt * BKB, m0, full + s);
      tma_load_2d(sb + s * B_ST, &tb, kt * BKB, 0, full + s);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = KIND == 0 ? make_idesc(BM, BN, 2, 1) : make_idesc(BM, BN, 1, 2);
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % ST;
      mbar_wait(full + s, (kt / ST) & 1);
      fence_after();
      const uint32_t a0 = smem_u32(sa + s * A_ST), b0 = smem_u32(sb + s * B_ST);
#pragma unroll
      for (int k = 0; k < BKB / 32; ++k) {
        const uint64_t ad = make_desc_sw128(a0 + k * 32);
        const uint64_t bd = make_desc_sw128(b0 + k * 32);
        if (KIND == 0) mma_tf32(tmem, ad, bd, idesc, (kt | k) ? 1u : 0u);
        else mma_i8(tmem, ad, bd, idesc, (kt | k) ? 1u : 0u);
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
      tmem_ld16(tmem + ((q * 32) << 16) + c0, v);
      tmem_wait_ld();
      if (KIND == 0)
        for (int j = 0; j < 16; ++j) reinterpret_cast<float*>(C)[(size_t)row * N + c0 + j] = __uint_as_float(v[j]);
      else
        for (int j = 0; j < 16; ++j) reinterpret_cast<int*>(C)[(size_t)row * N + c0 + j] = (int)v[j];
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_map(EncodeFn enc, void* ptr, uint64_t rows, uint64_t row_bytes, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {128, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

int main() {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t smem = ST * (A_ST + B_ST) + 8 * (2 * ST + 1) + 16;
  for (int kind = 0; kind < 2; ++kind) {
    const int esz = kind == 0 ? 4 : 1;
    const int M = 1024, N = 240, K = 2048, Kb = K * esz;
    std::vector<float> A((size_t)M * K), B((size_t)N * K);
    std::vector<int8_t> A8((size_t)M * K), B8((size_t)N * K);
    srand(1);
    for (size_t i = 0; i < A.size(); ++i) { A[i] = rand() / (float)RAND_MAX - 0.5f; A8[i] = (int8_t)(rand() % 255 - 127); }
    for (size_t i = 0; i < B.size(); ++i) { B[i] = rand() / (float)RAND_MAX - 0.5f; B8[i] = (int8_t)(rand() % 255 - 127); }
    void *dA, *dB, *dC;
    cudaMalloc(&dA, (size_t)M * Kb); cudaMalloc(&dB, (size_t)N * Kb); cudaMalloc(&dC, (size_t)M * N * 4);
    cudaMemcpy(dA, kind == 0 ? (void*)A.data() : (void*)A8.data(), (size_t)M * Kb, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, kind == 0 ? (void*)B.data() : (void*)B8.data(), (size_t)N * Kb, cudaMemcpyHostToDevice);
    CUtensorMap ta = make_map(enc, dA, M, Kb, BM), tb = make_map(enc, dB, N, Kb, BN);
    auto kern = kind == 0 ? k_gemm2<0> : k_gemm2<1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<M / BM, 192, smem>>>(ta, tb, dC, M, N, Kb);
    printf("kind %d launch: %s\n", kind, cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> C((size_t)M * N);
    std::vector<int> Ci((size_t)M * N);
    if (kind == 0) cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    else cudaMemcpy(Ci.data(), dC, Ci.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0; long bad = 0;
    for (int i = 0; i < M; i += 37)
      for (int j = 0; j < N; ++j) {
        double ref = 0; long refi = 0;
        for (int k = 0; k < K; ++k) {
          ref += (double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
          refi += (long)A8[(size_t)i * K + k] * B8[(size_t)j * K + k];
        }
        if (kind == 0) { maxerr = std::max(maxerr, std::fabs(ref - C[(size_t)i * N + j])); maxref = std::max(maxref, std::fabs(ref)); }
        else bad += (refi != Ci[(size_t)i * N + j]);
      }
    if (kind == 0) printf("tf32 max abs err %.3e rel %.3e\n", maxerr, maxerr / maxref);
    else printf("i8 mismatches %ld\n", bad);
    // timing on a big M
    const int Mb = 128 * 148 * 8;
    void* dA2; cudaMalloc(&dA2, (size_t)Mb * Kb); cudaMemset(dA2, 0, (size_t)Mb * Kb);
    void* dC2; cudaMalloc(&dC2, (size_t)Mb * N * 4);
    CUtensorMap ta2 = make_map(enc, dA2, Mb, Kb, BM);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<Mb / BM, 192, smem>>>(ta2, tb, dC2, Mb, N, Kb);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<Mb / BM, 192, smem>>>(ta2, tb, dC2, Mb, N, Kb);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("kind %d M=%d N=%d K=%d: %.3f ms/iter, %.1f T(FL)OP/s\n", kind, Mb, N, K, ms / 5, 2.0 * Mb * N * K / (ms / 5) / 1e9);
    printf("final: %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dA2); cudaFree(dC2);
  }
  return 0;
}
