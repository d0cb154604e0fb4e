// Standalone check of the tcgen05 kind::tf32 GEMM building blocks: C[M x N] = A[M x K] . B[N x K]^T
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc_common.cuh"
using namespace dpb::tc;

constexpr int BM = 128, BN = 240, BK = 32, STAGES = 3; // BK in tf32 elements (128 B per row)
constexpr int ACH = BK * 4 / 16;                        // 16-byte chunks per row per stage (8)
constexpr uint32_t A_STAGE = BM * BK * 4, B_STAGE = BN * BK * 4;

__global__ void __launch_bounds__(128, 1) k_tf32(const float* A, const float* B, float* C, int M, int N, int K) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* sa = smem;
  unsigned char* sb = smem + STAGES * A_STAGE;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sb + STAGES * B_STAGE);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + STAGES + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM;
  if (warp == 0) tmem_alloc<256>(tslot);
  if (tid == 0) {
    for (int s = 0; s <= STAGES; ++s) mbar_init(mbar + s, 1);
    fence_barrier_init();
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const int KT = K / BK;
  auto load = [&](int stage, int kt) {
    const int k0 = kt * BK;
    unsigned char* a = sa + stage * A_STAGE;
    unsigned char* b = sb + stage * B_STAGE;
    for (int idx = tid; idx < BM * ACH; idx += 128) {
      const int r = idx / ACH, c = idx % ACH;
      cp_async16(a + kmaj_off(r, c, BM), A + (size_t)(m0 + r) * K + k0 + c * 4);
    }
    for (int idx = tid; idx < BN * ACH; idx += 128) {
      const int r = idx / ACH, c = idx % ACH;
      cp_async16(b + kmaj_off(r, c, BN), B + (size_t)r * K + k0 + c * 4);
    }
  };
  const uint32_t idesc = make_idesc(BM, BN, 2, 1);
  uint32_t phase[STAGES] = {0, 0, 0};
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      const int st = nk % STAGES;
      if (nk >= STAGES) { mbar_wait(mbar + st, phase[st]); phase[st] ^= 1; }
      load(st, nk);
    }
    cp_commit();
    cp_wait<STAGES - 1>();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const int st = kt % STAGES;
      const uint32_t a0 = smem_u32(sa + st * A_STAGE), b0 = smem_u32(sb + st * B_STAGE);
#pragma unroll
      for (int k = 0; k < BK / 8; ++k) {  // UMMA K = 8 tf32 = 2 chunks
        const uint64_t ad = make_desc(a0 + k * 2 * (BM / 8) * 128, (BM / 8) * 128, 128);
        const uint64_t bd = make_desc(b0 + k * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
        mma_tf32(tmem, ad, bd, idesc, (kt | k) ? 1u : 0u);
      }
      commit(mbar + st);
    }
  }
  if (tid == 0) commit(mbar + STAGES);
  mbar_wait(mbar + STAGES, 0);
  fence_after();
  const int row = m0 + warp * 32 + lane;
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c0, v);
    tmem_wait_ld();
    for (int j = 0; j < 16 && c0 + j < N; ++j) C[(size_t)row * N + c0 + j] = __uint_as_float(v[j]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

int main() {
  const int M = 1024, N = 240, K = 2048;
  std::vector<float> A((size_t)M * K), B((size_t)N * K), C((size_t)M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f);
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f);
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, C.size() * 4);
  const size_t smem = STAGES * (A_STAGE + B_STAGE) + 8 * (STAGES + 1) + 16;
  cudaFuncSetAttribute(k_tf32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tf32<<<M / BM, 128, smem>>>(dA, dB, dC, M, N, K);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; i += 37)
    for (int j = 0; j < N; ++j) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
      maxerr = std::max(maxerr, std::fabs(ref - C[(size_t)i * N + j]));
      maxref = std::max(maxref, std::fabs(ref));
    }
  printf("max abs err %.3e (max |ref| %.3e) rel %.3e\n", maxerr, maxref, maxerr / maxref);
  // timing
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int Mb = 128 * 148 * 8;
  float *dA2; cudaMalloc(&dA2, (size_t)Mb * K * 4); cudaMemset(dA2, 0, (size_t)Mb * K * 4);
  float *dC2; cudaMalloc(&dC2, (size_t)Mb * N * 4);
  k_tf32<<<Mb / BM, 128, smem>>>(dA2, dB, dC2, Mb, N, K);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_tf32<<<Mb / BM, 128, smem>>>(dA2, dB, dC2, Mb, N, K);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("M=%d N=%d K=%d: %.3f ms/iter, %.1f TFLOP/s (tf32)\n", Mb, N, K, ms / 5, 2.0 * Mb * N * K / (ms / 5) / 1e9);
  printf("final: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
