// Do DFMA (SIMT) and DMMA (tensor) share the FP64 pipe on B200? Half the warps of every block
// run DFMA chains, the other half DMMA; compare against each alone.
#include <cstdio>
#include <cuda_runtime.h>
__device__ void dfma_part(double* out, int iters) {
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999, 1e-3);
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}
__device__ void dmma_part(double* out, int iters) {
  double acc[8][2];
  for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
  double s = 0; for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_mix(double* out, int it_f, int it_m, int mode) {
  const int w = threadIdx.x >> 5;
  if (mode == 0) dfma_part(out, it_f);
  else if (mode == 1) dmma_part(out, it_m);
  else { if (w & 1) dmma_part(out, it_m); else dfma_part(out, it_f); }
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, tpb = 256, itf = 20000, itm = 10000;
  for (int mode = 0; mode < 3; ++mode) {
    k_mix<<<blocks, tpb>>>(out, itf, itm, mode);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_mix<<<blocks, tpb>>>(out, itf, itm, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = blocks * (tpb / 32.0);
    double ff = 2.0 * 8 * itf * 32 * (mode == 2 ? warps / 2 : (mode == 0 ? warps : 0));
    double fm = 2.0 * 256 * 8 * (double)itm * (mode == 2 ? warps / 2 : (mode == 1 ? warps : 0));
    printf("mode %d (%s): %.3f ms  DFMA %.2f TF  DMMA %.2f TF  total %.2f TF\n", mode,
           mode == 0 ? "dfma" : mode == 1 ? "dmma" : "half/half", ms, ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9);
  }
  return 0;
}
