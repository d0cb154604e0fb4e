// FP64 pipe microbenchmark for B200 (sm_100a): DFMA (SIMT) and DMMA (mma.sync f64)
// throughput, used to set the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { acc[k][0] = 0; acc[k][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma1684_kernel(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) acc[k][q] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) s += acc[k][q];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) acc[k][q] = 0;
  double a[8], b[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + threadIdx.x * 1e-4 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]), "+d"(acc[k][2]), "+d"(acc[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) for (int q = 0; q < 4; ++q) s += acc[k][q];
  if (s == 12345.678) out[0] = s;
}

template <class K>
float time_it(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  double* out; CK(cudaMalloc(&out, 8));
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    int iters = 20000;
    float ms = time_it([&] { dfma_kernel<<<blocks, tpb>>>(out, iters, 0.999, 1e-3); });
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("DFMA  tpb %4d: %.3f ms  %.2f TFLOP/s\n", tpb, ms, flops / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * 4;
    int iters = 20000;
    float ms = time_it([&] { dmma884_kernel<<<blocks, tpb>>>(out, iters); });
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (tpb / 32);
    printf("DMMA m8n8k4   tpb %4d: %.3f ms  %.2f TFLOP/s\n", tpb, ms, flops / ms / 1e9);
    ms = time_it([&] { dmma1684_kernel<<<blocks, tpb>>>(out, iters); });
    flops = 2.0 * 16 * 8 * 4 * 4 * (double)iters * blocks * (tpb / 32);
    printf("DMMA m16n8k4  tpb %4d: %.3f ms  %.2f TFLOP/s\n", tpb, ms, flops / ms / 1e9);
    ms = time_it([&] { dmma16816_kernel<<<blocks, tpb>>>(out, iters / 4); });
    flops = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * blocks * (tpb / 32);
    printf("DMMA m16n8k16 tpb %4d: %.3f ms  %.2f TFLOP/s\n", tpb, ms, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
