// Device-side building blocks shared by the dp_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "host_common.hpp"

#define DPB_CUDA(x)                                                                        \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::dpb::CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));             \
  } while (0)

namespace dpb {

// Dynamic shared memory above 48 KB needs a per-function, per-device opt-in. Handles on several
// devices may live in one process (one per host thread), so the opt-in is recorded per
// (function, device, size) under a lock instead of a process-wide static flag.
void smem_optin_raw(const void* fn, size_t bytes);
template <class K>
inline void smem_optin(K* kern, size_t bytes) {
  smem_optin_raw(reinterpret_cast<const void*>(kern), bytes);
}

// Error codes raised by kernels into Workspace::err (first writer wins).
enum DevErr : int {
  DEV_OK = 0,
  DEV_OVERLAP = 1,     // r^2 < 1e-12 inside r_cut (env_mat.cpp:33)
  DEV_OVERFLOW = 2,    // more real neighbours of a type than max_nbr (env_mat.cpp:37-39)
  DEV_TABLE_LOW = 3,   // table input below x0 (table.cpp:21); cannot happen for s >= 0
  DEV_SHIFT_RANGE = 4, // image shift outside the packed key range
  DEV_ROW_CAP = 5,     // neighbour row longer than the sort capacity
  DEV_STALE = 6,       // list stale in MD (md.cpp:211-217)
  DEV_PBUF = 7,        // tabulate group buffer too small (grows at the next list rebuild)
  DEV_TABLE_VERIFY = 8, // GPU-built table does not reproduce the net at a node (table.cpp:133-147)
  DEV_LIST_CAP = 9,    // a row's entries exceed the chunk's entry capacity (sized from the list)
  DEV_ASYMMETRIC = 10, // list entry (i -> j, s) without its reverse (j -> i, -s)
  DEV_GCAP = 11,       // more real pairs than the compact pair-gradient buffer holds
};

// Cell as the kernels see it (geom.hpp:14-44).
struct DevCell {
  double h[9];
  double hinv[9];
  double vol;
  int per[3];
};

// Neighbour key: [type:6][j:28][s0+512:10][s1+512:10][s2+512:10]. Sorting keys ascending gives
// the stable type partition of the canonical (j, shift) order (env_mat.cpp:25, neighbor.cpp:10-17).
constexpr int KEY_SHIFT_BIAS = 512;
__host__ __device__ inline uint64_t make_key(int type, int j, int s0, int s1, int s2) {
  return (static_cast<uint64_t>(type) << 58) | (static_cast<uint64_t>(j) << 30) |
         (static_cast<uint64_t>(s0 + KEY_SHIFT_BIAS) << 20) |
         (static_cast<uint64_t>(s1 + KEY_SHIFT_BIAS) << 10) |
         static_cast<uint64_t>(s2 + KEY_SHIFT_BIAS);
}
__host__ __device__ inline int key_type(uint64_t k) { return static_cast<int>(k >> 58); }
__host__ __device__ inline int key_j(uint64_t k) {
  return static_cast<int>((k >> 30) & ((1u << 28) - 1));
}
__host__ __device__ inline void key_shift(uint64_t k, int* s) {
  s[0] = static_cast<int>((k >> 20) & 1023) - KEY_SHIFT_BIAS;
  s[1] = static_cast<int>((k >> 10) & 1023) - KEY_SHIFT_BIAS;
  s[2] = static_cast<int>(k & 1023) - KEY_SHIFT_BIAS;
}
// Key of the reverse entry (j -> i, -s) as seen in row j.
__host__ __device__ inline uint64_t with_key_j(uint64_t k, int j) {
  return (k & ~(static_cast<uint64_t>((1u << 28) - 1) << 30)) | (static_cast<uint64_t>(j) << 30);
}
__host__ __device__ inline uint64_t reverse_key(uint64_t k, int type_i, int i) {
  int s[3];
  key_shift(k, s);
  return make_key(type_i, i, -s[0], -s[1], -s[2]);
}

#ifdef __CUDACC__
// d = (r_j + s0 h0 + s1 h1 + s2 h2) - r_i evaluated exactly as the reference does: left to
// right, every product and sum rounded separately, no fused multiply-add (geom.hpp:61-69).
__device__ __forceinline__ void disp_exact(const DevCell& c, double3 ri, double3 rj, int s0,
                                           int s1, int s2, double* d) {
  const double rjv[3] = {rj.x, rj.y, rj.z};
  const double riv[3] = {ri.x, ri.y, ri.z};
#pragma unroll
  for (int x = 0; x < 3; ++x) {
    double img = __dadd_rn(rjv[x], __dmul_rn(static_cast<double>(s0), c.h[x]));
    img = __dadd_rn(img, __dmul_rn(static_cast<double>(s1), c.h[3 + x]));
    img = __dadd_rn(img, __dmul_rn(static_cast<double>(s2), c.h[6 + x]));
    d[x] = __dsub_rn(img, riv[x]);
  }
}

__device__ __forceinline__ double norm2_exact(const double* d) {
  return __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
}

// 32-byte vector accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256): one instruction per lane
// instead of two 16-byte ones; the address must be 32-byte aligned.
__device__ __forceinline__ double4 ldg4(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double4 ldc4(const double* p) { // coherent (data written earlier by this kernel)
  double4 v;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__device__ __forceinline__ double3 ld_pos(const double4* p, int j) {
  const double4 v = ldg4(reinterpret_cast<const double*>(p + j));
  return make_double3(v.x, v.y, v.z);
}

__device__ __forceinline__ void raise_err(int* err, int code) { atomicCAS(err, 0, code); }

// FP64 tanh without the branchy library path: t = (1 - e) / (1 + e), e = exp(-2|x|) in (0, 1],
// sign restored. Absolute error <= ~2.5e-16 everywhere (the value is only ever used next to O(1)
// terms: y = x + t, 1 - t^2), which keeps the FP64 path far inside its 1e-10 parity bar against
// glibc's tanh; ~2x fewer instructions and no divergence between the |x| regimes.
__device__ __forceinline__ double tanh_fp64(double x) {
  const double e = exp(-2.0 * fabs(x));
  return copysign(__ddiv_rn(1.0 - e, 1.0 + e), x);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
#endif // __CUDACC__

} // namespace dpb
