// Complex helpers for the sm_100a kernels.  A complex64 value is one 64-bit register pair, so ptxas
// can issue real×complex and complex+complex on the packed FP32x2 pipe (FFMA2/FADD2/FMUL2).
#pragma once
#include <cuda_runtime.h>

namespace hz {

template <typename R> struct Cx;
template <> struct Cx<float> { typedef float2 T; };
template <> struct Cx<double> { typedef double2 T; };

__device__ __forceinline__ unsigned long long f2_as_u64(float2 a) {
  return *reinterpret_cast<unsigned long long*>(&a);
}
__device__ __forceinline__ float2 u64_as_f2(unsigned long long a) {
  return *reinterpret_cast<float2*>(&a);
}

// ---- float2 (complex64) ---------------------------------------------------------------------
// Packed FP32x2 (FFMA2): every op is an fma.rn.f32x2 (a+b = 1·a+b, s·a = s·a+0), so no compiler
// mul/add contraction choice can make two unrolled copies round differently.
__device__ __forceinline__ float2 pk_fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_as_u64(a)), "l"(f2_as_u64(b)), "l"(f2_as_u64(c)));
  return u64_as_f2(d);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return pk_fma(make_float2(1.f, 1.f), a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return pk_fma(make_float2(-1.f, -1.f), b, a); }
__device__ __forceinline__ float2 cscale(float s, float2 a) { return pk_fma(make_float2(s, s), a, make_float2(0.f, 0.f)); }
__device__ __forceinline__ float2 cfma(float s, float2 a, float2 acc) { return pk_fma(make_float2(s, s), a, acc); }
// complex * complex (slow paths only)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 czero(float) { return make_float2(0.f, 0.f); }

// ---- double2 (complex128) -------------------------------------------------------------------
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cfma(double s, double2 a, double2 acc) {
  return make_double2(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 czero(double) { return make_double2(0.0, 0.0); }

// ---- loads ------------------------------------------------------------------------------------
__device__ __forceinline__ float2 ldg_c(const float2* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg_c(const double2* p) { return __ldg(p); }

__device__ __forceinline__ float2 shfl_up_c(float2 a, int d) {
  return u64_as_f2(__shfl_up_sync(0xffffffffu, f2_as_u64(a), d));
}
__device__ __forceinline__ float2 shfl_down_c(float2 a, int d) {
  return u64_as_f2(__shfl_down_sync(0xffffffffu, f2_as_u64(a), d));
}
__device__ __forceinline__ double2 shfl_up_c(double2 a, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, a.x, d), __shfl_up_sync(0xffffffffu, a.y, d));
}
__device__ __forceinline__ double2 shfl_down_c(double2 a, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, a.x, d), __shfl_down_sync(0xffffffffu, a.y, d));
}

__device__ __forceinline__ float2 make_cx(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 make_cx(double a, double b) { return make_double2(a, b); }
// 1/√w for G = v/(f h): one MUFU.RSQ (w = 1/v² is a normal positive number on valid rows)
__device__ __forceinline__ float rsqrt_r(float a) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}
__device__ __forceinline__ double rsqrt_r(double a) { return rsqrt(a); }

// ---- storage <-> compute conversion (mixed-precision residual: c64 storage, fp64 arithmetic) ----
__device__ __forceinline__ float2 to_cx(float2 a, float) { return a; }
__device__ __forceinline__ double2 to_cx(double2 a, double) { return a; }
__device__ __forceinline__ double2 to_cx(float2 a, double) { return make_double2((double)a.x, (double)a.y); }
__device__ __forceinline__ float2 from_cx(float2 a, float) { return a; }
__device__ __forceinline__ double2 from_cx(double2 a, double) { return a; }
__device__ __forceinline__ float2 from_cx(double2 a, float) { return make_float2((float)a.x, (float)a.y); }

}  // namespace hz
