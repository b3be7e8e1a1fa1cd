// Shared device helpers for the Flash PD-SSM sm_100a kernels.
// Layout conventions are those of include/pdssm.h:
//   scan tensors [B][H][L][c][N] (N fastest, c = 1 real or 2 re/im planes),
//   sequence s = b*H + h, chunk c covers [c*tau, min((c+1)*tau, L)).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pdssm.h"

namespace pdssm {

// device error word (PDSSM_CHECK_FINITE): bit 0 = out-of-range index, bit 1 = NaN/Inf.
// Internal linkage: every translation unit of the library has its own word (the units are
// compiled separately, without relocatable device code); pdssm_check_device reads and
// clears all of them (api_internal.cuh, PDSSM_DEFINE_ERRWORD).
static __device__ uint32_t g_err_word = 0;

enum : uint32_t { ERRBIT_RANGE = 1u, ERRBIT_NONFINITE = 2u };

__device__ __forceinline__ void report(uint32_t bit) { atomicOr(&g_err_word, bit); }

// ---------------------------------------------------------------- act dtypes
template <typename T> struct Act;
template <> struct Act<float> {
    static __device__ __forceinline__ float ld(const float* p) { return __ldg(p); }
    static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <> struct Act<__nv_bfloat16> {
    static __device__ __forceinline__ float ld(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }
    static __device__ __forceinline__ void st(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

template <typename T> __device__ __forceinline__ float ldact(const T* p) { return Act<T>::ld(p); }
template <typename T> __device__ __forceinline__ void stact(T* p, float v) { Act<T>::st(p, v); }
// plain (generic-pointer) load, valid for shared memory
__device__ __forceinline__ float ldact_s(const float* p) { return *p; }
__device__ __forceinline__ float ldact_s(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// ---------------------------------------------------------------- complex (split planes)
struct cpx {
    float re, im;
};
__device__ __forceinline__ cpx cmul(cpx a, cpx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
// conj(a) * b
__device__ __forceinline__ cpx cmulc(cpx a, cpx b) { return {a.re * b.re + a.im * b.im, a.re * b.im - a.im * b.re}; }
__device__ __forceinline__ cpx cadd(cpx a, cpx b) { return {a.re + b.re, a.im + b.im}; }

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace pdssm
