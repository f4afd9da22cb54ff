// Complex element helpers shared by the matvec and FFT kernels.
#pragma once

#include <cuda_runtime.h>

namespace aim {

// Complex element types: double2 (complex128 plans) and float2 (complex64
// plans, reading D16); Real<C> is the component type.
template <class C>
struct CxTraits;
template <>
struct CxTraits<double2> { using R = double; };
template <>
struct CxTraits<float2> { using R = float; };
template <class C>
using Real = typename CxTraits<C>::R;

template <class C>
__device__ __forceinline__ C mkc(Real<C> x, Real<C> y) {
    C v;
    v.x = x;
    v.y = y;
    return v;
}
template <class C>
__device__ __forceinline__ C cvt(double2 v) { return mkc<C>((Real<C>)v.x, (Real<C>)v.y); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
__device__ __forceinline__ float2 shfl_xor2(float2 v, int m) {
    return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
template <class C>
__device__ __forceinline__ C shfl_c(C v, int src) {
    return mkc<C>(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

}  // namespace aim
