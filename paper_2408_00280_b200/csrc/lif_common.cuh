// lif_common.cuh -- device-side building blocks of the fused LIF kernels (sm_100a).
//
// Shared by lif_forward.cuh and lif_backward.cuh only.  Nothing here is shared with
// oracle/ (the oracle is an independent fp64 C program).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace snn {

// ------------------------------------------------------------------------------------
// Per-launch constants (computed once on the host in fp32 -- SURVEY R9).
struct LifConsts {
    float k;        // 1 - 1/tau
    float s;        // dH/dX: 1/tau if decay_input else 1
    float c0;       // V_reset / tau: the constant of the charge
    float v_th;     // V_th
    float v_reset;  // V_reset
    float alpha;    // surrogate sharpness
    float atan_c;   // pi/2 * alpha (arctan surrogate)
    int   soft;     // soft reset
    int   detach;   // detach_reset
};

// ------------------------------------------------------------------------------------
// The per-step LIF arithmetic.  Written with explicit _rn intrinsics so the forward
// kernel and the RECOMPUTE backward (which re-runs the charge) execute the identical
// rounding sequence -> bitwise-identical H, S, V.

// Charge (Eq. 1 / north-star form): H = k V + (s X + c0).
__device__ __forceinline__ float lif_charge(const LifConsts& c, float V, float X) {
    return __fmaf_rn(c.k, V, __fmaf_rn(c.s, X, c.c0));
}
// Fire (Eq. 2): S = [H - V_th >= 0], evaluated as H >= V_th.  NaN -> 0.
__device__ __forceinline__ bool lif_fire(const LifConsts& c, float H) { return H >= c.v_th; }
// Reset: hard V = S ? V_reset : H (Eq. 1's (1-y), V_rest y);  soft V = H - V_th S.
__device__ __forceinline__ float lif_reset(const LifConsts& c, float H, bool S) {
    return S ? (c.soft ? __fsub_rn(H, c.v_th) : c.v_reset) : H;
}

// Surrogate derivative delta(u), u = H - V_th.
template <int SURR>
__device__ __forceinline__ float lif_surrogate(const LifConsts& c, float u);

// Sigmoid, in the |u| form: e = exp(-alpha|u|) in (0, 1].
template <>
__device__ __forceinline__ float lif_surrogate<0>(const LifConsts& c, float u) {
    const float e = expf(-c.alpha * fabsf(u));
    const float q = __fadd_rn(1.0f, e);
    return __fdiv_rn(__fmul_rn(c.alpha, e), __fmul_rn(q, q));
}
// Arctan: (alpha/2) / (1 + (pi/2 alpha u)^2).
template <>
__device__ __forceinline__ float lif_surrogate<1>(const LifConsts& c, float u) {
    const float z = __fmul_rn(c.atan_c, u);
    return __fdiv_rn(__fmul_rn(0.5f, c.alpha), __fmaf_rn(z, z, 1.0f));
}

// One reverse step of Eq. 3:
//   gH = gS delta + gV dV/dH,  dV/dH = hard: (1-S) + (V_reset - H) delta ; soft: 1 - V_th delta
// returns gH; caller writes gX = s gH and carries gV = k gH.
template <int SURR>
__device__ __forceinline__ float lif_grad_step(const LifConsts& c, float H, float gS, float gV) {
    const float u = __fsub_rn(H, c.v_th);
    const float d = lif_surrogate<SURR>(c, u);
    const bool S = lif_fire(c, H);
    float dVdH;
    if (c.soft) {
        dVdH = c.detach ? 1.0f : __fmaf_rn(-c.v_th, d, 1.0f);
    } else {
        const float base = S ? 0.0f : 1.0f;
        dVdH = c.detach ? base : __fmaf_rn(__fsub_rn(c.v_reset, H), d, base);
    }
    return __fmaf_rn(gS, d, __fmul_rn(gV, dVdH));
}

// ------------------------------------------------------------------------------------
// Vector I/O: VEC consecutive elements of type T as one (up to 128-bit) transaction.

template <typename T, int VEC>
struct alignas((sizeof(T) * VEC > 16) ? 16 : sizeof(T) * VEC) Pack {
    T v[VEC];
};

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

// Streaming loads: read once, never re-read by this kernel -> evict-first in L2 (.cs)
// and no L1 allocation.
template <typename T, int VEC>
__device__ __forceinline__ Pack<T, VEC> ld_stream(const T* p) {
    Pack<T, VEC> r;
    if constexpr (sizeof(Pack<T, VEC>) == 32) {
        int4 q[2];
        q[0] = __ldcs(reinterpret_cast<const int4*>(p));
        q[1] = __ldcs(reinterpret_cast<const int4*>(p) + 1);
        r = *reinterpret_cast<Pack<T, VEC>*>(q);
    } else if constexpr (sizeof(Pack<T, VEC>) == 16) {
        int4 q = __ldcs(reinterpret_cast<const int4*>(p));
        r = *reinterpret_cast<Pack<T, VEC>*>(&q);
    } else if constexpr (sizeof(Pack<T, VEC>) == 8) {
        int2 q = __ldcs(reinterpret_cast<const int2*>(p));
        r = *reinterpret_cast<Pack<T, VEC>*>(&q);
    } else if constexpr (sizeof(Pack<T, VEC>) == 4) {
        int q = __ldcs(reinterpret_cast<const int*>(p));
        r = *reinterpret_cast<Pack<T, VEC>*>(&q);
    } else {
        static_assert(sizeof(Pack<T, VEC>) == 2, "pack size");
        unsigned short q = __ldcs(reinterpret_cast<const unsigned short*>(p));
        r = *reinterpret_cast<Pack<T, VEC>*>(&q);
    }
    return r;
}

template <typename T, int VEC>
__device__ __forceinline__ void st_stream(T* p, const Pack<T, VEC>& r) {
    if constexpr (sizeof(Pack<T, VEC>) == 32) {
        const int4* q = reinterpret_cast<const int4*>(&r);
        __stcs(reinterpret_cast<int4*>(p), q[0]);
        __stcs(reinterpret_cast<int4*>(p) + 1, q[1]);
    } else if constexpr (sizeof(Pack<T, VEC>) == 16) {
        __stcs(reinterpret_cast<int4*>(p), *reinterpret_cast<const int4*>(&r));
    } else if constexpr (sizeof(Pack<T, VEC>) == 8) {
        __stcs(reinterpret_cast<int2*>(p), *reinterpret_cast<const int2*>(&r));
    } else if constexpr (sizeof(Pack<T, VEC>) == 4) {
        __stcs(reinterpret_cast<int*>(p), *reinterpret_cast<const int*>(&r));
    } else if constexpr (sizeof(Pack<T, VEC>) == 2) {
        __stcs(reinterpret_cast<unsigned short*>(p), *reinterpret_cast<const unsigned short*>(&r));
    } else {
        static_assert(sizeof(Pack<T, VEC>) == 1, "pack size");
        *reinterpret_cast<unsigned char*>(p) = *reinterpret_cast<const unsigned char*>(&r);
    }
}

// Load VEC elements at p (neuron n0 .. n0+VEC-1); `nvalid` < VEC only for the single
// ragged group at the end of the neuron range (scalar loads, zeros beyond N).
template <typename T, int VEC>
__device__ __forceinline__ Pack<T, VEC> ld_group(const T* p, int nvalid) {
    if (nvalid >= VEC) return ld_stream<T, VEC>(p);
    Pack<T, VEC> r;
#pragma unroll
    for (int i = 0; i < VEC; ++i) r.v[i] = (i < nvalid) ? p[i] : from_f32<T>(0.0f);
    return r;
}
template <typename T, int VEC>
__device__ __forceinline__ void st_group(T* p, const Pack<T, VEC>& r, int nvalid) {
    if (nvalid >= VEC) { st_stream<T, VEC>(p, r); return; }
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (i < nvalid) p[i] = r.v[i];
}

}  // namespace snn
