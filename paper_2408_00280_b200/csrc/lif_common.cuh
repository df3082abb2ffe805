// lif_common.cuh -- device-side building blocks of the fused LIF kernels (sm_100a):
// the per-step LIF arithmetic (one definition used by every kernel, so all paths round
// identically) and vector I/O helpers.  Nothing here is shared with oracle/ (the oracle is
// an independent fp64 C program).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace snn {

// ------------------------------------------------------------------------------------
// Per-launch constants, computed once on the host in fp32.
struct LifConsts {
    float k;          // 1 - 1/tau
    float s;          // dH/dX: 1/tau if decay_input else 1
    float c0;         // V_reset / tau: the constant of the charge
    float v_th;       // V_th
    float v_reset;    // V_reset
    float alpha;      // surrogate sharpness
    float ex2_scale;  // -alpha * log2(e): e^{-alpha|u|} = 2^{|u| ex2_scale}
    float atan_c;     // pi/2 * alpha (arctan surrogate)
    float half_alpha; // alpha / 2   (arctan surrogate numerator)
};

// Keep the constants in registers: without this ptxas re-reads them from the constant
// bank (LDC) inside the unrolled time loop, several instructions per neuron-step.
__device__ __forceinline__ void pin(LifConsts& c) {
    asm volatile("" : "+f"(c.k), "+f"(c.s), "+f"(c.c0), "+f"(c.v_th), "+f"(c.v_reset));
    asm volatile("" : "+f"(c.alpha), "+f"(c.ex2_scale), "+f"(c.atan_c), "+f"(c.half_alpha));
}

// Compile-time variant of the backward: bit 0 surrogate (0 sigmoid, 1 arctan), bit 1 soft
// reset, bit 2 detach_reset, bit 3 affine prologue, bit 4 residual prologue.  Branch-free inner loops.
template <int MODE>
struct Mode {
    static constexpr int SURR = MODE & 1;
    static constexpr bool SOFT = (MODE & 2) != 0;
    static constexpr bool DETACH = (MODE & 4) != 0;
    static constexpr bool AFF = (MODE & 8) != 0;   // affine prologue gradients (RECOMPUTE only)
    static constexpr bool RES = (MODE & 16) != 0;  // + residual add (implies AFF; TMA path only)
    // Paper-mode constants (decay_input = 0, V_reset = 0: s = 1, c0 = 0): the charge is
    // fma(k, V, X) and gX = gH -- the same values up to the sign of a zero (fma(1, -0, +0) is
    // +0), two fewer paired ops per backward step.  TMA RECOMPUTE backward (plain / affine /
    // residual).
    static constexpr bool P0 = (MODE & 32) != 0;
};

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2, ftz
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {  // MUFU.RCP, ftz
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------------------------------------
// The per-step LIF arithmetic (explicit _rn intrinsics: no compiler contraction choices,
// so the forward kernel and the RECOMPUTE backward, which re-runs the charge, produce
// bitwise-identical H, S, V -- DESIGN.md "Determinism").

// Charge (Eq. 1 / north-star form): H = k V + (s X + c0).
__device__ __forceinline__ float lif_charge(const LifConsts& c, float V, float X) {
    return __fmaf_rn(c.k, V, __fmaf_rn(c.s, X, c.c0));
}
// Fire (Eq. 2): S = [H - V_th >= 0], evaluated as H >= V_th.
// NaN H -> no spike.
__device__ __forceinline__ bool lif_fire(const LifConsts& c, float H) { return H >= c.v_th; }
// Reset: hard V = S ? V_reset : H (Eq. 1's (1 - y) and V_rest y terms);
// soft V = H - V_th S (BASELINE.json north_star).
template <bool SOFT>
__device__ __forceinline__ float lif_reset(const LifConsts& c, float H, bool S) {
    if constexpr (SOFT) return S ? __fsub_rn(H, c.v_th) : H;
    else return S ? c.v_reset : H;
}

// Surrogate derivative delta(u), u = H - V_th.
// Sigmoid in the |u| form: e = 2^{|u| ex2_scale} =
// e^{-alpha|u|} in [0, 1], so (1+e)^2 is in [1, 4] and the MUFU approximations are safe
// (ex2.approx / rcp.approx, ~2 ulp; e flushes to 0 only where delta < 1e-38).
// Arctan: (alpha/2) / (1 + (pi/2 alpha u)^2), denominator >= 1.
// Relative error ~1e-6, inside the parity bound (tests/parity.py).
template <int SURR>
__device__ __forceinline__ float lif_surrogate(const LifConsts& c, float u) {
    if constexpr (SURR == 0) {
        const float e = ex2_approx(__fmul_rn(fabsf(u), c.ex2_scale));
        const float q = __fadd_rn(1.0f, e);
        return __fmul_rn(__fmul_rn(c.alpha, e), rcp_approx(__fmul_rn(q, q)));
    } else {
        const float z = __fmul_rn(c.atan_c, u);
        return __fmul_rn(c.half_alpha, rcp_approx(__fmaf_rn(z, z, 1.0f)));
    }
}

// One reverse step of Eq. 3:
//   gH = gS delta + gV dV/dH,
//   dV/dH = hard: (1 - S) + (V_reset - H) delta ; soft: 1 - V_th delta (delta term dropped
//   when detach_reset).  Returns gH; the caller writes gX = s gH, gV <- k gH.
template <int MODE>
__device__ __forceinline__ float lif_grad_step(const LifConsts& c, float H, float gS, float gV) {
    using M = Mode<MODE>;
    const float u = __fsub_rn(H, c.v_th);
    const float d = lif_surrogate<M::SURR>(c, u);
    float dVdH;
    if constexpr (M::SOFT) {
        dVdH = M::DETACH ? 1.0f : __fmaf_rn(-c.v_th, d, 1.0f);
    } else {
        const float base = lif_fire(c, H) ? 0.0f : 1.0f;
        dVdH = M::DETACH ? base : __fmaf_rn(__fsub_rn(c.v_reset, H), d, base);
    }
    return __fmaf_rn(gS, d, __fmul_rn(gV, dVdH));
}

// ------------------------------------------------------------------------------------
// Paired fp32 arithmetic (sm_100 FFMA2 / FMUL2 / FADD2: two IEEE fp32 operations per
// instruction).  Each lane of a pair is rounded exactly like the scalar _rn intrinsic, so
// the paired and scalar paths are bitwise identical; pairs halve the FMA-pipe instruction
// count of the backward, which otherwise is issue-bound for bf16 io.
struct F2 {
    uint64_t v;
};
__device__ __forceinline__ F2 f2(float a, float b) {
    F2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ F2 f2(float a) { return f2(a, a); }
__device__ __forceinline__ void split(F2 a, float& x, float& y) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
}
__device__ __forceinline__ float lo(F2 a) { float x, y; split(a, x, y); return x; }
__device__ __forceinline__ float hi(F2 a) { float x, y; split(a, x, y); return y; }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
    F2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
    F2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
    F2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}

// Charge for two neurons: H = k V + (s X + c0)   (same roundings as lif_charge); P0: s = 1, c0 = 0.
template <bool P0 = false>
__device__ __forceinline__ F2 lif_charge2(const LifConsts& c, F2 V, F2 X) {
    if constexpr (P0) return fma2(f2(c.k), V, X);
    return fma2(f2(c.k), V, fma2(f2(c.s), X, f2(c.c0)));
}

// Surrogate for two neurons (same roundings as lif_surrogate, lane by lane).
template <int SURR>
__device__ __forceinline__ F2 lif_surrogate2(const LifConsts& c, F2 u) {
    if constexpr (SURR == 0) {
        const F2 t = mul2(f2(fabsf(lo(u)), fabsf(hi(u))), f2(c.ex2_scale));
        const F2 e = f2(ex2_approx(lo(t)), ex2_approx(hi(t)));
        const F2 q = add2(f2(1.0f), e);
        const F2 q2 = mul2(q, q);
        return mul2(mul2(f2(c.alpha), e), f2(rcp_approx(lo(q2)), rcp_approx(hi(q2))));
    } else {
        const F2 z = mul2(f2(c.atan_c), u);
        const F2 d = fma2(z, z, f2(1.0f));
        return mul2(f2(c.half_alpha), f2(rcp_approx(lo(d)), rcp_approx(hi(d))));
    }
}

// One reverse step of Eq. 3 for two neurons (same roundings as lif_grad_step).
template <int MODE>
__device__ __forceinline__ F2 lif_grad_step2(const LifConsts& c, F2 H, F2 gS, F2 gV) {
    using M = Mode<MODE>;
    const F2 u = sub2(H, f2(c.v_th));
    const F2 d = lif_surrogate2<M::SURR>(c, u);
    F2 dVdH;
    if constexpr (M::SOFT) {
        dVdH = M::DETACH ? f2(1.0f) : fma2(f2(-c.v_th), d, f2(1.0f));
    } else {
        const F2 base = f2(lif_fire(c, lo(H)) ? 0.0f : 1.0f, lif_fire(c, hi(H)) ? 0.0f : 1.0f);
        dVdH = M::DETACH ? base : fma2(sub2(f2(c.v_reset), H), d, base);
    }
    return fma2(gS, d, mul2(gV, dVdH));
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

// Step a row pointer by `ldb` bytes (a 64-bit IADD3 + IADD3.X pair; the kernels walk
// their output rows this way instead of scaling an element index every row).
template <typename T>
__device__ __forceinline__ T* step_bytes(T* p, int64_t ldb) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + ldb);
}

// Elements i, i+1 (i even) of a pack widened to fp32 as one pair.  bf16 -> fp32 is exact
// (the bf16 bits are the high half of the fp32 word), so for a bf16x2 word w the pair is
// (w << 16, w & 0xffff0000): two integer ops, where the generic per-element conversion costs
// the compiler a PRMT and two shifts.
template <typename T, int VEC>
__device__ __forceinline__ F2 load2(const Pack<T, VEC>& p, int i) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(&p.v[i]);
        F2 r;
        asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\t"
            "mov.b64 %0, {lo, hi};\n\t}" : "=l"(r.v) : "r"(w));
        return r;
    } else {
        return f2(to_f32(p.v[i]), to_f32(p.v[i + 1]));
    }
}

// Streaming loads: read once, never re-read by this kernel -> evict-first in L2 (.cs).
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

// Streaming stores (.cs: evict-first; the outputs are consumed by a later kernel).
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

// Store VEC elements at p whose address may not be aligned to the pack (rows of an odd
// row stride or an unaligned view): the widest aligned form, else element by element.
// `nvalid` < VEC for the ragged group at the end of the neuron range.  The alignment test is
// uniform across a warp (its lanes' groups are consecutive whole packs of one row).
template <typename T, int VEC>
__device__ __forceinline__ void st_any(T* p, const Pack<T, VEC>& r, int nvalid) {
    if (nvalid >= VEC && (reinterpret_cast<uintptr_t>(p) % sizeof(Pack<T, VEC>)) == 0) {
        st_stream<T, VEC>(p, r);
        return;
    }
    if constexpr (VEC % 2 == 0 && sizeof(T) * 2 <= 8) {
        using H = Pack<T, 2>;
        if (nvalid >= VEC && (reinterpret_cast<uintptr_t>(p) % sizeof(H)) == 0) {
#pragma unroll
            for (int i = 0; i < VEC; i += 2) {
                H h;
                h.v[0] = r.v[i];
                h.v[1] = r.v[i + 1];
                st_stream<T, 2>(p + i, h);
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (i < nvalid) __stcs(p + i, r.v[i]);
}

// Load VEC elements at p of any alignment (zeros beyond nvalid): the pack load when p is
// pack-aligned and the group full, else element by element.
template <typename T, int VEC>
__device__ __forceinline__ Pack<T, VEC> ld_any(const T* p, int nvalid) {
    if (nvalid >= VEC && (reinterpret_cast<uintptr_t>(p) % sizeof(Pack<T, VEC>)) == 0) return ld_stream<T, VEC>(p);
    Pack<T, VEC> r;
#pragma unroll
    for (int i = 0; i < VEC; ++i) r.v[i] = (i < nvalid) ? p[i] : from_f32<T>(0.0f);
    return r;
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
