// lif_kernels.cuh -- per-step helpers shared by every fused LIF kernel, and the GENERIC
// kernels (one thread per VEC-neuron group, register prefetch along T) used when the TMA
// path's alignment requirements do not hold (odd ld, unaligned views, tiny N).
//
// Temporal fusion: a thread owns its neurons for the whole time axis;
// V (forward) or the carried dL/dV (backward) lives in registers across the T loop and
// each [T, N] tensor is streamed exactly once.  No tensor cores: the op is elementwise-
// recurrent and HBM-bound.
#pragma once

#include "lif_common.cuh"

namespace snn {

constexpr int kCkpt = 16;           // SNN_LIF_CKPT_INTERVAL
constexpr int kBlock = 256;         // threads per CTA (generic kernels)
constexpr unsigned kFull = 0xffffffffu;

enum { SPK_U8 = 0, SPK_BITS = 1, SPK_IO = 2 };
enum { SAVE_H = 0, SAVE_RECOMPUTE = 1, SAVE_NONE = 2 };

// Peer handoff of a segment boundary (time split; lif_handoff.cuh).
// All pointers null = no handoff.  "peer" pointers are mapped addresses of the
// neighbour rank's buffers (CUDA IPC over NVLink); flags are per kHandoffBlock neurons.
struct Handoff {
    const float* recv_state;  // [N] local: written by the previous sender
    const int* recv_ready;    // [nblk] local: sender sets = epoch after writing recv_state
    int* recv_ack;            // [nblk] peer (the sender's send_ack): we set = epoch once consumed
    float* send_state;        // [N] peer: the next receiver's recv_state
    int* send_ready;          // [nblk] peer: the next receiver's recv_ready
    const int* send_ack;      // [nblk] local: the receiver acknowledges the previous epoch
    int epoch;                // > 0, increases by one per call
};

// Per-channel affine prologue folded into the LIF input: the layer input
// is X' = scale[c] X + shift[c] with c = (n / HW) % C (e.g. the BN affine of a conv
// output [T, B, C, H, W] flattened to N = B C H W).  scale = null: identity (the plain path;
// fma(1, X, 0) == X, so the arithmetic is unchanged).  Backward (RECOMPUTE only):
// dL/dX = scale[c] dL/dX', and per-neuron partials part_a[n] = sum_t dL/dX'[t,n] X[t,n],
// part_b[n] = sum_t dL/dX'[t,n], reduced per channel by affine_reduce_kernel.
struct Affine {
    const float* scale;   // [C] or null
    const float* shift;   // [C]
    int64_t C, HW;
    float* part_a;        // [N] backward output (per-neuron sum over t) or null
    float* part_b;        // [N]
    int seg;              // > 0: the backward reduces the partials itself into segments of `seg`
                          // neurons (affine_warp_segments) written to part_a/b[n / seg]; 0: per neuron
    const void* residual; // [T, ld] IO shortcut R added to the input (X' = a X + b + R) or null
    void* grad_residual;  // [T, ld] IO backward output dL/dR = dL/dX' (iff residual)
};

template <int VEC>
struct AffCoef {
    float a[VEC], b[VEC];
};

// AFF = false: the prologue is compiled out (the coefficients are never read).  One division
// per group (32-bit when the indices fit): the channel of n0 + i follows by stepping hw.
template <int VEC, bool AFF>
__device__ __forceinline__ AffCoef<VEC> load_affine(const Affine& af, int64_t n0, int nvalid) {
    AffCoef<VEC> co;
#pragma unroll
    for (int i = 0; i < VEC; ++i) { co.a[i] = 1.0f; co.b[i] = 0.0f; }
    if constexpr (AFF) {
        if (nvalid <= 0) return co;
        int64_t blk, hw;
        if (n0 + VEC <= (int64_t)UINT32_MAX && af.HW <= (int64_t)UINT32_MAX) {
            const uint32_t q = (uint32_t)n0 / (uint32_t)af.HW;
            blk = q;
            hw = (uint32_t)n0 - q * (uint32_t)af.HW;
        } else {
            blk = n0 / af.HW;
            hw = n0 - blk * af.HW;
        }
        int64_t ch = (af.C <= (int64_t)UINT32_MAX && blk <= (int64_t)UINT32_MAX)
                         ? (int64_t)((uint32_t)blk % (uint32_t)af.C) : blk % af.C;
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            if (i > 0 && ++hw == af.HW) {
                hw = 0;
                if (++ch == af.C) ch = 0;
            }
            if (i < nvalid) {
                co.a[i] = __ldg(af.scale + ch);
                co.b[i] = __ldg(af.shift + ch);
            }
        }
    }
    return co;
}

// Work distribution of a launch (host: launch_tiles).
struct Sched {
    int depth;      // steal requests kept in flight, 1..kMaxClc (0: the whole grid is resident)
    int prefetch;   // ring stages of the CTA's own tile to L2-prefetch before griddepcontrol.wait
};

struct FwdArgs {
    const void* x;        // [T, ld] IO
    const float* v_init;  // [N] or null
    void* spikes;         // per spike format
    float* saved;         // SAVE_H: [T, ldh]; RECOMPUTE: [ceil(T/kCkpt), ldh]
    float* v_final;       // [N] or null
    int64_t T, N, ld, ldh, nwords;
    int64_t spk_words_ld; // row stride (uint32 words) of bit-packed spikes: nwords, or the whole
                          // layer's when this launch covers a neuron chunk of it (time split)
    int x_off, r_off;     // unaligned TMA path: element offset of x / residual from their 1-D
                          // tensor maps' (16-byte aligned) base
    int ck0;              // RECOMPUTE: 1 = store checkpoint row 0 (V[-1]); 0 = skip it -- it would
                          // equal v_init / V_reset, which the backward reads instead (BwdArgs::ck0)
    LifConsts c;
    Handoff h;            // boundary V from / to the neighbour time segment (TMA path only)
    Affine af;            // input prologue (identity when af.scale == null)
#ifdef SNN_TRACE
    void* trace;          // TraceBuf (trace.cuh)
#endif
};

struct BwdArgs {
    const void* gS;             // [T, ld] IO
    const void* x;              // [T, ld] IO (RECOMPUTE)
    const float* saved;         // as FwdArgs::saved
    const float* grad_v_final;  // [N] or null
    void* gX;                   // [T, ld] IO
    float* grad_v_init;         // [N] or null
    int64_t T, N, ld, ldh;
    int x_off, g_off, r_off;    // unaligned TMA path: element offsets of x / gS / residual
    const float* v_init;        // RECOMPUTE with ck0 == 0: V[-1] of chunk 0 ([N], or null -> V_reset)
    int ck0;                    // 1: chunk 0's entry V is checkpoint row 0 (the forward stored it)
    LifConsts c;
    Handoff h;                  // boundary dL/dV from / to the neighbour segment (TMA path only)
    Affine af;                  // input prologue + its per-neuron gradient partials
#ifdef SNN_TRACE
    void* trace;                // TraceBuf (trace.cuh)
#endif
};

// ------------------------------------------------------------------------------------
// Affine gradients folded into the backward's tile epilogue: a warp's
// per-neuron partials (32 lanes x VEC = 2 neurons) are summed over segments of G consecutive
// neurons -- G = min(HW, 64) with G | HW, so a segment never crosses a (sample, channel) block of
// HW neurons and never leaves its warp -- in a fixed order (the lane's pair, then an xor-shuffle
// tree inside G/2 lanes); the segment starting at neuron n is written to seg_a/b[n / G].  No
// cross-warp synchronisation (the tile epilogue stays asynchronous between warps); the channel
// totals are summed by affine_segment_finish_kernel.  Deterministic run to run.
constexpr int kSegMax = 64;
template <int VEC>
__device__ __forceinline__ void affine_warp_segments(const float (&pa)[VEC], const float (&pb)[VEC], int nvalid,
                                                     int64_t n0, int G, int64_t nseg, float* seg_a, float* seg_b) {
    static_assert(VEC * 32 == kSegMax, "a warp covers one 64-neuron segment");
    float a = 0.0f, b = 0.0f;
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (i < nvalid) { a = __fadd_rn(a, pa[i]); b = __fadd_rn(b, pb[i]); }
    const int L = G / VEC;                     // lanes per segment, 1 .. 32
    for (int o = 1; o < L; o <<= 1) {
        a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = __fadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (((threadIdx.x & 31) % L) == 0) {
        const int64_t sidx = n0 / G;
        if (sidx < nseg) { seg_a[sidx] = a; seg_b[sidx] = b; }
    }
}

// ------------------------------------------------------------------------------------
// Forward step helpers.

// Eq. 1-2 + reset for this thread's VEC neurons: updates V, returns H in `hp` and the
// spike bits (bit i = neuron i of the group).
// AFF: the input is X' = fma(a, X, b); otherwise X itself.
// RES (with AFF): X' = fma(a, X, b) + R, R the residual shortcut row (rv).
template <bool AFF, bool RES = false, typename IO, int VEC>
__device__ __forceinline__ F2 input2(const AffCoef<VEC>& co, const Pack<IO, VEC>& xv, int i,
                                     const Pack<IO, VEC>* rv = nullptr) {
    F2 X2 = load2(xv, i);
    if constexpr (AFF) X2 = fma2(f2(co.a[i], co.a[i + 1]), X2, f2(co.b[i], co.b[i + 1]));
    if constexpr (RES) X2 = add2(X2, load2(*rv, i));
    return X2;
}
template <bool AFF, bool RES = false, typename IO, int VEC>
__device__ __forceinline__ float input1(const AffCoef<VEC>& co, const Pack<IO, VEC>& xv, int i,
                                        const Pack<IO, VEC>* rv = nullptr) {
    float X = to_f32(xv.v[i]);
    if constexpr (AFF) X = __fmaf_rn(co.a[i], X, co.b[i]);
    if constexpr (RES) X = __fadd_rn(X, to_f32(rv->v[i]));
    return X;
}

// P0 (paper-mode constants, s = 1, c0 = 0): the charge is fma(k, V, X) (Mode::P0).
template <bool SOFT, bool AFF, bool RES = false, bool P0 = false, typename IO, int VEC>
__device__ __forceinline__ unsigned fwd_compute(const LifConsts& c, float (&V)[VEC],
                                                const Pack<IO, VEC>& xv, Pack<float, VEC>& hp,
                                                const AffCoef<VEC>& co,
                                                const Pack<IO, VEC>* rv = nullptr) {
    unsigned bits = 0;
    if constexpr (VEC % 2 == 0) {   // paired FFMA2 charge, same roundings as the scalar path
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
            const F2 X2 = input2<AFF, RES>(co, xv, i, rv);
            const F2 H2 = lif_charge2<P0>(c, f2(V[i], V[i + 1]), X2);
            const float Ha = lo(H2), Hb = hi(H2);
            const bool Sa = lif_fire(c, Ha), Sb = lif_fire(c, Hb);
            V[i] = lif_reset<SOFT>(c, Ha, Sa);
            V[i + 1] = lif_reset<SOFT>(c, Hb, Sb);
            hp.v[i] = Ha;
            hp.v[i + 1] = Hb;
            bits |= ((unsigned)Sa << i) | ((unsigned)Sb << (i + 1));
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            const float H = lif_charge(c, V[i], input1<AFF, RES>(co, xv, i, rv));
            const bool S = lif_fire(c, H);
            V[i] = lif_reset<SOFT>(c, H, S);
            hp.v[i] = H;
            bits |= (unsigned)S << i;
        }
    }
    return bits;
}

// Re-run the charge / fire / reset (no outputs) -- the RECOMPUTE backward's forward pass.
template <bool SOFT, bool AFF, bool RES = false, bool P0 = false, typename IO, int VEC>
__device__ __forceinline__ void fwd_recompute_step(const LifConsts& c, float (&V)[VEC],
                                                   const Pack<IO, VEC>& xv, float (&h)[VEC],
                                                   const AffCoef<VEC>& co,
                                                   const Pack<IO, VEC>* rv = nullptr) {
    if constexpr (VEC % 2 == 0) {
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
            const F2 X2 = input2<AFF, RES>(co, xv, i, rv);
            const F2 H2 = lif_charge2<P0>(c, f2(V[i], V[i + 1]), X2);
            h[i] = lo(H2);
            h[i + 1] = hi(H2);
            V[i] = lif_reset<SOFT>(c, h[i], lif_fire(c, h[i]));
            V[i + 1] = lif_reset<SOFT>(c, h[i + 1], lif_fire(c, h[i + 1]));
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            h[i] = lif_charge(c, V[i], input1<AFF, RES>(co, xv, i, rv));
            V[i] = lif_reset<SOFT>(c, h[i], lif_fire(c, h[i]));
        }
    }
}

// Pack VEC spike bits of this lane into the warp's uint32 words and store them
// (SNN_SPK_BITS).  Lanes [w*L, (w+1)*L), L = 32/VEC, share word w of the warp; the warp's
// first neuron must be a multiple of 32 (group index g = warp-aligned).
template <int VEC>
__device__ __forceinline__ void store_spike_bits(uint32_t* row, int64_t g, unsigned bits,
                                                 int64_t nwords) {
    constexpr int L = 32 / VEC;
    const int lane = threadIdx.x & 31;
    uint32_t w;
    if constexpr (VEC == 1) {
        w = __ballot_sync(kFull, bits);
    } else {
        w = bits << ((lane % L) * VEC);
#pragma unroll
        for (int o = 1; o < L; o <<= 1) w |= __shfl_xor_sync(kFull, w, o);
    }
    if (lane % L == 0) {
        const int64_t word = ((g - lane) * VEC) / 32 + lane / L;
        if (word < nwords) __stcs(row + word, w);
    }
}

// Four u8 spikes (w: byte i = neuron i) at a global address of any alignment, branch-free
// (r2c): every case is a predicated store -- one 32-bit store when 4-aligned, two 16-bit ones
// when 2-aligned, byte / 16-bit / byte when odd -- so an unaligned row costs no per-row
// branches (streaming, evict-first like st_stream).
__device__ __forceinline__ void st_u8x4_any(uint8_t* p, uint32_t w) {
    const uint32_t a = (uint32_t)reinterpret_cast<uintptr_t>(p) & 3u;
    const uint32_t mid = (w >> 8) & 0xffffu;   // bytes 1..2 (the odd case's 16-bit store at p+1)
    asm volatile(
        "{\n\t.reg .pred q4, q2, q1;\n\t"
        "setp.eq.u32 q4, %1, 0;\n\t"
        "setp.eq.u32 q2, %1, 2;\n\t"
        "setp.eq.u32 q1, %5, 1;\n\t"
        "@q4 st.global.cs.u32 [%0], %2;\n\t"
        "@q2 st.global.cs.u16 [%0], %2;\n\t"
        "@q2 st.global.cs.u16 [%0+2], %3;\n\t"
        "@q1 st.global.cs.u8 [%0], %2;\n\t"
        "@q1 st.global.cs.u16 [%0+1], %4;\n\t"
        "@q1 st.global.cs.u8 [%0+3], %6;\n\t}"
        :: "l"(p), "r"(a), "r"(w), "r"(w >> 16), "r"(mid), "r"(a & 1u), "r"(w >> 24) : "memory");
}

// Store one time row's spikes.  `row` = spikes + t*ld (U8/IO) or words + t*nwords (BITS).
// Every lane of the warp must call this (BITS uses warp shuffles).
// UNAL: the row may not be pack-aligned (odd row stride / unaligned view): st_any.
template <typename IO, int VEC, int SFMT, bool UNAL = false>
__device__ __forceinline__ void store_spikes(void* row, int64_t g, int64_t n0, unsigned bits,
                                             int nvalid, int64_t nwords) {
    bits &= (nvalid >= VEC) ? ((VEC == 32) ? kFull : ((1u << VEC) - 1u)) : ((1u << nvalid) - 1u);
    if constexpr (SFMT == SPK_U8) {
        if (nvalid > 0) {
            Pack<uint8_t, VEC> sp;
#pragma unroll
            for (int i = 0; i < VEC; ++i) sp.v[i] = (uint8_t)((bits >> i) & 1u);
            if constexpr (UNAL && VEC == 4) {   // (bf16's 8 bytes as two of these: 7% slower than st_any)
                uint8_t* q = reinterpret_cast<uint8_t*>(row) + n0;
                if (nvalid >= VEC) st_u8x4_any(q, *reinterpret_cast<const uint32_t*>(&sp));
                else st_any<uint8_t, VEC>(q, sp, nvalid);
            } else if constexpr (UNAL) {
                st_any<uint8_t, VEC>(reinterpret_cast<uint8_t*>(row) + n0, sp, nvalid);
            } else {
                st_group<uint8_t, VEC>(reinterpret_cast<uint8_t*>(row) + n0, sp, nvalid);
            }
        }
    } else if constexpr (SFMT == SPK_IO) {
        if (nvalid > 0) {
            Pack<IO, VEC> sp;
#pragma unroll
            for (int i = 0; i < VEC; ++i) sp.v[i] = from_f32<IO>(((bits >> i) & 1u) ? 1.0f : 0.0f);
            if constexpr (UNAL) st_any<IO, VEC>(reinterpret_cast<IO*>(row) + n0, sp, nvalid);
            else st_group<IO, VEC>(reinterpret_cast<IO*>(row) + n0, sp, nvalid);
        }
    } else {
        store_spike_bits<VEC>(reinterpret_cast<uint32_t*>(row), g, bits, nwords);
    }
}

// Byte stride between consecutive spike rows.
template <typename IO, int SFMT>
__device__ __forceinline__ int64_t spike_row_bytes(const FwdArgs& a) {
    if constexpr (SFMT == SPK_U8) return a.ld;
    else if constexpr (SFMT == SPK_IO) return a.ld * (int64_t)sizeof(IO);
    else return a.spk_words_ld * 4;
}

// One reverse step of Eq. 3 for this thread's VEC neurons: returns gX[t] (io dtype) and
// carries gV <- k gH.
// AFF = with the affine prologue: gX = scale (s gH) and the per-neuron partials
// pa += (s gH) X_raw, pb += (s gH) accumulate over the time walk (xr = raw X of this row).
// RES (with AFF): also returns dL/dR = dL/dX' = s gH in *outr.
template <typename IO, int VEC, int MODE, bool AFF = false>
__device__ __forceinline__ Pack<IO, VEC> bwd_step(const LifConsts& c, float (&gV)[VEC],
                                                  const float (&h)[VEC], const Pack<IO, VEC>& gs,
                                                  const AffCoef<VEC>* co = nullptr,
                                                  const Pack<IO, VEC>* xr = nullptr,
                                                  float* pa = nullptr, float* pb = nullptr,
                                                  Pack<IO, VEC>* outr = nullptr) {
    constexpr bool RES = AFF && Mode<MODE>::RES;
    Pack<IO, VEC> out;
    if constexpr (VEC % 2 == 0) {   // paired FFMA2/FMUL2/FADD2, same roundings as scalar
#pragma unroll
        for (int i = 0; i < VEC; i += 2) {
            const F2 gH = lif_grad_step2<MODE>(c, f2(h[i], h[i + 1]),
                                               load2(gs, i),
                                               f2(gV[i], gV[i + 1]));
            F2 gx = Mode<MODE>::P0 ? gH : mul2(f2(c.s), gH);
            if constexpr (AFF) {
                const F2 x2 = load2(*xr, i);
                const F2 pa2 = fma2(gx, x2, f2(pa[i], pa[i + 1]));
                const F2 pb2 = add2(gx, f2(pb[i], pb[i + 1]));
                pa[i] = lo(pa2); pa[i + 1] = hi(pa2);
                pb[i] = lo(pb2); pb[i + 1] = hi(pb2);
                if constexpr (RES) {
                    outr->v[i] = from_f32<IO>(lo(gx));
                    outr->v[i + 1] = from_f32<IO>(hi(gx));
                }
                gx = mul2(f2(co->a[i], co->a[i + 1]), gx);
            }
            const F2 gv = mul2(f2(c.k), gH);
            out.v[i] = from_f32<IO>(lo(gx));
            out.v[i + 1] = from_f32<IO>(hi(gx));
            gV[i] = lo(gv);
            gV[i + 1] = hi(gv);
        }
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            const float gH = lif_grad_step<MODE>(c, h[i], to_f32(gs.v[i]), gV[i]);
            float gx = __fmul_rn(c.s, gH);
            if constexpr (AFF) {
                pa[i] = __fmaf_rn(gx, to_f32(xr->v[i]), pa[i]);
                pb[i] = __fadd_rn(gx, pb[i]);
                if constexpr (RES) outr->v[i] = from_f32<IO>(gx);
                gx = __fmul_rn(co->a[i], gx);
            }
            out.v[i] = from_f32<IO>(gx);
            gV[i] = __fmul_rn(c.k, gH);
        }
    }
    return out;
}

// ------------------------------------------------------------------------------------
// Generic forward: PF-deep register prefetch ring along T.
template <typename IO, int VEC, int SFMT, int SAVE, bool SOFT, bool AFF, int PF>
__global__ void __launch_bounds__(kBlock)
lif_forward_kernel(const FwdArgs a) {
    const int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int64_t n0 = g * VEC;
    const int nvalid = (int)max((int64_t)0, min((int64_t)VEC, a.N - n0));
    // Lanes past N stay alive (their warp's shuffles need them) but touch no memory.
    const IO* __restrict__ x = reinterpret_cast<const IO*>(a.x) + n0;
    LifConsts c = a.c;
    pin(c);
    const int64_t T = a.T, ld = a.ld;

    float V[VEC];
    if (a.v_init != nullptr && nvalid > 0) {
        Pack<float, VEC> v0 = ld_group<float, VEC>(a.v_init + n0, nvalid);
#pragma unroll
        for (int i = 0; i < VEC; ++i) V[i] = v0.v[i];
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) V[i] = c.v_reset;
    }
    const AffCoef<VEC> co = load_affine<VEC, AFF>(a.af, n0, nvalid);

    Pack<IO, VEC> buf[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j)
        if (j < T) buf[j] = ld_group<IO, VEC>(x + (int64_t)j * ld, nvalid);

    unsigned char* spk_row = reinterpret_cast<unsigned char*>(a.spikes);
    const int64_t spk_step = spike_row_bytes<IO, SFMT>(a);
    for (int64_t t0 = 0; t0 < T; t0 += PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int64_t t = t0 + j;
            if (t < T) {
                const Pack<IO, VEC> xv = buf[j];
                if (t + PF < T) buf[j] = ld_group<IO, VEC>(x + (t + PF) * ld, nvalid);
                if constexpr (SAVE == SAVE_RECOMPUTE) {
                    if ((t % kCkpt) == 0 && nvalid > 0 && (t > 0 || a.ck0)) {
                        Pack<float, VEC> ck;
#pragma unroll
                        for (int i = 0; i < VEC; ++i) ck.v[i] = V[i];
                        st_group<float, VEC>(a.saved + (t / kCkpt) * a.ldh + n0, ck, nvalid);
                    }
                }
                Pack<float, VEC> hp;
                const unsigned bits = fwd_compute<SOFT, AFF>(c, V, xv, hp, co);
                if constexpr (SAVE == SAVE_H) {
                    if (nvalid > 0) st_group<float, VEC>(a.saved + t * a.ldh + n0, hp, nvalid);
                }
                store_spikes<IO, VEC, SFMT>(spk_row, g, n0, bits, nvalid, a.nwords);
                spk_row += spk_step;
            }
        }
    }
    if (a.v_final != nullptr && nvalid > 0) {
        Pack<float, VEC> vf;
#pragma unroll
        for (int i = 0; i < VEC; ++i) vf.v[i] = V[i];
        st_group<float, VEC>(a.v_final + n0, vf, nvalid);
    }
}

// ------------------------------------------------------------------------------------
// Generic backward, SAVE_H: Eq. 3 over t = T-1..0 reading the saved H.
template <typename IO, int VEC, int MODE, int PF>
__global__ void __launch_bounds__(kBlock)
lif_backward_saveh_kernel(const BwdArgs a) {
    const int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int64_t n0 = g * VEC;
    const int nvalid = (int)max((int64_t)0, min((int64_t)VEC, a.N - n0));
    if (nvalid == 0) return;  // no warp collectives in the backward
    const IO* __restrict__ gs = reinterpret_cast<const IO*>(a.gS) + n0;
    const float* __restrict__ hs = a.saved + n0;
    IO* __restrict__ gx = reinterpret_cast<IO*>(a.gX) + n0;
    LifConsts c = a.c;
    pin(c);
    const int64_t T = a.T, ld = a.ld, ldh = a.ldh;

    float gV[VEC];
    if (a.grad_v_final != nullptr) {
        Pack<float, VEC> g0 = ld_group<float, VEC>(a.grad_v_final + n0, nvalid);
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = g0.v[i];
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = 0.0f;
    }

    Pack<IO, VEC> gbuf[PF];
    Pack<float, VEC> hbuf[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        const int64_t t = T - 1 - j;
        if (t >= 0) {
            gbuf[j] = ld_group<IO, VEC>(gs + t * ld, nvalid);
            hbuf[j] = ld_group<float, VEC>(hs + t * ldh, nvalid);
        }
    }
    for (int64_t t0 = T - 1; t0 >= 0; t0 -= PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int64_t t = t0 - j;
            if (t >= 0) {
                const Pack<IO, VEC> gv = gbuf[j];
                const Pack<float, VEC> hv = hbuf[j];
                if (t - PF >= 0) {
                    gbuf[j] = ld_group<IO, VEC>(gs + (t - PF) * ld, nvalid);
                    hbuf[j] = ld_group<float, VEC>(hs + (t - PF) * ldh, nvalid);
                }
                st_group<IO, VEC>(gx + t * ld, bwd_step<IO, VEC, MODE>(c, gV, hv.v, gv), nvalid);
            }
        }
    }
    if (a.grad_v_init != nullptr) {
        Pack<float, VEC> gi;
#pragma unroll
        for (int i = 0; i < VEC; ++i) gi.v[i] = gV[i];
        st_group<float, VEC>(a.grad_v_init + n0, gi, nvalid);
    }
}

// ------------------------------------------------------------------------------------
// V[-1] of the RECOMPUTE backward's chunk 0 when the forward did not store checkpoint row 0
// (ck0 == 0): the caller's v_init (the value the forward started from; any alignment), else
// V_reset.  Elements past nvalid are V_reset (never stored).
template <int VEC>
__device__ __forceinline__ Pack<float, VEC> entry_v0(const float* v_init, int64_t n0, int nvalid, float v_reset) {
    Pack<float, VEC> v;
#pragma unroll
    for (int i = 0; i < VEC; ++i) v.v[i] = (v_init != nullptr && i < nvalid) ? v_init[n0 + i] : v_reset;
    return v;
}

// Generic backward, SAVE_RECOMPUTE: per kCkpt-step chunk (last chunk first) reload the
// chunk's entry V checkpoint, re-run the forward charge over the chunk from x (identical
// instruction sequence -> bitwise-identical H), then walk the chunk backwards.
template <typename IO, int VEC, int MODE>
__global__ void __launch_bounds__(kBlock)
lif_backward_recompute_kernel(const BwdArgs a) {
    const int64_t g = (int64_t)blockIdx.x * kBlock + threadIdx.x;
    const int64_t n0 = g * VEC;
    const int nvalid = (int)max((int64_t)0, min((int64_t)VEC, a.N - n0));
    if (nvalid == 0) return;
    const IO* __restrict__ gs = reinterpret_cast<const IO*>(a.gS) + n0;
    const IO* __restrict__ xs = reinterpret_cast<const IO*>(a.x) + n0;
    const float* __restrict__ ck = a.saved + n0;
    IO* __restrict__ gx = reinterpret_cast<IO*>(a.gX) + n0;
    LifConsts c = a.c;
    pin(c);
    const int64_t T = a.T, ld = a.ld, ldh = a.ldh;

    float gV[VEC];
    if (a.grad_v_final != nullptr) {
        Pack<float, VEC> g0 = ld_group<float, VEC>(a.grad_v_final + n0, nvalid);
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = g0.v[i];
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = 0.0f;
    }

    constexpr bool AFF = Mode<MODE>::AFF;
    const AffCoef<VEC> co = load_affine<VEC, AFF>(a.af, n0, nvalid);
    float pa[VEC], pb[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) pa[i] = pb[i] = 0.0f;
    const int64_t nchunks = (T + kCkpt - 1) / kCkpt;
    // One chunk; FULL (16 rows) is branch-free so the rows' independent math interleaves,
    // a partial chunk (only the last one, when T % 16 != 0) keeps the per-row guards.
    auto chunk = [&](int64_t ch, auto full) {
        constexpr bool FULL = decltype(full)::value;
        const int64_t t0 = ch * kCkpt;
        const int len = FULL ? kCkpt : (int)min((int64_t)kCkpt, T - t0);
        const Pack<float, VEC> v0 = (ch > 0 || a.ck0) ? ld_group<float, VEC>(ck + ch * ldh, nvalid)
                                                      : entry_v0<VEC>(a.v_init, n0, nvalid, c.v_reset);
        Pack<IO, VEC> xb[kCkpt];
        Pack<IO, VEC> gb[kCkpt];
#pragma unroll
        for (int j = 0; j < kCkpt; ++j)
            if (FULL || j < len) xb[j] = ld_group<IO, VEC>(xs + (t0 + j) * ld, nvalid);
#pragma unroll
        for (int j = 0; j < kCkpt; ++j)
            if (FULL || j < len) gb[j] = ld_group<IO, VEC>(gs + (t0 + j) * ld, nvalid);

        float h[kCkpt][VEC];
        float V[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) V[i] = v0.v[i];
#pragma unroll
        for (int j = 0; j < kCkpt; ++j) {
            if (FULL || j < len) fwd_recompute_step<Mode<MODE>::SOFT, AFF>(c, V, xb[j], h[j], co);
        }
#pragma unroll
        for (int j = kCkpt - 1; j >= 0; --j) {
            if (FULL || j < len)
                st_group<IO, VEC>(gx + (t0 + j) * ld,
                                  bwd_step<IO, VEC, MODE, AFF>(c, gV, h[j], gb[j], &co, &xb[j], pa, pb),
                                  nvalid);
        }
    };
    for (int64_t ch = nchunks - 1; ch >= 0; --ch) {
        if ((ch + 1) * kCkpt <= T) chunk(ch, std::true_type{});
        else chunk(ch, std::false_type{});
    }
    if constexpr (AFF) {
        Pack<float, VEC> qa, qb;
#pragma unroll
        for (int i = 0; i < VEC; ++i) { qa.v[i] = pa[i]; qb.v[i] = pb[i]; }
        st_group<float, VEC>(a.af.part_a + n0, qa, nvalid);
        st_group<float, VEC>(a.af.part_b + n0, qb, nvalid);
    }
    if (a.grad_v_init != nullptr) {
        Pack<float, VEC> gi;
#pragma unroll
        for (int i = 0; i < VEC; ++i) gi.v[i] = gV[i];
        st_group<float, VEC>(a.grad_v_init + n0, gi, nvalid);
    }
}

}  // namespace snn
