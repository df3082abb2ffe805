// launch_tma.cuh -- host launchers of the persistent TMA kernels (lif_tma.cuh), templated
// on the io dtype and on UNAL (rows of the io tensors not 16-byte aligned: flat tensor maps);
// instantiated by fwd_tma_{f32,bf16}[_unal].cu and bwd_tma_{f32,bf16}[_unal].cu.
#pragma once

#include "internal.h"
#include "lif_tma.cuh"

#include <cstring>

namespace snn_host {

// Tile configurations: VEC neurons per consumer lane x NCONS
// consumer threads = W-neuron tile; R rows per stage; S stages in the smem ring.
// The SNN_{F32,BF16}_{FN,FS,RN,RS} and SNN_BF16_FV macros exist for A/B builds of other tile geometries
// (tools/variant_build.py); the product build takes the defaults.
#ifndef SNN_F32_FN
#define SNN_F32_FN 256
#endif
#ifndef SNN_F32_FS
#define SNN_F32_FS 3
#endif
#ifndef SNN_F32_RN
#define SNN_F32_RN 256
#endif
#ifndef SNN_F32_RS
#define SNN_F32_RS 3
#endif
#ifndef SNN_BF16_FN
#define SNN_BF16_FN 128
#endif
#ifndef SNN_BF16_FV
#define SNN_BF16_FV 8
#endif
#ifndef SNN_BF16_FS
#define SNN_BF16_FS 6
#endif
#ifndef SNN_BF16_RN
#define SNN_BF16_RN 256
#endif
#ifndef SNN_BF16_RS
#define SNN_BF16_RS 3
#endif
template <typename IO> struct TmaCfg;
template <> struct TmaCfg<float> {
    // forward: 1024-neuron tiles, 8 consumer warps, 32 KB stages x 3, 2 CTAs/SM (measured 5%
    // faster at T=512 than 512-neuron tiles with 4 warps and 16 KB x 6 stages)
    static constexpr int FV = 4, FN = SNN_F32_FN, FR = 8, FS = SNN_F32_FS;
    static constexpr int FN_RES = 128, FS_RES = 3;           // + residual rows: 32 KB stages
    static constexpr int RV = 2, RN = SNN_F32_RN, RS = SNN_F32_RS;   // backward RECOMPUTE: 66 KB chunks, FFMA2 pairs
    static constexpr int RS_RES = 2;                         // + residual rows: 99 KB chunks
    static constexpr int HV = 2, HN = 256, HR = 8, HS = 6;   // backward SAVE_H: 32 KB stages
};
template <> struct TmaCfg<__nv_bfloat16> {
    static constexpr int FV = SNN_BF16_FV, FN = SNN_BF16_FN, FR = 8, FS = SNN_BF16_FS;   // (8 warps x 2048-neuron tiles: slower on mid layers)
    static constexpr int FN_RES = 128, FS_RES = 3;
    static constexpr int RV = 2, RN = SNN_BF16_RN, RS = SNN_BF16_RS;   // 34 KB chunks, 2 CTAs/SM (VEC 4 x 128 lanes measured 6% slower at T=16)
    static constexpr int RS_RES = 2;                         // + residual rows: 51 KB chunks
    static constexpr int HV = 2, HN = 512, HR = 8, HS = 4;
};

// Tensor map of an io tensor [T, ld] (first N columns) with boxes of box_inner neurons x rows,
// and the element offset of its first element from 16 B below it (*off).  UNAL: no map -- the
// kernels copy those rows with 1-D bulk copies (lif_tma.cuh Region); *m is zeroed.
template <typename IO, bool UNAL>
bool encode_io(CUtensorMap* m, const void* base, const snn_lif_shape* s, int box_inner, int rows, int* off) {
    *off = (int)((reinterpret_cast<uintptr_t>(base) & 15u) / sizeof(IO));
    if constexpr (!UNAL) {
        return encode_2d(m, base, sizeof(IO), s->N, s->T, s->ld, box_inner, rows);
    } else {
        std::memset(m, 0, sizeof(*m));
        return true;
    }
}

// p0: paper-mode constants (s = 1, c0 = 0); used by the prologue variants only (for the plain
// forward the shorter charge measured no difference).
template <typename IO, bool UNAL>
snn_status launch_forward_tma(const snn_lif_shape* s, const snn::FwdArgs& a0, bool soft, bool p0, cudaStream_t st) {
    using C = TmaCfg<IO>;
    snn::FwdArgs a = a0;
    CUtensorMap tmx, tmr;
    // pro: 0 plain, 1 affine, 2 affine + residual (the residual doubles the stage, so that
    // variant has its own, shallower tile configuration).
    const bool res = a.af.residual != nullptr;
    const int bw = res ? snn::FwdTma<IO, C::FV, C::FN_RES, C::FR, C::FS_RES, 2>::BW
                       : snn::FwdTma<IO, C::FV, C::FN, C::FR, C::FS>::BW;
    if (!encode_io<IO, UNAL>(&tmx, a.x, s, bw, C::FR, &a.x_off))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for x%s", encode_detail());
    tmr = tmx;
    a.r_off = 0;
    if (res && !encode_io<IO, UNAL>(&tmr, a.af.residual, s, bw, C::FR, &a.r_off))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for the residual%s", encode_detail());
    auto go = [&](auto sfmt, auto save, auto sft, auto pro, auto pz) {
        constexpr int P = decltype(pro)::value;
        constexpr int NS = P == 2 ? C::FS_RES : C::FS;
        constexpr int NC = P == 2 ? C::FN_RES : C::FN;
        using K = snn::FwdTma<IO, C::FV, NC, C::FR, NS, P == 2 ? 2 : 1, UNAL>;
        auto k = snn::lif_forward_tma_kernel<IO, C::FV, decltype(sfmt)::value, decltype(save)::value,
                                             (bool)decltype(sft)::value, P >= 1, P == 2, NC, C::FR, NS, UNAL,
                                             (bool)decltype(pz)::value>;
        return launch_tiles(k, K::THREADS, K::SMEM, (s->N + K::W - 1) / K::W, (s->T + C::FR - 1) / C::FR,
                            st, "lif_forward_tma_kernel", tmx, tmr, a);
    };
    auto by_aff = [&](auto sfmt, auto save, auto sft) {
        if (a.af.scale == nullptr) return go(sfmt, save, sft, IC<0>{}, IC<0>{});
        if (a.af.residual == nullptr)
            return p0 ? go(sfmt, save, sft, IC<1>{}, IC<1>{}) : go(sfmt, save, sft, IC<1>{}, IC<0>{});
        if constexpr (decltype(save)::value == snn::SAVE_H)   // host rejects SAVE_H + residual
            return fail(SNN_ERR_UNSUPPORTED, "the residual prologue needs SAVE_RECOMPUTE or SAVE_NONE");
        else return p0 ? go(sfmt, save, sft, IC<2>{}, IC<1>{}) : go(sfmt, save, sft, IC<2>{}, IC<0>{});
    };
    auto by_soft = [&](auto sfmt, auto save) {
        return soft ? by_aff(sfmt, save, IC<1>{}) : by_aff(sfmt, save, IC<0>{});
    };
    auto by_save = [&](auto sfmt) {
        switch (s->save_mode) {
            case SNN_SAVE_H: return by_soft(sfmt, IC<snn::SAVE_H>{});
            case SNN_SAVE_RECOMPUTE: return by_soft(sfmt, IC<snn::SAVE_RECOMPUTE>{});
            default: return by_soft(sfmt, IC<snn::SAVE_NONE>{});
        }
    };
    switch (s->spike_fmt) {
        case SNN_SPK_U8: return by_save(IC<snn::SPK_U8>{});
        case SNN_SPK_BITS: return by_save(IC<snn::SPK_BITS>{});
        default: return by_save(IC<snn::SPK_IO>{});
    }
}

template <typename IO, int MODE, bool UNAL>
snn_status launch_backward_tma_mode(const snn_lif_shape* s, const snn::BwdArgs& a0, cudaStream_t st) {
    using C = TmaCfg<IO>;
    snn::BwdArgs a = a0;
    a.x_off = a.g_off = a.r_off = 0;
    if constexpr (MODE < 8) {   // SAVE_H has no affine-gradient or P0 variant (host never asks)
    if (s->save_mode == SNN_SAVE_H) {
        using Cfg = snn::BwdHTma<IO, C::HV, C::HN, C::HR, C::HS, UNAL>;
        CUtensorMap tmh, tmg;
        if (!encode_2d(&tmh, a.saved, 4, s->N, s->T, a.ldh, Cfg::BW, C::HR) ||
            !encode_io<IO, UNAL>(&tmg, a.gS, s, Cfg::BW, C::HR, &a.g_off))
            return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (SAVE_H backward)%s", encode_detail());
        auto k = snn::lif_backward_saveh_tma_kernel<IO, C::HV, MODE, C::HN, C::HR, C::HS, UNAL>;
        return launch_tiles(k, Cfg::THREADS, Cfg::SMEM, (s->N + Cfg::W - 1) / Cfg::W,
                            (s->T + C::HR - 1) / C::HR, st, "lif_backward_saveh_tma_kernel", tmh, tmg, a);
    }
    }
    constexpr bool RES = snn::Mode<MODE>::RES;
    constexpr int NS = RES ? C::RS_RES : C::RS;
    using Cfg = snn::BwdRecTma<IO, C::RV, C::RN, NS, RES, UNAL>;
    const int64_t nch = (s->T + snn::kCkpt - 1) / snn::kCkpt;
    CUtensorMap tmx, tmg, tmck, tmr;
    if (!encode_io<IO, UNAL>(&tmx, a.x, s, Cfg::BW, snn::kCkpt, &a.x_off) ||
        !encode_io<IO, UNAL>(&tmg, a.gS, s, Cfg::BW, snn::kCkpt, &a.g_off) ||
        !encode_2d(&tmck, a.saved, 4, s->N, nch, a.ldh, Cfg::BW, 1))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (RECOMPUTE backward)%s", encode_detail());
    tmr = tmx;
    if (RES && !encode_io<IO, UNAL>(&tmr, a.af.residual, s, Cfg::BW, snn::kCkpt, &a.r_off))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for the residual%s", encode_detail());
    auto k = snn::lif_backward_recompute_tma_kernel<IO, C::RV, MODE, C::RN, NS, UNAL>;
    return launch_tiles(k, Cfg::THREADS, Cfg::SMEM, (s->N + Cfg::W - 1) / Cfg::W, nch, st,
                        "lif_backward_recompute_tma_kernel", tmx, tmg, tmck, tmr, a);
}

template <typename IO, bool UNAL>
snn_status launch_backward_tma(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    switch (mode & 63) {
        case 0: return launch_backward_tma_mode<IO, 0, UNAL>(s, a, st);
        case 1: return launch_backward_tma_mode<IO, 1, UNAL>(s, a, st);
        case 2: return launch_backward_tma_mode<IO, 2, UNAL>(s, a, st);
        case 3: return launch_backward_tma_mode<IO, 3, UNAL>(s, a, st);
        case 4: return launch_backward_tma_mode<IO, 4, UNAL>(s, a, st);
        case 5: return launch_backward_tma_mode<IO, 5, UNAL>(s, a, st);
        case 6: return launch_backward_tma_mode<IO, 6, UNAL>(s, a, st);
        case 7: return launch_backward_tma_mode<IO, 7, UNAL>(s, a, st);
        case 8: return launch_backward_tma_mode<IO, 8, UNAL>(s, a, st);
        case 9: return launch_backward_tma_mode<IO, 9, UNAL>(s, a, st);
        case 10: return launch_backward_tma_mode<IO, 10, UNAL>(s, a, st);
        case 11: return launch_backward_tma_mode<IO, 11, UNAL>(s, a, st);
        case 12: return launch_backward_tma_mode<IO, 12, UNAL>(s, a, st);
        case 13: return launch_backward_tma_mode<IO, 13, UNAL>(s, a, st);
        case 14: return launch_backward_tma_mode<IO, 14, UNAL>(s, a, st);
        case 15: return launch_backward_tma_mode<IO, 15, UNAL>(s, a, st);
        case 24: return launch_backward_tma_mode<IO, 24, UNAL>(s, a, st);
        case 25: return launch_backward_tma_mode<IO, 25, UNAL>(s, a, st);
        case 26: return launch_backward_tma_mode<IO, 26, UNAL>(s, a, st);
        case 27: return launch_backward_tma_mode<IO, 27, UNAL>(s, a, st);
        case 28: return launch_backward_tma_mode<IO, 28, UNAL>(s, a, st);
        case 29: return launch_backward_tma_mode<IO, 29, UNAL>(s, a, st);
        case 30: return launch_backward_tma_mode<IO, 30, UNAL>(s, a, st);
        case 31: return launch_backward_tma_mode<IO, 31, UNAL>(s, a, st);
        case 32: return launch_backward_tma_mode<IO, 32, UNAL>(s, a, st);
        case 33: return launch_backward_tma_mode<IO, 33, UNAL>(s, a, st);
        case 34: return launch_backward_tma_mode<IO, 34, UNAL>(s, a, st);
        case 35: return launch_backward_tma_mode<IO, 35, UNAL>(s, a, st);
        case 36: return launch_backward_tma_mode<IO, 36, UNAL>(s, a, st);
        case 37: return launch_backward_tma_mode<IO, 37, UNAL>(s, a, st);
        case 38: return launch_backward_tma_mode<IO, 38, UNAL>(s, a, st);
        case 39: return launch_backward_tma_mode<IO, 39, UNAL>(s, a, st);
        case 40: return launch_backward_tma_mode<IO, 40, UNAL>(s, a, st);
        case 41: return launch_backward_tma_mode<IO, 41, UNAL>(s, a, st);
        case 42: return launch_backward_tma_mode<IO, 42, UNAL>(s, a, st);
        case 43: return launch_backward_tma_mode<IO, 43, UNAL>(s, a, st);
        case 44: return launch_backward_tma_mode<IO, 44, UNAL>(s, a, st);
        case 45: return launch_backward_tma_mode<IO, 45, UNAL>(s, a, st);
        case 46: return launch_backward_tma_mode<IO, 46, UNAL>(s, a, st);
        case 47: return launch_backward_tma_mode<IO, 47, UNAL>(s, a, st);
        case 56: return launch_backward_tma_mode<IO, 56, UNAL>(s, a, st);
        case 57: return launch_backward_tma_mode<IO, 57, UNAL>(s, a, st);
        case 58: return launch_backward_tma_mode<IO, 58, UNAL>(s, a, st);
        case 59: return launch_backward_tma_mode<IO, 59, UNAL>(s, a, st);
        case 60: return launch_backward_tma_mode<IO, 60, UNAL>(s, a, st);
        case 61: return launch_backward_tma_mode<IO, 61, UNAL>(s, a, st);
        case 62: return launch_backward_tma_mode<IO, 62, UNAL>(s, a, st);
        case 63: return launch_backward_tma_mode<IO, 63, UNAL>(s, a, st);
        default: return fail(SNN_ERR_UNSUPPORTED, "backward variant %d (residual without affine)", mode);
    }
}

}  // namespace snn_host
