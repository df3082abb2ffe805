// launch_tma.cuh -- host launchers of the persistent TMA kernels (lif_tma.cuh), templated
// on the io dtype; instantiated by fwd_tma_{f32,bf16}.cu and bwd_tma_{f32,bf16}.cu.
#pragma once

#include "internal.h"
#include "lif_tma.cuh"

namespace snn_host {

// Tile configurations: VEC neurons per consumer lane x NCONS
// consumer threads = W-neuron tile; R rows per stage; S stages in the smem ring.
template <typename IO> struct TmaCfg;
template <> struct TmaCfg<float> {
    // forward: 1024-neuron tiles, 8 consumer warps, 32 KB stages x 3, 2 CTAs/SM (measured 5%
    // faster at T=512 than 512-neuron tiles with 4 warps and 16 KB x 6 stages)
    static constexpr int FV = 4, FN = 256, FR = 8, FS = 3;
    static constexpr int FN_RES = 128, FS_RES = 3;           // + residual rows: 32 KB stages
    static constexpr int RV = 2, RN = 256, RS = 3;           // backward RECOMPUTE: 66 KB chunks, FFMA2 pairs
    static constexpr int RS_RES = 2;                         // + residual rows: 99 KB chunks
    static constexpr int HV = 2, HN = 256, HR = 8, HS = 6;   // backward SAVE_H: 32 KB stages
};
template <> struct TmaCfg<__nv_bfloat16> {
    static constexpr int FV = 8, FN = 128, FR = 8, FS = 6;   // (8 warps x 2048-neuron tiles: slower on mid layers)
    static constexpr int FN_RES = 128, FS_RES = 3;
    static constexpr int RV = 2, RN = 256, RS = 3;           // 34 KB chunks, 2 CTAs/SM (VEC 4 x 128 lanes measured 6% slower at T=16)
    static constexpr int RS_RES = 2;                         // + residual rows: 51 KB chunks
    static constexpr int HV = 2, HN = 512, HR = 8, HS = 4;
};

template <typename IO>
snn_status launch_forward_tma(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft,
                              cudaStream_t st) {
    using C = TmaCfg<IO>;
    CUtensorMap tmx, tmr;
    // pro: 0 plain, 1 affine, 2 affine + residual (the residual doubles the stage, so that
    // variant has its own, shallower tile configuration).
    const bool res = a.af.residual != nullptr;
    const int bw = res ? snn::FwdTma<IO, C::FV, C::FN_RES, C::FR, C::FS_RES, 2>::BW
                       : snn::FwdTma<IO, C::FV, C::FN, C::FR, C::FS>::BW;
    if (!encode_2d(&tmx, a.x, sizeof(IO), s->N, s->T, s->ld, bw, C::FR))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for x%s", encode_detail());
    tmr = tmx;
    if (res && !encode_2d(&tmr, a.af.residual, sizeof(IO), s->N, s->T, s->ld, bw, C::FR))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for the residual%s", encode_detail());
    auto go = [&](auto sfmt, auto save, auto sft, auto pro) {
        constexpr int P = decltype(pro)::value;
        constexpr int NS = P == 2 ? C::FS_RES : C::FS;
        constexpr int NC = P == 2 ? C::FN_RES : C::FN;
        using K = snn::FwdTma<IO, C::FV, NC, C::FR, NS, P == 2 ? 2 : 1>;
        auto k = snn::lif_forward_tma_kernel<IO, C::FV, decltype(sfmt)::value, decltype(save)::value,
                                             (bool)decltype(sft)::value, P >= 1, P == 2, NC, C::FR, NS>;
        return launch_tiles(k, K::THREADS, K::SMEM, (s->N + K::W - 1) / K::W, (s->T + C::FR - 1) / C::FR,
                            st, "lif_forward_tma_kernel", tmx, tmr, a);
    };
    auto by_aff = [&](auto sfmt, auto save, auto sft) {
        if (a.af.scale == nullptr) return go(sfmt, save, sft, IC<0>{});
        if (a.af.residual == nullptr) return go(sfmt, save, sft, IC<1>{});
        if constexpr (decltype(save)::value == snn::SAVE_H)   // host rejects SAVE_H + residual
            return fail(SNN_ERR_UNSUPPORTED, "the residual prologue needs SAVE_RECOMPUTE or SAVE_NONE");
        else return go(sfmt, save, sft, IC<2>{});
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

template <typename IO, int MODE>
snn_status launch_backward_tma_mode(const snn_lif_shape* s, const snn::BwdArgs& a, cudaStream_t st) {
    using C = TmaCfg<IO>;
    static_assert(MODE < 32 || (MODE & 24) == 0, "P0 variants are plain-path only");
    if constexpr (MODE < 8) {   // SAVE_H has no affine-gradient or P0 variant (host never asks)
    if (s->save_mode == SNN_SAVE_H) {
        using Cfg = snn::BwdHTma<IO, C::HV, C::HN, C::HR, C::HS>;
        CUtensorMap tmh, tmg;
        if (!encode_2d(&tmh, a.saved, 4, s->N, s->T, a.ldh, Cfg::BW, C::HR) ||
            !encode_2d(&tmg, a.gS, sizeof(IO), s->N, s->T, s->ld, Cfg::BW, C::HR))
            return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (SAVE_H backward)%s", encode_detail());
        auto k = snn::lif_backward_saveh_tma_kernel<IO, C::HV, MODE, C::HN, C::HR, C::HS>;
        return launch_tiles(k, Cfg::THREADS, Cfg::SMEM, (s->N + Cfg::W - 1) / Cfg::W,
                            (s->T + C::HR - 1) / C::HR, st, "lif_backward_saveh_tma_kernel", tmh, tmg, a);
    }
    }
    constexpr bool RES = snn::Mode<MODE>::RES;
    constexpr int NS = RES ? C::RS_RES : C::RS;
    using Cfg = snn::BwdRecTma<IO, C::RV, C::RN, NS, RES>;
    const int64_t nch = (s->T + snn::kCkpt - 1) / snn::kCkpt;
    CUtensorMap tmx, tmg, tmck, tmr;
    if (!encode_2d(&tmx, a.x, sizeof(IO), s->N, s->T, s->ld, Cfg::BW, snn::kCkpt) ||
        !encode_2d(&tmg, a.gS, sizeof(IO), s->N, s->T, s->ld, Cfg::BW, snn::kCkpt) ||
        !encode_2d(&tmck, a.saved, 4, s->N, nch, a.ldh, Cfg::BW, 1))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed (RECOMPUTE backward)%s", encode_detail());
    tmr = tmx;
    if (RES && !encode_2d(&tmr, a.af.residual, sizeof(IO), s->N, s->T, s->ld, Cfg::BW, snn::kCkpt))
        return fail(SNN_ERR_CUDA, "cuTensorMapEncodeTiled failed for the residual%s", encode_detail());
    auto k = snn::lif_backward_recompute_tma_kernel<IO, C::RV, MODE, C::RN, NS>;
    return launch_tiles(k, Cfg::THREADS, Cfg::SMEM, (s->N + Cfg::W - 1) / Cfg::W, nch, st,
                        "lif_backward_recompute_tma_kernel", tmx, tmg, tmck, tmr, a);
}

template <typename IO>
snn_status launch_backward_tma(const snn_lif_shape* s, const snn::BwdArgs& a, int mode,
                               cudaStream_t st) {
    switch (mode & 63) {
        case 0: return launch_backward_tma_mode<IO, 0>(s, a, st);
        case 1: return launch_backward_tma_mode<IO, 1>(s, a, st);
        case 2: return launch_backward_tma_mode<IO, 2>(s, a, st);
        case 3: return launch_backward_tma_mode<IO, 3>(s, a, st);
        case 4: return launch_backward_tma_mode<IO, 4>(s, a, st);
        case 5: return launch_backward_tma_mode<IO, 5>(s, a, st);
        case 6: return launch_backward_tma_mode<IO, 6>(s, a, st);
        case 7: return launch_backward_tma_mode<IO, 7>(s, a, st);
        case 8: return launch_backward_tma_mode<IO, 8>(s, a, st);
        case 9: return launch_backward_tma_mode<IO, 9>(s, a, st);
        case 10: return launch_backward_tma_mode<IO, 10>(s, a, st);
        case 11: return launch_backward_tma_mode<IO, 11>(s, a, st);
        case 12: return launch_backward_tma_mode<IO, 12>(s, a, st);
        case 13: return launch_backward_tma_mode<IO, 13>(s, a, st);
        case 14: return launch_backward_tma_mode<IO, 14>(s, a, st);
        case 15: return launch_backward_tma_mode<IO, 15>(s, a, st);
        case 24: return launch_backward_tma_mode<IO, 24>(s, a, st);
        case 25: return launch_backward_tma_mode<IO, 25>(s, a, st);
        case 26: return launch_backward_tma_mode<IO, 26>(s, a, st);
        case 27: return launch_backward_tma_mode<IO, 27>(s, a, st);
        case 28: return launch_backward_tma_mode<IO, 28>(s, a, st);
        case 29: return launch_backward_tma_mode<IO, 29>(s, a, st);
        case 30: return launch_backward_tma_mode<IO, 30>(s, a, st);
        case 31: return launch_backward_tma_mode<IO, 31>(s, a, st);
        case 32: return launch_backward_tma_mode<IO, 32>(s, a, st);
        case 33: return launch_backward_tma_mode<IO, 33>(s, a, st);
        case 34: return launch_backward_tma_mode<IO, 34>(s, a, st);
        case 35: return launch_backward_tma_mode<IO, 35>(s, a, st);
        case 36: return launch_backward_tma_mode<IO, 36>(s, a, st);
        case 37: return launch_backward_tma_mode<IO, 37>(s, a, st);
        case 38: return launch_backward_tma_mode<IO, 38>(s, a, st);
        case 39: return launch_backward_tma_mode<IO, 39>(s, a, st);
        default: return fail(SNN_ERR_UNSUPPORTED, "backward variant %d (residual without affine)", mode);
    }
}

}  // namespace snn_host
