// bwd_generic.cu -- launcher of the generic backward kernels (lif_kernels.cuh).  Threads
// own 8 bytes of io per row (2 fp32 / 4 bf16 neurons): the RECOMPUTE walk keeps
// 2 x kCkpt rows of x and gS in registers, so a narrow group keeps occupancy up.
#include "internal.h"
#include "lif_async.cuh"

namespace snn {
// ------------------------------------------------------------------------------------
// Affine prologue gradients: grad_scale[c] = sum_{b, hw} part_a[(b C + c) HW + hw], same for
// shift.  Two passes with a fixed partition and fixed summation orders, so the result is
// deterministic (bitwise run to run):
//   1. grid (S, C): CTA (j, c) sums piece j = flat indices [j L, min((j+1) L, B HW)) of channel
//      c's B x HW elements (per-thread strided sums, then a fixed shuffle/smem tree) and
//      writes its partial over the piece's first element (the CTA owns that piece; scratch);
//   2. warp c adds its S piece partials: lane l sums pieces l, l+32, ... in order, then a
//      fixed xor-shuffle tree.
// Both run under programmatic dependent launch (they wait for the backward in pdl_wait()).
__device__ __forceinline__ int64_t piece_first(int64_t j, int64_t L, int64_t C, int64_t HW, int64_t c) {
    const int64_t i = j * L;
    return ((i / HW) * C + c) * HW + i % HW;
}

__global__ void __launch_bounds__(256)
affine_partial_kernel(float* __restrict__ part_a, float* __restrict__ part_b, int64_t B, int64_t C,
                      int64_t HW, int64_t L) {
    pdl_wait();
    pdl_trigger();
    const int64_t c = blockIdx.y, j = blockIdx.x;
    const int64_t i0 = j * L, i1 = min(i0 + L, B * HW);
    float acc_a = 0.0f, acc_b = 0.0f;
    for (int64_t b = i0 / HW; b * HW < i1; ++b) {       // rows of this piece, each contiguous
        const int64_t lo = max(i0, b * HW) - b * HW, hi = min(i1, (b + 1) * HW) - b * HW;
        const int64_t base = (b * C + c) * HW;
        for (int64_t hw = lo + threadIdx.x; hw < hi; hw += blockDim.x) {
            acc_a = __fadd_rn(acc_a, part_a[base + hw]);
            acc_b = __fadd_rn(acc_b, part_b[base + hw]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc_a = __fadd_rn(acc_a, __shfl_xor_sync(0xffffffffu, acc_a, o));
        acc_b = __fadd_rn(acc_b, __shfl_xor_sync(0xffffffffu, acc_b, o));
    }
    __shared__ float sa[8], sb[8];
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { sa[warp] = acc_a; sb[warp] = acc_b; }
    __syncthreads();                                     // every read of the piece is done
    if (threadIdx.x == 0) {
        float ta = sa[0], tb = sb[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { ta = __fadd_rn(ta, sa[w]); tb = __fadd_rn(tb, sb[w]); }
        const int64_t n = piece_first(j, L, C, HW, c);
        part_a[n] = ta;
        part_b[n] = tb;
    }
}

__global__ void __launch_bounds__(256)
affine_finish_kernel(const float* __restrict__ part_a, const float* __restrict__ part_b, int64_t C,
                     int64_t HW, int64_t L, int64_t S, float* __restrict__ grad_scale,
                     float* __restrict__ grad_shift) {
    pdl_wait();
    const int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= C) return;                                   // whole warps exit together
    float ta = 0.0f, tb = 0.0f;
    for (int64_t j = lane; j < S; j += 32) {
        const int64_t n = piece_first(j, L, C, HW, c);
        ta = __fadd_rn(ta, part_a[n]);
        tb = __fadd_rn(tb, part_b[n]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ta = __fadd_rn(ta, __shfl_xor_sync(0xffffffffu, ta, o));
        tb = __fadd_rn(tb, __shfl_xor_sync(0xffffffffu, tb, o));
    }
    if (lane == 0) {
        grad_scale[c] = ta;
        grad_shift[c] = tb;
    }
}

// Per-channel sums of the segment partials the TMA backward wrote (affine_warp_segments):
// channel c owns segments ((b C + c) HW) / G + p, b < B, p < P = HW / G.  One CTA per channel:
// thread i sums flat (b, p) indices i, i + 256, ... in order, then a fixed shuffle tree and
// warp 0 adds the 8 warp partials in order -- deterministic.
__global__ void __launch_bounds__(256)
affine_segment_finish_kernel(const float* __restrict__ seg_a, const float* __restrict__ seg_b, int64_t B,
                             int64_t C, int64_t P, float* __restrict__ grad_scale, float* __restrict__ grad_shift) {
    pdl_wait();
    pdl_trigger();   // tiny: let the next kernel's launch and prologue overlap this one
    const int64_t c = blockIdx.x;
    float ta = 0.0f, tb = 0.0f;
    for (int64_t i = threadIdx.x; i < B * P; i += blockDim.x) {
        const int64_t s = ((i / P) * C + c) * P + i % P;
        ta = __fadd_rn(ta, seg_a[s]);
        tb = __fadd_rn(tb, seg_b[s]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ta = __fadd_rn(ta, __shfl_xor_sync(0xffffffffu, ta, o));
        tb = __fadd_rn(tb, __shfl_xor_sync(0xffffffffu, tb, o));
    }
    __shared__ float sa[8], sb[8];
    if ((threadIdx.x & 31) == 0) { sa[threadIdx.x >> 5] = ta; sb[threadIdx.x >> 5] = tb; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) { sa[0] = __fadd_rn(sa[0], sa[w]); sb[0] = __fadd_rn(sb[0], sb[w]); }
        grad_scale[c] = sa[0];
        grad_shift[c] = sb[0];
    }
}

}  // namespace snn

namespace snn_host {

namespace {
constexpr int kBwdPF = 8;

template <typename IO, int VEC, int MODE>
snn_status go_mode(const snn_lif_shape* s, const snn::BwdArgs& a, cudaStream_t st) {
    const int64_t groups = (s->N + VEC - 1) / VEC;
    const dim3 grid((unsigned)((groups + snn::kBlock - 1) / snn::kBlock));
    if constexpr (MODE < 8) {   // SAVE_H has no affine-gradient variant (host rejects it)
        if (s->save_mode == SNN_SAVE_H) {
            return launch_kernel(snn::lif_backward_saveh_kernel<IO, VEC, MODE, kBwdPF>, grid, dim3(snn::kBlock),
                                 0, st, false, "lif_backward_saveh_kernel", a);
        }
    }
    return launch_kernel(snn::lif_backward_recompute_kernel<IO, VEC, MODE>, grid, dim3(snn::kBlock), 0, st,
                         false, "lif_backward_recompute_kernel", a);
}

template <typename IO, int VEC>
snn_status go(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    switch (mode & 15) {
        case 0: return go_mode<IO, VEC, 0>(s, a, st);
        case 1: return go_mode<IO, VEC, 1>(s, a, st);
        case 2: return go_mode<IO, VEC, 2>(s, a, st);
        case 3: return go_mode<IO, VEC, 3>(s, a, st);
        case 4: return go_mode<IO, VEC, 4>(s, a, st);
        case 5: return go_mode<IO, VEC, 5>(s, a, st);
        case 6: return go_mode<IO, VEC, 6>(s, a, st);
        case 7: return go_mode<IO, VEC, 7>(s, a, st);
        case 8: return go_mode<IO, VEC, 8>(s, a, st);
        case 9: return go_mode<IO, VEC, 9>(s, a, st);
        case 10: return go_mode<IO, VEC, 10>(s, a, st);
        case 11: return go_mode<IO, VEC, 11>(s, a, st);
        case 12: return go_mode<IO, VEC, 12>(s, a, st);
        case 13: return go_mode<IO, VEC, 13>(s, a, st);
        case 14: return go_mode<IO, VEC, 14>(s, a, st);
        default: return go_mode<IO, VEC, 15>(s, a, st);
    }
}
}  // namespace

snn_status launch_backward_generic(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool vec,
                                   cudaStream_t st) {
    if (s->io_dtype == SNN_BF16)
        return vec ? go<__nv_bfloat16, 2>(s, a, mode, st) : go<__nv_bfloat16, 1>(s, a, mode, st);
    return vec ? go<float, 2>(s, a, mode, st) : go<float, 1>(s, a, mode, st);
}

snn_status launch_affine_segment_finish(const float* seg_a, const float* seg_b, int64_t B, int64_t C, int64_t HW,
                                        int G, float* grad_scale, float* grad_shift, cudaStream_t st) {
    if (C > INT32_MAX) return fail(SNN_ERR_INVALID_VALUE, "affine: too many channels");
    return launch_pdl(snn::affine_segment_finish_kernel, dim3((unsigned)C), dim3(256), st,
                      "affine_segment_finish_kernel", seg_a, seg_b, B, C, (int64_t)(HW / G), grad_scale, grad_shift);
}

snn_status launch_affine_reduce(float* part_a, float* part_b, int64_t B, int64_t C, int64_t HW,
                                float* grad_scale, float* grad_shift, cudaStream_t st) {
    // pieces of >= 2048 elements, about 4 CTAs per SM over all channels
    const int64_t M = B * HW;
    int64_t S = std::max<int64_t>(1, std::min<int64_t>((M + 2047) / 2048, (4 * num_sms() + C - 1) / C));
    const int64_t L = (M + S - 1) / S;
    S = (M + L - 1) / L;                                 // every piece non-empty
    if (C > 65535) return fail(SNN_ERR_INVALID_VALUE, "affine: C > 65535 channels");
    snn_status r = launch_pdl(snn::affine_partial_kernel, dim3((unsigned)S, (unsigned)C), dim3(256), st,
                              "affine_partial_kernel", part_a, part_b, B, C, HW, L);
    if (r != SNN_OK) return r;
    return launch_pdl(snn::affine_finish_kernel, dim3((unsigned)((C + 7) / 8)), dim3(256), st,
                      "affine_finish_kernel", (const float*)part_a, (const float*)part_b, C, HW, L, S,
                      grad_scale, grad_shift);
}

}  // namespace snn_host
