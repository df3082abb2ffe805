// bwd_generic.cu -- launcher of the generic backward kernels (lif_kernels.cuh).  Threads
// own 8 bytes of io per row (2 fp32 / 4 bf16 neurons): the RECOMPUTE walk keeps
// 2 x kCkpt rows of x and gS in registers, so a narrow group keeps occupancy up.
#include "internal.h"

namespace snn {
// ------------------------------------------------------------------------------------
// Affine prologue gradients: grad_scale[c] = sum_{b, hw} part_a[(b C + c) HW + hw], same for
// shift.  One CTA per channel, fixed per-thread strides and a fixed tree: deterministic.
__global__ void __launch_bounds__(256)
affine_reduce_kernel(const float* __restrict__ part_a, const float* __restrict__ part_b, int64_t B,
                     int64_t C, int64_t HW, float* __restrict__ grad_scale, float* __restrict__ grad_shift) {
    __shared__ float sa[256], sb[256];
    const int64_t ch = blockIdx.x;
    float acc_a = 0.0f, acc_b = 0.0f;
    const int64_t per = B * HW;
    for (int64_t i = threadIdx.x; i < per; i += blockDim.x) {
        const int64_t b = i / HW, hw = i % HW;
        const int64_t n = (b * C + ch) * HW + hw;
        acc_a = __fadd_rn(acc_a, part_a[n]);
        acc_b = __fadd_rn(acc_b, part_b[n]);
    }
    sa[threadIdx.x] = acc_a;
    sb[threadIdx.x] = acc_b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            sa[threadIdx.x] = __fadd_rn(sa[threadIdx.x], sa[threadIdx.x + w]);
            sb[threadIdx.x] = __fadd_rn(sb[threadIdx.x], sb[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        grad_scale[ch] = sa[0];
        grad_shift[ch] = sb[0];
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
            snn::lif_backward_saveh_kernel<IO, VEC, MODE, kBwdPF><<<grid, snn::kBlock, 0, st>>>(a);
            return launch_status("lif_backward_kernel");
        }
    }
    snn::lif_backward_recompute_kernel<IO, VEC, MODE><<<grid, snn::kBlock, 0, st>>>(a);
    return launch_status("lif_backward_kernel");
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
        return vec ? go<__nv_bfloat16, 4>(s, a, mode, st) : go<__nv_bfloat16, 1>(s, a, mode, st);
    return vec ? go<float, 2>(s, a, mode, st) : go<float, 1>(s, a, mode, st);
}

snn_status launch_affine_reduce(const float* part_a, const float* part_b, int64_t B, int64_t C,
                                int64_t HW, float* grad_scale, float* grad_shift, cudaStream_t st) {
    snn::affine_reduce_kernel<<<(unsigned)C, 256, 0, st>>>(part_a, part_b, B, C, HW, grad_scale, grad_shift);
    return launch_status("affine_reduce_kernel");
}

}  // namespace snn_host
