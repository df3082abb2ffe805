// bwd_generic.cu -- launcher of the generic backward kernels (lif_kernels.cuh).  Threads
// own 8 bytes of io per row (2 fp32 / 4 bf16 neurons): the RECOMPUTE walk keeps
// 2 x kCkpt rows of x and gS in registers, so a narrow group keeps occupancy up.
#include "internal.h"

namespace snn_host {

namespace {
constexpr int kBwdPF = 8;

template <typename IO, int VEC, int MODE>
snn_status go_mode(const snn_lif_shape* s, const snn::BwdArgs& a, cudaStream_t st) {
    const int64_t groups = (s->N + VEC - 1) / VEC;
    const dim3 grid((unsigned)((groups + snn::kBlock - 1) / snn::kBlock));
    if (s->save_mode == SNN_SAVE_H)
        snn::lif_backward_saveh_kernel<IO, VEC, MODE, kBwdPF><<<grid, snn::kBlock, 0, st>>>(a);
    else
        snn::lif_backward_recompute_kernel<IO, VEC, MODE><<<grid, snn::kBlock, 0, st>>>(a);
    return launch_status("lif_backward_kernel");
}

template <typename IO, int VEC>
snn_status go(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    switch (mode & 7) {
        case 0: return go_mode<IO, VEC, 0>(s, a, st);
        case 1: return go_mode<IO, VEC, 1>(s, a, st);
        case 2: return go_mode<IO, VEC, 2>(s, a, st);
        case 3: return go_mode<IO, VEC, 3>(s, a, st);
        case 4: return go_mode<IO, VEC, 4>(s, a, st);
        case 5: return go_mode<IO, VEC, 5>(s, a, st);
        case 6: return go_mode<IO, VEC, 6>(s, a, st);
        default: return go_mode<IO, VEC, 7>(s, a, st);
    }
}
}  // namespace

snn_status launch_backward_generic(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool vec,
                                   cudaStream_t st) {
    if (s->io_dtype == SNN_BF16)
        return vec ? go<__nv_bfloat16, 4>(s, a, mode, st) : go<__nv_bfloat16, 1>(s, a, mode, st);
    return vec ? go<float, 2>(s, a, mode, st) : go<float, 1>(s, a, mode, st);
}

}  // namespace snn_host
