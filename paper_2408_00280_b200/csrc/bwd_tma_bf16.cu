// bwd_tma_bf16.cu -- instantiates the persistent TMA backward kernels for __nv_bfloat16 io, aligned rows
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_bf16(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool unal, cudaStream_t st) {
    if (unal) return launch_backward_tma_unal_bf16(s, a, mode, st);
    return launch_backward_tma<__nv_bfloat16, false>(s, a, mode, st);
}
}  // namespace snn_host
