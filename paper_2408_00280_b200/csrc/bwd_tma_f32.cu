// bwd_tma_f32.cu -- instantiates the persistent TMA backward kernels for float io, aligned rows
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_f32(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool unal, cudaStream_t st) {
    if (unal) return launch_backward_tma_unal_f32(s, a, mode, st);
    return launch_backward_tma<float, false>(s, a, mode, st);
}
}  // namespace snn_host
