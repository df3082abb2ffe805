// bwd_tma_f32.cu -- instantiates the persistent TMA backward kernels for float io
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_f32(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    return launch_backward_tma<float>(s, a, mode, st);
}
}  // namespace snn_host
