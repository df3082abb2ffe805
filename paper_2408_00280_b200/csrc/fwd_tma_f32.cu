// fwd_tma_f32.cu -- instantiates the persistent TMA forward kernels for float io
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_forward_tma_f32(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, cudaStream_t st) {
    return launch_forward_tma<float>(s, a, soft, st);
}
}  // namespace snn_host
