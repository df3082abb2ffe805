// fwd_tma_f32.cu -- instantiates the persistent TMA forward kernels for float io, aligned rows
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_forward_tma_f32(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0, bool unal,
                                  cudaStream_t st) {
    if (unal) return launch_forward_tma_unal_f32(s, a, soft, p0, st);
    return launch_forward_tma<float, false>(s, a, soft, p0, st);
}
}  // namespace snn_host
