// bwd_tma_f32_unal.cu -- the persistent TMA backward kernels for float io rows that are not
// 16-byte aligned (1-D tensor maps; lif_tma.cuh UNAL).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_unal_f32(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    return launch_backward_tma<float, true>(s, a, mode, st);
}
}  // namespace snn_host
