// fwd_tma_f32_unal.cu -- the persistent TMA forward kernels for float io rows that are not
// 16-byte aligned (1-D tensor maps; lif_tma.cuh UNAL).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_forward_tma_unal_f32(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0,
                                       cudaStream_t st) {
    return launch_forward_tma<float, true>(s, a, soft, p0, st);
}
}  // namespace snn_host
