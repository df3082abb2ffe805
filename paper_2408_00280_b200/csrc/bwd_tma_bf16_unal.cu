// bwd_tma_bf16_unal.cu -- the persistent TMA backward kernels for __nv_bfloat16 io rows that are not
// 16-byte aligned (1-D tensor maps; lif_tma.cuh UNAL).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_unal_bf16(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    return launch_backward_tma<__nv_bfloat16, true>(s, a, mode, st);
}
}  // namespace snn_host
