// bwd_tma_bf16.cu -- instantiates the persistent TMA backward kernels for __nv_bfloat16 io
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_backward_tma_bf16(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st) {
    return launch_backward_tma<__nv_bfloat16>(s, a, mode, st);
}
}  // namespace snn_host
