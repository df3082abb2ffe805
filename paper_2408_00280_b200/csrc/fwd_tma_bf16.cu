// fwd_tma_bf16.cu -- instantiates the persistent TMA forward kernels for __nv_bfloat16 io, aligned rows
// (one translation unit per variant family so the library builds in parallel).
#include "launch_tma.cuh"

namespace snn_host {
snn_status launch_forward_tma_bf16(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0, bool unal,
                                  cudaStream_t st) {
    if (unal) return launch_forward_tma_unal_bf16(s, a, soft, p0, st);
    return launch_forward_tma<__nv_bfloat16, false>(s, a, soft, p0, st);
}
}  // namespace snn_host
