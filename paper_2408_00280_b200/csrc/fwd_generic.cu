// fwd_generic.cu -- launcher of the generic forward kernels (lif_kernels.cuh): one thread
// per VEC-neuron group with a register prefetch ring along T.  Used when the TMA path's
// alignment requirements do not hold.
#include "internal.h"

namespace snn_host {

namespace {
constexpr int kFwdPF = 8;  // rows in flight per thread

template <typename IO, int VEC>
snn_status go(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, cudaStream_t st) {
    const int64_t groups = (s->N + VEC - 1) / VEC;
    const dim3 grid((unsigned)((groups + snn::kBlock - 1) / snn::kBlock));
    auto go_aff = [&](auto sfmt, auto save, auto sft, auto aff) {
        return launch_kernel(snn::lif_forward_kernel<IO, VEC, decltype(sfmt)::value, decltype(save)::value,
                                                     (bool)decltype(sft)::value, (bool)decltype(aff)::value, kFwdPF>,
                             grid, dim3(snn::kBlock), 0, st, false, "lif_forward_kernel", a);
    };
    auto launch = [&](auto sfmt, auto save, auto sft) {
        return a.af.scale != nullptr ? go_aff(sfmt, save, sft, IC<1>{}) : go_aff(sfmt, save, sft, IC<0>{});
    };
    auto by_soft = [&](auto sfmt, auto save) {
        return soft ? launch(sfmt, save, IC<1>{}) : launch(sfmt, save, IC<0>{});
    };
    auto by_save = [&](auto sfmt) {
        switch (s->save_mode) {
            case SNN_SAVE_H: return by_soft(sfmt, IC<snn::SAVE_H>{});
            case SNN_SAVE_RECOMPUTE: return by_soft(sfmt, IC<snn::SAVE_RECOMPUTE>{});
            default: return by_soft(sfmt, IC<snn::SAVE_NONE>{});
        }
    };
    switch (s->spike_fmt) {
        case SNN_SPK_U8: return by_save(IC<snn::SPK_U8>{});
        case SNN_SPK_BITS: return by_save(IC<snn::SPK_BITS>{});
        default: return by_save(IC<snn::SPK_IO>{});
    }
}
}  // namespace

snn_status launch_forward_generic(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool vec,
                                  cudaStream_t st) {
    if (s->io_dtype == SNN_BF16)
        return vec ? go<__nv_bfloat16, 4>(s, a, soft, st) : go<__nv_bfloat16, 1>(s, a, soft, st);
    return vec ? go<float, 4>(s, a, soft, st) : go<float, 1>(s, a, soft, st);
}

}  // namespace snn_host
