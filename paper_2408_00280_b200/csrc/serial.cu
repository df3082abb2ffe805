// serial.cu -- the paper's "Serial (CUDA)" baseline (Fig. 3; Fig. 5
// caption PAPER.md:419): ONE kernel launch per time step, the membrane state round-tripped
// through HBM between steps.  It is the comparison point temporal fusion removes, not the
// method: per neuron-step it moves X + V_in + V_out + S + H (forward) and gS + H + gV_in +
// gV_out + gX (backward) and pays T launches.  It runs the same per-step arithmetic as the
// fused kernels (lif_common.cuh), so fused == serial bitwise (tested).
#include "internal.h"

namespace snn {

template <typename IO, bool SOFT>
__global__ void __launch_bounds__(256)
lif_serial_forward_step_kernel(const IO* __restrict__ x_t, float* __restrict__ V, uint8_t* __restrict__ s_t,
                               float* __restrict__ h_t, int64_t N, LifConsts c) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float H = lif_charge(c, V[n], to_f32(x_t[n]));
    const bool S = lif_fire(c, H);
    V[n] = lif_reset<SOFT>(c, H, S);
    s_t[n] = (uint8_t)S;
    h_t[n] = H;
}

template <typename IO, int MODE>
__global__ void __launch_bounds__(256)
lif_serial_backward_step_kernel(const IO* __restrict__ gs_t, const float* __restrict__ h_t,
                                float* __restrict__ gV, IO* __restrict__ gx_t, int64_t N, LifConsts c) {
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const float gH = lif_grad_step<MODE>(c, h_t[n], to_f32(gs_t[n]), gV[n]);
    gx_t[n] = from_f32<IO>(__fmul_rn(c.s, gH));
    gV[n] = __fmul_rn(c.k, gH);
}

}  // namespace snn

namespace snn_host {

snn_status launch_serial_forward_step(int io_dtype, bool soft, const void* x_t, float* V, uint8_t* s_t,
                                      float* h_t, int64_t N, const snn::LifConsts& c, cudaStream_t st) {
    const dim3 grid((unsigned)((N + 255) / 256));
    auto go = [&](auto io, auto sft) {
        using IO = decltype(io);
        snn::lif_serial_forward_step_kernel<IO, (bool)decltype(sft)::value>
            <<<grid, 256, 0, st>>>(reinterpret_cast<const IO*>(x_t), V, s_t, h_t, N, c);
    };
    if (io_dtype == SNN_BF16) { if (soft) go(__nv_bfloat16{}, IC<1>{}); else go(__nv_bfloat16{}, IC<0>{}); }
    else { if (soft) go(float{}, IC<1>{}); else go(float{}, IC<0>{}); }
    return launch_status("lif_serial_forward_step_kernel");
}

snn_status launch_serial_backward_step(int io_dtype, int mode, const void* gs_t, const float* h_t,
                                       float* gV, void* gx_t, int64_t N, const snn::LifConsts& c,
                                       cudaStream_t st) {
    const dim3 grid((unsigned)((N + 255) / 256));
    auto go = [&](auto io, auto md) {
        using IO = decltype(io);
        snn::lif_serial_backward_step_kernel<IO, decltype(md)::value><<<grid, 256, 0, st>>>(
            reinterpret_cast<const IO*>(gs_t), h_t, gV, reinterpret_cast<IO*>(gx_t), N, c);
    };
    auto by_mode = [&](auto io) {
        switch (mode & 7) {
            case 0: go(io, IC<0>{}); break;
            case 1: go(io, IC<1>{}); break;
            case 2: go(io, IC<2>{}); break;
            case 3: go(io, IC<3>{}); break;
            case 4: go(io, IC<4>{}); break;
            case 5: go(io, IC<5>{}); break;
            case 6: go(io, IC<6>{}); break;
            default: go(io, IC<7>{}); break;
        }
    };
    if (io_dtype == SNN_BF16) by_mode(__nv_bfloat16{}); else by_mode(float{});
    return launch_status("lif_serial_backward_step_kernel");
}

}  // namespace snn_host
