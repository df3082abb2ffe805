// snn_lif_api.cu -- the C ABI of include/snn_lif.h: argument validation, variant
// selection and kernel launch.  The library never allocates, frees or synchronises.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <type_traits>
#include <utility>

#include "../../include/snn_lif.h"
#include "lif_kernels.cuh"

namespace {

thread_local char g_err[512] = "";

snn_status fail(snn_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
snn_status fail(snn_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

constexpr int64_t kLdhAlign = 16;  // saved-row stride alignment (elements)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

snn_status check_params(const snn_lif_params* p) {
    if (!p) return fail(SNN_ERR_NULL_POINTER, "params is NULL");
    if (!std::isfinite(p->tau) || !(p->tau >= 1.0f))
        return fail(SNN_ERR_INVALID_VALUE, "tau must be finite and >= 1 (got %g)", (double)p->tau);
    if (!std::isfinite(p->v_th) || !std::isfinite(p->v_reset) || !(p->v_th > p->v_reset))
        return fail(SNN_ERR_INVALID_VALUE, "need finite v_th > v_reset (got v_th=%g v_reset=%g)",
                    (double)p->v_th, (double)p->v_reset);
    if (!std::isfinite(p->alpha) || !(p->alpha > 0.0f))
        return fail(SNN_ERR_INVALID_VALUE, "alpha must be finite and > 0 (got %g)", (double)p->alpha);
    if (p->reset_mode != SNN_RESET_HARD && p->reset_mode != SNN_RESET_SOFT)
        return fail(SNN_ERR_INVALID_VALUE, "reset_mode %d", p->reset_mode);
    if (p->surrogate != SNN_SURR_SIGMOID && p->surrogate != SNN_SURR_ATAN)
        return fail(SNN_ERR_INVALID_VALUE, "surrogate %d", p->surrogate);
    if ((p->decay_input != 0 && p->decay_input != 1) || (p->detach_reset != 0 && p->detach_reset != 1))
        return fail(SNN_ERR_INVALID_VALUE, "decay_input / detach_reset must be 0 or 1");
    return SNN_OK;
}

snn_status check_shape(const snn_lif_shape* s) {
    if (!s) return fail(SNN_ERR_NULL_POINTER, "shape is NULL");
    if (s->T < 1 || s->N < 1) return fail(SNN_ERR_INVALID_VALUE, "T=%lld N=%lld must be >= 1",
                                          (long long)s->T, (long long)s->N);
    if (s->ld < s->N) return fail(SNN_ERR_INVALID_VALUE, "ld=%lld < N=%lld", (long long)s->ld,
                                  (long long)s->N);
    // T*ld (and T*ldh of the saved buffer) must fit in int64 byte offsets.
    const int64_t big = s->ld > s->N + kLdhAlign ? s->ld : s->N + kLdhAlign;
    if (s->T > (INT64_MAX / 8) / big)
        return fail(SNN_ERR_INVALID_VALUE, "dimension overflow: T*ld too large");
    if (s->io_dtype != SNN_F32 && s->io_dtype != SNN_BF16)
        return fail(SNN_ERR_INVALID_VALUE, "io_dtype %d", s->io_dtype);
    if (s->spike_fmt < SNN_SPK_U8 || s->spike_fmt > SNN_SPK_IO)
        return fail(SNN_ERR_INVALID_VALUE, "spike_fmt %d", s->spike_fmt);
    if (s->save_mode < SNN_SAVE_H || s->save_mode > SNN_SAVE_NONE)
        return fail(SNN_ERR_INVALID_VALUE, "save_mode %d", s->save_mode);
    return SNN_OK;
}

snn::LifConsts make_consts(const snn_lif_params* p) {
    snn::LifConsts c;
    const float inv_tau = 1.0f / p->tau;  // IEEE fp32 division
    c.k = 1.0f - inv_tau;
    c.s = p->decay_input ? inv_tau : 1.0f;
    c.c0 = p->v_reset * inv_tau;
    c.v_th = p->v_th;
    c.v_reset = p->v_reset;
    c.alpha = p->alpha;
    c.atan_c = 1.57079632679489662f * p->alpha;
    c.soft = p->reset_mode == SNN_RESET_SOFT;
    c.detach = p->detach_reset;
    return c;
}

int64_t saved_ld(const snn_lif_shape* s) { return round_up(s->N, kLdhAlign); }

int64_t saved_rows(const snn_lif_shape* s) {
    if (s->save_mode == SNN_SAVE_H) return s->T;
    if (s->save_mode == SNN_SAVE_RECOMPUTE) return (s->T + snn::kCkpt - 1) / snn::kCkpt;
    return 0;
}

size_t io_size(int dt) { return dt == SNN_BF16 ? 2 : 4; }

snn_status launch_status(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(SNN_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return SNN_OK;
}

template <int V> using IC = std::integral_constant<int, V>;

// Forward prefetch depth along T (rows in flight per thread).
constexpr int kFwdPF = 8;
constexpr int kBwdPF = 8;

template <typename IO, int VEC>
snn_status launch_forward(const snn_lif_shape* s, const snn::FwdArgs& a, cudaStream_t st) {
    const int64_t groups = (s->N + VEC - 1) / VEC;
    const dim3 grid((unsigned)((groups + snn::kBlock - 1) / snn::kBlock));
    auto go = [&](auto sfmt, auto save) {
        snn::lif_forward_kernel<IO, VEC, decltype(sfmt)::value, decltype(save)::value, kFwdPF>
            <<<grid, snn::kBlock, 0, st>>>(a);
    };
    auto by_save = [&](auto sfmt) {
        switch (s->save_mode) {
            case SNN_SAVE_H: go(sfmt, IC<snn::SAVE_H>{}); break;
            case SNN_SAVE_RECOMPUTE: go(sfmt, IC<snn::SAVE_RECOMPUTE>{}); break;
            default: go(sfmt, IC<snn::SAVE_NONE>{}); break;
        }
    };
    switch (s->spike_fmt) {
        case SNN_SPK_U8: by_save(IC<snn::SPK_U8>{}); break;
        case SNN_SPK_BITS: by_save(IC<snn::SPK_BITS>{}); break;
        default: by_save(IC<snn::SPK_IO>{}); break;
    }
    return launch_status("lif_forward_kernel");
}

template <typename IO, int VEC>
snn_status launch_backward(const snn_lif_shape* s, int surrogate, const snn::BwdArgs& a,
                           cudaStream_t st) {
    const int64_t groups = (s->N + VEC - 1) / VEC;
    const dim3 grid((unsigned)((groups + snn::kBlock - 1) / snn::kBlock));
    auto go = [&](auto surr) {
        constexpr int SURR = decltype(surr)::value;
        if (s->save_mode == SNN_SAVE_H)
            snn::lif_backward_saveh_kernel<IO, VEC, SURR, kBwdPF><<<grid, snn::kBlock, 0, st>>>(a);
        else
            snn::lif_backward_recompute_kernel<IO, VEC, SURR><<<grid, snn::kBlock, 0, st>>>(a);
    };
    if (surrogate == SNN_SURR_SIGMOID) go(IC<0>{}); else go(IC<1>{});
    return launch_status("lif_backward_kernel");
}

}  // namespace

extern "C" {

const char* snn_status_string(snn_status st) {
    switch (st) {
        case SNN_OK: return "SNN_OK";
        case SNN_ERR_INVALID_VALUE: return "SNN_ERR_INVALID_VALUE";
        case SNN_ERR_NULL_POINTER: return "SNN_ERR_NULL_POINTER";
        case SNN_ERR_MISALIGNED: return "SNN_ERR_MISALIGNED";
        case SNN_ERR_UNSUPPORTED: return "SNN_ERR_UNSUPPORTED";
        case SNN_ERR_CUDA: return "SNN_ERR_CUDA";
        case SNN_ERR_NCCL: return "SNN_ERR_NCCL";
    }
    return "SNN_ERR_UNKNOWN";
}

const char* snn_last_error_message(void) { return g_err; }

int snn_lif_abi_version(void) { return SNN_LIF_ABI_VERSION; }

size_t snn_lif_saved_bytes(const snn_lif_params* p, const snn_lif_shape* s) {
    if (check_params(p) != SNN_OK || check_shape(s) != SNN_OK) return 0;
    return (size_t)saved_rows(s) * (size_t)saved_ld(s) * sizeof(float);
}

snn_status snn_lif_forward(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                           const float* v_init, void* spikes, void* saved, float* v_final,
                           void* stream) {
    g_err[0] = 0;
    snn_status st;
    if ((st = check_params(p)) != SNN_OK) return st;
    if ((st = check_shape(s)) != SNN_OK) return st;
    if (!x) return fail(SNN_ERR_NULL_POINTER, "x is NULL");
    if (!spikes) return fail(SNN_ERR_NULL_POINTER, "spikes is NULL");
    if (s->save_mode != SNN_SAVE_NONE && !saved)
        return fail(SNN_ERR_NULL_POINTER, "saved is NULL but save_mode needs it");
    const size_t esz = io_size(s->io_dtype);
    const size_t ssz = s->spike_fmt == SNN_SPK_U8 ? 1 : s->spike_fmt == SNN_SPK_BITS ? 4 : esz;
    if (!aligned(x, esz) || !aligned(spikes, ssz) || (v_init && !aligned(v_init, 4)) ||
        (v_final && !aligned(v_final, 4)) || (saved && s->save_mode != SNN_SAVE_NONE && !aligned(saved, 16)))
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size "
                                        "(saved needs 16 B)");

    snn::FwdArgs a;
    a.x = x; a.v_init = v_init; a.spikes = spikes;
    a.saved = s->save_mode == SNN_SAVE_NONE ? nullptr : static_cast<float*>(saved);
    a.v_final = v_final;
    a.T = s->T; a.N = s->N; a.ld = s->ld; a.ldh = saved_ld(s); a.nwords = (s->N + 31) / 32;
    a.c = make_consts(p);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);

    const int vec = s->io_dtype == SNN_BF16 ? 8 : 4;
    bool fast = (s->ld % vec) == 0 && aligned(x, 16) && (!v_init || aligned(v_init, 16)) &&
                (!v_final || aligned(v_final, 16));
    if (s->spike_fmt == SNN_SPK_U8 || s->spike_fmt == SNN_SPK_IO) fast = fast && aligned(spikes, 16);
    if (s->io_dtype == SNN_BF16) {
        return fast ? launch_forward<__nv_bfloat16, 8>(s, a, cs)
                    : launch_forward<__nv_bfloat16, 1>(s, a, cs);
    }
    return fast ? launch_forward<float, 4>(s, a, cs) : launch_forward<float, 1>(s, a, cs);
}

snn_status snn_lif_backward(const snn_lif_params* p, const snn_lif_shape* s,
                            const void* grad_spikes, const void* x, const float* v_init,
                            const void* saved, const float* grad_v_final, void* grad_x,
                            float* grad_v_init, void* stream) {
    g_err[0] = 0;
    snn_status st;
    if ((st = check_params(p)) != SNN_OK) return st;
    if ((st = check_shape(s)) != SNN_OK) return st;
    if (s->save_mode == SNN_SAVE_NONE)
        return fail(SNN_ERR_INVALID_VALUE, "backward needs a forward run with SAVE_H or SAVE_RECOMPUTE");
    if (!grad_spikes) return fail(SNN_ERR_NULL_POINTER, "grad_spikes is NULL");
    if (!grad_x) return fail(SNN_ERR_NULL_POINTER, "grad_x is NULL");
    if (!saved) return fail(SNN_ERR_NULL_POINTER, "saved is NULL");
    if (s->save_mode == SNN_SAVE_RECOMPUTE && !x)
        return fail(SNN_ERR_NULL_POINTER, "x is required with SAVE_RECOMPUTE");
    const size_t esz = io_size(s->io_dtype);
    if (!aligned(grad_spikes, esz) || !aligned(grad_x, esz) || (x && !aligned(x, esz)) ||
        !aligned(saved, 16) || (grad_v_final && !aligned(grad_v_final, 4)) ||
        (grad_v_init && !aligned(grad_v_init, 4)))
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size "
                                        "(saved needs 16 B)");
    (void)v_init;  // the RECOMPUTE checkpoints already hold V[-1]

    snn::BwdArgs a;
    a.gS = grad_spikes; a.x = x; a.saved = static_cast<const float*>(saved);
    a.grad_v_final = grad_v_final; a.gX = grad_x; a.grad_v_init = grad_v_init;
    a.T = s->T; a.N = s->N; a.ld = s->ld; a.ldh = saved_ld(s);
    a.c = make_consts(p);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);

    // Backward threads own 8 bytes of io per row (2 fp32 / 4 bf16 neurons): the reverse
    // walk keeps 2 x kCkpt rows of x and gS in registers, so a narrower group keeps
    // occupancy up.
    const int vec = s->io_dtype == SNN_BF16 ? 4 : 2;
    const bool fast = (s->ld % vec) == 0 && aligned(grad_spikes, 16) && aligned(grad_x, 16) &&
                      (!x || s->save_mode != SNN_SAVE_RECOMPUTE || aligned(x, 16)) &&
                      (!grad_v_final || aligned(grad_v_final, 16)) &&
                      (!grad_v_init || aligned(grad_v_init, 16));
    if (s->io_dtype == SNN_BF16) {
        return fast ? launch_backward<__nv_bfloat16, 4>(s, p->surrogate, a, cs)
                    : launch_backward<__nv_bfloat16, 1>(s, p->surrogate, a, cs);
    }
    return fast ? launch_backward<float, 2>(s, p->surrogate, a, cs)
                : launch_backward<float, 1>(s, p->surrogate, a, cs);
}

}  // extern "C"
