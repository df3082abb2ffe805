// snn_lif_api.cu -- the C ABI of include/snn_lif.h: argument validation, constants,
// variant selection.  Kernel launches live in fwd_*/bwd_* translation units.
// The library never allocates, frees or synchronises.
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <mutex>
#include <utility>

#include "internal.h"
#include "trace.cuh"
#include "lif_handoff.cuh"

namespace snn_host {

namespace {
thread_local char g_err[512] = "";
thread_local char g_enc[256] = "";
}

snn_status fail(snn_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

Recorder*& current_recorder() {
    static thread_local Recorder* rec = nullptr;
    return rec;
}

snn_status replay(const RecordedLaunch& r, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = r.grid;
    cfg.blockDim = r.block;
    cfg.dynamicSmemBytes = r.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = r.pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelExC(&cfg, r.func, const_cast<void**>(r.args.data()));
    if (e != cudaSuccess) return fail(SNN_ERR_CUDA, "plan replay launch failed: %s", cudaGetErrorString(e));
    return launch_status("plan replay");
}

snn_status launch_status(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SNN_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return SNN_OK;
}

const SchedKnobs& sched_knobs() {
    static const SchedKnobs k = [] {
        SchedKnobs r;
        auto env = [](const char* n, int* v) {
            if (const char* e = std::getenv(n)) *v = std::atoi(e);
        };
        env("SNN_LIF_CLC_DEPTH", &r.max_depth);
        env("SNN_LIF_PREFETCH", &r.prefetch_max_stages);
        r.max_depth = std::max(1, std::min(r.max_depth, 4));
        return r;
    }();
    return k;
}

int num_sms() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return n;
}

// ---- tensor maps (TMA descriptors), encoded per call on the host --------------------

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}
}  // namespace

bool tma_available() { return encode_fn() != nullptr; }

bool encode_2d(CUtensorMap* m, const void* base, size_t esz, int64_t inner, int64_t outer,
               int64_t ld, int box_inner, int box_outer) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const CUtensorMapDataType dt = esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                            : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    const cuuint64_t strides[1] = {(cuuint64_t)(ld * (int64_t)esz)};
    const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    const cuuint32_t estr[2] = {1, 1};
    auto encode = [&] {
        return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    CUresult r = encode();
    if (r == CUDA_ERROR_INVALID_CONTEXT) {
        // A thread whose first CUDA call is this driver entry point (e.g. torch's autograd
        // worker) has no current context yet: let the runtime bind the device's primary one.
        cudaFree(nullptr);
        r = encode();
    }
    if (r != CUDA_SUCCESS)
        snprintf(g_enc, sizeof(g_enc), " [CUresult %d: base %p map %p dims %lld x %lld ld %lld box %d x %d]",
                 (int)r, base, (void*)m, (long long)inner, (long long)outer, (long long)ld, box_inner,
                 box_outer);
    return r == CUDA_SUCCESS;
}

const char* encode_detail() { return g_enc; }

int cached_occupancy(const void* k, int threads, int smem, int (*prep)(const void*, int, int)) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, k});
    if (it != cache.end()) return it->second;
    const int occ = prep(k, threads, smem);
    cache[{dev, k}] = occ;
    return occ;
}

int tma_vec_forward(int io_dtype) { return io_dtype == SNN_BF16 ? 8 : 4; }
int tma_vec_backward(int io_dtype) { return 2; }

}  // namespace snn_host

using namespace snn_host;

namespace {

constexpr int64_t kLdhAlign = 16;  // saved-row stride alignment (elements)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
size_t io_size(int dt) { return dt == SNN_BF16 ? 2 : 4; }

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
    if (s->T < 1 || s->N < 1)
        return fail(SNN_ERR_INVALID_VALUE, "T=%lld N=%lld must be >= 1", (long long)s->T, (long long)s->N);
    if (s->ld < s->N)
        return fail(SNN_ERR_INVALID_VALUE, "ld=%lld < N=%lld", (long long)s->ld, (long long)s->N);
    // T*ld (and T*ldh of the saved buffer) must fit in int64 byte offsets.
    const int64_t big = s->ld > s->N + kLdhAlign ? s->ld : s->N + kLdhAlign;
    if (s->T > (INT64_MAX / 8) / big) return fail(SNN_ERR_INVALID_VALUE, "dimension overflow: T*ld too large");
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
    c.ex2_scale = -p->alpha * 1.44269504088896341f;   // -alpha log2(e)
    c.atan_c = 1.57079632679489662f * p->alpha;        // pi/2 alpha
    c.half_alpha = 0.5f * p->alpha;
    return c;
}

int mode_of(const snn_lif_params* p) {
    return (p->surrogate == SNN_SURR_ATAN ? 1 : 0) | (p->reset_mode == SNN_RESET_SOFT ? 2 : 0) |
           (p->detach_reset ? 4 : 0);
}

int64_t saved_ld(const snn_lif_shape* s) { return round_up(s->N, kLdhAlign); }

int64_t saved_rows(const snn_lif_shape* s) {
    if (s->save_mode == SNN_SAVE_H) return s->T;
    if (s->save_mode == SNN_SAVE_RECOMPUTE) return (s->T + snn::kCkpt - 1) / snn::kCkpt;
    return 0;
}

// Which kernel family runs (SNN_LIF_NO_TMA=1 forces the generic kernels: tests cover both).
// The TMA kernels take every shape: rows of the io tensors ([T, ld]: x, grad_spikes, grad_x,
// spikes, residual) that are 16-B aligned with a 16-B row stride get 2-D tensor maps (ALIGNED);
// otherwise (odd ld, an unaligned column view) 1-D maps over the flat storage (UNALIGNED), whose
// int32 element coordinates bound T*ld.  [N] vectors and the saved state need no alignment
// beyond their element (saved: 16 B, validated).
enum class Path { GENERIC, ALIGNED, UNALIGNED };
Path tma_path(const snn_lif_shape* s, std::initializer_list<const void*> rows) {
    const char* e = std::getenv("SNN_LIF_NO_TMA");
    if ((e && e[0] == '1') || !tma_available()) return Path::GENERIC;
    if (s->N > INT32_MAX || s->T > INT32_MAX) return Path::GENERIC;
    const int64_t q = 16 / (int64_t)io_size(s->io_dtype);
    bool al = s->ld % q == 0;
    for (const void* p : rows)
        if (p && !aligned(p, 16)) al = false;
    if (al) return Path::ALIGNED;
    if (s->T > (INT32_MAX - 16) / s->ld) return Path::GENERIC;   // 1-D coordinates are int32
    return Path::UNALIGNED;
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

}  // extern "C"

namespace {

bool handoff_valid(const snn_lif_handoff* h) {
    if (!h) return true;
    if (h->epoch < 1) return false;
    if (h->recv_state && !h->recv_ready) return false;
    if (h->send_state && !h->send_ready) return false;
    if (h->send_state && !h->send_ack) return false;
    return true;
}

snn::Handoff to_dev(const snn_lif_handoff* h) {
    snn::Handoff d = {};
    if (h) {
        d.recv_state = h->recv_state; d.recv_ready = h->recv_ready; d.recv_ack = h->recv_ack;
        d.send_state = h->send_state; d.send_ready = h->send_ready; d.send_ack = h->send_ack;
        d.epoch = h->epoch;
    }
    return d;
}

bool affine_valid(const snn_lif_affine* af, const snn_lif_shape* s) {
    if (!af) return true;
    if (!af->scale || !af->shift || af->C < 1 || af->HW < 1) return false;
    if (af->C > INT64_MAX / af->HW || s->N % (af->C * af->HW) != 0) return false;
    return true;
}

snn::Affine to_dev(const snn_lif_affine* af) {
    snn::Affine d = {};
    if (af) {
        d.scale = af->scale; d.shift = af->shift; d.C = af->C; d.HW = af->HW;
        d.residual = af->residual; d.grad_residual = af->grad_residual;
    }
    return d;
}

}  // namespace

namespace snn_host {

#ifdef SNN_TRACE
// Trace builds only (trace.cuh): one device buffer of per-CTA records, allocated on first use.
static void* trace_buf() {
    static void* buf = nullptr;
    if (!buf && cudaMalloc(&buf, sizeof(snn::TraceBuf)) == cudaSuccess) cudaMemset(buf, 0, 64);
    return buf;
}
extern "C" int snn_trace_read(void* host, int max_records) {
    void* b = trace_buf();
    unsigned int n = 0;
    if (!b || cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(&n, b, sizeof(n), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    if (n > (unsigned)snn::kTraceRecords) n = snn::kTraceRecords;
    if ((int)n > max_records) n = (unsigned)max_records;
    if (n && cudaMemcpy(host, static_cast<char*>(b) + offsetof(snn::TraceBuf, rec), n * sizeof(snn::TraceRec),
                        cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    cudaMemset(b, 0, 64);
    cudaDeviceSynchronize();
    return (int)n;
}
#endif

snn_status forward_impl(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                        const float* v_init, const snn_lif_handoff* handoff, void* spikes, void* saved,
                        float* v_final, void* stream, const snn_lif_affine* affine, const ChunkView* cv) {
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
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size (saved needs 16 B)");

    snn::FwdArgs a{};
    a.x = x; a.v_init = v_init; a.spikes = spikes;
    a.saved = s->save_mode == SNN_SAVE_NONE ? nullptr : static_cast<float*>(saved);
    // RECOMPUTE checkpoint row 0 (V[-1]) is stored only for the fused handoff, where V[-1]
    // arrives from the neighbour inside the kernel.  Elsewhere it is v_init or V_reset, which
    // the backward entry points receive themselves: a layer with T <= 16 stores no checkpoint.
    a.ck0 = handoff != nullptr ? 1 : 0;
    a.v_final = v_final;
    a.T = s->T; a.N = s->N; a.ld = s->ld; a.ldh = saved_ld(s); a.nwords = (s->N + 31) / 32;
    a.spk_words_ld = a.nwords;
    if (cv) { a.ldh = cv->ldh; a.spk_words_ld = cv->spk_words_ld; }
#ifdef SNN_TRACE
    a.trace = trace_buf();
#endif
    a.c = make_consts(p);
    const bool soft = p->reset_mode == SNN_RESET_SOFT;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (!handoff_valid(handoff)) return fail(SNN_ERR_INVALID_VALUE, "handoff: epoch < 1 or missing flags");
    if (!affine_valid(affine, s))
        return fail(SNN_ERR_INVALID_VALUE, "affine: need scale/shift, C >= 1, HW >= 1, N %% (C*HW) == 0");
    a.h = to_dev(handoff);
    a.af = to_dev(affine);
    const void* res = affine ? affine->residual : nullptr;
    if (res) {
        if (!aligned(res, esz)) return fail(SNN_ERR_MISALIGNED, "residual is not aligned to its element size");
        if (s->save_mode == SNN_SAVE_H)
            return fail(SNN_ERR_UNSUPPORTED, "the residual prologue needs save_mode SAVE_RECOMPUTE or SAVE_NONE");
    }

    const Path path = tma_path(s, {x, s->spike_fmt == SNN_SPK_BITS ? nullptr : spikes, res});
    const bool p0 = !p->decay_input && p->v_reset == 0.0f;   // paper-mode constants (Mode::P0)
    if (path != Path::GENERIC)
        return s->io_dtype == SNN_BF16 ? launch_forward_tma_bf16(s, a, soft, p0, path == Path::UNALIGNED, cs)
                                       : launch_forward_tma_f32(s, a, soft, p0, path == Path::UNALIGNED, cs);
    if (res)
        return fail(SNN_ERR_UNSUPPORTED, "the residual prologue runs on the TMA kernels only (SNN_LIF_NO_TMA "
                                         "is set, or T*ld exceeds int32 coordinates with unaligned rows)");
    if (handoff)
        return fail(SNN_ERR_UNSUPPORTED, "the fused handoff runs on the TMA kernels only (SNN_LIF_NO_TMA is "
                                         "set, or T*ld exceeds int32 coordinates with unaligned rows)");
    const int vec = 4;   // bf16 and fp32: 4 neurons per thread (bf16 x 8 measured 5% slower, fp32 x 2 2x slower)
    bool fast = (s->ld % vec) == 0 && aligned(x, 16) && (!v_init || aligned(v_init, 16)) &&
                (!v_final || aligned(v_final, 16));
    if (s->spike_fmt == SNN_SPK_U8 || s->spike_fmt == SNN_SPK_IO) fast = fast && aligned(spikes, 16);
    return launch_forward_generic(s, a, soft, fast, cs);
}

snn_status backward_impl(const snn_lif_params* p, const snn_lif_shape* s,
                         const void* grad_spikes, const void* x, const float* v_init, const void* saved,
                         const float* grad_v_final, const snn_lif_handoff* handoff, void* grad_x,
                         float* grad_v_init, void* stream, const snn_lif_affine* affine,
                         float* part_a, float* part_b, const ChunkView* cv, int* seg_out) {
    if (seg_out) *seg_out = 0;
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
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size (saved needs 16 B)");
    snn::BwdArgs a{};
    a.gS = grad_spikes; a.x = x; a.saved = static_cast<const float*>(saved);
    a.grad_v_final = grad_v_final; a.gX = grad_x; a.grad_v_init = grad_v_init;
    a.T = s->T; a.N = s->N; a.ld = s->ld; a.ldh = cv ? cv->ldh : saved_ld(s);
    a.v_init = v_init;
    a.ck0 = handoff != nullptr ? 1 : 0;   // as forward_impl stored it
    if (v_init && !aligned(v_init, 4)) return fail(SNN_ERR_MISALIGNED, "v_init is not 4-byte aligned");
#ifdef SNN_TRACE
    a.trace = trace_buf();
#endif
    a.c = make_consts(p);
    int mode = mode_of(p);
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (!handoff_valid(handoff)) return fail(SNN_ERR_INVALID_VALUE, "handoff: epoch < 1 or missing flags");
    a.h = to_dev(handoff);
    if (affine) {
        if (!affine_valid(affine, s))
            return fail(SNN_ERR_INVALID_VALUE, "affine: need scale/shift, C >= 1, HW >= 1, N %% (C*HW) == 0");
        if (s->save_mode != SNN_SAVE_RECOMPUTE)
            return fail(SNN_ERR_UNSUPPORTED, "affine backward needs save_mode SAVE_RECOMPUTE");
        if (!part_a || !part_b) return fail(SNN_ERR_NULL_POINTER, "affine backward needs part_a / part_b");
        if (!aligned(part_a, 16) || !aligned(part_b, 16))
            return fail(SNN_ERR_MISALIGNED, "part_a / part_b must be 16-byte aligned");
        a.af = to_dev(affine);
        a.af.part_a = part_a;
        a.af.part_b = part_b;
        a.af.seg = 0;   // set below when the TMA kernels fold the channel reduction in
        mode |= 8;
        if ((affine->residual == nullptr) != (affine->grad_residual == nullptr))
            return fail(SNN_ERR_NULL_POINTER, "residual and grad_residual go together");
        if (affine->residual) {
            if (!aligned(affine->residual, esz) || !aligned(affine->grad_residual, esz))
                return fail(SNN_ERR_MISALIGNED, "residual / grad_residual not aligned to their element size");
            mode |= 16;
        }
    }
    const void* res = (mode & 16) ? affine->residual : nullptr;
    void* gres = (mode & 16) ? affine->grad_residual : nullptr;

    const Path path = tma_path(s, {grad_spikes, grad_x, s->save_mode == SNN_SAVE_RECOMPUTE ? x : nullptr, res, gres});
    if (path != Path::GENERIC) {
        // paper-mode constants on the RECOMPUTE path (plain, affine, residual): the P0 variants
        // (lif_common.cuh Mode::P0; the SAVE_H kernel has no P0 instantiation)
        const int tmode = (s->save_mode == SNN_SAVE_RECOMPUTE && !p->decay_input && p->v_reset == 0.0f)
                              ? (mode | 32) : mode;
        if (affine && seg_out) a.af.seg = *seg_out = affine_segment(affine->HW);
        return s->io_dtype == SNN_BF16 ? launch_backward_tma_bf16(s, a, tmode, path == Path::UNALIGNED, cs)
                                       : launch_backward_tma_f32(s, a, tmode, path == Path::UNALIGNED, cs);
    }
    if (res)
        return fail(SNN_ERR_UNSUPPORTED, "the residual prologue runs on the TMA kernels only (SNN_LIF_NO_TMA "
                                         "is set, or T*ld exceeds int32 coordinates with unaligned rows)");
    if (handoff)
        return fail(SNN_ERR_UNSUPPORTED, "the fused handoff runs on the TMA kernels only (SNN_LIF_NO_TMA is "
                                         "set, or T*ld exceeds int32 coordinates with unaligned rows)");
    const int vec = 2;   // bf16 and fp32: 2 neurons per thread (bf16 x 4 held too many registers)
    const bool fast = (s->ld % vec) == 0 && aligned(grad_spikes, 16) && aligned(grad_x, 16) &&
                      (!x || s->save_mode != SNN_SAVE_RECOMPUTE || aligned(x, 16)) &&
                      (!grad_v_final || aligned(grad_v_final, 16)) &&
                      (!grad_v_init || aligned(grad_v_init, 16));
    return launch_backward_generic(s, a, mode, fast, cs);
}

int64_t saved_row_stride(const snn_lif_shape* s) { return saved_ld(s); }

// Segment length of the affine reduction folded into the TMA backward's tile epilogue
// (lif_kernels.cuh affine_warp_segments): G = min(HW, 64) when it divides the channel block of
// HW neurons (HW a multiple of 64, or a power of two >= 2); 0 = the per-neuron partials + the
// two-pass reduction.
int affine_segment(int64_t HW) {
    if (HW >= snn::kSegMax) return HW % snn::kSegMax == 0 ? snn::kSegMax : 0;
    return (HW >= 2 && (HW & (HW - 1)) == 0) ? (int)HW : 0;
}

}  // namespace snn_host

extern "C" {

snn_status snn_lif_forward(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                           const float* v_init, void* spikes, void* saved, float* v_final,
                           void* stream) {
    NvtxRange r("snn_lif_forward");
    return forward_impl(p, s, x, v_init, nullptr, spikes, saved, v_final, stream);
}

snn_status snn_lif_backward(const snn_lif_params* p, const snn_lif_shape* s,
                            const void* grad_spikes, const void* x, const float* v_init,
                            const void* saved, const float* grad_v_final, void* grad_x,
                            float* grad_v_init, void* stream) {
    NvtxRange r("snn_lif_backward");
    return backward_impl(p, s, grad_spikes, x, v_init, saved, grad_v_final, nullptr, grad_x, grad_v_init, stream);
}

snn_status snn_lif_forward_affine(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                                  const float* v_init, const snn_lif_affine* af, void* spikes,
                                  void* saved, float* v_final, void* stream) {
    if (!af) return fail(SNN_ERR_NULL_POINTER, "affine is NULL");
    NvtxRange r("snn_lif_forward_affine");
    return forward_impl(p, s, x, v_init, nullptr, spikes, saved, v_final, stream, af);
}

snn_status snn_lif_backward_affine(const snn_lif_params* p, const snn_lif_shape* s,
                                   const void* grad_spikes, const void* x, const float* v_init, const void* saved,
                                   const float* grad_v_final, const snn_lif_affine* af, void* grad_x,
                                   float* grad_v_init, float* part_a, float* part_b,
                                   float* grad_scale, float* grad_shift, void* stream) {
    if (!af) return fail(SNN_ERR_NULL_POINTER, "affine is NULL");
    if (!grad_scale || !grad_shift) return fail(SNN_ERR_NULL_POINTER, "grad_scale / grad_shift is NULL");
    NvtxRange r("snn_lif_backward_affine");
    int seg = 0;
    snn_status st = backward_impl(p, s, grad_spikes, x, v_init, saved, grad_v_final, nullptr, grad_x, grad_v_init,
                                  stream, af, part_a, part_b, nullptr, &seg);
    if (st != SNN_OK) return st;
    if (seg > 0)   // the backward already reduced each tile into channel segments: one tiny finish
        return launch_affine_segment_finish(part_a, part_b, s->N / (af->C * af->HW), af->C, af->HW, seg,
                                            grad_scale, grad_shift, static_cast<cudaStream_t>(stream));
    return launch_affine_reduce(part_a, part_b, s->N / (af->C * af->HW), af->C, af->HW, grad_scale,
                                grad_shift, static_cast<cudaStream_t>(stream));
}

int64_t snn_lif_handoff_blocks(int64_t N) {
    return N < 1 ? 0 : (N + snn::kHandoffBlock - 1) / snn::kHandoffBlock;
}

snn_status snn_lif_forward_handoff(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                                   const float* v_init, const snn_lif_handoff* h, void* spikes,
                                   void* saved, float* v_final, void* stream) {
    if (!h) return fail(SNN_ERR_NULL_POINTER, "handoff is NULL");
    NvtxRange r("snn_lif_forward_handoff");
    return forward_impl(p, s, x, v_init, h, spikes, saved, v_final, stream);
}

snn_status snn_lif_backward_handoff(const snn_lif_params* p, const snn_lif_shape* s,
                                    const void* grad_spikes, const void* x, const void* saved,
                                    const float* grad_v_final, const snn_lif_handoff* h, void* grad_x,
                                    float* grad_v_init, void* stream) {
    if (!h) return fail(SNN_ERR_NULL_POINTER, "handoff is NULL");
    NvtxRange r("snn_lif_backward_handoff");
    return backward_impl(p, s, grad_spikes, x, nullptr, saved, grad_v_final, h, grad_x, grad_v_init, stream);
}

snn_status snn_lif_serial_forward_step(const snn_lif_params* p, int io_dtype, int64_t N,
                                       const void* x_t, float* v, uint8_t* spikes_t, float* h_t,
                                       void* stream) {
    g_err[0] = 0;
    snn_status st;
    if ((st = check_params(p)) != SNN_OK) return st;
    if (N < 1) return fail(SNN_ERR_INVALID_VALUE, "N=%lld must be >= 1", (long long)N);
    if (io_dtype != SNN_F32 && io_dtype != SNN_BF16) return fail(SNN_ERR_INVALID_VALUE, "io_dtype %d", io_dtype);
    if (!x_t || !v || !spikes_t || !h_t) return fail(SNN_ERR_NULL_POINTER, "a required pointer is NULL");
    if (!aligned(x_t, io_size(io_dtype)) || !aligned(v, 4) || !aligned(h_t, 4))
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size");
    return launch_serial_forward_step(io_dtype, p->reset_mode == SNN_RESET_SOFT, x_t, v, spikes_t, h_t, N,
                                      make_consts(p), static_cast<cudaStream_t>(stream));
}

snn_status snn_lif_serial_backward_step(const snn_lif_params* p, int io_dtype, int64_t N,
                                        const void* grad_spikes_t, const float* h_t, float* grad_v,
                                        void* grad_x_t, void* stream) {
    g_err[0] = 0;
    snn_status st;
    if ((st = check_params(p)) != SNN_OK) return st;
    if (N < 1) return fail(SNN_ERR_INVALID_VALUE, "N=%lld must be >= 1", (long long)N);
    if (io_dtype != SNN_F32 && io_dtype != SNN_BF16) return fail(SNN_ERR_INVALID_VALUE, "io_dtype %d", io_dtype);
    if (!grad_spikes_t || !h_t || !grad_v || !grad_x_t)
        return fail(SNN_ERR_NULL_POINTER, "a required pointer is NULL");
    const size_t esz = io_size(io_dtype);
    if (!aligned(grad_spikes_t, esz) || !aligned(grad_x_t, esz) || !aligned(h_t, 4) || !aligned(grad_v, 4))
        return fail(SNN_ERR_MISALIGNED, "a pointer is not aligned to its element size");
    return launch_serial_backward_step(io_dtype, mode_of(p), grad_spikes_t, h_t, grad_v, grad_x_t, N,
                                       make_consts(p), static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ---- plans: record once, replay many times (include/snn_lif.h snn_lif_plan_*) -----------

struct snn_lif_plan {
    int device = -1;
    bool has_backward = false;
    std::vector<snn_host::RecordedLaunch> fwd, bwd;
};

namespace {

// Run `body` with a Recorder installed on this thread; its launches land in `out`.
template <typename F>
snn_status record_into(std::vector<snn_host::RecordedLaunch>& out, F body) {
    snn_host::Recorder rec;
    snn_host::Recorder*& slot = snn_host::current_recorder();
    snn_host::Recorder* prev = slot;
    slot = &rec;
    const snn_status st = body();
    slot = prev;
    if (st == SNN_OK) out = std::move(rec.launches);
    return st;
}

snn_status replay_all(const snn_lif_plan* plan, const std::vector<snn_host::RecordedLaunch>& v, void* stream) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != plan->device)
        return fail(SNN_ERR_INVALID_VALUE, "plan was created on device %d, current device is %d", plan->device, dev);
    for (const auto& r : v) {
        const snn_status st = snn_host::replay(r, static_cast<cudaStream_t>(stream));
        if (st != SNN_OK) return st;
    }
    return SNN_OK;
}

}  // namespace

extern "C" {

snn_status snn_lif_plan_create(snn_lif_plan** out, const snn_lif_params* p, const snn_lif_shape* s,
                               const void* x, const float* v_init, void* spikes, void* saved,
                               float* v_final, const void* grad_spikes, const float* grad_v_final,
                               void* grad_x, float* grad_v_init) {
    g_err[0] = 0;
    if (!out) return fail(SNN_ERR_NULL_POINTER, "plan output pointer is NULL");
    *out = nullptr;
    if ((grad_spikes == nullptr) != (grad_x == nullptr))
        return fail(SNN_ERR_NULL_POINTER, "grad_spikes and grad_x go together (both NULL: forward-only plan)");
    auto plan = std::make_unique<snn_lif_plan>();
    snn_status st = record_into(plan->fwd, [&] {   // validation first: nothing touches the device on error
        return forward_impl(p, s, x, v_init, nullptr, spikes, saved, v_final, nullptr);
    });
    if (st != SNN_OK) return st;
    if (grad_spikes) {
        st = record_into(plan->bwd, [&] {
            return backward_impl(p, s, grad_spikes, x, v_init, saved, grad_v_final, nullptr, grad_x, grad_v_init,
                                 nullptr);
        });
        if (st != SNN_OK) return st;
        plan->has_backward = true;
    }
    if (cudaGetDevice(&plan->device) != cudaSuccess) return fail(SNN_ERR_CUDA, "cudaGetDevice failed");
    *out = plan.release();
    return SNN_OK;
}

snn_status snn_lif_plan_create_affine(snn_lif_plan** out, const snn_lif_params* p, const snn_lif_shape* s,
                                      const void* x, const float* v_init, const snn_lif_affine* af,
                                      void* spikes, void* saved, float* v_final, const void* grad_spikes,
                                      const float* grad_v_final, void* grad_x, float* grad_v_init,
                                      float* part_a, float* part_b, float* grad_scale, float* grad_shift) {
    g_err[0] = 0;
    if (!out) return fail(SNN_ERR_NULL_POINTER, "plan output pointer is NULL");
    *out = nullptr;
    if (!af) return fail(SNN_ERR_NULL_POINTER, "affine is NULL");
    if ((grad_spikes == nullptr) != (grad_x == nullptr))
        return fail(SNN_ERR_NULL_POINTER, "grad_spikes and grad_x go together (both NULL: forward-only plan)");
    auto plan = std::make_unique<snn_lif_plan>();
    snn_status st = record_into(plan->fwd, [&] {
        return snn_lif_forward_affine(p, s, x, v_init, af, spikes, saved, v_final, nullptr);
    });
    if (st != SNN_OK) return st;
    if (grad_spikes) {
        st = record_into(plan->bwd, [&] {
            return snn_lif_backward_affine(p, s, grad_spikes, x, v_init, saved, grad_v_final, af, grad_x, grad_v_init,
                                           part_a, part_b, grad_scale, grad_shift, nullptr);
        });
        if (st != SNN_OK) return st;
        plan->has_backward = true;
    }
    if (cudaGetDevice(&plan->device) != cudaSuccess) return fail(SNN_ERR_CUDA, "cudaGetDevice failed");
    *out = plan.release();
    return SNN_OK;
}

snn_status snn_lif_plan_forward(const snn_lif_plan* plan, void* stream) {
    g_err[0] = 0;
    if (!plan) return fail(SNN_ERR_NULL_POINTER, "plan is NULL");
    return replay_all(plan, plan->fwd, stream);
}

snn_status snn_lif_plan_backward(const snn_lif_plan* plan, void* stream) {
    g_err[0] = 0;
    if (!plan) return fail(SNN_ERR_NULL_POINTER, "plan is NULL");
    if (!plan->has_backward) return fail(SNN_ERR_INVALID_VALUE, "forward-only plan (created without grad buffers)");
    return replay_all(plan, plan->bwd, stream);
}

void snn_lif_plan_destroy(snn_lif_plan* plan) { delete plan; }

}  // extern "C"
