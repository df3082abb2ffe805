// host_stream.cu -- snn_lif_fwd_bwd_host: a layer's forward + backward over HOST buffers,
// streamed through device staging slots in neuron chunks (include/snn_lif.h).  Pure runtime:
// every element of the path still runs in the kernels behind snn_lif_forward/backward; this
// file only orders 2-D copies and launches on three streams so that host->device,
// the kernels and device->host overlap (neurons are independent).
#include <cstdint>

#include "internal.h"

namespace snn_host {
namespace {

constexpr int64_t kChunkAlign = 512;   // whole TMA tiles, whole 32-bit spike words
constexpr size_t kAlign = 256;

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Plan {
    int64_t nc = 0;          // neurons per chunk (last one may be shorter)
    int64_t nch = 0;         // chunk count
    int nslots = 0;
    size_t esz = 0;
    // per-slot byte offsets and the slot size
    size_t off_x = 0, off_g = 0, off_s = 0, off_gx = 0, off_saved = 0, slot = 0;
    snn_lif_shape cs{};      // shape of a full chunk in its slot (ld = nc)
};

size_t spike_row_bytes(const snn_lif_shape* s, int64_t n, int64_t ld) {
    switch (s->spike_fmt) {
        case SNN_SPK_U8: return (size_t)ld;
        case SNN_SPK_BITS: return (size_t)((n + 31) / 32) * 4;
        default: return (size_t)ld * (s->io_dtype == SNN_BF16 ? 2 : 4);
    }
}

bool make_plan(const snn_lif_params* p, const snn_lif_shape* s, int64_t chunk_neurons, int nslots,
               Plan* pl) {
    if (!p || !s || s->T < 1 || s->N < 1 || s->ld < s->N) return false;
    pl->esz = s->io_dtype == SNN_BF16 ? 2 : 4;
    int64_t nc = chunk_neurons;
    if (nc <= 0) nc = (int64_t)((32ull << 20) / ((size_t)s->T * pl->esz));
    nc = std::max<int64_t>(kChunkAlign, (nc + kChunkAlign - 1) / kChunkAlign * kChunkAlign);
    nc = std::min<int64_t>(nc, (s->N + kChunkAlign - 1) / kChunkAlign * kChunkAlign);
    pl->nc = nc;
    pl->nch = (s->N + nc - 1) / nc;
    pl->nslots = nslots <= 0 ? 3 : nslots;
    if (pl->nslots < 2 || pl->nslots > 8) return false;
    pl->nslots = (int)std::min<int64_t>(pl->nslots, std::max<int64_t>(2, pl->nch));
    pl->cs = *s;
    pl->cs.N = nc;
    pl->cs.ld = nc;
    const size_t tensor = round_up((size_t)s->T * nc * pl->esz, kAlign);
    pl->off_x = 0;
    pl->off_g = pl->off_x + tensor;
    pl->off_gx = pl->off_g + tensor;
    pl->off_s = pl->off_gx + tensor;
    pl->off_saved = pl->off_s + round_up((size_t)s->T * spike_row_bytes(s, nc, nc), kAlign);
    pl->slot = pl->off_saved + round_up(snn_lif_saved_bytes(p, &pl->cs), kAlign);
    return true;
}

struct Resources {   // streams / events of one call (created and destroyed inside it)
    cudaStream_t in = nullptr, out = nullptr;
    cudaStream_t caller = nullptr;   // the caller's kernel stream (its queued chunks read the slots)
    cudaEvent_t start = nullptr;
    cudaEvent_t ready[8] = {}, computed[8] = {}, drained[8] = {};
    ~Resources() {
        // Every exit -- success or an error half-way through the chunk loop -- first drains
        // the copies and kernels already queued: they read and write the caller's host
        // buffers and workspace, which the caller may free as soon as this call returns.
        if (in) cudaStreamSynchronize(in);
        if (caller) cudaStreamSynchronize(caller);
        if (out) cudaStreamSynchronize(out);
        for (int i = 0; i < 8; ++i) {
            if (ready[i]) cudaEventDestroy(ready[i]);
            if (computed[i]) cudaEventDestroy(computed[i]);
            if (drained[i]) cudaEventDestroy(drained[i]);
        }
        if (start) cudaEventDestroy(start);
        if (in) cudaStreamDestroy(in);
        if (out) cudaStreamDestroy(out);
    }
};

#define SNN_CUDA_TRY(expr, what)                                                          \
    do {                                                                                  \
        const cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess) return fail(SNN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

}  // namespace
}  // namespace snn_host

using namespace snn_host;

extern "C" {

size_t snn_lif_host_workspace_bytes(const snn_lif_params* p, const snn_lif_shape* s,
                                    int64_t chunk_neurons, int nslots) {
    Plan pl;
    if (!make_plan(p, s, chunk_neurons, nslots, &pl)) return 0;
    return pl.slot * (size_t)pl.nslots;
}

snn_status snn_lif_fwd_bwd_host(const snn_lif_params* p, const snn_lif_shape* s, const void* x_host,
                                const void* g_host, void* spikes_host, void* gx_host,
                                int64_t chunk_neurons, int nslots, void* workspace,
                                size_t workspace_bytes, void* stream) {
    if (!p || !s) return fail(SNN_ERR_NULL_POINTER, "params / shape is NULL");
    if (!x_host || !g_host || !spikes_host || !gx_host || !workspace)
        return fail(SNN_ERR_NULL_POINTER, "a host buffer or the workspace is NULL");
    if (s->T < 1 || s->N < 1 || s->ld < s->N) return fail(SNN_ERR_INVALID_VALUE, "need T, N >= 1 and ld >= N");
    if (s->save_mode != SNN_SAVE_H && s->save_mode != SNN_SAVE_RECOMPUTE)
        return fail(SNN_ERR_INVALID_VALUE, "save_mode must be SAVE_H or SAVE_RECOMPUTE");
    Plan pl;
    if (!make_plan(p, s, chunk_neurons, nslots, &pl))
        return fail(SNN_ERR_INVALID_VALUE, "bad chunk_neurons / nslots (nslots in [2, 8])");
    if (workspace_bytes < pl.slot * (size_t)pl.nslots)
        return fail(SNN_ERR_INVALID_VALUE, "workspace too small: %zu < %zu bytes", workspace_bytes,
                    pl.slot * (size_t)pl.nslots);
    if (reinterpret_cast<uintptr_t>(workspace) % kAlign != 0)
        return fail(SNN_ERR_MISALIGNED, "workspace must be 256-byte aligned");

    NvtxRange range("snn_lif_fwd_bwd_host");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    Resources r;
    r.caller = cs;
    SNN_CUDA_TRY(cudaStreamCreateWithFlags(&r.in, cudaStreamNonBlocking), "cudaStreamCreate");
    SNN_CUDA_TRY(cudaStreamCreateWithFlags(&r.out, cudaStreamNonBlocking), "cudaStreamCreate");
    SNN_CUDA_TRY(cudaEventCreateWithFlags(&r.start, cudaEventDisableTiming), "cudaEventCreate");
    for (int i = 0; i < pl.nslots; ++i) {
        SNN_CUDA_TRY(cudaEventCreateWithFlags(&r.ready[i], cudaEventDisableTiming), "cudaEventCreate");
        SNN_CUDA_TRY(cudaEventCreateWithFlags(&r.computed[i], cudaEventDisableTiming), "cudaEventCreate");
        SNN_CUDA_TRY(cudaEventCreateWithFlags(&r.drained[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    // the workspace may still be in use by earlier work on the caller's stream
    SNN_CUDA_TRY(cudaEventRecord(r.start, cs), "cudaEventRecord");
    SNN_CUDA_TRY(cudaStreamWaitEvent(r.in, r.start, 0), "cudaStreamWaitEvent");

    const size_t hrow = (size_t)s->ld * pl.esz;                  // host row pitch of x / g / gx
    const size_t hspk = spike_row_bytes(s, s->N, s->ld);         // host row pitch of spikes
    unsigned char* ws = static_cast<unsigned char*>(workspace);
    for (int64_t c = 0; c < pl.nch; ++c) {
        const int sl = (int)(c % pl.nslots);
        const int64_t n0 = c * pl.nc, n = std::min<int64_t>(pl.nc, s->N - n0);
        unsigned char* base = ws + (size_t)sl * pl.slot;
        void* dx = base + pl.off_x;
        void* dg = base + pl.off_g;
        void* dgx = base + pl.off_gx;
        void* ds = base + pl.off_s;
        void* dsaved = base + pl.off_saved;
        snn_lif_shape sh = pl.cs;
        sh.N = n;                                                // ld stays nc (slot pitch)
        const size_t drow = (size_t)pl.nc * pl.esz;
        const size_t width = (size_t)n * pl.esz;

        // host -> device, once the slot's previous chunk has left the device
        if (c >= pl.nslots) SNN_CUDA_TRY(cudaStreamWaitEvent(r.in, r.drained[sl], 0), "cudaStreamWaitEvent");
        SNN_CUDA_TRY(cudaMemcpy2DAsync(dx, drow, static_cast<const unsigned char*>(x_host) + n0 * pl.esz,
                                       hrow, width, s->T, cudaMemcpyHostToDevice, r.in), "copy x in");
        SNN_CUDA_TRY(cudaMemcpy2DAsync(dg, drow, static_cast<const unsigned char*>(g_host) + n0 * pl.esz,
                                       hrow, width, s->T, cudaMemcpyHostToDevice, r.in), "copy grad_spikes in");
        SNN_CUDA_TRY(cudaEventRecord(r.ready[sl], r.in), "cudaEventRecord");

        // the fused kernels on the caller's stream
        SNN_CUDA_TRY(cudaStreamWaitEvent(cs, r.ready[sl], 0), "cudaStreamWaitEvent");
        snn_status st = snn_lif_forward(p, &sh, dx, nullptr, ds, dsaved, nullptr, stream);
        if (st != SNN_OK) return st;   // ~Resources drains every queued copy first
        st = snn_lif_backward(p, &sh, dg, dx, nullptr, dsaved, nullptr, dgx, nullptr, stream);
        if (st != SNN_OK) return st;
        SNN_CUDA_TRY(cudaEventRecord(r.computed[sl], cs), "cudaEventRecord");

        // device -> host
        SNN_CUDA_TRY(cudaStreamWaitEvent(r.out, r.computed[sl], 0), "cudaStreamWaitEvent");
        const size_t srow_dev = spike_row_bytes(s, n, pl.nc);   // bits rows: ceil(n/32) words
        const size_t sw = s->spike_fmt == SNN_SPK_BITS ? (size_t)((n + 31) / 32) * 4
                        : s->spike_fmt == SNN_SPK_U8 ? (size_t)n : width;
        const size_t soff = s->spike_fmt == SNN_SPK_BITS ? (size_t)(n0 / 32) * 4
                          : s->spike_fmt == SNN_SPK_U8 ? (size_t)n0 : (size_t)n0 * pl.esz;
        SNN_CUDA_TRY(cudaMemcpy2DAsync(static_cast<unsigned char*>(spikes_host) + soff, hspk, ds, srow_dev,
                                       sw, s->T, cudaMemcpyDeviceToHost, r.out), "copy spikes out");
        SNN_CUDA_TRY(cudaMemcpy2DAsync(static_cast<unsigned char*>(gx_host) + n0 * pl.esz, hrow, dgx, drow,
                                       width, s->T, cudaMemcpyDeviceToHost, r.out), "copy grad_x out");
        SNN_CUDA_TRY(cudaEventRecord(r.drained[sl], r.out), "cudaEventRecord");
    }
    SNN_CUDA_TRY(cudaStreamSynchronize(r.out), "cudaStreamSynchronize");
    SNN_CUDA_TRY(cudaStreamSynchronize(cs), "cudaStreamSynchronize");
    return SNN_OK;
}

}  // extern "C"
