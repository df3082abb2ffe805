// internal.h -- host-side glue shared by the translation units of libsnn_lif.so
// (not part of the public ABI; include/snn_lif.h is).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <type_traits>
#include <vector>

#include "../../include/snn_lif.h"
#include "lif_kernels.cuh"

namespace snn_host {

// NVTX range over a C-ABI call (forward / backward / time-split chunks show up as
// named ranges in an Nsight timeline).  Header-only NVTX v3: without an attached tool a push /
// pop is a null function-pointer check.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Thread-local error detail (snn_last_error_message) + status.
snn_status fail(snn_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
snn_status launch_status(const char* what);

int num_sms();

// 2-D tensor map over a row-major [outer, inner] tensor (row stride ld elements);
// box = box_inner x box_outer elements; out-of-range elements read as zero.
bool encode_2d(CUtensorMap* m, const void* base, size_t esz, int64_t inner, int64_t outer,
               int64_t ld, int box_inner, int box_outer);
bool tma_available();
const char* encode_detail();   // why the last encode_2d on this thread failed

template <int V> using IC = std::integral_constant<int, V>;

// ---- launch recording (snn_lif_plan_*): with a Recorder installed on the calling thread,
// the launch helpers below store each launch -- kernel, geometry and a copy of every
// argument -- instead of enqueuing it; a plan replays them later with cudaLaunchKernelExC.
struct RecordedLaunch {
    const void* func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    bool pdl = false;
    std::vector<std::shared_ptr<void>> arg_store;   // one heap copy per parameter (alignment kept)
    std::vector<void*> args;                        // pointers into arg_store, in order
};
struct Recorder {
    std::vector<RecordedLaunch> launches;
};
Recorder*& current_recorder();   // thread-local; nullptr = launch immediately

template <typename P>
void record_arg(RecordedLaunch& r, const P& v) {
    std::shared_ptr<void> p(new P(v), [](void* q) { delete static_cast<P*>(q); });
    r.args.push_back(p.get());
    r.arg_store.push_back(std::move(p));
}

// SNN_LIF_NO_PDL=1: launch without programmatic dependent launch (A/B measurements only; the
// kernels' griddepcontrol instructions are no-ops then).
inline bool pdl_disabled() {
    static const bool off = [] {
        const char* e = std::getenv("SNN_LIF_NO_PDL");
        return e && e[0] == '1';
    }();
    return off;
}

// Launch kernel `k` (PDL attribute when `pdl`), or record it when a Recorder is installed.
template <typename... Params, typename... Args>
snn_status launch_kernel(void (*k)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                         bool pdl, const char* what, const Args&... args) {
    static_assert(sizeof...(Params) == sizeof...(Args), "kernel arity");
    if (Recorder* rec = current_recorder()) {
        RecordedLaunch r;
        r.func = reinterpret_cast<const void*>(k);
        r.grid = grid; r.block = block; r.smem = smem; r.pdl = pdl;
        (record_arg<std::remove_cv_t<std::remove_reference_t<Params>>>(r, args), ...);
        rec->launches.push_back(std::move(r));
        return SNN_OK;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (lif_async.cuh)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl && !pdl_disabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k, static_cast<Params>(args)...);
    if (e != cudaSuccess) return fail(SNN_ERR_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
    return launch_status(what);
}

// Replay one recorded launch on `st`.
snn_status replay(const RecordedLaunch& r, cudaStream_t st);

// Opt the kernel into its dynamic shared memory and return resident CTAs per SM.
template <typename Kernel>
int prepare(Kernel k, int threads, int smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem) != cudaSuccess || occ < 1)
        occ = 1;
    return occ;
}

// Resident CTAs per SM of kernel `k` (cudaFuncSetAttribute + occupancy query), cached per
// (device, kernel) -- the attribute must be set once per kernel, not per signature.
int cached_occupancy(const void* k, int threads, int smem, int (*prep)(const void*, int, int));

// Tile launch: one CTA per tile; resident CTAs steal the tiles of pending CTAs through
// cluster launch control (lif_tma.cuh), so the grid behaves persistently, with one steal
// request in flight.  Short tiles (<= 4 ring stages) L2-prefetch the CTA's own first ring
// stages before griddepcontrol.wait (hides the first DRAM round trip behind the predecessor's
// tail; measured +4% on cfg2, but -3% sustained when tiles of 8 or more stages do, T >= 128;
// an evict-first hint on the prefetch does not change that).
// Environment overrides (A/B timing, tools/trace_timeline.py): SNN_LIF_CLC_DEPTH (requests
// in flight, 1..4), SNN_LIF_PREFETCH (0: never prefetch; >0: prefetch tiles of up to that
// many stages).
struct SchedKnobs {
    int max_depth = 1;
    int prefetch_max_stages = 4;
};
const SchedKnobs& sched_knobs();

template <typename Kernel, typename... Args>
snn_status launch_tiles(Kernel k, int threads, int smem, int64_t ntiles, int64_t stages_per_tile,
                        cudaStream_t st, const char* what, const Args&... args) {
    const int occ = cached_occupancy(reinterpret_cast<const void*>(k), threads, smem, [](const void* kk, int t, int sm) {
        return prepare(reinterpret_cast<Kernel>(const_cast<void*>(kk)), t, sm);
    });
    if (ntiles > INT32_MAX) return fail(SNN_ERR_INVALID_VALUE, "too many tiles");
    const SchedKnobs& kn = sched_knobs();
    const int64_t resident = (int64_t)occ * num_sms();
    snn::Sched sc;
    // Steal requests in flight: none when every CTA is resident from the start (nothing can
    // ever be pending, and a CTA would only wait for the failed responses before exiting).
    sc.depth = ntiles <= resident
                   ? 0
                   : (int)std::max<int64_t>(1, std::min<int64_t>(kn.max_depth, (8 + stages_per_tile - 1) / stages_per_tile));
    sc.prefetch = stages_per_tile <= kn.prefetch_max_stages ? 1 << 20 : 0;
    return launch_kernel(k, dim3((unsigned)ntiles), dim3(threads), (size_t)smem, st, true, what, args..., sc);
}

// Plain launch with programmatic dependent launch allowed: the kernel must call pdl_wait()
// before touching global memory.
template <typename Kernel, typename... Args>
snn_status launch_pdl(Kernel k, dim3 grid, dim3 block, cudaStream_t st, const char* what,
                      const Args&... args) {
    return launch_kernel(k, grid, block, 0, st, true, what, args...);
}

// ---- the validated entry points behind the C ABI (snn_lif_api.cu) --------------------
// A launch over a neuron chunk [a, a + n) of a wider layer passes the chunk's shape and
// pointers (x + a, spikes + a, ...) plus the whole layer's row strides of the saved state and
// of bit-packed spike rows (the time split, comm.cu).
struct ChunkView {
    int64_t ldh;            // saved-state row stride (floats) of the whole layer
    int64_t spk_words_ld;   // bit-packed spike row stride (uint32 words) of the whole layer
};
snn_status forward_impl(const snn_lif_params* p, const snn_lif_shape* s, const void* x,
                        const float* v_init, const snn_lif_handoff* handoff, void* spikes, void* saved,
                        float* v_final, void* stream, const snn_lif_affine* affine = nullptr,
                        const ChunkView* cv = nullptr);
snn_status backward_impl(const snn_lif_params* p, const snn_lif_shape* s, const void* grad_spikes,
                         const void* x, const float* v_init, const void* saved, const float* grad_v_final,
                         const snn_lif_handoff* handoff, void* grad_x, float* grad_v_init, void* stream,
                         const snn_lif_affine* affine = nullptr, float* part_a = nullptr,
                         float* part_b = nullptr, const ChunkView* cv = nullptr, int* seg_out = nullptr);
int affine_segment(int64_t HW);
int64_t saved_row_stride(const snn_lif_shape* s);   // round_up(N, 16)

// ---- launchers (one translation unit each, compiled in parallel) -------------------
// Generic path: any alignment; `vec` selects the 128-bit vector variant.
snn_status launch_forward_generic(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool vec,
                                  cudaStream_t st);
snn_status launch_backward_generic(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool vec,
                                   cudaStream_t st);
// TMA path, any N; unal = the io rows are not 16-B aligned (1-D tensor maps).  The _unal
// halves live in their own translation units (parallel build).
// p0: paper-mode constants (decay_input = 0, V_reset = 0) -- the prologue variants' short charge.
snn_status launch_forward_tma_f32(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0, bool unal,
                                  cudaStream_t st);
snn_status launch_forward_tma_bf16(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0, bool unal,
                                   cudaStream_t st);
snn_status launch_backward_tma_f32(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool unal, cudaStream_t st);
snn_status launch_backward_tma_bf16(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, bool unal, cudaStream_t st);
snn_status launch_forward_tma_unal_f32(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0,
                                       cudaStream_t st);
snn_status launch_forward_tma_unal_bf16(const snn_lif_shape* s, const snn::FwdArgs& a, bool soft, bool p0,
                                        cudaStream_t st);
snn_status launch_backward_tma_unal_f32(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st);
snn_status launch_backward_tma_unal_bf16(const snn_lif_shape* s, const snn::BwdArgs& a, int mode, cudaStream_t st);
int tma_vec_forward(int io_dtype);
// Channel sums of the per-tile segment partials of the fused affine backward (G neurons each).
snn_status launch_affine_segment_finish(const float* seg_a, const float* seg_b, int64_t B, int64_t C, int64_t HW,
                                        int G, float* grad_scale, float* grad_shift, cudaStream_t st);
// part_a / part_b are scratch: the reduction overwrites some of their entries.
snn_status launch_affine_reduce(float* part_a, float* part_b, int64_t B, int64_t C,
                                int64_t HW, float* grad_scale, float* grad_shift, cudaStream_t st);
// Serial (one launch per time step) baseline of Fig. 3 -- comparison only (serial.cu).
snn_status launch_serial_forward_step(int io_dtype, bool soft, const void* x_t, float* V, uint8_t* s_t,
                                      float* h_t, int64_t N, const snn::LifConsts& c, cudaStream_t st);
snn_status launch_serial_backward_step(int io_dtype, int mode, const void* gs_t, const float* h_t,
                                       float* gV, void* gx_t, int64_t N, const snn::LifConsts& c,
                                       cudaStream_t st);
int tma_vec_backward(int io_dtype);

}  // namespace snn_host
