// trace.cuh -- per-CTA timeline stamps of the TMA kernels, compiled in only with
// -DSNN_TRACE (tools/variant_build.py --name trace -DSNN_TRACE builds that variant as a separate library; the product
// library has none of this).  Each CTA claims one record with an atomic and its first consumer
// warp writes: kernel kind, grid size, SM id, T, N, %globaltimer at entry, after
// griddepcontrol.wait, when the first ring stage landed, at exit, and the tiles it ran.
// The buffer pointer rides in FwdArgs/BwdArgs::trace (set by forward_impl/backward_impl);
// read back with snn_trace_read (snn_lif_api.cu, SNN_TRACE builds only).
#pragma once

#include <stdint.h>

namespace snn {

#ifdef SNN_TRACE
constexpr int kTraceRecords = 1 << 16;
struct TraceRec {
    uint32_t kind, grid, smid, tiles;
    int64_t T, N;
    uint64_t t_entry, t_wait, t_first, t_end;
    int32_t first_stolen, last_tile;   // tile indices: the first taken over from a pending CTA, the last run
    uint64_t t_issue;                  // the producer issued the first stage's loads
};
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
__device__ __forceinline__ uint64_t* trace_issue_slot() {
    __shared__ uint64_t slot;
    return &slot;
}
// producer: stamp the first issue (the slot is zeroed by thread 0 before the CTA's first barrier)
__device__ __forceinline__ void trace_issue() {
    uint64_t* p = trace_issue_slot();
    if (*p == 0) *p = gtimer();
}
struct TraceBuf {   // device memory, allocated by snn_trace_read's first call
    unsigned int count, pad[15];
    TraceRec rec[kTraceRecords];
};

struct TraceCta {
    uint64_t t_entry = 0, t_wait = 0, t_first = 0;
    uint32_t tiles = 0;
    int32_t first_stolen = -1, last_tile = -1;
    __device__ __forceinline__ void entry() {
        t_entry = gtimer();
        if (threadIdx.x == 0) *trace_issue_slot() = 0;
    }
    __device__ __forceinline__ void waited() { t_wait = gtimer(); }
    __device__ __forceinline__ void stage() {
        if (t_first == 0) t_first = gtimer();
    }
    __device__ __forceinline__ void tile(int t) {
        if (tiles == 1) first_stolen = t;
        last_tile = t;
        ++tiles;
    }
    // first consumer warp, lane 0
    __device__ __forceinline__ void done(void* buf, uint32_t kind, int64_t T, int64_t N) {
        if ((threadIdx.x & 31) != 0 || buf == nullptr) return;
        TraceBuf* b = static_cast<TraceBuf*>(buf);
        const unsigned i = atomicAdd(&b->count, 1u);
        if (i >= (unsigned)kTraceRecords) return;
        TraceRec r;
        r.kind = kind; r.grid = gridDim.x; r.smid = smid(); r.tiles = tiles;
        r.T = T; r.N = N;
        r.t_entry = t_entry; r.t_wait = t_wait; r.t_first = t_first; r.t_end = gtimer();
        r.first_stolen = first_stolen; r.last_tile = last_tile;
        r.t_issue = *trace_issue_slot();
        b->rec[i] = r;
    }
};
#else
__device__ __forceinline__ void trace_issue() {}
struct TraceCta {
    __device__ __forceinline__ void entry() {}
    __device__ __forceinline__ void waited() {}
    __device__ __forceinline__ void stage() {}
    __device__ __forceinline__ void tile(int) {}
    __device__ __forceinline__ void done(void*, uint32_t, int64_t, int64_t) {}
};
#endif

}  // namespace snn
