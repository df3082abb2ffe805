// lif_async.cuh -- sm_100a async-copy primitives (mbarrier + cp.async.bulk) used by the
// persistent, warp-specialised LIF kernels in lif_tma.cuh.
#pragma once

#include <stdint.h>

namespace snn {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

// Make the barrier inits visible to the async (TMA) proxy before first use.
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Producer: arrive once and announce `bytes` of incoming transaction.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Wait until the phase with the given parity has completed (fresh barrier: parity 1
// counts as complete, which is what lets the producer fill an empty ring).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// L2 policy: streamed once -> evict first.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 1-D bulk async copy global -> shared (UBLKCP), completion counted on `bar` in bytes.
// dst / src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 2-D TMA tile load (UTMALDG): box at coordinates (c0 = neuron, c1 = time row) of the
// tensor described by `tmap` (a __grid_constant__ CUtensorMap) into shared memory.
// Out-of-range elements are zero-filled and still counted in the transaction bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// L2 prefetch of the box at (c0, c1) (no shared-memory destination, no barrier).  Issued
// before griddepcontrol.wait for a CTA's first ring stages: a prefetch returns nothing to the
// program and L2 is the point of coherence, so a line the predecessor kernel writes afterwards
// is simply updated there; the loads after the wait then find their lines (and their
// translations) close by instead of paying the first DRAM + page-walk round trip serially.
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1)
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// ---- programmatic dependent launch ---------------------------------------------------
// Kernels are launched with cudaLaunchAttributeProgrammaticStreamSerialization: a kernel
// may start (barrier init, descriptor prefetch) while its predecessor drains, and blocks
// in pdl_wait() -- before touching global memory -- until the predecessor has completed
// and flushed.  A CTA calls pdl_trigger() once no tile is left to steal, so the successor
// fills SMs freed during this kernel's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- cluster launch control (sm_100): hardware work stealing ------------------------
// The grid has one CTA per tile.  A running CTA that finishes a tile asks the hardware to
// cancel a CTA that has not started yet and takes over its tile (its blockIdx.x); when no
// CTA is pending the request fails and the CTA drains.  Fast SMs therefore take more
// tiles, which balances per-SM speed differences without a global atomic counter.
struct ClcSlot {
    uint4 resp;      // 16-byte try_cancel response (written by the async proxy)
    uint64_t bar;    // completion barrier (16 transaction bytes)
};

__device__ __forceinline__ void clc_init(ClcSlot* c) { mbar_init(&c->bar, 1); }

// Issue an asynchronous steal request (one thread).  Its answer is read with
// clc_next_tile; issuing early hides the round trip behind the current tile.
__device__ __forceinline__ void clc_request(ClcSlot* c) {
    mbar_arrive_expect_tx(&c->bar, 16);
    asm volatile(
        "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];"
        ::"r"(smem_u32(&c->resp)), "r"(smem_u32(&c->bar))
        : "memory");
}

// Waits for the outstanding request: the stolen tile (blockIdx.x of the cancelled CTA)
// or -1 when no CTA was pending.  One thread only.  The proxy fence orders this generic
// read of the response before the async write of the slot's next request.
__device__ __forceinline__ int clc_next_tile(ClcSlot* c, uint32_t& phase) {
    mbar_wait(&c->bar, phase);
    phase ^= 1u;
    uint32_t ok, x;
    asm volatile(
        "{\n\t.reg .b128 r;\n\t.reg .pred p;\n\t"
        "ld.shared.b128 r, [%2];\n\t"
        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "@p clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n\t}"
        : "=r"(ok), "=r"(x)
        : "r"(smem_u32(&c->resp))
        : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    return ok ? (int)x : -1;
}

}  // namespace snn
