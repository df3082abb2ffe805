// lif_handoff.cuh -- fused boundary handoff of the time-segment split (
// PAPER.md:252 "inter-GPU communication enables cross-device operator fusion").
//
// Rank d runs the fused kernel on its time segment.  For every neuron tile the kernel
//  * at tile start: waits until the previous rank has published that tile's boundary
//    state (recv_ready[blk] >= epoch, acquire at system scope), then reads it from local
//    memory (the previous rank wrote it over NVLink);
//  * at tile end: waits until the next rank acknowledged the previous epoch of that block
//    (send_ack[blk] >= epoch - 1: credit-based flow control, so a fast rank never
//    overwrites a buffer still being read), stores its carry-out straight into the next
//    rank's buffer (send_state: a peer-mapped pointer), then -- after a consumer-wide
//    barrier -- releases send_ready[blk] = epoch at system scope, and acknowledges its own
//    receive (recv_ack[blk] = epoch).
// The transfer is per tile inside the compute kernel: no per-chunk launches, no NCCL, and
// the wavefront lag between ranks is one tile.  Spin loops sleep (__nanosleep) and trap
// after a long timeout instead of hanging the GPU.
#pragma once

#include <stdint.h>

#include "lif_kernels.cuh"

namespace snn {

constexpr int kHandoffBlock = 256;   // neurons per flag (every TMA tile is a multiple)

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag_ge(const int* p, int epoch) {
    const long long t0 = clock64();
    while (ld_acquire_sys(p) < epoch) {
        __nanosleep(200);
        if (clock64() - t0 > (1ll << 37)) __trap();   // ~60 s: a lost peer is a fault, not a hang
    }
}

// Consumer barrier (all NCONS consumer threads; the producer warp has its own role).
template <int NCONS>
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"r"(NCONS) : "memory");
}

// Tile start: the boundary state of this lane's VEC neurons from the previous rank.
template <int VEC>
__device__ __forceinline__ void handoff_recv(const Handoff& h, int64_t N, int64_t n0, int nvalid,
                                             float (&out)[VEC]) {
    const int lane = threadIdx.x & 31;
    if (lane == 0 && n0 < N) wait_flag_ge(h.recv_ready + n0 / kHandoffBlock, h.epoch);   // warp inside one block
    __syncwarp();
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (i < nvalid) out[i] = __ldcv(h.recv_state + n0 + i);   // bypass stale L1
}

// Tile end: publish this tile's carry-out to the next rank and acknowledge the receive.
template <int VEC, int NCONS>
__device__ __forceinline__ void handoff_send(const Handoff& h, int tile, int W, int64_t N, int64_t n0,
                                             int nvalid, const float (&val)[VEC]) {
    const int lane = threadIdx.x & 31;
    if (h.send_state != nullptr) {
        if (lane == 0 && n0 < N) wait_flag_ge(h.send_ack + n0 / kHandoffBlock, h.epoch - 1);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < VEC; ++i)
            if (i < nvalid) h.send_state[n0 + i] = val[i];
    }
    consumers_sync<NCONS>();   // every consumer's stores (and receive loads) are done
    if (threadIdx.x == 32) {   // first consumer thread
        const int64_t nblk = (N + kHandoffBlock - 1) / kHandoffBlock;
        const int64_t b0 = (int64_t)tile * W / kHandoffBlock;
        const int64_t b1 = min(nblk, b0 + W / kHandoffBlock);
        __threadfence_system();
        for (int64_t b = b0; b < b1; ++b) {
            if (h.send_ready != nullptr) st_release_sys(h.send_ready + b, h.epoch);
            if (h.recv_ack != nullptr) st_release_sys(h.recv_ack + b, h.epoch);
        }
    }
}

}  // namespace snn
