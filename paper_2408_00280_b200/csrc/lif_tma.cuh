// lif_tma.cuh -- persistent, warp-specialised fused LIF kernels for sm_100a, fed by the
// Tensor Memory Accelerator.
//
// Why this shape:
//  * The path is HBM-bound (a few flops per byte), so what matters is keeping enough
//    bytes in flight per SM (Little's law: ~6.5 TB/s x ~1-2 us ~= 50-100 KB per SM)
//    independently of how many registers the recurrence needs.  One producer lane issues
//    2-D TMA tile loads (cp.async.bulk.tensor.2d -> UTMALDG; box = up to 256 neurons x R
//    time rows, 4-16 KB per instruction) into a shared-memory ring; completion is counted
//    in bytes on an mbarrier.  The ring size, not the register file, sets the bytes in
//    flight, and the TMA engine (not the LSU) does the address generation.
//  * One CTA per W-neuron tile, made persistent by cluster launch control: a resident CTA
//    that finishes a tile cancels a not-yet-started CTA and takes its tile (hardware work
//    stealing, clusterlaunchcontrol.try_cancel).  Every consumer thread still owns its
//    neurons for the whole time axis (temporal fusion); the machine is
//    filled in one wave, faster SMs take more tiles, and the tail is < one tile.
//  * Consumer warps read their neurons from the ring (conflict-free 4-16 B per lane), run
//    the recurrence in registers and store outputs straight to HBM with coalesced
//    streaming stores, then release the ring slot (one mbarrier arrive per warp).
//  * Ragged T (not a multiple of the row block) and a ragged last tile are handled by the
//    TMA's zero fill; consumers do not store past T / N.  A ragged last VEC group (N not a
//    multiple of VEC) stores element by element.
//  * UNAL (unaligned) variants: a 2-D tensor map needs 16-byte row strides and a 16-byte
//    aligned base, and a TMA box must start on a 16-byte boundary; an odd row stride (e.g. a
//    contiguous [T, N] with N % 4 != 0 in fp32) or an unaligned column view breaks both.  Those
//    tensors get a flat tensor map -- one row over the whole [T, ld] storage, base aligned down
//    to 16 B.  Per time row the producer loads the tile's span aligned DOWN to 16 B: the tile's
//    256-neuron boxes plus one 16-byte tail box (smem rows [NB*BW + 16 B, padded to 128 B]);
//    the row's element shift m (0..3 fp32, 0..7 bf16) is read past by the consumers, with
//    pack loads when m keeps the pack aligned and element loads otherwise, and they store with
//    the widest aligned form per row (st_any).  ~3% more smem and bytes than the aligned
//    kernel; everything else is the same code.
//
// Smem layout of one tensor's row-block: NB boxes of [rows][BW] (BW = min(W, 256)).
#pragma once

#include <cuda.h>

#include <type_traits>

#include "lif_async.cuh"
#include "lif_handoff.cuh"
#include "lif_kernels.cuh"
#include "trace.cuh"

namespace snn {

#ifdef SNN_TRACE
#define SNN_TRACE_BUF(a) ((a).trace)
#else
#define SNN_TRACE_BUF(a) nullptr
#endif

// Shared-memory control block of a ring with S stages.
template <int S>
struct Barriers {
    uint64_t full[S];    // producer -> consumers: stage landed (TMA bytes counted)
    uint64_t empty[S];   // consumers -> producer: stage released (one arrive per warp)
    int tile[S];         // tile index the stage belongs to; -1 = no more work
    ClcSlot clc[4];      // cluster-launch-control response slots (work stealing)
};

constexpr int kMaxClc = 4;

constexpr int kAlignSlack = 1024;

// Dynamic smem, re-based to 1024 B (TMA destinations must be >=128 B aligned).
__device__ __forceinline__ unsigned char* smem_base() {
    extern __shared__ __align__(1024) unsigned char dyn_smem[];
    const uint32_t a = smem_u32(dyn_smem);
    return dyn_smem + ((1024u - (a & 1023u)) & 1023u);
}

template <int S>
__device__ __forceinline__ void init_barriers(Barriers<S>* b, uint32_t consumer_warps) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&b->full[s], 1);
            mbar_init(&b->empty[s], consumer_warps);
        }
        for (int i = 0; i < kMaxClc; ++i) clc_init(&b->clc[i]);
        fence_mbar_init();
    }
    __syncthreads();
}

// Producer skeleton shared by the kernels.  The CTA processes its own tile (blockIdx.x)
// first, then tiles of pending CTAs it cancels through cluster launch control.  sc.depth
// (1..kMaxClc) steal requests are kept in flight; the default is one: more lets a CTA hoard
// tiles it cannot start yet while others run dry at the end of the grid (r2, per-CTA
// timelines of tools/trace_timeline.py: the last CTA ended 4-5 us after the median one at
// depth 4, ~2 us at depth 1; cfg2 +4%).  Each tile is `nstages` ring stages;
// `bytes(tile, j)` is stage j's transaction byte count and `issue(stage_ptr, tile, j, bar)`
// issues its TMA loads.  Ends with a tile = -1 sentinel stage; every outstanding request is
// drained before returning (its response is an async smem write) and a late success is still
// processed.  Request number q lives in slot q % depth (each slot has at most one in flight).
// WARP = false: run by one thread.  WARP = true: run by the whole producer warp in lockstep --
// every lane waits and tracks the same state, lane 0 alone writes the stage metadata, arms the
// barriers and sends the steal requests, and `issue` is called on every lane (the unaligned
// kernels spread their per-row TMA loads over the lanes: one thread issues ~one UTMALDG per
// 50 ns, too few for rows that each need their own loads).
template <int S, int STAGE_BYTES, bool WARP = false, typename Bytes, typename Issue>
__device__ __forceinline__ void produce(unsigned char* smem, Barriers<S>* bar, int64_t nstages,
                                        const Sched& sc, Bytes bytes, Issue issue) {
    const bool leader = !WARP || (threadIdx.x & 31) == 0;
    const int depth = sc.depth;
    uint32_t k = 0;
    uint32_t phases = 0;   // bit i = parity of CLC slot i (a bit set, not an array: no local memory)
    int issued = 0, consumed = 0;
    bool stop = false;
    for (int i = 0; i < depth; ++i, ++issued)
        if (leader) clc_request(&bar->clc[i]);
    int tile = (int)blockIdx.x;
    while (true) {
        for (int64_t j = 0; j < nstages; ++j, ++k) {
            const int s = k % S;
            mbar_wait(&bar->empty[s], ((k / S) & 1) ^ 1);
            if (leader) {
                bar->tile[s] = tile;
                mbar_arrive_expect_tx(&bar->full[s], bytes(tile, j));
            }
            if constexpr (WARP) __syncwarp();
            issue(smem + s * STAGE_BYTES, tile, j, &bar->full[s]);
            trace_issue();
        }
        tile = -1;
        while (consumed < issued) {
            const int i = consumed % depth;
            uint32_t ph = (phases >> i) & 1u;
            const int r = clc_next_tile(&bar->clc[i], ph);
            phases ^= 1u << i;
            ++consumed;
            if (r >= 0) {
                tile = r;
                if (!stop) {
                    if (leader) clc_request(&bar->clc[issued % depth]);
                    ++issued;
                }
                break;
            }
            stop = true;   // no CTA pending: issue no more requests, drain the rest
        }
        if (tile < 0) {
            if (leader) pdl_trigger();   // nothing left to steal: let the next kernel start filling SMs
            const int s = k % S;
            mbar_wait(&bar->empty[s], ((k / S) & 1) ^ 1);
            if (leader) {
                bar->tile[s] = -1;
                mbar_arrive(&bar->full[s]);
            }
            return;
        }
    }
}

// Element offset of neuron nt (VEC-aligned, < W) at row r of a [NB][ROWS][BW] region.
template <int VEC, int BW, int ROWS>
__device__ __forceinline__ int box_off(int nt, int r) {
    return ((nt / BW) * ROWS + r) * BW + (nt % BW);
}

// One io tensor's rows of a stage.  Aligned: NB 2-D tensor-map boxes, smem [NB][ROWS][BW]
// (rows past T zero-filled by the TMA).  UNAL: per time row ONE 1-D bulk copy
// (cp.async.bulk, UBLKCP) of the tile span [c0, c0 + W) of that row shifted down to a 16-byte
// boundary, W*esz + 16 bytes (truncated at the view's last 16-byte chunk, which holds its last
// element: nothing past the allocation is read), into smem row r at r * RP (RP = W*esz + 16 B,
// 128-B aligned rows); only the `rows` valid rows are loaded (tx_bytes counts the same).
template <typename IO, int BW, int ROWS, int NB, bool UNAL>
struct Region {
    static constexpr int Q = 16 / (int)sizeof(IO);
    static constexpr int WB = NB * BW * (int)sizeof(IO);          // tile span bytes
    // UNAL smem row pitch: 16-B aligned rows (the bulk-copy destination rule).  (r2: was + 128 B,
    // which pushed the bf16 backward's 3-stage ring past two CTAs per SM: 45% of aligned speed.)
    static constexpr int RP = WB + 16;
    static constexpr int RPE = RP / (int)sizeof(IO);
    static constexpr int BYTES = UNAL ? ROWS * RP : WB * ROWS;

    // The flat extent of an io view x [T, ld] (first N columns): its aligned-down base and the
    // end of the 16-byte chunk holding its last element.
    struct Flat {
        uintptr_t x;     // the view's first element
        uintptr_t end;   // round_up(address past its last element, 16)
    };
    __device__ static __forceinline__ Flat flat(const void* x, int64_t T, int64_t N, int64_t ld) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(x);
        return Flat{a, (a + (uintptr_t)(((T - 1) * ld + N) * (int64_t)sizeof(IO)) + 15) & ~uintptr_t(15)};
    }
    // UNAL: source address and byte count of time row t's copy.
    __device__ static __forceinline__ uint32_t row_copy(const Flat& f, int64_t t, int64_t c0, int64_t ld,
                                                        uintptr_t* src) {
        const uintptr_t s = (f.x + (uintptr_t)((t * ld + c0) * (int64_t)sizeof(IO))) & ~uintptr_t(15);
        *src = s;
        const uintptr_t lim = f.end - s;
        return (uint32_t)(lim < (uintptr_t)(WB + 16) ? lim : (uintptr_t)(WB + 16));
    }
    __device__ static __forceinline__ uint32_t tx_bytes(const Flat& f, int64_t t0, int rows, int64_t c0, int64_t ld) {
        if constexpr (!UNAL) {
            return (uint32_t)(WB * ROWS);
        } else {
            uint32_t b = 0;
            uintptr_t src;
            for (int r = 0; r < rows; ++r) b += row_copy(f, t0 + r, c0, ld, &src);
            return b;
        }
    }
    // rows t0 .. t0 + rows - 1 of tile columns c0 ..  Aligned: one thread, tensor map tm.
    // UNAL: every lane of the producer warp; lane (r + lane0) % 32 copies row r.
    __device__ static __forceinline__ void load(unsigned char* dst, const void* tm, const Flat& f, int64_t c0,
                                                int64_t t0, int rows, int64_t ld, uint64_t* fb, uint64_t pol,
                                                int lane0 = 0) {
        if constexpr (!UNAL) {
#pragma unroll
            for (int b = 0; b < NB; ++b)
                tma_load_2d(dst + b * BW * ROWS * (int)sizeof(IO), tm, (int)(c0 + b * BW), (int)t0, fb, pol);
        } else {
            const int lane = threadIdx.x & 31;
#pragma unroll 1
            for (int r = (lane - lane0) & 31; r < rows; r += 32) {
                uintptr_t src;
                const uint32_t n = row_copy(f, t0 + r, c0, ld, &src);
                bulk_g2s(dst + r * RP, reinterpret_cast<const void*>(src), n, fb, pol);
            }
        }
    }
};

// 16 bytes of shared memory at p, s = p's byte shift (1..15, warp-uniform) past the 16-B
// aligned address b below it: the two aligned chunks at b and b + 16 (two conflict-free LDS.128 per
// lane), realigned in registers -- a word select for s % 4 == 0 (fp32 rows), PRMT byte
// permutes otherwise (bf16 rows at an odd element).  (r2c: per-word or per-element loads at a
// 16-byte-lane stride hit the same bank 4-way, i.e. 4-8x the shared-memory cycles of an
// aligned row.)  The caller's row has >= 16 readable bytes past its last element (RP).
__device__ __forceinline__ uint4 lds_realign16(const void* p, uint32_t s) {
    const uint4* b = reinterpret_cast<const uint4*>(reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15));
    const uint4 lo = b[0], hi = b[1];
    const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t o[4];
    const uint32_t sel = (s & 3u) == 2u ? 0x5432u : ((s & 3u) == 1u ? 0x4321u : 0x6543u);
    auto pick = [&](auto q) {
        constexpr int Q = decltype(q)::value;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            o[k] = (s & 3u) == 0u ? w[k + Q] : __byte_perm(w[k + Q], w[k + Q + 1], sel);
    };
    switch (s >> 2) {   // warp-uniform
        case 0: pick(std::integral_constant<int, 0>{}); break;
        case 1: pick(std::integral_constant<int, 1>{}); break;
        case 2: pick(std::integral_constant<int, 2>{}); break;
        default: pick(std::integral_constant<int, 3>{}); break;
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// VEC elements from shared memory at q of any element alignment, with the widest loads the
// address allows (16 / 8 / 4 bytes; element loads only for 2-byte-aligned bf16); 16-byte
// packs are realigned from two aligned chunks (lds_realign16).  The choice is warp-uniform:
// every lane's q has the same misalignment.
template <typename IO, int VEC>
__device__ __forceinline__ Pack<IO, VEC> lds_widest(const IO* q) {
    constexpr int B = (int)sizeof(Pack<IO, VEC>);
    const uint32_t a = smem_u32(q);
    Pack<IO, VEC> r;
    if (a % B == 0) return *reinterpret_cast<const Pack<IO, VEC>*>(q);
    if constexpr (B == 16) {   // (an 8-byte-aligned row keeps the two LDS.64: measured faster)
        if (a % 8 != 0) {
            const uint4 v = lds_realign16(q, a & 15u);
            *reinterpret_cast<uint4*>(&r) = v;
            return r;
        }
    }
    if constexpr (B >= 16) {
        if (a % 8 == 0) {
#pragma unroll
            for (int i = 0; i < B / 8; ++i)
                reinterpret_cast<uint2*>(&r)[i] = reinterpret_cast<const uint2*>(q)[i];
            return r;
        }
    }
    if constexpr (B >= 8) {
        if (a % 4 == 0) {
#pragma unroll
            for (int i = 0; i < B / 4; ++i)
                reinterpret_cast<uint32_t*>(&r)[i] = reinterpret_cast<const uint32_t*>(q)[i];
            return r;
        }
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i) r.v[i] = q[i];
    return r;
}

// Branch-free variant for the unaligned-row kernels' 16-byte packs (r2c): the two aligned
// chunks at shared address b and b + 16, rotated by s >> 2 words through a two-level SEL network
// and byte-shifted by s & 3 with PRMT (bf16 only; fp32 shifts are whole words).  Every row of an
// unaligned launch takes the same instruction sequence whatever its shift -- the branchy
// per-row dispatch (and the uniform-register re-materialisations of its basic blocks) cost more
// issue slots than these SELs (ncu: 2.4x the aligned kernel's instructions, 14% of them R2UR).
template <typename IO, int VEC>
__device__ __forceinline__ Pack<IO, VEC> lds_rot16(uint32_t b, uint32_t s) {
    static_assert(sizeof(Pack<IO, VEC>) == 16, "16-byte packs");
    uint32_t w[8];
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(b));
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+16];"
                 : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(b));
    constexpr bool BYTES = sizeof(IO) < 4;
    constexpr int NT = BYTES ? 5 : 4;   // rotated words needed
    const uint32_t q = s >> 2;
    uint32_t u[NT + 2], t[NT];
#pragma unroll
    for (int k = 0; k < NT + 2; ++k) u[k] = (q & 1u) ? w[k + 1] : w[k];
#pragma unroll
    for (int k = 0; k < NT; ++k) t[k] = (q & 2u) ? u[k + 2] : u[k];
    Pack<IO, VEC> r;
    uint32_t* o = reinterpret_cast<uint32_t*>(&r);
    if constexpr (BYTES) {
        const uint32_t sel = 0x3210u + 0x1111u * (s & 3u);
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = __byte_perm(t[k], t[k + 1], sel);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = t[k];
    }
    return r;
}

// The backward's narrower packs, branch-free likewise (r2c): 8 bytes (fp32 pairs; always
// 4-byte aligned) from the two aligned 8-byte words around them and a SEL; 4 bytes (bf16
// pairs; 2-byte aligned) from two aligned words and a PRMT.  a = the pack's shared address.
__device__ __forceinline__ uint2 lds_rot8(uint32_t a) {
    const uint32_t b = a & ~7u;
    uint32_t w0, w1, w2, w3;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(b));
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2+8];" : "=r"(w2), "=r"(w3) : "r"(b));
    const bool sh = (a & 4u) != 0u;
    return make_uint2(sh ? w1 : w0, sh ? w2 : w1);
}
__device__ __forceinline__ uint32_t lds_rot4(uint32_t a) {
    const uint32_t b = a & ~3u;
    uint32_t w0, w1;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(b));
    asm volatile("ld.shared.u32 %0, [%1+4];" : "=r"(w1) : "r"(b));
    return __byte_perm(w0, w1, 0x3210u + 0x1111u * (a & 3u));
}

// A consumer lane's view of one tensor's rows in a stage: src(j) = the lane's VEC elements of
// row j.  Aligned: box layout, pack loads.  UNAL: row-major with the row's element shift
// m_j = (m0 + j*dm) mod Q (m0 = the first row's, dm = ld mod Q); pack loads where the shift keeps
// the pack aligned, element loads otherwise (a warp-uniform choice per row).
template <typename IO, int VEC, int BW, int RPE, bool UNAL>
struct RowSrc {
    const IO* p;   // aligned: the lane's element of row 0 (box layout); UNAL: row 0 base + lane offset
    int m0, dm;
    __device__ __forceinline__ Pack<IO, VEC> operator()(int j) const {
        if constexpr (!UNAL) {
            return *reinterpret_cast<const Pack<IO, VEC>*>(p + j * BW);
        } else {
            constexpr int Q = 16 / (int)sizeof(IO);
            if constexpr (sizeof(Pack<IO, VEC>) == 16) {   // the lane's chunk is 16-B aligned
                return lds_rot16<IO, VEC>(smem_u32(p) + (uint32_t)(j * RPE * (int)sizeof(IO)),
                                          (uint32_t)(((m0 + j * dm) & (Q - 1)) * (int)sizeof(IO)));
            } else if constexpr (sizeof(Pack<IO, VEC>) == 8 || sizeof(Pack<IO, VEC>) == 4) {
                const IO* q = p + j * RPE + ((m0 + j * dm) & (Q - 1));
                Pack<IO, VEC> r;
                if constexpr (sizeof(Pack<IO, VEC>) == 8) *reinterpret_cast<uint2*>(&r) = lds_rot8(smem_u32(q));
                else *reinterpret_cast<uint32_t*>(&r) = lds_rot4(smem_u32(q));
                return r;
            } else {
                const IO* q = p + j * RPE + ((m0 + j * dm) & (Q - 1));
                return lds_widest<IO, VEC>(q);
            }
        }
    }
};

// The lane's RowSrc for rows starting at time t0 of a region at `base` (stage smem).
template <typename IO, int VEC, int BW, int ROWS, int NB, bool UNAL>
__device__ __forceinline__ RowSrc<IO, VEC, BW, Region<IO, BW, ROWS, NB, UNAL>::RPE, UNAL>
row_src(const unsigned char* base, int nt, int64_t t0, int64_t ld, int off) {
    constexpr int Q = 16 / (int)sizeof(IO);
    RowSrc<IO, VEC, BW, Region<IO, BW, ROWS, NB, UNAL>::RPE, UNAL> s;
    if constexpr (!UNAL) {
        s.p = reinterpret_cast<const IO*>(base) + ((nt / BW) * ROWS) * BW + (nt % BW);
        s.m0 = s.dm = 0;
    } else {
        s.p = reinterpret_cast<const IO*>(base) + nt;
        s.m0 = (int)((off + t0 * ld) & (Q - 1));
        s.dm = (int)(ld & (Q - 1));
    }
    return s;
}

// Store a consumer's VEC outputs of one row: the plain streaming pack store on the aligned
// path, the widest aligned form on the unaligned one; a ragged last group (nvalid < VEC)
// element by element either way (a pack store would spill into the neighbouring columns).
template <bool UNAL, typename T, int VEC>
__device__ __forceinline__ void st_out(T* p, const Pack<T, VEC>& r, int nvalid) {
    if constexpr (UNAL && sizeof(Pack<T, VEC>) == 8 && sizeof(T) == 4) {   // fp32 pairs: 4-B aligned
        if (nvalid >= VEC) {
            const uint2 v = *reinterpret_cast<const uint2*>(&r);
            asm volatile(
                "{\n\t.reg .pred q8;\n\t"
                "setp.eq.u32 q8, %1, 0;\n\t"
                "@q8 st.global.cs.v2.u32 [%0], {%2, %3};\n\t"
                "@!q8 st.global.cs.u32 [%0], %2;\n\t"
                "@!q8 st.global.cs.u32 [%0+4], %3;\n\t}"
                :: "l"(p), "r"((uint32_t)reinterpret_cast<uintptr_t>(p) & 7u), "r"(v.x), "r"(v.y) : "memory");
        } else {
            st_any<T, VEC>(p, r, nvalid);
        }
    } else if constexpr (UNAL && sizeof(Pack<T, VEC>) == 4 && sizeof(T) == 2) {   // bf16 pairs: 2-B aligned
        if (nvalid >= VEC) {
            const uint32_t v = *reinterpret_cast<const uint32_t*>(&r);
            asm volatile(
                "{\n\t.reg .pred q4;\n\t"
                "setp.eq.u32 q4, %1, 0;\n\t"
                "@q4 st.global.cs.u32 [%0], %2;\n\t"
                "@!q4 st.global.cs.u16 [%0], %2;\n\t"
                "@!q4 st.global.cs.u16 [%0+2], %3;\n\t}"
                :: "l"(p), "r"((uint32_t)reinterpret_cast<uintptr_t>(p) & 3u), "r"(v), "r"(v >> 16) : "memory");
        } else {
            st_any<T, VEC>(p, r, nvalid);
        }
    } else if constexpr (UNAL) {
        st_any<T, VEC>(p, r, nvalid);
    } else if (nvalid >= VEC) {
        st_stream<T, VEC>(p, r);
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i)
            if (i < nvalid) __stcs(p + i, r.v[i]);
    }
}

// [N] fp32 vectors (carries, partials): any alignment, ragged last group.
template <int VEC>
__device__ __forceinline__ void load_vec(const float* p, int nvalid, float (&out)[VEC]) {
    const Pack<float, VEC> v = ld_any<float, VEC>(p, nvalid);
#pragma unroll
    for (int i = 0; i < VEC; ++i)
        if (i < nvalid) out[i] = v.v[i];
}
template <int VEC>
__device__ __forceinline__ void store_vec(float* p, int nvalid, const float (&in)[VEC]) {
    Pack<float, VEC> v;
#pragma unroll
    for (int i = 0; i < VEC; ++i) v.v[i] = in[i];
    st_any<float, VEC>(p, v, nvalid);
}

__device__ __forceinline__ int group_valid(int64_t n0, int64_t N, int vec) {
    const int64_t r = N - n0;
    return r <= 0 ? 0 : (r >= vec ? vec : (int)r);
}

// ------------------------------------------------------------------------------------
// Forward.  Stage = R time rows of a W-neuron tile.  Warp 0 lane 0 = producer;
// warps 1..NCONS/32 = consumers, each lane owning VEC neurons.
// NIN = 2: the stage also holds the residual rows R at R_OFF.
template <typename IO, int VEC, int NCONS, int R, int S, int NIN = 1, bool UNAL = false>
struct FwdTma {
    static constexpr int W = NCONS * VEC;
    static constexpr int BW = W < 256 ? W : 256;
    static constexpr int NB = W / BW;
    using Reg = Region<IO, BW, R, NB, UNAL>;
    static constexpr int R_OFF = Reg::BYTES;
    static constexpr int STAGE_BYTES = NIN * Reg::BYTES;
    static constexpr int SMEM = S * STAGE_BYTES + (int)sizeof(Barriers<S>) + kAlignSlack;
    static constexpr int THREADS = NCONS + 32;
    static_assert(W % BW == 0 && BW % VEC == 0, "tile geometry");
};

template <typename IO, int VEC, int SFMT, int SAVE, bool SOFT, bool AFF, bool RES, int NCONS, int R, int S,
          bool UNAL, bool P0 = false>
__global__ void __launch_bounds__(NCONS + 32)
lif_forward_tma_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmr,
                       const FwdArgs a, const Sched sc) {
    static_assert(!RES || AFF, "the residual prologue rides on the affine one");
    using Cfg = FwdTma<IO, VEC, NCONS, R, S, RES ? 2 : 1, UNAL>;
    using Reg = typename Cfg::Reg;
    constexpr int W = Cfg::W, BW = Cfg::BW, NB = Cfg::NB;
    unsigned char* smem = smem_base();
    auto* bar = reinterpret_cast<Barriers<S>*>(smem + S * Cfg::STAGE_BYTES);
    TraceCta tr;
    tr.entry();
    init_barriers<S>(bar, NCONS / 32);
    const int64_t T = a.T, N = a.N;
    const int64_t nrb = (T + R - 1) / R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {   // before the wait: kernel-parameter descriptors, L2 prefetch of the own tile
        tma_prefetch_desc(&tmx);
        if constexpr (RES) tma_prefetch_desc(&tmr);
        if constexpr (!UNAL) {
            const int c0 = (int)blockIdx.x * W;
            for (int j = 0; j < sc.prefetch && j < S && j < nrb; ++j)
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    tma_prefetch_2d(&tmx, c0 + b * BW, j * R);
                    if constexpr (RES) tma_prefetch_2d(&tmr, c0 + b * BW, j * R);
                }
        }
    }
    pdl_wait();   // predecessor complete before any global-memory access
    tr.waited();

    if (warp == 0) {  // ---------------- producer (one lane; the whole warp for unaligned rows)
        if (UNAL || lane == 0) {
            const uint64_t pol = policy_evict_first();
            const auto fx = Reg::flat(a.x, T, N, a.ld);
            const auto fr = Reg::flat(a.af.residual, T, N, a.ld);
            auto rows_of = [&](int64_t rb) { return (int)min((int64_t)R, T - rb * R); };
            produce<S, Cfg::STAGE_BYTES, UNAL>(
                smem, bar, nrb, sc,
                [&](int tile, int64_t rb) {
                    const int64_t c0 = (int64_t)tile * W;
                    uint32_t b = Reg::tx_bytes(fx, rb * R, rows_of(rb), c0, a.ld);
                    if constexpr (RES) b += Reg::tx_bytes(fr, rb * R, rows_of(rb), c0, a.ld);
                    return b;
                },
                [&](unsigned char* stg, int tile, int64_t rb, uint64_t* fb) {
                    Reg::load(stg, &tmx, fx, (int64_t)tile * W, rb * R, rows_of(rb), a.ld, fb, pol);
                    if constexpr (RES)
                        Reg::load(stg + Cfg::R_OFF, &tmr, fr, (int64_t)tile * W, rb * R, rows_of(rb), a.ld, fb, pol, R);
                });
        }
        return;
    }

    // ---------------- consumers
    LifConsts c = a.c;
    pin(c);
    const int ct = threadIdx.x - 32;
    const int64_t spk_step = spike_row_bytes<IO, SFMT>(a);
    uint32_t k = 0;
    while (true) {
        int s = k % S;
        mbar_wait(&bar->full[s], (k / S) & 1);
        const int tile = bar->tile[s];
        if (tile < 0) break;
        tr.stage();
        tr.tile(tile);
        const int64_t g = (int64_t)tile * NCONS + ct;
        const int64_t n0 = g * VEC;
        const int nvalid = group_valid(n0, N, VEC);
        const bool tile_full = (int64_t)(tile + 1) * W <= N;   // uniform across the CTA
        float V[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) V[i] = c.v_reset;
        if (a.h.recv_state != nullptr) {            // segment boundary from the previous rank
            handoff_recv<VEC>(a.h, N, n0, nvalid, V);
        } else if (a.v_init != nullptr && nvalid > 0) {
            load_vec<VEC>(a.v_init + n0, nvalid, V);
        }
        const AffCoef<VEC> co = load_affine<VEC, AFF>(a.af, n0, nvalid);
        unsigned char* spk_row = reinterpret_cast<unsigned char*>(a.spikes);
        float* h_row = a.saved + n0;   // SAVE_H: advanced one row per step
        for (int64_t rb = 0; rb < nrb; ++rb, ++k) {
            if (rb > 0) {
                s = k % S;
                mbar_wait(&bar->full[s], (k / S) & 1);
            }
            const int rows = (int)min((int64_t)R, T - rb * R);
            const unsigned char* stg = smem + s * Cfg::STAGE_BYTES;
            const auto xs = row_src<IO, VEC, BW, R, NB, UNAL>(stg, ct * VEC, rb * R, a.ld, a.x_off);
            const auto rsrc = row_src<IO, VEC, BW, R, NB, UNAL>(stg + Cfg::R_OFF, ct * VEC, rb * R, a.ld, a.r_off);
            // F: a full stage of a full tile (guard-free).  A partial stage keeps per-row guards:
            // unlike the backward (bwd_chunk_masked), masking every row here measured slower
            // (bf16 T=10: 31 -> 39 us), the forward's V chain being serial anyway.
            auto rowloop = [&](auto full) {
            constexpr bool F = decltype(full)::value;
            const int nv = F ? VEC : nvalid;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                if (F || r < rows) {
                    const Pack<IO, VEC> xv = xs(r);
                    Pack<IO, VEC> rv;
                    if constexpr (RES) rv = rsrc(r);
                    if constexpr (SAVE == SAVE_RECOMPUTE) {
                        // checkpoint the V entering step t when t % kCkpt == 0 (the saved rows are
                        // padded to 16 floats: a ragged group's pack store stays inside its row)
                        const int64_t t = rb * R + r;
                        if ((t % kCkpt) == 0 && nv > 0 && (t > 0 || a.ck0)) {
                            Pack<float, VEC> ck;
#pragma unroll
                            for (int i = 0; i < VEC; ++i) ck.v[i] = V[i];
                            st_stream<float, VEC>(h_row + (t / kCkpt) * a.ldh, ck);
                        }
                    }
                    Pack<float, VEC> hp;
                    const unsigned bits = fwd_compute<SOFT, AFF, RES, P0>(c, V, xv, hp, co, &rv);
                    if constexpr (SAVE == SAVE_H) {
                        if (nv > 0) st_stream<float, VEC>(h_row, hp);
                        h_row += a.ldh;
                    }
                    // (r2: a warp-cooperative funnel-shift store of unaligned u8 rows -- one aligned word
                    // per lane instead of byte stores -- measured 10-20% slower; not used)
                    store_spikes<IO, VEC, SFMT, UNAL>(spk_row, g, n0, bits, nv, a.nwords);
                    spk_row += spk_step;
                }
            }
            };
            if (rows == R && tile_full) rowloop(std::true_type{}); else rowloop(std::false_type{});
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->empty[s]);
        }
        if (a.h.send_state != nullptr || a.h.recv_ack != nullptr)   // uniform across the CTA
            handoff_send<VEC, NCONS>(a.h, tile, W, N, n0, nvalid, V);
        if (a.v_final != nullptr && nvalid > 0) store_vec<VEC>(a.v_final + n0, nvalid, V);
    }
    if (warp == 1) tr.done(SNN_TRACE_BUF(a), 1u, T, N);
}

// ------------------------------------------------------------------------------------
// Backward, RECOMPUTE.  Stage = one kCkpt-step chunk of the tile: x rows, gS rows and the
// chunk's entry-V checkpoint row.  Chunks of a tile are streamed last-first.
// RES: the stage also holds the chunk's residual rows at R_OFF.
template <typename IO, int VEC, int NCONS, int S, bool RES = false, bool UNAL = false>
struct BwdRecTma {
    static constexpr int W = NCONS * VEC;
    static constexpr int BW = W < 256 ? W : 256;
    static constexpr int NB = W / BW;
    using Reg = Region<IO, BW, kCkpt, NB, UNAL>;
    static constexpr int CK_BOX_BYTES = BW * 4;
    static constexpr int NIN = RES ? 3 : 2;
    static constexpr int X_OFF = 0;
    static constexpr int G_OFF = Reg::BYTES;
    static constexpr int R_OFF = 2 * Reg::BYTES;
    static constexpr int CK_OFF = NIN * Reg::BYTES;
    static constexpr int STAGE_BYTES = NIN * Reg::BYTES + NB * CK_BOX_BYTES;
    static constexpr int SMEM = S * STAGE_BYTES + (int)sizeof(Barriers<S>) + kAlignSlack;
    static constexpr int THREADS = NCONS + 32;
    static_assert(W % BW == 0 && BW % VEC == 0 && STAGE_BYTES % 128 == 0, "tile geometry");
};

// Reverse walk over rows [0, rows) of one chunk.  h = recomputed H; gsm = gS rows in smem;
// gxp = gX at the chunk's LAST row, walked backwards by ldb bytes.
// RES: grp = dL/dR at the chunk's last row, walked like gxp.
template <typename IO, int VEC, int MODE, int ROWS_MAX, bool UNAL, typename GS, typename XS>
__device__ __forceinline__ void bwd_chunk(const LifConsts& c, float (&gV)[VEC],
                                          const float (&h)[ROWS_MAX][VEC], const GS& gsm,
                                          IO* gxp, int64_t ldb, int rows, int nvalid,
                                          const AffCoef<VEC>& co, const XS& xs, float* pa, float* pb,
                                          IO* grp = nullptr) {
#pragma unroll
    for (int j = ROWS_MAX - 1; j >= 0; --j) {
        if (j < rows) {
            const Pack<IO, VEC> gv = gsm(j);
            Pack<IO, VEC> out, outr;
            if constexpr (Mode<MODE>::AFF) {
                const Pack<IO, VEC> xr = xs(j);
                out = bwd_step<IO, VEC, MODE, true>(c, gV, h[j], gv, &co, &xr, pa, pb, &outr);
            } else {
                out = bwd_step<IO, VEC, MODE>(c, gV, h[j], gv);
            }
            if (nvalid > 0) st_out<UNAL>(gxp, out, nvalid);
            gxp = step_bytes(gxp, -ldb);
            if constexpr (Mode<MODE>::RES) {
                if (nvalid > 0) st_out<UNAL>(grp, outr, nvalid);
                grp = step_bytes(grp, -ldb);
            }
        }
    }
}

// Partial chunk (rows < ROWS_MAX, or a ragged last tile): every row of the ROWS_MAX block is
// computed unconditionally -- rows past T were zero-filled by the TMA (or hold a previous
// stage's values on the unaligned path), so their arithmetic stays independent of the carried
// gV until the select -- and only the carry update (a select on the uniform `act`) and the
// stores are conditional.  One basic block per chunk lets the compiler interleave the rows'
// independent surrogate math, which a per-row branch (the old guarded loop) serialised: T=10
// cost as much as T=16.  gx0 / gr0 = row 0 of the chunk.
template <typename IO, int VEC, int MODE, int ROWS_MAX, bool UNAL, typename GS, typename XS>
__device__ __forceinline__ void bwd_chunk_masked(const LifConsts& c, float (&gV)[VEC],
                                                 const float (&h)[kCkpt][VEC], const GS& gsm,
                                                 IO* gx0, int64_t ldb, int rows, int nvalid,
                                                 const AffCoef<VEC>& co, const XS& xs, float* pa, float* pb,
                                                 IO* gr0 = nullptr) {
#pragma unroll
    for (int j = ROWS_MAX - 1; j >= 0; --j) {
        const bool act = j < rows;   // uniform across the CTA
        const Pack<IO, VEC> gv = gsm(j);
        Pack<IO, VEC> out, outr;
        float g2[VEC], pa2[VEC], pb2[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) { g2[i] = gV[i]; pa2[i] = pa[i]; pb2[i] = pb[i]; }
        if constexpr (Mode<MODE>::AFF) {
            const Pack<IO, VEC> xr = xs(j);
            out = bwd_step<IO, VEC, MODE, true>(c, g2, h[j], gv, &co, &xr, pa2, pb2, &outr);
        } else {
            out = bwd_step<IO, VEC, MODE>(c, g2, h[j], gv);
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            gV[i] = act ? g2[i] : gV[i];
            if constexpr (Mode<MODE>::AFF) { pa[i] = act ? pa2[i] : pa[i]; pb[i] = act ? pb2[i] : pb[i]; }
        }
        if (act && nvalid > 0) {
            st_out<UNAL>(step_bytes(gx0, j * ldb), out, nvalid);
            if constexpr (Mode<MODE>::RES) st_out<UNAL>(step_bytes(gr0, j * ldb), outr, nvalid);
        }
    }
}

template <typename IO, int VEC, int MODE, int ROWS_MAX, typename XS>
__device__ __forceinline__ void recompute_chunk(const LifConsts& c, float (&V)[VEC],
                                                float (&h)[kCkpt][VEC], const XS& xs, int rows,
                                                const AffCoef<VEC>& co, const XS& rs) {
#pragma unroll
    for (int j = 0; j < ROWS_MAX; ++j) {
        if (j < rows) {
            const Pack<IO, VEC> xv = xs(j);
            Pack<IO, VEC> rv;
            if constexpr (Mode<MODE>::RES) rv = rs(j);
            fwd_recompute_step<Mode<MODE>::SOFT, Mode<MODE>::AFF, Mode<MODE>::RES, Mode<MODE>::P0>(c, V, xv, h[j],
                                                                                               co, &rv);
        }
    }
}

template <typename IO, int VEC, int MODE, int NCONS, int S, bool UNAL>
__global__ void __launch_bounds__(NCONS + 32)
lif_backward_recompute_tma_kernel(const __grid_constant__ CUtensorMap tmx,
                                  const __grid_constant__ CUtensorMap tmg,
                                  const __grid_constant__ CUtensorMap tmck,
                                  const __grid_constant__ CUtensorMap tmr, const BwdArgs a,
                                  const Sched sc) {
    constexpr bool RES = Mode<MODE>::RES;
    static_assert(!RES || Mode<MODE>::AFF, "the residual prologue rides on the affine one");
    using Cfg = BwdRecTma<IO, VEC, NCONS, S, RES, UNAL>;
    using Reg = typename Cfg::Reg;
    constexpr int W = Cfg::W, BW = Cfg::BW, NB = Cfg::NB;
    unsigned char* smem = smem_base();
    auto* bar = reinterpret_cast<Barriers<S>*>(smem + S * Cfg::STAGE_BYTES);
    TraceCta tr;
    tr.entry();
    init_barriers<S>(bar, NCONS / 32);
    const int64_t T = a.T, N = a.N, ld = a.ld;
    const int64_t nch = (T + kCkpt - 1) / kCkpt;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {   // before the wait: kernel-parameter descriptors, L2 prefetch of the own tile
        tma_prefetch_desc(&tmx); tma_prefetch_desc(&tmg); tma_prefetch_desc(&tmck);
        if constexpr (RES) tma_prefetch_desc(&tmr);
        const int c0 = (int)blockIdx.x * W;
        for (int j = 0; j < sc.prefetch && j < S && j < nch; ++j) {
            const int ch = (int)nch - 1 - j;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if (ch > 0 || a.ck0) tma_prefetch_2d(&tmck, c0 + b * BW, ch);
                if constexpr (!UNAL) {
                    tma_prefetch_2d(&tmx, c0 + b * BW, ch * kCkpt);
                    tma_prefetch_2d(&tmg, c0 + b * BW, ch * kCkpt);
                    if constexpr (RES) tma_prefetch_2d(&tmr, c0 + b * BW, ch * kCkpt);
                }
            }
        }
    }
    pdl_wait();   // predecessor complete before any global-memory access
    tr.waited();

    if (warp == 0) {  // ---------------- producer: chunks of a tile, last first (whole warp if unaligned)
        if (UNAL || lane == 0) {
            const uint64_t pol = policy_evict_first();
            auto rows_of = [&](int64_t j) {
                const int64_t ch = nch - 1 - j;
                return (int)min((int64_t)kCkpt, T - ch * kCkpt);
            };
            const auto fx = Reg::flat(a.x, T, N, ld);
            const auto fg = Reg::flat(a.gS, T, N, ld);
            const auto fr = Reg::flat(a.af.residual, T, N, ld);
            produce<S, Cfg::STAGE_BYTES, UNAL>(
                smem, bar, nch, sc,
                [&](int tile, int64_t j) {
                    const int64_t t0 = (nch - 1 - j) * kCkpt, c0 = (int64_t)tile * W;
                    const bool ck = t0 > 0 || a.ck0;   // chunk 0 without a stored V[-1]: no checkpoint box
                    uint32_t b = (ck ? (uint32_t)(NB * Cfg::CK_BOX_BYTES) : 0u) + Reg::tx_bytes(fx, t0, rows_of(j), c0, ld) +
                                 Reg::tx_bytes(fg, t0, rows_of(j), c0, ld);
                    if constexpr (RES) b += Reg::tx_bytes(fr, t0, rows_of(j), c0, ld);
                    return b;
                },
                [&](unsigned char* stg, int tile, int64_t j, uint64_t* fb) {
                    const int64_t ch = nch - 1 - j;
                    const int rows = rows_of(j);
                    const int64_t c0 = (int64_t)tile * W;
                    if (lane == 0 && (ch > 0 || a.ck0)) {
#pragma unroll
                        for (int b = 0; b < NB; ++b)   // checkpoints: the saved rows are always 16-B aligned
                            tma_load_2d(stg + Cfg::CK_OFF + b * Cfg::CK_BOX_BYTES, &tmck, (int)(c0 + b * BW), (int)ch,
                                        fb, pol);
                    }
                    Reg::load(stg + Cfg::X_OFF, &tmx, fx, c0, ch * kCkpt, rows, ld, fb, pol);
                    Reg::load(stg + Cfg::G_OFF, &tmg, fg, c0, ch * kCkpt, rows, ld, fb, pol, kCkpt);
                    if constexpr (RES) Reg::load(stg + Cfg::R_OFF, &tmr, fr, c0, ch * kCkpt, rows, ld, fb, pol, 2 * kCkpt);
                });
        }
        return;
    }

    // ---------------- consumers
    LifConsts c = a.c;
    pin(c);
    const int ct = threadIdx.x - 32;
    const int nt = ct * VEC;
    const int ckoff = box_off<VEC, BW, 1>(nt, 0);
    IO* gx = reinterpret_cast<IO*>(a.gX);
    const int64_t ldb = ld * (int64_t)sizeof(IO);
    uint32_t k = 0;
    while (true) {
        int s = k % S;
        mbar_wait(&bar->full[s], (k / S) & 1);
        const int tile = bar->tile[s];
        if (tile < 0) break;
        tr.stage();
        tr.tile(tile);
        const int64_t n0 = (int64_t)tile * W + nt;
        const int nvalid = group_valid(n0, N, VEC);
        const bool tile_full = (int64_t)(tile + 1) * W <= N;   // uniform across the CTA
        const AffCoef<VEC> co = load_affine<VEC, Mode<MODE>::AFF>(a.af, n0, nvalid);
        float pa[VEC], pb[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) pa[i] = pb[i] = 0.0f;
        float gV[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = 0.0f;
        if (a.h.recv_state != nullptr) {            // dL/dV from the later segment's rank
            handoff_recv<VEC>(a.h, N, n0, nvalid, gV);
        } else if (a.grad_v_final != nullptr && nvalid > 0) {
            load_vec<VEC>(a.grad_v_final + n0, nvalid, gV);
        }
        for (int64_t ch = nch - 1; ch >= 0; --ch, ++k) {
            if (ch < nch - 1) {
                s = k % S;
                mbar_wait(&bar->full[s], (k / S) & 1);
            }
            const int64_t t0 = ch * kCkpt;
            const int rows = (int)min((int64_t)kCkpt, T - t0);
            const unsigned char* stg = smem + s * Cfg::STAGE_BYTES;
            const auto xs = row_src<IO, VEC, BW, kCkpt, NB, UNAL>(stg + Cfg::X_OFF, nt, t0, ld, a.x_off);
            const auto gsm = row_src<IO, VEC, BW, kCkpt, NB, UNAL>(stg + Cfg::G_OFF, nt, t0, ld, a.g_off);
            const auto rs = row_src<IO, VEC, BW, kCkpt, NB, UNAL>(stg + Cfg::R_OFF, nt, t0, ld, a.r_off);
            const Pack<float, VEC> v0 =
                (ch > 0 || a.ck0)
                    ? *reinterpret_cast<const Pack<float, VEC>*>(reinterpret_cast<const float*>(stg + Cfg::CK_OFF) + ckoff)
                    : entry_v0<VEC>(a.v_init, n0, nvalid, c.v_reset);
            float V[VEC];
#pragma unroll
            for (int i = 0; i < VEC; ++i) V[i] = v0.v[i];
            float h[kCkpt][VEC];
            IO* gxp = gx + (t0 + rows - 1) * ld + n0;
            IO* grp = nullptr;
            if constexpr (RES) grp = reinterpret_cast<IO*>(a.af.grad_residual) + (t0 + rows - 1) * ld + n0;
            if (rows == kCkpt && tile_full) {   // full chunk of a full tile: guard-free code
                recompute_chunk<IO, VEC, MODE, kCkpt>(c, V, h, xs, kCkpt, co, rs);
                bwd_chunk<IO, VEC, MODE, kCkpt, UNAL>(c, gV, h, gsm, gxp, ldb, kCkpt, VEC, co, xs, pa, pb, grp);
            } else if (rows == kCkpt / 2 && tile_full) {   // half chunk (T % 16 == 8, e.g. T = 8): guard-free too
                constexpr int HR = kCkpt / 2;
                recompute_chunk<IO, VEC, MODE, HR>(c, V, h, xs, HR, co, rs);
                bwd_chunk<IO, VEC, MODE, HR, UNAL>(c, gV, reinterpret_cast<const float(&)[HR][VEC]>(h), gsm, gxp, ldb,
                                                   HR, VEC, co, xs, pa, pb, grp);
            } else {                            // partial chunk or ragged tile: masked rows
                IO* gx0 = gx + t0 * ld + n0;
                IO* gr0 = RES ? reinterpret_cast<IO*>(a.af.grad_residual) + t0 * ld + n0 : nullptr;
                if (rows <= kCkpt / 4) {
                    recompute_chunk<IO, VEC, MODE, kCkpt / 4>(c, V, h, xs, kCkpt / 4, co, rs);
                    bwd_chunk_masked<IO, VEC, MODE, kCkpt / 4, UNAL>(c, gV, h, gsm, gx0, ldb, rows, nvalid, co, xs, pa,
                                                                     pb, gr0);
                } else if (rows <= kCkpt / 2) {
                    recompute_chunk<IO, VEC, MODE, kCkpt / 2>(c, V, h, xs, kCkpt / 2, co, rs);
                    bwd_chunk_masked<IO, VEC, MODE, kCkpt / 2, UNAL>(c, gV, h, gsm, gx0, ldb, rows, nvalid, co, xs, pa,
                                                                     pb, gr0);
                } else {
                    recompute_chunk<IO, VEC, MODE, kCkpt>(c, V, h, xs, kCkpt, co, rs);
                    bwd_chunk_masked<IO, VEC, MODE, kCkpt, UNAL>(c, gV, h, gsm, gx0, ldb, rows, nvalid, co, xs, pa, pb,
                                                                 gr0);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->empty[s]);
        }
        if (a.h.send_state != nullptr || a.h.recv_ack != nullptr)   // uniform across the CTA
            handoff_send<VEC, NCONS>(a.h, tile, W, N, n0, nvalid, gV);
        if constexpr (Mode<MODE>::AFF) {
            if (a.af.seg > 0) {   // uniform: fold the per-channel reduction into the tile epilogue
                if constexpr (VEC * 32 == kSegMax)
                    affine_warp_segments<VEC>(pa, pb, nvalid, n0, a.af.seg, N / a.af.seg, a.af.part_a, a.af.part_b);
            } else if (nvalid > 0) {
                store_vec<VEC>(a.af.part_a + n0, nvalid, pa);
                store_vec<VEC>(a.af.part_b + n0, nvalid, pb);
            }
        }
        if (a.grad_v_init != nullptr && nvalid > 0) store_vec<VEC>(a.grad_v_init + n0, nvalid, gV);
    }
    if (warp == 1) tr.done(SNN_TRACE_BUF(a), 2u, T, N);
}

// ------------------------------------------------------------------------------------
// Backward, SAVE_H.  Stage = R time rows of H (fp32) and gS; row blocks streamed last-first.
template <typename IO, int VEC, int NCONS, int R, int S, bool UNAL = false>
struct BwdHTma {
    static constexpr int W = NCONS * VEC;
    static constexpr int BW = W < 256 ? W : 256;
    static constexpr int NB = W / BW;
    static constexpr int HBOX = BW * R * 4;
    using Reg = Region<IO, BW, R, NB, UNAL>;
    static constexpr int G_OFF = NB * HBOX;
    static constexpr int STAGE_BYTES = NB * HBOX + Reg::BYTES;
    static constexpr int SMEM = S * STAGE_BYTES + (int)sizeof(Barriers<S>) + kAlignSlack;
    static constexpr int THREADS = NCONS + 32;
    static_assert(W % BW == 0 && BW % VEC == 0 && STAGE_BYTES % 128 == 0, "tile geometry");
};

template <typename IO, int VEC, int MODE, int NCONS, int R, int S, bool UNAL>
__global__ void __launch_bounds__(NCONS + 32)
lif_backward_saveh_tma_kernel(const __grid_constant__ CUtensorMap tmh,
                              const __grid_constant__ CUtensorMap tmg, const BwdArgs a,
                              const Sched sc) {
    using Cfg = BwdHTma<IO, VEC, NCONS, R, S, UNAL>;
    using Reg = typename Cfg::Reg;
    constexpr int W = Cfg::W, BW = Cfg::BW, NB = Cfg::NB;
    unsigned char* smem = smem_base();
    auto* bar = reinterpret_cast<Barriers<S>*>(smem + S * Cfg::STAGE_BYTES);
    TraceCta tr;
    tr.entry();
    init_barriers<S>(bar, NCONS / 32);
    const int64_t T = a.T, N = a.N, ld = a.ld;
    const int64_t nrb = (T + R - 1) / R;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {   // before the wait: kernel-parameter descriptors, L2 prefetch of the own tile
        tma_prefetch_desc(&tmh); tma_prefetch_desc(&tmg);
        const int c0 = (int)blockIdx.x * W;
        for (int j = 0; j < sc.prefetch && j < S && j < nrb; ++j) {
            const int rb = (int)nrb - 1 - j;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                tma_prefetch_2d(&tmh, c0 + b * BW, rb * R);
                if constexpr (!UNAL) tma_prefetch_2d(&tmg, c0 + b * BW, rb * R);
            }
        }
    }
    pdl_wait();   // predecessor complete before any global-memory access
    tr.waited();

    if (warp == 0) {   // producer (whole warp if unaligned)
        if (UNAL || lane == 0) {
            const uint64_t pol = policy_evict_first();
            auto rows_of = [&](int64_t j) {
                const int64_t rb = nrb - 1 - j;
                return (int)min((int64_t)R, T - rb * R);
            };
            const auto fg = Reg::flat(a.gS, T, N, ld);
            produce<S, Cfg::STAGE_BYTES, UNAL>(
                smem, bar, nrb, sc,
                [&](int tile, int64_t j) {
                    return (uint32_t)(NB * Cfg::HBOX) +
                           Reg::tx_bytes(fg, (nrb - 1 - j) * R, rows_of(j), (int64_t)tile * W, ld);
                },
                [&](unsigned char* stg, int tile, int64_t j, uint64_t* fb) {
                    const int64_t rb = nrb - 1 - j;
                    const int64_t c0 = (int64_t)tile * W;
                    if (lane == 0) {
#pragma unroll
                        for (int b = 0; b < NB; ++b)   // H: the saved rows are always 16-B aligned
                            tma_load_2d(stg + b * Cfg::HBOX, &tmh, (int)(c0 + b * BW), (int)(rb * R), fb, pol);
                    }
                    Reg::load(stg + Cfg::G_OFF, &tmg, fg, c0, rb * R, rows_of(j), ld, fb, pol);
                });
        }
        return;
    }

    LifConsts c = a.c;
    pin(c);
    const int ct = threadIdx.x - 32;
    const int nt = ct * VEC;
    const int roff = box_off<VEC, BW, R>(nt, 0);
    IO* gx = reinterpret_cast<IO*>(a.gX);
    const int64_t ldb = ld * (int64_t)sizeof(IO);
    uint32_t k = 0;
    while (true) {
        int s = k % S;
        mbar_wait(&bar->full[s], (k / S) & 1);
        const int tile = bar->tile[s];
        if (tile < 0) break;
        tr.stage();
        tr.tile(tile);
        const int64_t n0 = (int64_t)tile * W + nt;
        const int nvalid = group_valid(n0, N, VEC);
        const bool tile_full = (int64_t)(tile + 1) * W <= N;   // uniform across the CTA
        float gV[VEC];
#pragma unroll
        for (int i = 0; i < VEC; ++i) gV[i] = 0.0f;
        if (a.h.recv_state != nullptr) {            // dL/dV from the later segment's rank
            handoff_recv<VEC>(a.h, N, n0, nvalid, gV);
        } else if (a.grad_v_final != nullptr && nvalid > 0) {
            load_vec<VEC>(a.grad_v_final + n0, nvalid, gV);
        }
        for (int64_t rb = nrb - 1; rb >= 0; --rb, ++k) {
            if (rb < nrb - 1) {
                s = k % S;
                mbar_wait(&bar->full[s], (k / S) & 1);
            }
            const int rows = (int)min((int64_t)R, T - rb * R);
            const unsigned char* stg = smem + s * Cfg::STAGE_BYTES;
            const float* hs = reinterpret_cast<const float*>(stg) + roff;
            const auto gsm = row_src<IO, VEC, BW, R, NB, UNAL>(stg + Cfg::G_OFF, nt, rb * R, ld, a.g_off);
            IO* gxp = gx + (rb * R + rows - 1) * ld + n0;
            auto walk = [&](auto full) {
                constexpr bool F = decltype(full)::value;
#pragma unroll
                for (int r = R - 1; r >= 0; --r) {
                    if (F || r < rows) {
                        const Pack<float, VEC> hv = *reinterpret_cast<const Pack<float, VEC>*>(hs + r * BW);
                        const Pack<IO, VEC> gv = gsm(r);
                        const Pack<IO, VEC> out = bwd_step<IO, VEC, MODE>(c, gV, hv.v, gv);
                        if (F || nvalid > 0) st_out<UNAL>(gxp, out, F ? VEC : nvalid);
                        gxp = step_bytes(gxp, -ldb);
                    }
                }
            };
            // (a masked walk, as the RECOMPUTE backward's partial chunks use, measured slower here)
            if (rows == R && tile_full) walk(std::true_type{}); else walk(std::false_type{});
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar->empty[s]);
        }
        if (a.h.send_state != nullptr || a.h.recv_ack != nullptr)   // uniform across the CTA
            handoff_send<VEC, NCONS>(a.h, tile, W, N, n0, nvalid, gV);
        if (a.grad_v_init != nullptr && nvalid > 0) store_vec<VEC>(a.grad_v_init + n0, nvalid, gV);
    }
    if (warp == 1) tr.done(SNN_TRACE_BUF(a), 3u, T, N);
}

}  // namespace snn
