// comm.cu -- the paper's time-segment split behind the C ABI (include/snn_lif.h
// snn_comm_* / snn_lif_*_tsplit).
//
// Rank d of an NCCL communicator owns time steps [t_d, t_{d+1}) of every neuron (ranks are
// ordered like time).  Forward: rank d receives the previous segment's post-reset V [N]
// fp32 from rank d-1, runs the fused forward over its segment and sends its final V to rank
// d+1 ("the boundary membrane state is handed to the next rank", BASELINE north_star (3)).
// Backward mirrors it: dL/dV arrives from d+1 and grad_v_init leaves to d-1.  To give the k
// ranks concurrent work on one layer the neuron axis is cut into n_chunks
// chunks processed in the same order everywhere: rank d starts chunk m once chunk m's
// boundary has arrived -- a wavefront of efficiency M/(M+k-1).
//
// Streams: the kernels run on the caller's stream, the NCCL point-to-point operations on the
// communicator's own stream, ordered by events (recv(m) -> kernel(m) -> send(m)); the two
// streams fork from and join back into the caller's stream, so a call is capturable into a
// CUDA graph and the compute of chunk m+1 overlaps the transfer of chunk m.
//
// NCCL is resolved at run time (dlopen): the library loads and every non-NCCL entry point
// works without it; inside a process that already loaded NCCL (torch) that same copy is used.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>
#include <nccl_device.h>   // ncclWindow_t, ncclGetPeerPointer (the symmetric-window handoff below)

#include "internal.h"

namespace snn_host {
namespace {

struct NcclApi {
    bool ok = false;
    char why[256] = "";
    int version = 0;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    // symmetric memory windows (NCCL >= 2.27; optional: the window handoff needs them)
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*MemFree)(void*) = nullptr;
    ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclTeam_t (*TeamLsa)(ncclComm_t) = nullptr;
    bool windows = false;
};

// libnccl.so.2: the copy already in the process (torch's) if any, else $SNN_NCCL_LIBRARY, else
// the loader's search path.
const NcclApi& nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = std::getenv("SNN_NCCL_LIBRARY");
        if (!h && env && env[0]) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            snprintf(api.why, sizeof(api.why), "cannot load libnccl.so.2: %s", dlerror());
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
#define SNN_NCCL_SYM(field, name)                                                  \
        api.field = reinterpret_cast<decltype(api.field)>(sym(name));                  \
        if (!api.field) { snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name); return; }
        SNN_NCCL_SYM(GetVersion, "ncclGetVersion")
        SNN_NCCL_SYM(GetUniqueId, "ncclGetUniqueId")
        SNN_NCCL_SYM(CommInitRank, "ncclCommInitRank")
        SNN_NCCL_SYM(CommDestroy, "ncclCommDestroy")
        SNN_NCCL_SYM(CommGetAsyncError, "ncclCommGetAsyncError")
        SNN_NCCL_SYM(Send, "ncclSend")
        SNN_NCCL_SYM(Recv, "ncclRecv")
        SNN_NCCL_SYM(GroupStart, "ncclGroupStart")
        SNN_NCCL_SYM(GroupEnd, "ncclGroupEnd")
        SNN_NCCL_SYM(GetErrorString, "ncclGetErrorString")
#undef SNN_NCCL_SYM
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.MemAlloc = reinterpret_cast<decltype(api.MemAlloc)>(sym("ncclMemAlloc"));
        api.MemFree = reinterpret_cast<decltype(api.MemFree)>(sym("ncclMemFree"));
        api.CommWindowRegister = reinterpret_cast<decltype(api.CommWindowRegister)>(sym("ncclCommWindowRegister"));
        api.CommWindowDeregister =
            reinterpret_cast<decltype(api.CommWindowDeregister)>(sym("ncclCommWindowDeregister"));
        api.TeamLsa = reinterpret_cast<decltype(api.TeamLsa)>(sym("ncclTeamLsa"));
        api.windows = api.AllReduce && api.MemAlloc && api.MemFree && api.CommWindowRegister &&
                      api.CommWindowDeregister && api.TeamLsa;
        api.GetVersion(&api.version);
        api.ok = true;
    });
    return api;
}

}  // namespace
}  // namespace snn_host

using namespace snn_host;

struct snn_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = -1;
    cudaStream_t cs = nullptr;                     // NCCL operations
    cudaEvent_t fork = nullptr, join = nullptr;
    std::vector<cudaEvent_t> recv_ev, done_ev;     // per chunk
    float* scratch = nullptr;                      // connection warm-up
};

namespace {

#define SNN_NCCL_TRY(expr, what)                                                                   \
    do {                                                                                           \
        const ncclResult_t r_ = (expr);                                                            \
        if (r_ != ncclSuccess)                                                                     \
            return fail(SNN_ERR_NCCL, "%s: %s", what, nccl_api().GetErrorString(r_));                   \
    } while (0)
#define SNN_CUDA_OK(expr, what)                                                                    \
    do {                                                                                           \
        const cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess) return fail(SNN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

snn_status ensure_events(snn_comm* c, int n) {
    while ((int)c->recv_ev.size() < n) {
        cudaEvent_t a, b;
        SNN_CUDA_OK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "cudaEventCreate");
        SNN_CUDA_OK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "cudaEventCreate");
        c->recv_ev.push_back(a);
        c->done_ev.push_back(b);
    }
    return SNN_OK;
}

// Neuron chunk m of M over N: boundaries on multiples of 512 (whole TMA tiles and whole
// 32-bit spike words), the first (units mod M) chunks one unit longer.
constexpr int64_t kChunkAlign = 512;
void chunk_range(int64_t N, int M, int m, int64_t* a, int64_t* b) {
    const int64_t units = (N + kChunkAlign - 1) / kChunkAlign;
    const int64_t q = units / M, r = units % M;
    const int64_t lo = m * q + std::min<int64_t>(m, r);
    const int64_t hi = lo + q + (m < r ? 1 : 0);
    *a = std::min(N, lo * kChunkAlign);
    *b = std::min(N, hi * kChunkAlign);
}

int effective_chunks(int64_t N, int n_chunks) {
    const int64_t units = (N + kChunkAlign - 1) / kChunkAlign;
    return (int)std::max<int64_t>(1, std::min<int64_t>(n_chunks, units));
}

snn_status check_comm(const snn_comm* c) {
    if (!c) return fail(SNN_ERR_NULL_POINTER, "comm is NULL");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != c->device)
        return fail(SNN_ERR_INVALID_VALUE, "comm was created on device %d, current device is %d", c->device, dev);
    return SNN_OK;
}

size_t io_bytes(int dt) { return dt == SNN_BF16 ? 2 : 4; }

// Pointer of column a in a [T, ld] tensor of element size esz (or bit-packed spike words).
template <typename P>
P* col(P* base, int64_t a, size_t esz) {
    return base ? reinterpret_cast<P*>(reinterpret_cast<uintptr_t>(base) + (uintptr_t)(a * (int64_t)esz)) : nullptr;
}

}  // namespace

extern "C" {

snn_status snn_nccl_unique_id(void* out) {
    if (!out) return fail(SNN_ERR_NULL_POINTER, "out is NULL");
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(SNN_ERR_NCCL, "%s", api.why);
    ncclUniqueId id;
    SNN_NCCL_TRY(api.GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == SNN_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
    return SNN_OK;
}

snn_status snn_comm_create(snn_comm** out, const void* unique_id, int nranks, int rank) {
    if (!out) return fail(SNN_ERR_NULL_POINTER, "out is NULL");
    *out = nullptr;
    if (!unique_id) return fail(SNN_ERR_NULL_POINTER, "unique_id is NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(SNN_ERR_INVALID_VALUE, "need 0 <= rank < nranks (rank=%d nranks=%d)", rank, nranks);
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(SNN_ERR_NCCL, "%s", api.why);
    auto c = std::make_unique<snn_comm>();
    c->nranks = nranks;
    c->rank = rank;
    SNN_CUDA_OK(cudaGetDevice(&c->device), "cudaGetDevice");
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    SNN_NCCL_TRY(api.CommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank");
    auto cleanup = [&] { api.CommDestroy(c->comm); c->comm = nullptr; };
    cudaError_t e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&c->scratch, 4 * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(c->scratch, 0, 4 * sizeof(float));
    if (e != cudaSuccess) {
        cleanup();
        return fail(SNN_ERR_CUDA, "comm resources: %s", cudaGetErrorString(e));
    }
    // Connect both neighbours in both directions now (NCCL sets point-to-point connections up
    // lazily, at their first use): the time-split calls then never pay the handshake.
    if (nranks > 1) {
        for (int dir = 0; dir < 2; ++dir) {
            const int to = dir == 0 ? rank + 1 : rank - 1, from = dir == 0 ? rank - 1 : rank + 1;
            ncclResult_t r = api.GroupStart();
            if (r == ncclSuccess && to >= 0 && to < nranks) r = api.Send(c->scratch, 1, ncclFloat32, to, c->comm, c->cs);
            if (r == ncclSuccess && from >= 0 && from < nranks)
                r = api.Recv(c->scratch + 1, 1, ncclFloat32, from, c->comm, c->cs);
            const ncclResult_t r2 = api.GroupEnd();
            if (r == ncclSuccess) r = r2;
            if (r != ncclSuccess) {
                cleanup();
                return fail(SNN_ERR_NCCL, "neighbour connection: %s", api.GetErrorString(r));
            }
        }
        e = cudaStreamSynchronize(c->cs);
        if (e != cudaSuccess) {
            cleanup();
            return fail(SNN_ERR_CUDA, "neighbour connection: %s", cudaGetErrorString(e));
        }
    }
    *out = c.release();
    return SNN_OK;
}

snn_status snn_comm_destroy(snn_comm* c) {
    if (!c) return SNN_OK;
    snn_status st = SNN_OK;
    if (c->cs) cudaStreamSynchronize(c->cs);
    if (c->comm) {
        const ncclResult_t r = nccl_api().CommDestroy(c->comm);
        if (r != ncclSuccess) st = fail(SNN_ERR_NCCL, "ncclCommDestroy: %s", nccl_api().GetErrorString(r));
    }
    for (auto ev : c->recv_ev) cudaEventDestroy(ev);
    for (auto ev : c->done_ev) cudaEventDestroy(ev);
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->join) cudaEventDestroy(c->join);
    if (c->scratch) cudaFree(c->scratch);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
    return st;
}

snn_status snn_comm_info(const snn_comm* c, int* nranks, int* rank) {
    if (!c) return fail(SNN_ERR_NULL_POINTER, "comm is NULL");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    return SNN_OK;
}

}  // extern "C"

namespace {

// The shared chunk loop.  dir = +1 (forward: receive from rank-1, send to rank+1) or -1
// (backward: receive from rank+1, send to rank-1).  `launch(m, a, b, recv_ptr_or_null)` enqueues
// chunk m's kernel on the caller's stream and returns its status; `in` / `out` are the [N]
// boundary buffers (the chunk's slice [a, b) is sent / received).
template <typename Launch>
snn_status tsplit_loop(snn_comm* c, int64_t N, int M, int dir, float* in, float* out, cudaStream_t st,
                       Launch launch) {
    const NcclApi& api = nccl_api();
    const int from = c->rank - dir, to = c->rank + dir;
    const bool has_from = c->nranks > 1 && from >= 0 && from < c->nranks;
    const bool has_to = c->nranks > 1 && to >= 0 && to < c->nranks;
    if (!has_from && !has_to) {   // k = 1: the plain chunked kernels
        for (int m = 0; m < M; ++m) {
            int64_t a, b;
            chunk_range(N, M, m, &a, &b);
            const snn_status s = launch(m, a, b, false);
            if (s != SNN_OK) return s;
        }
        return SNN_OK;
    }
    snn_status s;
    if ((s = ensure_events(c, M)) != SNN_OK) return s;
    // fork the comm stream off the caller's stream (earlier work on it -- e.g. the producer of
    // x, or a previous call reading the same boundary buffers -- comes first)
    SNN_CUDA_OK(cudaEventRecord(c->fork, st), "cudaEventRecord");
    SNN_CUDA_OK(cudaStreamWaitEvent(c->cs, c->fork, 0), "cudaStreamWaitEvent");
    int64_t a0, b0;
    chunk_range(N, M, 0, &a0, &b0);
    if (has_from) {
        SNN_NCCL_TRY(api.Recv(in + a0, (size_t)(b0 - a0), ncclFloat32, from, c->comm, c->cs), "ncclRecv");
        SNN_CUDA_OK(cudaEventRecord(c->recv_ev[0], c->cs), "cudaEventRecord");
    }
    for (int m = 0; m < M; ++m) {
        int64_t a, b;
        chunk_range(N, M, m, &a, &b);
        if (has_from) SNN_CUDA_OK(cudaStreamWaitEvent(st, c->recv_ev[m], 0), "cudaStreamWaitEvent");
        {
            NvtxRange chunk("tsplit chunk");
            if ((s = launch(m, a, b, has_from)) != SNN_OK) return s;
        }
        SNN_CUDA_OK(cudaEventRecord(c->done_ev[m], st), "cudaEventRecord");
        SNN_CUDA_OK(cudaStreamWaitEvent(c->cs, c->done_ev[m], 0), "cudaStreamWaitEvent");
        // chunk m's boundary out, and the next chunk's boundary in, as one NCCL group
        int64_t a1 = 0, b1 = 0;
        const bool next_in = has_from && m + 1 < M;
        if (next_in) chunk_range(N, M, m + 1, &a1, &b1);
        SNN_NCCL_TRY(api.GroupStart(), "ncclGroupStart");
        ncclResult_t r = ncclSuccess;
        if (has_to) r = api.Send(out + a, (size_t)(b - a), ncclFloat32, to, c->comm, c->cs);
        if (r == ncclSuccess && next_in) r = api.Recv(in + a1, (size_t)(b1 - a1), ncclFloat32, from, c->comm, c->cs);
        const ncclResult_t r2 = api.GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(SNN_ERR_NCCL, "boundary exchange of chunk %d: %s", m,
                        api.GetErrorString(r != ncclSuccess ? r : r2));
        if (next_in) SNN_CUDA_OK(cudaEventRecord(c->recv_ev[m + 1], c->cs), "cudaEventRecord");
    }
    // join: the caller's stream waits for the last send (the boundary buffers may be reused)
    SNN_CUDA_OK(cudaEventRecord(c->join, c->cs), "cudaEventRecord");
    SNN_CUDA_OK(cudaStreamWaitEvent(st, c->join, 0), "cudaStreamWaitEvent");
    ncclResult_t ae = ncclSuccess;
    if (api.CommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
        return fail(SNN_ERR_NCCL, "communicator error: %s", api.GetErrorString(ae));
    return SNN_OK;
}

// Validate a whole-layer call without enqueuing anything: run it with a launch recorder
// installed (internal.h), so every check and tensor-map encode happens and no kernel launches.
template <typename F>
snn_status dry_run(F body) {
    Recorder rec;
    Recorder*& slot = current_recorder();
    Recorder* prev = slot;
    slot = &rec;
    const snn_status st = body();
    slot = prev;
    return st;
}

snn_status tsplit_common_checks(snn_comm* c, const snn_lif_shape* s, int n_chunks) {
    snn_status st;
    if ((st = check_comm(c)) != SNN_OK) return st;
    if (!s) return fail(SNN_ERR_NULL_POINTER, "shape is NULL");
    if (n_chunks < 1) return fail(SNN_ERR_INVALID_VALUE, "n_chunks=%d must be >= 1", n_chunks);
    if (n_chunks > s->N) return fail(SNN_ERR_INVALID_VALUE, "n_chunks=%d > N=%lld", n_chunks, (long long)s->N);
    if (c->nranks > 1 && !nccl_api().ok) return fail(SNN_ERR_NCCL, "%s", nccl_api().why);
    return SNN_OK;
}

}  // namespace

extern "C" {

snn_status snn_lif_forward_tsplit(snn_comm* c, const snn_lif_params* p, const snn_lif_shape* s,
                                  int n_chunks, const void* x, void* spikes, void* saved,
                                  float* v_in_ws, float* v_out_ws, void* stream) {
    NvtxRange range("snn_lif_forward_tsplit");
    snn_status st;
    if ((st = tsplit_common_checks(c, s, n_chunks)) != SNN_OK) return st;
    const bool first = c->rank == 0, last = c->rank == c->nranks - 1;
    if (!first && !v_in_ws) return fail(SNN_ERR_NULL_POINTER, "v_in_ws is required on ranks > 0 (receive buffer)");
    if (!last && !v_out_ws) return fail(SNN_ERR_NULL_POINTER, "v_out_ws is required on ranks < nranks-1 (send buffer)");
    // whole-layer validation first: a non-OK status means nothing was enqueued
    if ((st = dry_run([&] { return forward_impl(p, s, x, v_in_ws, nullptr, spikes, saved, v_out_ws, stream); })) !=
        SNN_OK)
        return st;
    const int M = effective_chunks(s->N, n_chunks);
    const size_t esz = io_bytes(s->io_dtype);
    const ChunkView cv{saved_row_stride(s), (s->N + 31) / 32};
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    return tsplit_loop(c, s->N, M, +1, v_in_ws, v_out_ws, cs, [&](int, int64_t a, int64_t b, bool) {
        snn_lif_shape sc = *s;
        sc.N = b - a;
        void* spk = s->spike_fmt == SNN_SPK_BITS ? col(spikes, a / 32, 4)
                  : col(spikes, a, s->spike_fmt == SNN_SPK_U8 ? 1 : esz);
        // rank 0 starts from v_in_ws (the layer's v_init) when given, else V_reset
        const float* vin = v_in_ws ? v_in_ws + a : nullptr;
        return forward_impl(p, &sc, col(x, a, esz), vin, nullptr, spk, col(saved, a, 4),
                            v_out_ws ? v_out_ws + a : nullptr, stream, nullptr, &cv);
    });
}

snn_status snn_lif_backward_tsplit(snn_comm* c, const snn_lif_params* p, const snn_lif_shape* s,
                                   int n_chunks, const void* grad_spikes, const void* x,
                                   const float* v_in_ws, const void* saved, void* grad_x,
                                   float* g_in_ws, float* g_out_ws, void* stream) {
    NvtxRange range("snn_lif_backward_tsplit");
    snn_status st;
    if ((st = tsplit_common_checks(c, s, n_chunks)) != SNN_OK) return st;
    const bool first = c->rank == 0, last = c->rank == c->nranks - 1;
    if (!last && !g_in_ws) return fail(SNN_ERR_NULL_POINTER, "g_in_ws is required on ranks < nranks-1 (receive buffer)");
    if (!first && !g_out_ws) return fail(SNN_ERR_NULL_POINTER, "g_out_ws is required on ranks > 0 (send buffer)");
    if ((st = dry_run([&] {
             return backward_impl(p, s, grad_spikes, x, v_in_ws, saved, g_in_ws, nullptr, grad_x, g_out_ws, stream);
         })) != SNN_OK)
        return st;
    const int M = effective_chunks(s->N, n_chunks);
    const size_t esz = io_bytes(s->io_dtype);
    const ChunkView cv{saved_row_stride(s), (s->N + 31) / 32};
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    return tsplit_loop(c, s->N, M, -1, g_in_ws, g_out_ws, cs, [&](int, int64_t a, int64_t b, bool) {
        snn_lif_shape sc = *s;
        sc.N = b - a;
        // the last rank starts from g_in_ws (the layer's grad_v_final) when given, else 0
        const float* gin = g_in_ws ? g_in_ws + a : nullptr;
        // chunk 0's V[-1]: the slice of v_in_ws the forward started from (received from d-1, or
        // rank 0's v_init), else V_reset
        const float* vin = v_in_ws ? v_in_ws + a : nullptr;
        return backward_impl(p, &sc, col(grad_spikes, a, esz), col(x, a, esz), vin, col(saved, a, 4), gin, nullptr,
                             col(grad_x, a, esz), g_out_ws ? g_out_ws + a : nullptr, stream, nullptr, nullptr,
                             nullptr, &cv);
    });
}

}  // extern "C"

// ---- the fused boundary handoff over NCCL symmetric windows -------------
// Every rank allocates one buffer with ncclMemAlloc holding the receive sides of both
// directions -- [fwd state N f32 | fwd ready nblk | fwd ack nblk | bwd state N f32 | bwd ready
// nblk | bwd ack nblk], each part 256-B aligned, identical offsets on every rank -- and
// registers it as a symmetric window on the snn_comm's communicator.  The neighbours' parts are
// then plain load/store addresses of this process (ncclGetPeerPointer: the LSA team's flat
// mapping over NVLink), handed to the kernels' existing snn_lif_handoff struct: the kernels
// store each tile's carry-out straight into the neighbour's buffer and release its flag, as
// with CUDA IPC (lif_handoff.cuh), but the peers come from the NCCL communicator.

struct snn_handoff_window {
    snn_comm* comm = nullptr;
    void* buf = nullptr;
    size_t bytes = 0;
    ncclWindow_t win = nullptr;
    int64_t N = 0, nblk = 0;
    size_t off[6] = {};
    char* local = nullptr;
    char* prev = nullptr;   // rank-1's buffer (NULL on rank 0)
    char* next = nullptr;   // rank+1's buffer (NULL on the last rank)
    int epoch[2] = {0, 0};
};

namespace snn_window {
__global__ void window_peer_ptrs(ncclWindow_t w, int p0, int p1, void** out) {
    out[0] = p0 >= 0 ? ncclGetPeerPointer(w, 0, p0) : nullptr;
    out[1] = p1 >= 0 ? ncclGetPeerPointer(w, 0, p1) : nullptr;
}
}  // namespace snn_window

namespace {

size_t round256(size_t b) { return (b + 255) & ~size_t(255); }

void window_free(snn_handoff_window* w) {
    const NcclApi& api = nccl_api();
    if (w->win) api.CommWindowDeregister(w->comm->comm, w->win);
    if (w->buf) api.MemFree(w->buf);
    delete w;
}

}  // namespace

extern "C" {

snn_status snn_handoff_window_create(snn_comm* c, int64_t N, snn_handoff_window** out) {
    NvtxRange range("snn_handoff_window_create");
    if (!out) return fail(SNN_ERR_NULL_POINTER, "out is NULL");
    *out = nullptr;
    snn_status st;
    if ((st = check_comm(c)) != SNN_OK) return st;
    if (N < 1) return fail(SNN_ERR_INVALID_VALUE, "N=%lld must be >= 1", (long long)N);
    const NcclApi& api = nccl_api();
    if (!api.ok) return fail(SNN_ERR_NCCL, "%s", api.why);
    if (!api.windows) return fail(SNN_ERR_UNSUPPORTED, "libnccl.so.2 (version %d) has no symmetric-window API", api.version);
    // every neighbour must be a load/store peer (the LSA team: same node, NVLink / P2P)
    const ncclTeam_t lsa = api.TeamLsa(c->comm);
    for (int peer : {c->rank - 1, c->rank + 1}) {
        if (peer < 0 || peer >= c->nranks) continue;
        const int i = lsa.rank + (peer - c->rank);
        if (lsa.stride != 1 || i < 0 || i >= lsa.nRanks)
            return fail(SNN_ERR_UNSUPPORTED,
                        "rank %d is not a load/store peer of rank %d (LSA team of %d ranks): use the NCCL "
                        "send/recv split (snn_lif_*_tsplit) or CUDA IPC peers",
                        peer, c->rank, lsa.nRanks);
    }
    auto w = new snn_handoff_window();
    w->comm = c;
    w->N = N;
    w->nblk = (N + SNN_LIF_HANDOFF_BLOCK - 1) / SNN_LIF_HANDOFF_BLOCK;
    const size_t part[6] = {round256(4 * (size_t)N), round256(4 * (size_t)w->nblk), round256(4 * (size_t)w->nblk),
                            round256(4 * (size_t)N), round256(4 * (size_t)w->nblk), round256(4 * (size_t)w->nblk)};
    for (int i = 0; i < 6; ++i) {
        w->off[i] = w->bytes;
        w->bytes += part[i];
    }
    w->bytes = (w->bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    ncclResult_t r = api.MemAlloc(&w->buf, w->bytes);
    if (r == ncclSuccess) r = api.CommWindowRegister(c->comm, w->buf, w->bytes, &w->win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
        window_free(w);
        return fail(SNN_ERR_NCCL, "symmetric window (ncclMemAlloc / ncclCommWindowRegister): %s", api.GetErrorString(r));
    }
    void** ptrs = nullptr;
    cudaError_t e = cudaMemsetAsync(w->buf, 0, w->bytes, c->cs);
    if (e == cudaSuccess) e = cudaMalloc(&ptrs, 2 * sizeof(void*));
    if (e == cudaSuccess) {
        snn_window::window_peer_ptrs<<<1, 1, 0, c->cs>>>(w->win, c->rank > 0 ? c->rank - 1 : -1,
                                             c->rank + 1 < c->nranks ? c->rank + 1 : -1, ptrs);
        e = cudaGetLastError();
    }
    void* host[2] = {nullptr, nullptr};
    if (e == cudaSuccess) e = cudaMemcpyAsync(host, ptrs, sizeof(host), cudaMemcpyDeviceToHost, c->cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->cs);
    if (ptrs) cudaFree(ptrs);
    if (e != cudaSuccess) {
        window_free(w);
        return fail(SNN_ERR_CUDA, "symmetric window setup: %s", cudaGetErrorString(e));
    }
    w->local = static_cast<char*>(w->buf);
    w->prev = static_cast<char*>(host[0]);
    w->next = static_cast<char*>(host[1]);
    // every rank's buffer is zeroed before any rank's kernel can publish into it
    if (c->nranks > 1) {
        r = api.AllReduce(c->scratch, c->scratch, 1, ncclFloat32, ncclSum, c->comm, c->cs);
        if (r != ncclSuccess) {
            window_free(w);
            return fail(SNN_ERR_NCCL, "window barrier: %s", api.GetErrorString(r));
        }
        e = cudaStreamSynchronize(c->cs);
        if (e != cudaSuccess) {
            window_free(w);
            return fail(SNN_ERR_CUDA, "window barrier: %s", cudaGetErrorString(e));
        }
    }
    *out = w;
    return SNN_OK;
}

snn_status snn_handoff_window_next(snn_handoff_window* w, int direction, snn_lif_handoff* h) {
    if (!w || !h) return fail(SNN_ERR_NULL_POINTER, "window or handoff is NULL");
    if (direction != 0 && direction != 1) return fail(SNN_ERR_INVALID_VALUE, "direction %d: 0 forward, 1 backward", direction);
    std::memset(h, 0, sizeof(*h));
    h->epoch = ++w->epoch[direction];
    // forward (0): receive V from rank-1 into my fwd part, send into rank+1's fwd part;
    // backward (1): receive dL/dV from rank+1 into my bwd part, send into rank-1's bwd part.
    const size_t st = direction == 0 ? w->off[0] : w->off[3], rd = direction == 0 ? w->off[1] : w->off[4],
                 ak = direction == 0 ? w->off[2] : w->off[5];
    char* from = direction == 0 ? w->prev : w->next;
    char* to = direction == 0 ? w->next : w->prev;
    if (from) {
        h->recv_state = reinterpret_cast<const float*>(w->local + st);
        h->recv_ready = reinterpret_cast<const int*>(w->local + rd);
        h->recv_ack = reinterpret_cast<int*>(from + ak);   // the sender's ack flags
    }
    if (to) {
        h->send_state = reinterpret_cast<float*>(to + st);
        h->send_ready = reinterpret_cast<int*>(to + rd);
        h->send_ack = reinterpret_cast<const int*>(w->local + ak);
    }
    return SNN_OK;
}

snn_status snn_handoff_window_pointer(const snn_handoff_window* w, int which, void** ptr) {
    if (!w || !ptr) return fail(SNN_ERR_NULL_POINTER, "window or ptr is NULL");
    if (which < -1 || which > 1) return fail(SNN_ERR_INVALID_VALUE, "which=%d: -1 previous, 0 own, 1 next", which);
    *ptr = which < 0 ? w->prev : which > 0 ? w->next : w->local;
    return SNN_OK;
}

snn_status snn_handoff_window_destroy(snn_handoff_window* w) {
    if (!w) return SNN_OK;
    snn_comm* c = w->comm;
    snn_status st = SNN_OK;
    cudaDeviceSynchronize();   // this rank's kernels are done with every buffer they touch
    if (c->nranks > 1) {       // ... and every other rank's too, before anything is freed
        const ncclResult_t r = nccl_api().AllReduce(c->scratch, c->scratch, 1, ncclFloat32, ncclSum, c->comm, c->cs);
        if (r != ncclSuccess) st = fail(SNN_ERR_NCCL, "window barrier: %s", nccl_api().GetErrorString(r));
        cudaStreamSynchronize(c->cs);
    }
    window_free(w);
    return st;
}

}  // extern "C"
