/*
 * snn_lif.h -- C ABI of the B200 (sm_100a) temporally fused LIF library
 *              (libsnn_lif.so, built from paper_2408_00280_b200/csrc/).
 *
 * The method: "temporal fusion" (arXiv 2408.00280) -- every LIF layer
 * runs all T time steps of its neurons inside ONE kernel launch, each neuron's state
 * held in registers across the time loop ("assigns each neuron's computation to an
 * individual GPU thread, amalgamating memory operations for each layer across all time
 * steps within the GPU kernel"), forward (Eq. 1-2) and backward
 * (Eq. 3) alike (Fig. 2 caption).  The paper's programming model
 * (Listing 1) exposes fusedForwardLIF(x, args) /
 * fusedBackwardLIF(grad_y, args); snn_lif_forward / snn_lif_backward are those two calls.
 *
 * ----------------------------------------------------------------------------------
 * Conventions shared by every entry point
 *
 *  Layout.  Time-major, row-major [T, N] with row stride `ld` elements (ld >= N), i.e.
 *  element (t, n) at t*ld + n (the paper's "memory alignment post-concatenation",
 *  PAPER.md:217-218; Listing 1 caption: x "aggregates a tensor for all neurons i across
 *  each time step t").  ld > N lets a caller pass a neuron-shard view
 *  (column range) of a wider tensor.  [N] vectors are dense fp32.
 *
 *  Ownership.  Every data pointer is a DEVICE pointer owned by the caller (PyTorch
 *  allocates).  The device calls never allocate, free or synchronise; every call only
 *  enqueues kernels on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *  stream) and returns.  Outputs are valid once that stream's work completes.  The one
 *  exception is the host-buffer runtime call snn_lif_fwd_bwd_host (host pointers, its own
 *  copy streams, blocking), documented where it is declared.
 *
 *  Errors.  Arguments are validated synchronously, before anything is enqueued; a
 *  non-OK status means nothing was launched.  A launch failure is reported as
 *  SNN_ERR_CUDA (from cudaGetLastError); faults inside a kernel surface at the
 *  caller's next synchronisation, as for any CUDA call.  snn_last_error_message()
 *  returns a thread-local detail string for the last non-OK status of this thread.
 *
 *  Alignment.  Element alignment is mandatory (SNN_ERR_MISALIGNED otherwise).  The
 *  128-bit vector fast path additionally needs 16-byte-aligned base pointers and
 *  ld % (16 / sizeof(io element)) == 0; otherwise a scalar path runs (never an error).
 *
 *  Determinism.  Identical inputs and build give bitwise-identical outputs, and chained
 *  segments (v_final -> v_init forward, grad_v_init -> grad_v_final backward) are
 *  bitwise equal to one whole-axis call.  SAVE_H and
 *  SAVE_RECOMPUTE produce bitwise-identical gradients.
 *
 *  Threading.  No global mutable state besides the thread-local error string; calls on
 *  different streams may run concurrently.
 */
#ifndef SNN_LIF_H
#define SNN_LIF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNN_LIF_ABI_VERSION 4

typedef enum {
    SNN_OK = 0,
    SNN_ERR_INVALID_VALUE = 1,  /* a size, flag or hyper-parameter is out of range      */
    SNN_ERR_NULL_POINTER = 2,   /* a required pointer is NULL                            */
    SNN_ERR_MISALIGNED = 3,     /* a pointer is not aligned to its element size          */
    SNN_ERR_UNSUPPORTED = 4,    /* a valid but unimplemented combination                 */
    SNN_ERR_CUDA = 5,           /* the CUDA runtime reported an error at launch          */
    SNN_ERR_NCCL = 6            /* NCCL reported an error (time split), or is unavailable */
} snn_status;

/* dtype of x, grad_spikes, grad_x (and of spikes when spike_fmt == SNN_SPK_IO).
 * Arithmetic is always fp32: bf16 values are widened exactly on load and
 * results rounded to nearest-even on store. */
typedef enum { SNN_F32 = 0, SNN_BF16 = 1 } snn_dtype;

/* Reset after a spike.  HARD: V = V_reset (Eq. 1's (1 - y) and V_rest*y terms,
 * PAPER.md:165).  SOFT: V = H - V_th (BASELINE.json north_star; not in the paper). */
typedef enum { SNN_RESET_HARD = 0, SNN_RESET_SOFT = 1 } snn_reset_mode;

/* Surrogate derivative delta(u), u = H - V_th.
 * SIGMOID: alpha e^{-alpha|u|} / (1 + e^{-alpha|u|})^2 (alpha = 4).
 * ATAN:    (alpha/2) / (1 + (pi/2 alpha u)^2) (SpikingJelly convention). */
typedef enum { SNN_SURR_SIGMOID = 0, SNN_SURR_ATAN = 1 } snn_surrogate;

/* Spike output format (values are exactly 0 or 1):
 *   U8   uint8  [T, ld]
 *   BITS uint32 [T, ceil(N/32)] (dense rows; bit j of word w is neuron 32w + j;
 *        bits of neurons >= N are 0)
 *   IO   io dtype [T, ld] (fp32 or bf16 1.0/0.0 -- the form a following conv consumes) */
typedef enum { SNN_SPK_U8 = 0, SNN_SPK_BITS = 1, SNN_SPK_IO = 2 } snn_spike_fmt;

/* What the forward keeps for the backward (the paper never shows it: Listing 1 stores
 * only args):
 *   SAVE_H          fp32 pre-reset potential H[t, n] for every step;
 *   SAVE_RECOMPUTE  fp32 post-reset V every SNN_LIF_CKPT_INTERVAL steps; the backward
 *                   re-runs the forward charge from those checkpoints and x, bitwise;
 *   SAVE_NONE       nothing (inference). */
typedef enum { SNN_SAVE_H = 0, SNN_SAVE_RECOMPUTE = 1, SNN_SAVE_NONE = 2 } snn_save_mode;

#define SNN_LIF_CKPT_INTERVAL 16

/* Hyper-parameters (the paper's Eq. 1 and the north star's charge are one
 * family).  With k = 1 - 1/tau and s = (decay_input ? 1/tau : 1):
 *     H[t] = k V[t-1] + V_reset/tau + s X[t]       (charge; Eq. 1 at V_reset = 0, s = 1)
 *     S[t] = (H[t] >= V_th)                         (fire, Eq. 2)
 *     V[t] = HARD ? (S ? V_reset : H) : H - V_th S  (reset)
 * Paper mode: tau = 1.25 (k_tau = 0.2), v_th = 0.3, v_reset = 0,
 * HARD, decay_input = 0, detach_reset = 0, SIGMOID, alpha = 4. */
typedef struct {
    float tau;          /* >= 1 (finite).  k = 1 - 1/tau computed in fp32       */
    float v_th;         /* > v_reset                                             */
    float v_reset;      /* reset value, and V[-1] when v_init is NULL          */
    int   reset_mode;   /* snn_reset_mode                                                     */
    int   decay_input;  /* 1: H = V + (X - (V - V_reset))/tau (north star); 0: paper Eq. 1    */
    int   detach_reset; /* 0: gradient flows through the reset (Eq. 3's -v delta term); 1: not */
    int   surrogate;    /* snn_surrogate                                                      */
    float alpha;        /* > 0 (finite)                                                       */
} snn_lif_params;

typedef struct {
    int64_t T;          /* >= 1 time steps                                                    */
    int64_t N;          /* >= 1 neurons                                                       */
    int64_t ld;         /* >= N; row stride (elements) of x, spikes (U8/IO), grad_spikes, grad_x */
    int     io_dtype;   /* snn_dtype                                                          */
    int     spike_fmt;  /* snn_spike_fmt                                                      */
    int     save_mode;  /* snn_save_mode                                                      */
} snn_lif_shape;

/* Bytes of the opaque `saved` buffer for (params, shape); 0 for SAVE_NONE or an invalid
 * shape.  The buffer must be 16-byte aligned; its layout is private and valid only for
 * the same (params, shape) pair and the same x / v_init. */
size_t snn_lif_saved_bytes(const snn_lif_params* params, const snn_lif_shape* shape);

/* Forward over all T steps in one launch (fusedForwardLIF; Eq. 1-2).
 *   x        [T, ld] io dtype             input currents x_i^(t)               (read)
 *   v_init   [N] fp32 or NULL -> v_reset   carry-in V[-1]          (read)
 *   spikes   per shape->spike_fmt          S[t, n] = y_i^(t)                     (write)
 *   saved    snn_lif_saved_bytes() bytes, NULL iff SAVE_NONE                    (write)
 *   v_final  [N] fp32 or NULL              carry-out V[T-1], post-reset          (write)
 * x must not alias any output. */
snn_status snn_lif_forward(const snn_lif_params* params, const snn_lif_shape* shape,
                           const void* x, const float* v_init, void* spikes, void* saved,
                           float* v_final, void* stream);

/* Backward (surrogate BPTT) over t = T-1..0 in one launch (fusedBackwardLIF,
 * PAPER.md:302; Eq. 3):
 *   gH[t] = gS[t] delta[t] + gV dV/dH[t];  grad_x[t] = s gH[t];  gV <- k gH[t]
 * with dV/dH = HARD: (1 - S) + (V_reset - H) delta;  SOFT: 1 - V_th delta
 * (the delta term dropped when detach_reset).
 *   grad_spikes  [T, ld] io dtype   dL/dS[t] from the next layer (the paper's grad y)  (read)
 *   x            [T, ld] io dtype   required iff SAVE_RECOMPUTE, else ignored (may be NULL)
 *   v_init       [N] fp32 or NULL   RECOMPUTE: the SAME pointer and contents given to the forward
 *                                   (NULL iff the forward's was NULL): V[-1] is not checkpointed,
 *                                   the backward re-reads it here (for T <= 16 the forward
 *                                   stores no checkpoint at all).  Ignored for SAVE_H.   (read)
 *   saved        the forward's saved buffer (same params/shape)                   (read)
 *   grad_v_final [N] fp32 or NULL -> 0   dL/dV[T-1] from a later time segment      (read)
 *   grad_x       [T, ld] io dtype   dL/dX[t]; must not alias any input            (write)
 *   grad_v_init  [N] fp32 or NULL   dL/dV[-1], the carry to an earlier segment     (write)
 * SAVE_NONE -> SNN_ERR_INVALID_VALUE. */
snn_status snn_lif_backward(const snn_lif_params* params, const snn_lif_shape* shape,
                            const void* grad_spikes, const void* x, const float* v_init,
                            const void* saved, const float* grad_v_final, void* grad_x,
                            float* grad_v_init, void* stream);

/* ---- Time-segment split with the boundary handoff fused into the kernels (SURVEY 8(f)
 * f1; rank d owns time steps [t_d, t_{d+1}) of every neuron, the boundary
 * membrane state goes forward in time and dL/dV backward).  Per neuron tile the kernel
 * waits for the previous rank's boundary state (ready flag, acquire at system scope),
 * computes the tile over the whole local segment, stores its carry-out straight into the
 * next rank's buffer through a peer-mapped pointer (CUDA IPC over NVLink) and releases
 * that tile's flag -- no separate collective, wavefront lag = one tile.
 * Flags are int32, one per SNN_LIF_HANDOFF_BLOCK neurons (snn_lif_handoff_blocks(N)
 * words), zero-initialised by the caller before the first call; `epoch` starts at 1 and
 * increases by one per call on every rank.  Credit-based flow control (ack flags) stops
 * a fast rank from overwriting a buffer the receiver has not read yet.
 * Forward: recv_* carry V (the previous segment's v_final), send_* the next segment's
 *          v_init.  Backward: recv_* carry dL/dV from the LATER segment, send_* go to the
 *          earlier one.  NULL recv_state = first segment (v_init / grad_v_final apply);
 *          NULL send_state = last segment.
 * SAVE_RECOMPUTE state written by snn_lif_forward_handoff holds V[-1] (it arrives inside the
 * kernel), so it pairs with snn_lif_backward_handoff only -- and snn_lif_forward's with
 * snn_lif_backward (which re-reads V[-1] from its v_init); likewise the affine pair below
 * (v_init: the forward's, as for snn_lif_backward).
 * Requires the TMA path (16-byte-aligned pointers, ld a multiple of 16 bytes, N a
 * multiple of 8 for bf16 / 4 for fp32), else SNN_ERR_UNSUPPORTED. */
#define SNN_LIF_HANDOFF_BLOCK 256

typedef struct {
    const float* recv_state;   /* [N] fp32, local: written by the sending rank            */
    const int32_t* recv_ready; /* [blocks], local: sender sets = epoch when written       */
    int32_t* recv_ack;         /* [blocks], peer: the sender's send_ack; we set = epoch    */
    float* send_state;         /* [N] fp32, peer: the receiving rank's recv_state          */
    int32_t* send_ready;       /* [blocks], peer: the receiving rank's recv_ready          */
    const int32_t* send_ack;   /* [blocks], local: the receiver's acknowledgements         */
    int32_t epoch;             /* >= 1, +1 per call                                        */
} snn_lif_handoff;

int64_t snn_lif_handoff_blocks(int64_t N);

snn_status snn_lif_forward_handoff(const snn_lif_params* params, const snn_lif_shape* shape,
                                   const void* x, const float* v_init, const snn_lif_handoff* handoff,
                                   void* spikes, void* saved, float* v_final, void* stream);
snn_status snn_lif_backward_handoff(const snn_lif_params* params, const snn_lif_shape* shape,
                                    const void* grad_spikes, const void* x, const void* saved,
                                    const float* grad_v_final, const snn_lif_handoff* handoff,
                                    void* grad_x, float* grad_v_init, void* stream);

/* ---- Time-segment split over NCCL (Eq. 4b
 * "each GPU handles a time segment, and the boundary membrane state (and, in
 * backward, the boundary dV gradient) is handed to the next rank", BASELINE north_star (3)).
 *
 * An snn_comm wraps an NCCL communicator whose rank order is time order: rank d owns local
 * time steps [t_d, t_{d+1}) of every neuron of a layer (x is the [T_d, ld] segment).
 *   snn_nccl_unique_id  writes the 128-byte ncclUniqueId (one rank calls it and ships the
 *                       bytes to the others, e.g. over torch.distributed).
 *   snn_comm_create     collective over the nranks processes (blocks until all joined); binds
 *                       the CUDA device current at the call; connects the neighbour ranks in
 *                       both directions up front.  *out = NULL on failure.
 *   snn_comm_destroy    synchronises the comm's stream and frees everything (NULL is a no-op).
 * NCCL is loaded at run time (the process's libnccl.so.2, else $SNN_NCCL_LIBRARY): without it
 * these calls return SNN_ERR_NCCL and every other entry point still works.  The comm owns
 * one CUDA stream, a few events and 16 bytes of device memory -- no layer buffers.
 *
 * snn_lif_forward_tsplit: the fused forward of this rank's segment, the neuron axis cut into
 * n_chunks chunks (boundaries on multiples of 512 neurons; n_chunks is clamped to
 * ceil(N/512)) processed in the same order on every rank, so the ranks form a wavefront
 * (efficiency n_chunks / (n_chunks + nranks - 1)).  Per chunk: receive its V [chunk] fp32
 * from rank-1 into v_in_ws, run the fused forward kernel from it, send the chunk's final V
 * (v_out_ws) to rank+1.  The kernels run on `stream`; the NCCL send / recv run on the comm's
 * stream, event-ordered against it and joined back before the call's work on `stream` ends
 * (capturable into a CUDA graph).  Every rank passes the same params, N, ld, io_dtype,
 * spike_fmt, save_mode and n_chunks; T may differ (the partition of the time axis).
 *   x, spikes, saved   as snn_lif_forward over the local segment (saved: snn_lif_saved_bytes
 *                      of this local shape)
 *   v_in_ws  [N] fp32  rank > 0: receive buffer (required); rank 0: the layer's v_init, or NULL
 *   v_out_ws [N] fp32  rank < nranks-1: send buffer (required); last rank: the layer's final V
 *                      (v_final), or NULL
 * snn_lif_backward_tsplit: the mirror image -- per chunk receive dL/dV from rank+1 into
 * g_in_ws, run the fused backward, send grad_v_init (g_out_ws) to rank-1.
 *   grad_spikes, x, saved, grad_x  as snn_lif_backward over the local segment
 *   v_in_ws  [N] fp32  the forward's v_in_ws, unchanged since (each chunk's V[-1]); NULL iff
 *                      the forward's was NULL (rank 0 without v_init)
 *   g_in_ws  [N] fp32  rank < nranks-1: receive buffer (required); last rank: the layer's
 *                      grad_v_final, or NULL (0)
 *   g_out_ws [N] fp32  rank > 0: send buffer (required); rank 0: the layer's grad_v_init, or NULL
 * The result is bitwise identical to one whole-axis snn_lif_forward / snn_lif_backward on one
 * GPU (the boundary state travels in fp32, exactly the register state).
 * With nranks = 1 both calls are the chunked single-GPU kernels.  Errors: as snn_lif_forward
 * / snn_lif_backward (validated for the whole segment before anything is enqueued), plus
 * SNN_ERR_INVALID_VALUE for n_chunks < 1 or > N, or a device other than the comm's;
 * SNN_ERR_NCCL if NCCL fails (work already enqueued for earlier chunks stays enqueued). */
#define SNN_NCCL_UNIQUE_ID_BYTES 128

typedef struct snn_comm snn_comm;

snn_status snn_nccl_unique_id(void* out /* SNN_NCCL_UNIQUE_ID_BYTES bytes */);
snn_status snn_comm_create(snn_comm** out, const void* unique_id, int nranks, int rank);
snn_status snn_comm_destroy(snn_comm* comm);
snn_status snn_comm_info(const snn_comm* comm, int* nranks, int* rank);
snn_status snn_lif_forward_tsplit(snn_comm* comm, const snn_lif_params* params, const snn_lif_shape* shape,
                                  int n_chunks, const void* x, void* spikes, void* saved,
                                  float* v_in_ws, float* v_out_ws, void* stream);
snn_status snn_lif_backward_tsplit(snn_comm* comm, const snn_lif_params* params, const snn_lif_shape* shape,
                                   int n_chunks, const void* grad_spikes, const void* x, const float* v_in_ws,
                                   const void* saved, void* grad_x, float* g_in_ws, float* g_out_ws,
                                   void* stream);

/* ---- The fused boundary handoff over NCCL symmetric windows (PAPER.md:252
 * "inter-GPU communication enables cross-device operator fusion and data exchange along the
 * temporal dimension").  The buffers and peer pointers that snn_lif_forward_handoff /
 * snn_lif_backward_handoff need, taken from an snn_comm instead of CUDA IPC: each rank
 * allocates one buffer with ncclMemAlloc holding the receive side of both directions (state
 * [N] fp32, ready and ack flags [snn_lif_handoff_blocks(N)] int32, per direction) and
 * registers it as a symmetric window (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC); the
 * neighbours' buffers are then ordinary load/store addresses of this process
 * (ncclGetPeerPointer over the communicator's LSA team -- NVLink / P2P peers of one node).
 *   snn_handoff_window_create  collective over the comm's ranks; N = neurons of the layer
 *                              (the same on every rank); zeroes the buffers and returns once
 *                              every rank has.  SNN_ERR_UNSUPPORTED when a time neighbour is
 *                              not a load/store peer (another node, or no P2P path) or the
 *                              process's NCCL has no window API; SNN_ERR_NCCL on NCCL errors.
 *   snn_handoff_window_next    fills *handoff for this rank's next call in `direction`
 *                              (0 forward: V from rank-1, to rank+1; 1 backward: dL/dV from
 *                              rank+1, to rank-1) with epoch = 1, 2, ... per direction; pass
 *                              it to the matching snn_lif_*_handoff call.  Every rank makes
 *                              the same sequence of calls.
 *   snn_handoff_window_pointer the base of this rank's buffer (which = 0) or of its previous
 *                              (-1) / next (+1) neighbour's as mapped here (NULL without one).
 *   snn_handoff_window_destroy synchronises the comm's stream, deregisters and frees
 *                              (collective; NULL is a no-op).  Destroy windows before their comm. */
typedef struct snn_handoff_window snn_handoff_window;

snn_status snn_handoff_window_create(snn_comm* comm, int64_t N, snn_handoff_window** out);
snn_status snn_handoff_window_next(snn_handoff_window* window, int direction, snn_lif_handoff* handoff);
snn_status snn_handoff_window_pointer(const snn_handoff_window* window, int which, void** ptr);
snn_status snn_handoff_window_destroy(snn_handoff_window* window);

/* ---- Producer fusion ("fold the preceding BN affine / residual add into
 * the LIF prologue"): a per-channel affine prologue folded into the LIF input -- the
 * layer's current is X' = scale[c] X + shift[c] (+ R) with c = (n / HW) % C, e.g. the
 * BatchNorm affine of a conv output [T, B, C, H, W] flattened to N = B C H W, plus
 * optionally a residual shortcut R (the spiking-ResNet block's LIF input BN(conv) + R) --
 * so neither the normalised tensor nor the sum is ever written to / re-read from HBM.
 * The backward returns dL/dX = scale[c] dL/dX', dL/dR = dL/dX' (when R is given) and the
 * per-channel sums the BN backward needs, grad_scale[c] = sum_{t,n in c} dL/dX'[t,n] X[t,n]
 * and grad_shift[c] = sum dL/dX'[t,n] (per-neuron partials in caller scratch, then a
 * deterministic fixed-order reduction).
 * Requirements: N % (C * HW) == 0; backward needs save_mode SAVE_RECOMPUTE.  With a
 * residual: forward save_mode SAVE_RECOMPUTE or SAVE_NONE, and the TMA path (16-byte-aligned
 * pointers, ld a multiple of 16 bytes, N a multiple of 8 for bf16 / 4 for fp32; the
 * backward: N a multiple of 2), else SNN_ERR_UNSUPPORTED.  The backward must get the same
 * residual the forward got (the RECOMPUTE backward re-derives X'). */
typedef struct {
    const float* scale;   /* [C] fp32 */
    const float* shift;   /* [C] fp32 */
    int64_t C;            /* channels (>= 1)                                          */
    int64_t HW;           /* neurons per channel per sample (>= 1)                    */
    const void* residual; /* [T, ld] io dtype shortcut R added to the input, or NULL  (read) */
    void* grad_residual;  /* backward only: [T, ld] io dtype dL/dR, required iff residual;
                             ignored by the forward                                  (write) */
} snn_lif_affine;

snn_status snn_lif_forward_affine(const snn_lif_params* params, const snn_lif_shape* shape,
                                  const void* x, const float* v_init, const snn_lif_affine* affine,
                                  void* spikes, void* saved, float* v_final, void* stream);
/* part_a, part_b: [N] fp32 caller scratch (16-B aligned; contents undefined on return);
 * grad_scale, grad_shift: [C] fp32 outputs, bitwise deterministic run to run. */
snn_status snn_lif_backward_affine(const snn_lif_params* params, const snn_lif_shape* shape,
                                   const void* grad_spikes, const void* x, const float* v_init, const void* saved,
                                   const float* grad_v_final, const snn_lif_affine* affine,
                                   void* grad_x, float* grad_v_init, float* part_a, float* part_b,
                                   float* grad_scale, float* grad_shift, void* stream);

/* ---- Baseline, not the method: the paper's "Serial (CUDA)" training of Fig. 3
 * (Fig. 5 caption PAPER.md:419) -- ONE time step per call, the membrane
 * state round-tripped through caller memory between steps, for the fused-vs-serial
 * comparison (bench.py --serial).  Same per-step arithmetic as the fused kernels, so T
 * chained calls are bitwise equal to one snn_lif_forward / snn_lif_backward (SAVE_H).
 *   x_t        [N] io dtype   input currents of step t                       (read)
 *   v          [N] fp32       in: V[t-1] (post-reset), out: V[t]              (read/write)
 *   spikes_t   [N] uint8      S[t]                                             (write)
 *   h_t        [N] fp32       H[t] (pre-reset; what the serial backward reads) (write)
 * Backward step (call for t = T-1 .. 0):
 *   grad_spikes_t [N] io dtype, h_t [N] fp32                                   (read)
 *   grad_v     [N] fp32       in: dL/dV[t], out: dL/dV[t-1]                    (read/write)
 *   grad_x_t   [N] io dtype   dL/dX[t]                                         (write)
 * Contiguous [N] vectors; errors as for snn_lif_forward. */
snn_status snn_lif_serial_forward_step(const snn_lif_params* params, int io_dtype, int64_t N,
                                       const void* x_t, float* v, uint8_t* spikes_t, float* h_t,
                                       void* stream);
snn_status snn_lif_serial_backward_step(const snn_lif_params* params, int io_dtype, int64_t N,
                                        const void* grad_spikes_t, const float* h_t, float* grad_v,
                                        void* grad_x_t, void* stream);

/* ---- Host-buffer training step (runtime, not a kernel): one layer's forward + backward
 * over HOST buffers, as a user without the tensors on the device calls it (bench.py's e2e).
 * The neuron axis is cut into chunks of `chunk_neurons` columns (neurons are independent,
 * PAPER.md:191-193); each chunk goes host -> device (x, grad_spikes), through
 * snn_lif_forward + snn_lif_backward, and device -> host (spikes, grad_x), with up to
 * `nslots` chunks in flight on three streams (copy-in, the caller's `stream` for the
 * kernels, copy-out), so both PCIe directions and the kernels overlap.
 *   x_host, grad_spikes_host  [T, ld] io dtype      host memory (pinned for full speed)  (read)
 *   spikes_host               per spike_fmt, row stride ld (u8/io) or ceil(N/32) words (write)
 *   grad_x_host               [T, ld] io dtype                                        (write)
 *   workspace                 device memory of snn_lif_host_workspace_bytes() bytes,
 *                             256-B aligned, caller-owned (the staging slots)
 * Carries: V[-1] = v_reset and dL/dV[T-1] = 0 (use the device calls for carries).
 * chunk_neurons <= 0 picks ~32 MiB of x per chunk; it is rounded up to a multiple of 512.
 * nslots in [2, 8] (<= 0: 3).  save_mode must be SAVE_H or SAVE_RECOMPUTE (saved state stays
 * in the slot).  The call BLOCKS until every output is in host memory; the copy streams and
 * events it needs are created and destroyed inside the call.  Errors: as snn_lif_forward,
 * plus SNN_ERR_INVALID_VALUE for a too-small workspace. */
size_t snn_lif_host_workspace_bytes(const snn_lif_params* params, const snn_lif_shape* shape,
                                    int64_t chunk_neurons, int nslots);
snn_status snn_lif_fwd_bwd_host(const snn_lif_params* params, const snn_lif_shape* shape,
                                const void* x_host, const void* grad_spikes_host, void* spikes_host,
                                void* grad_x_host, int64_t chunk_neurons, int nslots,
                                void* workspace, size_t workspace_bytes, void* stream);

/* ---- Plans (runtime, not new arithmetic): validate a layer's call once -- parameters,
 * shape, buffers, kernel variant, TMA tensor maps, launch geometry -- and replay it with
 * nothing but the launches.  For fixed-shape loops (serving, a training step whose
 * activations live in the same buffers every iteration) the per-call host work drops to
 * the launch itself.  Same kernels, same results, bit for bit, as snn_lif_forward /
 * snn_lif_backward with the same arguments.
 *   snn_lif_plan_create  binds the forward's buffers (as snn_lif_forward) and, when
 *                        grad_spikes / grad_x are non-NULL, the backward's (as
 *                        snn_lif_backward; both NULL = forward-only plan).  Errors as those
 *                        calls (nothing is launched); *plan = NULL on failure.
 *   snn_lif_plan_forward / _backward  enqueue the recorded launches on `stream`; the
 *                        buffers' CONTENTS may change between replays, their addresses
 *                        may not.  Must run with the device current at creation
 *                        (SNN_ERR_INVALID_VALUE otherwise).  _backward on a forward-only
 *                        plan: SNN_ERR_INVALID_VALUE.
 *   snn_lif_plan_destroy frees the host-side plan (no device memory is owned). */
typedef struct snn_lif_plan snn_lif_plan;

snn_status snn_lif_plan_create(snn_lif_plan** plan, const snn_lif_params* params,
                               const snn_lif_shape* shape, const void* x, const float* v_init,
                               void* spikes, void* saved, float* v_final, const void* grad_spikes,
                               const float* grad_v_final, void* grad_x, float* grad_v_init);
/* The same for the affine / residual prologue calls (snn_lif_forward_affine /
 * snn_lif_backward_affine's arguments; the backward's scratch and per-channel outputs are
 * bound too).  A forward-only affine plan is BN-folded inference. */
snn_status snn_lif_plan_create_affine(snn_lif_plan** plan, const snn_lif_params* params,
                                      const snn_lif_shape* shape, const void* x, const float* v_init,
                                      const snn_lif_affine* affine, void* spikes, void* saved,
                                      float* v_final, const void* grad_spikes, const float* grad_v_final,
                                      void* grad_x, float* grad_v_init, float* part_a, float* part_b,
                                      float* grad_scale, float* grad_shift);
snn_status snn_lif_plan_forward(const snn_lif_plan* plan, void* stream);
snn_status snn_lif_plan_backward(const snn_lif_plan* plan, void* stream);
void snn_lif_plan_destroy(snn_lif_plan* plan);

/* Status name, e.g. "SNN_ERR_INVALID_VALUE" (static storage). */
const char* snn_status_string(snn_status status);

/* Detail for the last non-OK status returned on the calling thread ("" if none). */
const char* snn_last_error_message(void);

/* SNN_LIF_ABI_VERSION of the built library. */
int snn_lif_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SNN_LIF_H */
