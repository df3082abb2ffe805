"""ctypes binding of include/snn_lif.h (argument marshalling only).

Loads the in-tree ``libsnn_lif.so``.  There is no fallback: if the library is missing or
fails to load, importing this module raises, naming the fix (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# SNN_LIF_LIBRARY: load another build of the same library (A/B timing of kernel changes,
# tools/kbench.py); it is still this package's CUDA library, never a fallback.
LIB_PATH = os.environ.get("SNN_LIF_LIBRARY") or os.path.join(_PKG, "libsnn_lif.so")

# enums (include/snn_lif.h)
SNN_OK = 0
STATUS_NAMES = {0: "SNN_OK", 1: "SNN_ERR_INVALID_VALUE", 2: "SNN_ERR_NULL_POINTER",
                3: "SNN_ERR_MISALIGNED", 4: "SNN_ERR_UNSUPPORTED", 5: "SNN_ERR_CUDA",
                6: "SNN_ERR_NCCL"}
SNN_F32, SNN_BF16 = 0, 1
SNN_RESET_HARD, SNN_RESET_SOFT = 0, 1
SNN_SURR_SIGMOID, SNN_SURR_ATAN = 0, 1
SNN_SPK_U8, SNN_SPK_BITS, SNN_SPK_IO = 0, 1, 2
SNN_SAVE_H, SNN_SAVE_RECOMPUTE, SNN_SAVE_NONE = 0, 1, 2
SNN_LIF_CKPT_INTERVAL = 16

# Every symbol include/snn_lif.h declares (checked by tests/test_abi.py).
EXPORTED_SYMBOLS = (
    "snn_lif_saved_bytes", "snn_lif_forward", "snn_lif_backward", "snn_status_string",
    "snn_last_error_message", "snn_lif_abi_version", "snn_lif_serial_forward_step",
    "snn_lif_serial_backward_step", "snn_lif_handoff_blocks", "snn_lif_forward_handoff",
    "snn_lif_backward_handoff", "snn_lif_forward_affine", "snn_lif_backward_affine",
    "snn_lif_host_workspace_bytes", "snn_lif_fwd_bwd_host", "snn_lif_plan_create", "snn_lif_plan_create_affine",
    "snn_lif_plan_forward", "snn_lif_plan_backward", "snn_lif_plan_destroy",
    "snn_nccl_unique_id", "snn_comm_create", "snn_comm_destroy", "snn_comm_info",
    "snn_lif_forward_tsplit", "snn_lif_backward_tsplit",
    "snn_handoff_window_create", "snn_handoff_window_next", "snn_handoff_window_pointer",
    "snn_handoff_window_destroy",
)
SNN_NCCL_UNIQUE_ID_BYTES = 128
SNN_LIF_HANDOFF_BLOCK = 256


class snn_lif_params(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_float), ("v_th", ctypes.c_float), ("v_reset", ctypes.c_float),
                ("reset_mode", ctypes.c_int), ("decay_input", ctypes.c_int),
                ("detach_reset", ctypes.c_int), ("surrogate", ctypes.c_int),
                ("alpha", ctypes.c_float)]


class snn_lif_shape(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int64), ("N", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("io_dtype", ctypes.c_int), ("spike_fmt", ctypes.c_int),
                ("save_mode", ctypes.c_int)]


class snn_lif_affine(ctypes.Structure):
    _fields_ = [("scale", ctypes.c_void_p), ("shift", ctypes.c_void_p), ("C", ctypes.c_int64),
                ("HW", ctypes.c_int64), ("residual", ctypes.c_void_p), ("grad_residual", ctypes.c_void_p)]


ABI_VERSION = 4   # include/snn_lif.h SNN_LIF_ABI_VERSION these structs mirror


class snn_lif_handoff(ctypes.Structure):
    _fields_ = [("recv_state", ctypes.c_void_p), ("recv_ready", ctypes.c_void_p),
                ("recv_ack", ctypes.c_void_p), ("send_state", ctypes.c_void_p),
                ("send_ready", ctypes.c_void_p), ("send_ack", ctypes.c_void_p),
                ("epoch", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build the CUDA library first "
                          "(python -c 'import __graft_entry__ as g; g.build()'); "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(snn_lif_params)
    S = ctypes.POINTER(snn_lif_shape)
    vp, fp = ctypes.c_void_p, ctypes.c_void_p
    lib.snn_lif_saved_bytes.argtypes = [P, S]
    lib.snn_lif_saved_bytes.restype = ctypes.c_size_t
    lib.snn_lif_forward.argtypes = [P, S, vp, fp, vp, vp, fp, vp]
    lib.snn_lif_forward.restype = ctypes.c_int
    lib.snn_lif_backward.argtypes = [P, S, vp, vp, fp, vp, fp, vp, fp, vp]
    lib.snn_lif_backward.restype = ctypes.c_int
    lib.snn_status_string.argtypes = [ctypes.c_int]
    lib.snn_status_string.restype = ctypes.c_char_p
    lib.snn_last_error_message.argtypes = []
    lib.snn_last_error_message.restype = ctypes.c_char_p
    lib.snn_lif_abi_version.argtypes = []
    lib.snn_lif_abi_version.restype = ctypes.c_int
    if lib.snn_lif_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI version {lib.snn_lif_abi_version()}, the binding "
                          f"expects {ABI_VERSION}: rebuild the library")
    i64 = ctypes.c_int64
    lib.snn_lif_serial_forward_step.argtypes = [P, ctypes.c_int, i64, vp, vp, vp, vp, vp]
    lib.snn_lif_serial_forward_step.restype = ctypes.c_int
    lib.snn_lif_serial_backward_step.argtypes = [P, ctypes.c_int, i64, vp, vp, vp, vp, vp]
    lib.snn_lif_serial_backward_step.restype = ctypes.c_int
    Hp = ctypes.POINTER(snn_lif_handoff)
    lib.snn_lif_handoff_blocks.argtypes = [i64]
    lib.snn_lif_handoff_blocks.restype = i64
    lib.snn_lif_forward_handoff.argtypes = [P, S, vp, fp, Hp, vp, vp, fp, vp]
    lib.snn_lif_forward_handoff.restype = ctypes.c_int
    lib.snn_lif_backward_handoff.argtypes = [P, S, vp, vp, vp, fp, Hp, vp, fp, vp]
    lib.snn_lif_backward_handoff.restype = ctypes.c_int
    Ap = ctypes.POINTER(snn_lif_affine)
    lib.snn_lif_forward_affine.argtypes = [P, S, vp, fp, Ap, vp, vp, fp, vp]
    lib.snn_lif_forward_affine.restype = ctypes.c_int
    lib.snn_lif_backward_affine.argtypes = [P, S, vp, vp, fp, vp, fp, Ap, vp, fp, fp, fp, fp, fp, vp]
    lib.snn_lif_backward_affine.restype = ctypes.c_int
    lib.snn_lif_host_workspace_bytes.argtypes = [P, S, ctypes.c_int64, ctypes.c_int]
    lib.snn_lif_host_workspace_bytes.restype = ctypes.c_size_t
    lib.snn_lif_fwd_bwd_host.argtypes = [P, S, vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int, vp,
                                         ctypes.c_size_t, vp]
    lib.snn_lif_fwd_bwd_host.restype = ctypes.c_int
    lib.snn_lif_plan_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), P, S, vp, fp, vp, vp, fp, vp, fp, vp, fp]
    lib.snn_lif_plan_create.restype = ctypes.c_int
    lib.snn_lif_plan_create_affine.argtypes = [ctypes.POINTER(ctypes.c_void_p), P, S, vp, fp, Ap, vp, vp, fp,
                                               vp, fp, vp, fp, fp, fp, fp, fp]
    lib.snn_lif_plan_create_affine.restype = ctypes.c_int
    lib.snn_lif_plan_forward.argtypes = [vp, vp]
    lib.snn_lif_plan_forward.restype = ctypes.c_int
    lib.snn_lif_plan_backward.argtypes = [vp, vp]
    lib.snn_lif_plan_backward.restype = ctypes.c_int
    lib.snn_lif_plan_destroy.argtypes = [vp]
    lib.snn_lif_plan_destroy.restype = None
    ci = ctypes.c_int
    lib.snn_nccl_unique_id.argtypes = [vp]
    lib.snn_nccl_unique_id.restype = ci
    lib.snn_comm_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), vp, ci, ci]
    lib.snn_comm_create.restype = ci
    lib.snn_comm_destroy.argtypes = [vp]
    lib.snn_comm_destroy.restype = ci
    lib.snn_comm_info.argtypes = [vp, ctypes.POINTER(ci), ctypes.POINTER(ci)]
    lib.snn_comm_info.restype = ci
    lib.snn_lif_forward_tsplit.argtypes = [vp, P, S, ci, vp, vp, vp, fp, fp, vp]
    lib.snn_lif_forward_tsplit.restype = ci
    lib.snn_lif_backward_tsplit.argtypes = [vp, P, S, ci, vp, vp, fp, vp, vp, fp, fp, vp]
    lib.snn_lif_backward_tsplit.restype = ci
    lib.snn_handoff_window_create.argtypes = [vp, i64, ctypes.POINTER(ctypes.c_void_p)]
    lib.snn_handoff_window_create.restype = ci
    lib.snn_handoff_window_next.argtypes = [vp, ci, Hp]
    lib.snn_handoff_window_next.restype = ci
    lib.snn_handoff_window_pointer.argtypes = [vp, ci, ctypes.POINTER(ctypes.c_void_p)]
    lib.snn_handoff_window_pointer.restype = ci
    lib.snn_handoff_window_destroy.argtypes = [vp]
    lib.snn_handoff_window_destroy.restype = ci
    return lib


lib = _load()


class SNNError(RuntimeError):
    def __init__(self, status: int):
        name = lib.snn_status_string(status).decode()
        detail = lib.snn_last_error_message().decode()
        super().__init__(f"{name}: {detail}")
        self.status = status


def check(status: int) -> None:
    if status != SNN_OK:
        raise SNNError(status)


def snn_lif_saved_bytes(params: snn_lif_params, shape: snn_lif_shape) -> int:
    return lib.snn_lif_saved_bytes(ctypes.byref(params), ctypes.byref(shape))


def snn_lif_forward(params, shape, x, v_init, spikes, saved, v_final, stream) -> None:
    """Raw entry point; pointer arguments are ints (device addresses) or None."""
    check(lib.snn_lif_forward(ctypes.byref(params), ctypes.byref(shape), x, v_init, spikes,
                              saved, v_final, stream))


def snn_lif_backward(params, shape, grad_spikes, x, v_init, saved, grad_v_final, grad_x,
                     grad_v_init, stream) -> None:
    check(lib.snn_lif_backward(ctypes.byref(params), ctypes.byref(shape), grad_spikes, x, v_init,
                               saved, grad_v_final, grad_x, grad_v_init, stream))


def snn_lif_serial_forward_step(params, io_dtype, N, x_t, v, spikes_t, h_t, stream) -> None:
    check(lib.snn_lif_serial_forward_step(ctypes.byref(params), io_dtype, N, x_t, v, spikes_t, h_t,
                                          stream))


def snn_lif_serial_backward_step(params, io_dtype, N, grad_spikes_t, h_t, grad_v, grad_x_t,
                                 stream) -> None:
    check(lib.snn_lif_serial_backward_step(ctypes.byref(params), io_dtype, N, grad_spikes_t, h_t,
                                           grad_v, grad_x_t, stream))


def snn_lif_forward_handoff(params, shape, x, v_init, handoff, spikes, saved, v_final, stream) -> None:
    check(lib.snn_lif_forward_handoff(ctypes.byref(params), ctypes.byref(shape), x, v_init,
                                      ctypes.byref(handoff), spikes, saved, v_final, stream))


def snn_lif_backward_handoff(params, shape, grad_spikes, x, saved, grad_v_final, handoff, grad_x,
                             grad_v_init, stream) -> None:
    check(lib.snn_lif_backward_handoff(ctypes.byref(params), ctypes.byref(shape), grad_spikes, x,
                                       saved, grad_v_final, ctypes.byref(handoff), grad_x,
                                       grad_v_init, stream))


def snn_lif_forward_affine(params, shape, x, v_init, affine, spikes, saved, v_final, stream) -> None:
    check(lib.snn_lif_forward_affine(ctypes.byref(params), ctypes.byref(shape), x, v_init,
                                     ctypes.byref(affine), spikes, saved, v_final, stream))


def snn_lif_backward_affine(params, shape, grad_spikes, x, v_init, saved, grad_v_final, affine, grad_x,
                            grad_v_init, part_a, part_b, grad_scale, grad_shift, stream) -> None:
    check(lib.snn_lif_backward_affine(ctypes.byref(params), ctypes.byref(shape), grad_spikes, x, v_init, saved,
                                      grad_v_final, ctypes.byref(affine), grad_x, grad_v_init, part_a,
                                      part_b, grad_scale, grad_shift, stream))


def snn_lif_host_workspace_bytes(params, shape, chunk_neurons, nslots) -> int:
    return int(lib.snn_lif_host_workspace_bytes(ctypes.byref(params), ctypes.byref(shape),
                                                chunk_neurons, nslots))


def snn_lif_fwd_bwd_host(params, shape, x_host, grad_spikes_host, spikes_host, grad_x_host,
                         chunk_neurons, nslots, workspace, workspace_bytes, stream) -> None:
    check(lib.snn_lif_fwd_bwd_host(ctypes.byref(params), ctypes.byref(shape), x_host, grad_spikes_host,
                                   spikes_host, grad_x_host, chunk_neurons, nslots, workspace,
                                   workspace_bytes, stream))


def snn_lif_plan_create(params, shape, x, v_init, spikes, saved, v_final, grad_spikes, grad_v_final,
                        grad_x, grad_v_init) -> int:
    """Returns the opaque plan handle (an int)."""
    h = ctypes.c_void_p()
    check(lib.snn_lif_plan_create(ctypes.byref(h), ctypes.byref(params), ctypes.byref(shape), x, v_init,
                                  spikes, saved, v_final, grad_spikes, grad_v_final, grad_x, grad_v_init))
    return h.value


def snn_lif_plan_forward(plan, stream) -> None:
    check(lib.snn_lif_plan_forward(plan, stream))


def snn_lif_plan_backward(plan, stream) -> None:
    check(lib.snn_lif_plan_backward(plan, stream))


def snn_lif_plan_destroy(plan) -> None:
    lib.snn_lif_plan_destroy(plan)


def snn_lif_plan_create_affine(params, shape, x, v_init, affine, spikes, saved, v_final, grad_spikes,
                               grad_v_final, grad_x, grad_v_init, part_a, part_b, grad_scale,
                               grad_shift) -> int:
    h = ctypes.c_void_p()
    check(lib.snn_lif_plan_create_affine(ctypes.byref(h), ctypes.byref(params), ctypes.byref(shape), x, v_init,
                                         ctypes.byref(affine), spikes, saved, v_final, grad_spikes, grad_v_final,
                                         grad_x, grad_v_init, part_a, part_b, grad_scale, grad_shift))
    return h.value


# ---- time split over NCCL (include/snn_lif.h snn_comm_* / snn_lif_*_tsplit)

def snn_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(SNN_NCCL_UNIQUE_ID_BYTES)
    check(lib.snn_nccl_unique_id(buf))
    return buf.raw


def snn_comm_create(unique_id: bytes, nranks: int, rank: int) -> int:
    if len(unique_id) != SNN_NCCL_UNIQUE_ID_BYTES:
        raise ValueError("unique_id must be 128 bytes")
    h = ctypes.c_void_p()
    check(lib.snn_comm_create(ctypes.byref(h), ctypes.create_string_buffer(unique_id, len(unique_id)), nranks, rank))
    return h.value


def snn_comm_destroy(comm) -> None:
    check(lib.snn_comm_destroy(comm))


def snn_lif_forward_tsplit(comm, params, shape, n_chunks, x, spikes, saved, v_in_ws, v_out_ws, stream) -> None:
    check(lib.snn_lif_forward_tsplit(comm, ctypes.byref(params), ctypes.byref(shape), n_chunks, x, spikes, saved,
                                     v_in_ws, v_out_ws, stream))


def snn_lif_backward_tsplit(comm, params, shape, n_chunks, grad_spikes, x, v_in_ws, saved, grad_x, g_in_ws,
                            g_out_ws, stream) -> None:
    check(lib.snn_lif_backward_tsplit(comm, ctypes.byref(params), ctypes.byref(shape), n_chunks, grad_spikes, x,
                                      v_in_ws, saved, grad_x, g_in_ws, g_out_ws, stream))


# ---- fused handoff over NCCL symmetric windows (include/snn_lif.h snn_handoff_window_*)

def snn_handoff_window_create(comm, N: int) -> int:
    h = ctypes.c_void_p()
    check(lib.snn_handoff_window_create(comm, N, ctypes.byref(h)))
    return h.value


def snn_handoff_window_next(window, direction: int) -> snn_lif_handoff:
    h = snn_lif_handoff()
    check(lib.snn_handoff_window_next(window, direction, ctypes.byref(h)))
    return h


def snn_handoff_window_pointer(window, which: int) -> int:
    p = ctypes.c_void_p()
    check(lib.snn_handoff_window_pointer(window, which, ctypes.byref(p)))
    return p.value or 0


def snn_handoff_window_destroy(window) -> None:
    check(lib.snn_handoff_window_destroy(window))
