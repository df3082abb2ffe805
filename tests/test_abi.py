"""The C-ABI library loads and exports every symbol include/snn_lif.h declares; host-side
validation (which runs before any launch) rejects bad arguments.  No GPU needed: every
call here returns an error status before touching the device."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "snn_lif.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(snn_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__._build_module().build()
    from paper_2408_00280_b200 import _lib
    return _lib


def test_every_declared_symbol_is_exported(lib):
    decl = declared_functions()
    assert decl, "no declarations parsed"
    for name in decl:
        assert hasattr(lib.lib, name), f"{name} declared in snn_lif.h but not exported"
    assert sorted(lib.EXPORTED_SYMBOLS) == decl


def test_abi_version_and_status_strings(lib):
    assert lib.lib.snn_lif_abi_version() == lib.ABI_VERSION == 4
    assert lib.lib.snn_status_string(0) == b"SNN_OK"
    assert lib.lib.snn_status_string(3) == b"SNN_ERR_MISALIGNED"


def _p(lib, **kw):
    d = dict(tau=1.25, v_th=0.3, v_reset=0.0, reset_mode=0, decay_input=0, detach_reset=0,
             surrogate=0, alpha=4.0)
    d.update(kw)
    return lib.snn_lif_params(**d)


def _s(lib, **kw):
    d = dict(T=8, N=1024, ld=1024, io_dtype=0, spike_fmt=0, save_mode=1)
    d.update(kw)
    return lib.snn_lif_shape(**d)


def test_saved_bytes(lib):
    # RECOMPUTE: ceil(T/16) rows of round_up(N, 16) floats; SAVE_H: T rows; NONE: 0
    assert lib.snn_lif_saved_bytes(_p(lib), _s(lib, T=40, N=1000, ld=1000)) == 3 * 1008 * 4
    assert lib.snn_lif_saved_bytes(_p(lib), _s(lib, T=40, N=1000, ld=1000, save_mode=0)) == 40 * 1008 * 4
    assert lib.snn_lif_saved_bytes(_p(lib), _s(lib, save_mode=2)) == 0
    assert lib.snn_lif_saved_bytes(_p(lib, tau=0.5), _s(lib)) == 0


@pytest.mark.parametrize("pkw,skw,code", [
    (dict(tau=0.9), {}, 1), (dict(tau=float("nan")), {}, 1), (dict(v_th=0.0), {}, 1),
    (dict(alpha=0.0), {}, 1), (dict(reset_mode=2), {}, 1), (dict(surrogate=7), {}, 1),
    (dict(decay_input=2), {}, 1),
    ({}, dict(T=0), 1), ({}, dict(N=0), 1), ({}, dict(ld=10), 1), ({}, dict(io_dtype=5), 1),
    ({}, dict(spike_fmt=3), 1), ({}, dict(save_mode=9), 1),
    ({}, dict(T=1 << 40, N=1 << 30, ld=1 << 30), 1),
])
def test_forward_validation(lib, pkw, skw, code):
    st = lib.lib.snn_lif_forward(ctypes.byref(_p(lib, **pkw)), ctypes.byref(_s(lib, **skw)),
                                 16, None, 16, 16, None, None)
    assert st == code
    assert lib.lib.snn_last_error_message()


def test_null_and_misaligned_pointers(lib):
    P, S = ctypes.byref(_p(lib)), ctypes.byref(_s(lib))
    assert lib.lib.snn_lif_forward(P, S, None, None, 16, 16, None, None) == 2
    assert lib.lib.snn_lif_forward(P, S, 16, None, None, 16, None, None) == 2
    assert lib.lib.snn_lif_forward(P, S, 16, None, 16, None, None, None) == 2   # saved needed
    assert lib.lib.snn_lif_forward(P, S, 18, None, 16, 16, None, None) == 3     # x not 4-aligned
    assert lib.lib.snn_lif_forward(P, S, 16, None, 16, 24, None, None) == 3     # saved not 16-aligned
    # backward
    assert lib.lib.snn_lif_backward(P, S, None, 16, None, 16, None, 16, None, None) == 2
    assert lib.lib.snn_lif_backward(P, S, 16, None, None, 16, None, 16, None, None) == 2  # x for RECOMPUTE
    Sn = ctypes.byref(_s(lib, save_mode=2))
    assert lib.lib.snn_lif_backward(P, Sn, 16, 16, None, 16, None, 16, None, None) == 1


def test_python_errors_are_loud(lib):
    err = lib.SNNError(1)
    assert "SNN_ERR_INVALID_VALUE" in str(err)


def test_plan_validation_before_any_device_work(lib):
    """snn_lif_plan_create validates like snn_lif_forward / _backward and returns before any
    launch; replaying a NULL plan is an error, not a crash."""
    P, S = ctypes.byref(_p(lib)), ctypes.byref(_s(lib))
    h = ctypes.c_void_p()
    assert lib.lib.snn_lif_plan_create(None, P, S, 16, None, 16, 16, None, None, None, None, None) == 2
    assert lib.lib.snn_lif_plan_create(ctypes.byref(h), ctypes.byref(_p(lib, tau=0.5)), S, 16, None, 16, 16,
                                       None, None, None, None, None) == 1
    assert h.value is None
    # grad_spikes without grad_x (and vice versa)
    assert lib.lib.snn_lif_plan_create(ctypes.byref(h), P, S, 16, None, 16, 16, None, 16, None, None, None) == 2
    assert lib.lib.snn_lif_plan_create(ctypes.byref(h), P, S, 16, None, 16, 16, None, None, None, 16, None) == 2
    assert lib.lib.snn_lif_plan_create(ctypes.byref(h), P, S, None, None, 16, 16, None, None, None, None, None) == 2
    assert lib.lib.snn_lif_plan_forward(None, None) == 2
    assert lib.lib.snn_lif_plan_backward(None, None) == 2
    lib.lib.snn_lif_plan_destroy(None)


def test_comm_and_tsplit_validation(lib):
    """The NCCL time-split entry points validate before touching NCCL or the device."""
    P, S = ctypes.byref(_p(lib)), ctypes.byref(_s(lib))
    h = ctypes.c_void_p()
    uid = ctypes.create_string_buffer(128)
    assert lib.lib.snn_nccl_unique_id(None) == 2
    assert lib.lib.snn_comm_create(None, uid, 1, 0) == 2
    assert lib.lib.snn_comm_create(ctypes.byref(h), None, 1, 0) == 2
    assert lib.lib.snn_comm_create(ctypes.byref(h), uid, 0, 0) == 1
    assert lib.lib.snn_comm_create(ctypes.byref(h), uid, 2, 2) == 1
    assert lib.lib.snn_comm_create(ctypes.byref(h), uid, 2, -1) == 1
    assert h.value is None
    assert lib.lib.snn_comm_destroy(None) == 0
    assert lib.lib.snn_comm_info(None, None, None) == 2
    assert lib.lib.snn_lif_forward_tsplit(None, P, S, 1, 16, 16, 16, None, None, None) == 2
    assert lib.lib.snn_lif_backward_tsplit(None, P, S, 1, 16, 16, None, 16, 16, None, None, None) == 2
    assert b"comm is NULL" in lib.lib.snn_last_error_message()


def test_handoff_window_validation(lib):
    """The NCCL-window handoff entry points validate their handles before any NCCL or device work."""
    h = ctypes.c_void_p()
    assert lib.lib.snn_handoff_window_create(None, 1024, ctypes.byref(h)) == 2
    assert lib.lib.snn_handoff_window_create(None, 1024, None) == 2
    assert h.value is None
    ho = lib.snn_lif_handoff()
    assert lib.lib.snn_handoff_window_next(None, 0, ctypes.byref(ho)) == 2
    assert lib.lib.snn_handoff_window_pointer(None, 0, ctypes.byref(h)) == 2
    assert lib.lib.snn_handoff_window_destroy(None) == 0


def test_nccl_unique_id_from_the_process_nccl(lib):
    """snn_nccl_unique_id resolves NCCL at run time (no GPU needed) and returns 128 bytes."""
    uid = lib.snn_nccl_unique_id()
    assert len(uid) == 128 and any(uid)


def test_affine_validation(lib):
    """snn_lif_forward_affine / snn_lif_backward_affine (ABI 4: the backward takes the forward's
    v_init) validate before any launch."""
    P, S = ctypes.byref(_p(lib)), ctypes.byref(_s(lib))
    ok = lib.snn_lif_affine(scale=16, shift=16, C=4, HW=256, residual=None, grad_residual=None)
    bad_div = lib.snn_lif_affine(scale=16, shift=16, C=3, HW=256, residual=None, grad_residual=None)
    no_scale = lib.snn_lif_affine(scale=None, shift=16, C=4, HW=256, residual=None, grad_residual=None)
    f = lib.lib.snn_lif_forward_affine
    assert f(P, S, 16, None, None, 16, 16, None, None) == 2                      # affine NULL
    assert f(P, S, 16, None, ctypes.byref(bad_div), 16, 16, None, None) == 1     # N % (C HW) != 0
    assert f(P, S, 16, None, ctypes.byref(no_scale), 16, 16, None, None) == 1
    assert f(P, S, 16, 18, ctypes.byref(ok), 16, 16, None, None) == 3            # v_init misaligned
    b = lib.lib.snn_lif_backward_affine
    #       P  S  gS  x   v_init saved gvf  af            gx  gvi  pa  pb  gsc gsh  stream
    assert b(P, S, 16, 16, None, 16, None, None, 16, None, 16, 16, 16, 16, None) == 2          # affine NULL
    assert b(P, S, 16, 16, None, 16, None, ctypes.byref(ok), 16, None, 16, 16, None, 16, None) == 2  # grad_scale
    assert b(P, S, 16, 16, None, 16, None, ctypes.byref(ok), 16, None, None, 16, 16, 16, None) == 2  # part_a
    assert b(P, S, 16, 16, 18, 16, None, ctypes.byref(ok), 16, None, 16, 16, 16, 16, None) == 3     # v_init
    assert b(P, S, 16, 16, None, 16, None, ctypes.byref(bad_div), 16, None, 16, 16, 16, 16, None) == 1
    Sh = ctypes.byref(_s(lib, save_mode=0))
    assert b(P, Sh, 16, 16, None, 16, None, ctypes.byref(ok), 16, None, 16, 16, 16, 16, None) == 4  # SAVE_H


def test_backward_v_init_alignment(lib):
    P, S = ctypes.byref(_p(lib)), ctypes.byref(_s(lib))
    assert lib.lib.snn_lif_backward(P, S, 16, 16, 18, 16, None, 16, None, None) == 3
