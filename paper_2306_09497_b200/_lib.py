"""ctypes binding of libswe_b200.so (the C ABI in include/swe_b200.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libswe_b200.so")

SWE_OK, SWE_ESHAPE, SWE_ENOCONV, SWE_ENONFINITE, SWE_ECUDA, SWE_ENCCL = range(6)

# every symbol include/swe_b200.h declares
EXPORTS = (
    "swe_plan_create", "swe_plan_destroy", "swe_plan_info", "swe_plan_grid", "swe_plan_bytes",
    "swe_synthesis", "swe_analysis", "swe_uv_from_vortdiv", "swe_vortdiv_from_uv",
    "swe_tendency", "swe_imex_step", "swe_truncate_pad", "swe_state_stats",
    "swe_kernel_launches", "swe_last_error", "swe_profile", "swe_profile_read",
    "swe_set_option", "swe_ke_spectrum", "swe_window_maxdiff", "swe_grid_sqdiff",
    "swe_settls_step", "swe_departure_points", "swe_interpolate", "swe_imex_sweep",
    "swe_stepper_cfg_size", "swe_synthesis_pair", "swe_grad_grid", "swe_imex_step_async",
    "swe_imex_step_async_io", "swe_plan_status", "swe_imex_sweep_async",
)


class StepperCfgC(ctypes.Structure):
    """swe_stepper_cfg (mirror of StepperConfig, steppers.py:31-50)."""

    _fields_ = [("dt", ctypes.c_double), ("visc_order", ctypes.c_int),
                ("visc_nu", ctypes.c_double), ("coriolis_implicit", ctypes.c_int),
                ("include_nonlinear", ctypes.c_int), ("implicit_tol", ctypes.c_double),
                ("implicit_max_iter", ctypes.c_int), ("implicit_solver", ctypes.c_int),
                ("select_batch", ctypes.c_int)]


class NoConvergence(RuntimeError):
    pass


class NonFinite(RuntimeError):
    pass


_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and prototype the library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_2306_09497_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    proto = {
        "swe_plan_create": (I, [I, D, D, D, I, ctypes.POINTER(P)]),
        "swe_plan_destroy": (None, [P]),
        "swe_plan_info": (I, [P, ctypes.POINTER(I), ctypes.POINTER(I), ctypes.POINTER(I)]),
        "swe_plan_grid": (I, [P, P, P]),
        "swe_plan_bytes": (ctypes.c_longlong, [P]),
        "swe_synthesis": (I, [P, P, P, I, P]),
        "swe_analysis": (I, [P, P, P, I, P]),
        "swe_uv_from_vortdiv": (I, [P, P, P, P, P, I, P]),
        "swe_vortdiv_from_uv": (I, [P, P, P, P, P, I, P]),
        "swe_tendency": (I, [P, I, P, P, P, I, P]),
        "swe_imex_step": (I, [P, P, P, I, ctypes.POINTER(StepperCfgC), I, P, P, P]),
        "swe_truncate_pad": (I, [P, P, P, P, I, P]),
        "swe_state_stats": (I, [P, P, I, P, P, P]),
        "swe_kernel_launches": (ctypes.c_longlong, []),
        "swe_last_error": (ctypes.c_char_p, []),
        "swe_profile": (I, [I]),
        "swe_profile_read": (I, [P, P, P]),
        "swe_set_option": (I, [ctypes.c_char_p, I]),
        "swe_ke_spectrum": (I, [P, P, I, P, P]),
        "swe_window_maxdiff": (I, [P, P, P, P, I, P, P]),
        "swe_grid_sqdiff": (I, [P, P, ctypes.c_longlong, P, P]),
        "swe_settls_step": (I, [P, P, P, P, I, ctypes.POINTER(StepperCfgC), P, P]),
        "swe_departure_points": (I, [P, P, P, P, P, I, D, I, P, P, P]),
        "swe_interpolate": (I, [P, P, P, P, I, P, P]),
        "swe_imex_sweep": (I, [P, P, P, I, P, ctypes.POINTER(StepperCfgC), P, P]),
        "swe_stepper_cfg_size": (I, []),
        "swe_synthesis_pair": (I, [P, P, P, P, I, P]),
        "swe_grad_grid": (I, [P, P, P, P, I, P]),
        "swe_imex_step_async": (I, [P, P, P, I, ctypes.POINTER(StepperCfgC), I, P]),
        "swe_imex_step_async_io": (I, [P, P, ctypes.c_longlong, P, ctypes.c_longlong, P, I,
                                       ctypes.POINTER(StepperCfgC), I, P]),
        "swe_plan_status": (I, [P, ctypes.POINTER(I), I, P]),
        "swe_imex_sweep_async": (I, [P, P, P, I, P, ctypes.POINTER(StepperCfgC), P]),
    }
    for name, (res, args) in proto.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.swe_stepper_cfg_size() != ctypes.sizeof(StepperCfgC):
        raise RuntimeError(f"{path}: swe_stepper_cfg is {lib.swe_stepper_cfg_size()} bytes, "
                           f"the binding's is {ctypes.sizeof(StepperCfgC)} (stale library?)")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().swe_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = ""):
    """Map C return codes to the reference's exception types."""
    if rc == SWE_OK:
        return
    msg = last_error()
    if rc == SWE_ESHAPE:
        raise ValueError(msg or what)
    if rc == SWE_ENOCONV:
        raise NoConvergence(msg)
    if rc == SWE_ENONFINITE:
        raise NonFinite(msg)
    raise RuntimeError(f"{what}: {msg}")


def kernel_launches() -> int:
    return int(load().swe_kernel_launches())


def set_option(key: str, value: int):
    """Tuning switch (e.g. fft_path: 0 auto, 1 warp-per-row, 2 lane=row)."""
    check(load().swe_set_option(key.encode(), int(value)), "swe_set_option")


KERNEL_CLASSES =("legendre_synthesis", "legendre_analysis", "fft_grid", "spectral")


def profile(enable: bool):
    check(load().swe_profile(1 if enable else 0), "swe_profile")


def profile_read():
    """{class: (device ms, algorithmic work, launches)} since profile(True)."""
    import numpy as np
    ms = np.zeros(4)
    work = np.zeros(4)
    cnt = np.zeros(4, dtype=np.int64)
    check(load().swe_profile_read(ms.ctypes.data_as(ctypes.c_void_p),
                                  work.ctypes.data_as(ctypes.c_void_p),
                                  cnt.ctypes.data_as(ctypes.c_void_p)), "swe_profile_read")
    return {k: (float(ms[i]), float(work[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}
