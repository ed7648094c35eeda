"""ctypes mirror of include/frir.h and the loader of the in-tree libfrir.so.

The library is the product: there is no CPU fallback.  If the shared object
is missing, every entry point raises :class:`FrirLibraryError` (run
``python -c "import __graft_entry__ as g; g.build()"`` to build it).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libfrir.so"

FRIR_OK, FRIR_EINVAL, FRIR_ECUDA, FRIR_ERANGE, FRIR_ENOMEM = 0, -1, -2, -3, -4
STAGE_GEOM, STAGE_DELAY, STAGE_RENDER, STAGE_ALL = 1, 2, 4, 7
TAB_H1, TAB_H2, TAB_SOS, TAB_COMP_D, TAB_COMP_W = 0, 1, 2, 3, 4
TAB_KAPPA, TAB_U, TAB_ZPHASE, TAB_PPOW, TAB_LPCOEF, TAB_GW = 5, 6, 7, 8, 9, 10

c_int32, c_int64, c_uint64, c_double = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
c_void_p = ctypes.c_void_p


class FrirLibraryError(RuntimeError):
    """libfrir.so is missing or failed; the CUDA path has no fallback."""


class FrirPlanDesc(ctypes.Structure):
    _fields_ = [
        ("sample_rate", c_int32), ("r_h", c_int32), ("r_l", c_int32), ("up", c_int32),
        ("down", c_int32), ("half1", c_int32), ("len1", c_int32), ("half2", c_int32),
        ("len2", c_int32), ("t0", c_int32), ("sup", c_int32), ("nb", c_int32),
        ("horizon", c_int32), ("lt_max", c_int32), ("pad_", c_int32),
        ("sos", c_double * 6), ("c1", c_double), ("c2", c_double),
    ]


class FrirJob(ctypes.Structure):
    _fields_ = [
        ("room", c_double * 3), ("center", c_double * 3), ("d0", c_double), ("az", c_double),
        ("el", c_double), ("t60", c_double), ("c0", c_double), ("alpha", c_double),
        ("beta", c_double), ("perturb_lo", c_double), ("perturb_hi", c_double), ("tau", c_double),
        ("seed", c_uint64), ("source_index", c_int32), ("n_images", c_int32),
        ("mic_off", c_int32), ("n_mics", c_int32),
        ("n_images_hi", c_int32), ("normalize", c_int32), ("kind", c_int32), ("lattice", c_int32),
        ("early_lo_ms", c_double), ("early_hi_ms", c_double), ("duration", c_double),
        ("reflection", c_double),
        ("img_off", c_int64), ("item_off", c_int64), ("out_off", c_int64),
        ("chan_off", c_int32), ("out_stride", c_int32), ("L", c_int32), ("n1", c_int32),
        ("n2", c_int32), ("pad_", c_int32),
        ("r", c_double), ("rr_max", c_double), ("alpha3", c_double), ("b3a3", c_double),
        ("log2r", c_double), ("e_lo", c_int32), ("e_hi", c_int32),
        ("key", c_uint64 * 4),
    ]


class FrirBatch(ctypes.Structure):
    _fields_ = [
        ("jobs", c_void_p), ("n_jobs", c_int32), ("total_channels", c_int32),
        ("chan_job", c_void_p), ("chan_order", c_void_p), ("mics", c_void_p),
        ("draw_dist", c_void_p), ("draw_az", c_void_p), ("draw_el", c_void_p),
        ("draw_refl", c_void_p),
        ("total_images", c_int64), ("total_items", c_int64), ("total_out", c_int64),
        ("max_rows", c_int32), ("max_windows", c_int32),
    ]


class FrirSceneSpec(ctypes.Structure):
    _fields_ = [
        ("room_length", c_double * 2), ("room_width", c_double * 2), ("room_height", c_double * 2),
        ("t60", c_double * 2), ("distance", c_double * 2), ("elevation", c_double * 2),
        ("center", c_double * 3), ("aperture", c_double), ("c0", c_double), ("alpha3", c_double),
        ("b3a3", c_double), ("n_sources", c_int32), ("n_mics", c_int32), ("num_images", c_int32),
        ("out_stride", c_int32),
    ]


JOB_DTYPE = np.dtype(FrirJob)

# (name, restype, argtypes) of every symbol include/frir.h declares.
MIX_POWER_CHUNKS = 32  # FRIR_MIX_POWER_CHUNKS
ABI_VERSION = 3  # FRIR_ABI_VERSION
KIND_FRAM, KIND_ISM, KIND_TRAIN = 0, 1, 2  # FRIR_KIND_*
STAGE_RATIO_SAMPLE, STAGE_RESCALE, STAGE_REFLECTIONS = 0, 1, 2  # frir_stage_eval ops

SIGNATURES = [
    ("frir_plan_create", c_int32, [c_int32, ctypes.POINTER(c_void_p)]),
    ("frir_plan_describe", c_int32, [c_void_p, ctypes.POINTER(FrirPlanDesc)]),
    ("frir_plan_destroy", c_int32, [c_void_p]),
    ("frir_design_describe", c_int32, [c_int32, ctypes.POINTER(FrirPlanDesc)]),
    ("frir_design_table", c_int32, [c_int32, c_int32, c_void_p, c_int64, ctypes.POINTER(c_int64)]),
    ("frir_philox_doubles", c_int32, [c_uint64, c_uint64, c_uint64, c_uint64, c_int64, c_void_p]),
    ("frir_jobs_prepare", c_int32,
     [c_int32, c_void_p, c_int32, c_int32, ctypes.POINTER(FrirBatch), c_void_p, c_void_p]),
    ("frir_workspace_size", ctypes.c_size_t, [c_void_p, ctypes.POINTER(FrirBatch)]),
    ("frir_simulate", c_int32,
     [c_void_p, ctypes.POINTER(FrirBatch), c_void_p, ctypes.c_size_t, c_void_p, c_void_p,
      c_void_p, c_void_p]),
    ("frir_simulate_stages", c_int32,
     [c_void_p, ctypes.POINTER(FrirBatch), c_void_p, ctypes.c_size_t, c_void_p, c_void_p,
      c_void_p, c_void_p, c_int32]),
    ("frir_launch_count", c_int32, [c_void_p, ctypes.POINTER(FrirBatch), c_int32]),
    ("frir_mix_convolve_scratch", c_int64, [c_int32, c_int32, c_int32, c_int64, c_int64, ctypes.POINTER(c_int64)]),
    ("frir_mix_convolve", c_int32,
     [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
      c_void_p, c_int64, c_void_p, c_int32, c_int32, c_int32, c_int64, c_int64, c_void_p, c_int64, c_void_p,
      c_int64, c_void_p]),
    ("frir_mix_powers", c_int32,
     [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    ("frir_mix_gains", c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    ("frir_mix_combine", c_int32,
     [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_int64, c_int64, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p]),
    ("frir_sample_scene_jobs", c_int32,
     [c_void_p, ctypes.POINTER(FrirSceneSpec), c_uint64, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
      c_void_p]),
    ("frir_edc", c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p]),
    ("frir_t60", c_int32,
     [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_double, c_double, c_double,
      c_double, c_void_p, c_void_p]),
    ("frir_edc_f64", c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_void_p]),
    ("frir_t60_f64", c_int32,
     [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int64, c_void_p, c_double, c_double, c_double,
      c_double, c_void_p, c_void_p]),
    ("frir_stage_eval", c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    ("frir_philox_uniform", c_int32,
     [c_uint64, c_uint64, c_uint64, c_int64, c_int64, c_double, c_double, c_void_p, c_void_p]),
    ("frir_image_set", c_int32,
     [c_void_p, ctypes.POINTER(FrirBatch), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
      c_void_p]),
    ("frir_impulse_train_scratch", c_int64, [c_int32, c_int32, c_int32]),
    ("frir_impulse_train", c_int32,
     [c_void_p, c_void_p, c_int32, c_int32, c_double, c_double, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
      c_int64, c_void_p]),
    ("frir_early_window", c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    ("frir_train_nonzeros", c_int32, [c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    ("frir_simulate_train", c_int32,
     [c_void_p, ctypes.POINTER(FrirBatch), c_void_p, ctypes.c_size_t, c_void_p, c_int64, c_int32, c_void_p, c_void_p,
      c_void_p]),
    ("frir_last_error", ctypes.c_char_p, []),
    ("frir_abi_version", c_int32, []),
    ("frir_struct_size", c_int64, [c_int32]),
    ("frir_debug_status", c_int32, []),
]

_lib = None


def lib():
    """Load libfrir.so once; raise FrirLibraryError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("FRIR_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise FrirLibraryError(
            f"{path} not found: the CUDA extension is not built (no CPU fallback exists); "
            "run __graft_entry__.build()"
        )
    try:
        handle = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise FrirLibraryError(f"cannot load {path}: {exc}") from exc
    for name, restype, argtypes in SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if handle.frir_abi_version() != ABI_VERSION:
        raise FrirLibraryError("libfrir ABI version mismatch")
    for which, ty in ((0, FrirJob), (1, FrirBatch), (2, FrirPlanDesc)):
        if handle.frir_struct_size(which) != ctypes.sizeof(ty):
            raise FrirLibraryError(f"struct layout mismatch for {ty.__name__}")
    _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().frir_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str) -> None:
    """Map a status code to the reference's exception types."""
    if status == FRIR_OK:
        return
    msg = last_error()
    if status == FRIR_EINVAL:
        raise ValueError(msg)
    raise FrirLibraryError(f"{what} failed ({status}): {msg}")


def design_describe(sample_rate: int) -> FrirPlanDesc:
    d = FrirPlanDesc()
    check(lib().frir_design_describe(int(sample_rate), ctypes.byref(d)), "frir_design_describe")
    return d


def design_table(sample_rate: int, which: int) -> np.ndarray:
    n = c_int64(0)
    check(lib().frir_design_table(int(sample_rate), which, None, 0, ctypes.byref(n)), "frir_design_table")
    out = np.empty(n.value, dtype=np.float64)
    check(lib().frir_design_table(int(sample_rate), which, out.ctypes.data, n.value, ctypes.byref(n)),
          "frir_design_table")
    return out


def philox_doubles(seed: int, source_index: int, stage: int, first: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    check(lib().frir_philox_doubles(seed, source_index, stage, first, n, out.ctypes.data),
          "frir_philox_doubles")
    return out
