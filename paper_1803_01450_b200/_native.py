"""ctypes binding of the C-ABI library ``libmlamr_b200.so`` (include/mlamr_b200.h).

The product path has no fallback: if the CUDA library is missing or fails
to load, :func:`lib` raises and nothing runs on the CPU instead.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLAMR_LIB") or os.path.join(HERE, "_lib", "libmlamr_b200.so")

MAX_LAYERS = 4
ST_CFL = 1
ST_GEOMETRY = 2
ST_NONFINITE = 4
ST_BATHY = 8
BC_KIND = {"wall": 0, "outflow": 1}
SIDES = ("left", "right", "bottom", "top")

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dp = ctypes.POINTER(ctypes.c_double)
c_vp = ctypes.c_void_p


class Params(ctypes.Structure):
    """mlamr_params (include/mlamr_b200.h)."""
    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
        ("gravity", ctypes.c_double),
        ("dry_tolerance", ctypes.c_double),
        ("densities", ctypes.c_double * MAX_LAYERS),
    ]


class Level(ctypes.Structure):
    """mlamr_level (include/mlamr_b200.h)."""
    _fields_ = [
        ("num_patches", ctypes.c_int32),
        ("num_layers", ctypes.c_int32),
        ("level_nx", ctypes.c_int32),
        ("level_ny", ctypes.c_int32),
        ("dx", ctypes.c_double),
        ("dy", ctypes.c_double),
        ("field_stride", ctypes.c_int64),
        ("box", c_vp),
        ("offset", c_vp),
        ("state", c_vp),
        ("bathy", c_vp),
        ("own", c_vp),
        ("gown", c_vp),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "mlamr_version": (ctypes.c_int, []),
    "mlamr_build_info": (ctypes.c_char_p, []),
    "mlamr_paint_owner": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, c_vp]),
    "mlamr_step": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_int, Params, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mlamr_step_finalize": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_double,
                                           Params, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp]),
    "mlamr_tile_list": (ctypes.c_longlong, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp]),
    "mlamr_memset": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_longlong, c_vp]),
    "mlamr_sum_partials": (ctypes.c_int, [c_vp, ctypes.c_longlong, ctypes.c_int, ctypes.c_double, c_vp, c_vp,
                                          ctypes.c_int, c_vp]),
    "mlamr_max_speed_tiles": (ctypes.c_int, [Level, c_vp, c_vp, ctypes.c_int, ctypes.c_int, Params, c_vp, c_vp]),
    "mlamr_fill_ghosts": (ctypes.c_int, [Level, ctypes.POINTER(Level), c_vp, ctypes.c_double,
                                         ctypes.c_int, ctypes.c_int, c_i32p, Params, c_vp, c_vp,
                                         ctypes.c_int, c_vp]),
    "mlamr_ghost_plan": (ctypes.c_int, [Level, c_vp, c_vp, ctypes.c_int, c_vp]),
    "mlamr_fill_ghosts_planned": (ctypes.c_int, [Level, ctypes.POINTER(Level), c_vp, ctypes.c_double,
                                                 ctypes.c_int, ctypes.c_int, c_i32p, Params, c_vp, c_vp, c_vp,
                                                 c_vp, ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int, c_vp,
                                                 c_vp, ctypes.c_int, c_vp]),
    "mlamr_plan_interp_cells": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp,
                                               c_vp]),
    "mlamr_fill_bathymetry": (ctypes.c_int, [Level, c_vp, c_i32p, c_vp]),
    "mlamr_average_down": (ctypes.c_int, [Level, Level, ctypes.c_int, ctypes.c_int, Params, c_vp,
                                          ctypes.c_int, c_vp, c_vp]),
    "mlamr_regrid_fill": (ctypes.c_int, [Level, Level, Level, ctypes.c_int, ctypes.c_int, Params,
                                         c_vp, ctypes.c_int, c_vp, c_vp, ctypes.c_int, c_vp]),
    "mlamr_derefine_delta": (ctypes.c_int, [Level, Level, c_vp, ctypes.c_int, ctypes.c_int, Params,
                                            c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_vp]),
    "mlamr_interpolate_box": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             c_vp, ctypes.c_int, ctypes.c_int, Params,
                                             c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mlamr_level_reduce": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp,
                                          ctypes.c_int, c_vp]),
    "mlamr_pack_interiors": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                            c_vp]),
    "mlamr_level_reduce_planned": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, c_vp,
                                                  ctypes.c_int, c_vp, c_vp, c_vp]),
    "mlamr_flag_cells": (ctypes.c_int, [Level, c_vp, Params, c_vp, c_vp, c_vp, ctypes.c_int, c_vp,
                                        ctypes.c_int, c_vp]),
    "mlamr_copy_segments": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, c_vp, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, c_vp]),
    "mlamr_flags_reference": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             c_vp, c_vp, c_vp, c_vp]),
    "mlamr_cluster_sat": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, c_vp,
                                         ctypes.c_int]),
    "mlamr_chop_boxes": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        c_vp, ctypes.c_int]),
    "mlamr_step_tile": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_vp, c_vp]),
    "mlamr_set_step_form": (ctypes.c_int, [ctypes.c_int]),
    "mlamr_boxes_meet_any": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, ctypes.c_int, ctypes.c_int, c_vp]),
    "mlamr_selftest_div": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int, c_vp, c_vp, c_vp]),
    "mlamr_flags_bernoulli": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong,
                                             ctypes.c_ulonglong, ctypes.c_double, ctypes.c_int, c_vp, c_vp, c_vp,
                                             c_vp]),
    "mlamr_flags_gradient_raw": (ctypes.c_int, [Level, c_vp, Params, ctypes.c_uint, ctypes.c_double, c_vp, c_vp,
                                                c_vp, c_vp, c_vp]),
    "mlamr_flags_finish": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp,
                                          c_vp]),
    "mlamr_flags_gradient": (ctypes.c_int, [Level, c_vp, Params, ctypes.c_uint, ctypes.c_double, ctypes.c_int,
                                            c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mlamr_copy_pairs_of_plan": (ctypes.c_int, [Level, c_vp, c_vp, c_vp, ctypes.c_int, c_vp, ctypes.c_int, c_vp,
                                                c_vp]),
    "mlamr_fill_copy_pairs": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, ctypes.c_int, c_vp, c_vp]),
    "mlamr_check_bathymetry": (ctypes.c_int, [Level, Level, ctypes.c_int, ctypes.c_int, ctypes.c_double, c_vp,
                                              ctypes.c_int64, c_vp, c_vp, c_vp]),
    "mlamr_average_down_flat": (ctypes.c_int, [Level, Level, ctypes.c_int, ctypes.c_int, Params, c_vp,
                                               ctypes.c_int64, c_vp, c_vp]),
    "mlamr_pt_create": (ctypes.c_void_p, [Params, c_vp, c_vp]),
    "mlamr_pt_destroy": (None, [c_vp]),
    "mlamr_pt_set_level": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "mlamr_pt_set_level_bathymetry": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp]),
    "mlamr_pt_upload_patches": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mlamr_pt_download": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_vp, c_vp]),
    "mlamr_pt_num_patches": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "mlamr_pt_max_speed": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp]),
    "mlamr_pt_stash": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_double]),
    "mlamr_pt_clear_stash": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "mlamr_pt_fill_ghosts": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_double]),
    "mlamr_pt_step_level": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, c_vp, c_vp]),
    "mlamr_pt_average_down": (ctypes.c_int, [c_vp, ctypes.c_int]),
    "mlamr_pt_regrid": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp]),
    "mlamr_pt_composite_mass": (ctypes.c_int, [c_vp, c_vp]),
    "mlamr_pt_check_finite": (ctypes.c_int, [c_vp]),
    "mlamr_pt_status": (ctypes.c_int, [c_vp]),
    "mlamr_sat_u8": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp, c_vp]),
    "mlamr_pack_frame": (ctypes.c_int, [Level, c_vp, ctypes.c_int, c_vp, c_vp, ctypes.c_int, ctypes.c_int,
                                        c_vp, c_vp]),
    "mlamr_cluster_flags": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, c_vp,
                                           c_vp, ctypes.c_int]),
}

_lib = None


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or broken (no CPU fallback exists)."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from None
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def step_tile(max_patch_nx: int, num_layers: int) -> tuple:
    """(rows, columns) of the step tiles for a level whose widest patch
    interior is ``max_patch_nx`` cells (the library picks the shape)."""
    ty, tx = ctypes.c_int(), ctypes.c_int()
    lib().mlamr_step_tile(int(max_patch_nx), int(num_layers), ctypes.byref(ty), ctypes.byref(tx))
    return ty.value, tx.value


LAUNCHES = [0]


def check(rc: int, what: str) -> None:
    """Count the kernels a C-ABI compute entry point launches: one each,
    except mlamr_step, which writes its tile descriptors first
    (k_make_desc, csrc/k_step.cu)."""
    LAUNCHES[0] += 2 if what in ("mlamr_step", "step") else 1
    if rc != 0:
        raise NativeLibraryError(f"{what} failed to launch (cuda error {rc})")


def make_params(num_layers: int, densities, gravity: float, dry_tolerance: float) -> Params:
    p = Params()
    p.num_layers = num_layers
    p.gravity = gravity
    p.dry_tolerance = dry_tolerance
    for m in range(MAX_LAYERS):
        p.densities[m] = densities[m] if m < len(densities) else 0.0
    return p


def bc_array(boundaries: dict):
    arr = (ctypes.c_int32 * 4)(*[BC_KIND[boundaries[s]] for s in SIDES])
    return arr
