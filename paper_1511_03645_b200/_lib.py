"""ctypes binding of libadjamr_b200.so (C ABI in include/adjamr_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every call raises ``NativeUnavailableError``.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADJAMR_LIB") or os.path.join(HERE, "libadjamr_b200.so")

# constants mirrored from the header
ADJ_OK, ADJ_ERR_CFL, ADJ_ERR_NONFINITE, ADJ_ERR_SCHEDULING = 0, 1, 2, 3
ADJ_ERR_OUT_OF_RANGE, ADJ_ERR_BAD_ARG, ADJ_ERR_CUDA = 4, 5, -1
SYS_AC1D, SYS_AC2D, SYS_SWE2D = 0, 1, 2
FORM_WAVE, FORM_FWAVE = 0, 1
LIMITERS = {"none": 0, "minmod": 1, "MC": 2, "superbee": 3}
VARIANT_EXACT, VARIANT_FAST = 0, 1
EDGE_XLO, EDGE_XHI, EDGE_YLO, EDGE_YHI = 1, 2, 4, 8
BC_WALL, BC_OUTFLOW, BC_PERIODIC = 0, 1, 2
BC_CODES = {"wall": BC_WALL, "outflow": BC_OUTFLOW, "periodic": BC_PERIODIC}
RECT_COPY, RECT_COARSE = 0, 1
STEP_KEEP_NONFINITE, STEP_NO_SPEED_OUT, STEP_TWO_ROWS, STEP_COUNTER_ZERO, STEP_PHYS_IN = 1, 2, 4, 8, 16
STEP_WET_DRY = 32
STEP_UNIFORM_MAT = 64


class NativeUnavailableError(RuntimeError):
    """The CUDA extension could not be loaded or no GPU is present."""


class NativeError(RuntimeError):
    """A native call failed with a CUDA or argument error."""


# numpy mirrors of the device tables (layout must match the header)
PATCH_DTYPE = np.dtype([("offset", "<i8"), ("flag_word", "<i8"), ("nx", "<i4"), ("ny", "<i4"),
                        ("pitch", "<i4"), ("lo_x", "<i4"), ("lo_y", "<i4"), ("edges", "<i4"),
                        ("pad0", "<i4"), ("pad1", "<i4")])
TILE_DTYPE = np.dtype([("patch", "<i4"), ("i0", "<i4"), ("j0", "<i4"), ("ni", "<i4"),
                       ("nj", "<i4"), ("pad", "<i4")])
RECT_DTYPE = np.dtype([("kind", "<i4"), ("dst_patch", "<i4"), ("src_patch", "<i4"), ("di0", "<i4"),
                       ("dj0", "<i4"), ("ni", "<i4"), ("nj", "<i4"), ("si0", "<i4"), ("sj0", "<i4"),
                       ("pad", "<i4")])
assert PATCH_DTYPE.itemsize == 48 and TILE_DTYPE.itemsize == 24 and RECT_DTYPE.itemsize == 40

P, D, I32, I64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64


class AdjGhostPlan(C.Structure):
    _fields_ = [("dst", P), ("src", P), ("meta", P), ("c_base", P), ("c_step", P), ("c_wx", P), ("c_wy", P),
                ("n", I32), ("nc", I32)]


class AdjGhostPlanBuildArgs(C.Structure):
    _fields_ = [("plan", AdjGhostPlan), ("rects", P), ("rect_cell0", P), ("patches", P), ("coarse_patches", P),
                ("axis_w", P), ("axis_i", P), ("edge_patches", P), ("owner", P), ("counter", P),
                ("nrect", I32), ("rect_cells", I32), ("nedge", I32), ("ndim", I32), ("m", I32),
                ("ghost", I32), ("ghost_coarse", I32), ("max_ghost_cells", I32),
                ("bc", I32 * 4), ("normal_comp", I32 * 2), ("stream", P)]


class AdjGhostPlanFillArgs(C.Structure):
    _fields_ = [("plan", AdjGhostPlan), ("q", P), ("q_coarse_old", P), ("q_coarse_new", P),
                ("comp_stride", I64), ("coarse_comp_stride", I64),
                ("ndim", I32), ("m", I32), ("time_mode", I32), ("pad", I32),
                ("w_time", D), ("w_time_dev", P), ("stream", P)]


class AdjStepRestrict(C.Structure):
    _fields_ = [("q_coarse", P), ("cell", P), ("base", P), ("coarse_comp_stride", I64), ("ratio", I32),
                ("pad", I32)]


class AdjJobFill(C.Structure):
    _fields_ = [("entry_off", P), ("dst", P), ("src", P), ("meta", P), ("c_base", P), ("c_step", P),
                ("c_wx", P), ("c_wy", P), ("cache", P), ("q_coarse_old", P), ("q_coarse_new", P),
                ("coarse_comp_stride", I64), ("n", I32), ("cache_mode", I32), ("time_mode", I32), ("pad", I32),
                ("w_time", D), ("w_time_dev", P)]


class AdjStepArgs(C.Structure):
    _fields_ = [("q_in", P), ("q_out", P), ("aux", P), ("patches", P), ("tiles", P),
                ("speed_max", P), ("nonfinite", P), ("work_counter", P), ("static_speed", P), ("job_offsets", P),
                ("njob", I32), ("pad2", I32), ("comp_stride", I64), ("aux_stride", I64),
                ("npatch", I32), ("ntile", I32), ("ndim", I32), ("ghost", I32),
                ("system", I32), ("form", I32), ("reversed", I32), ("limiter", I32),
                ("variant", I32), ("flags", I32),
                ("dt", D), ("dtdx", D), ("dtdy", D), ("gravity", D), ("stream", P), ("prefill", AdjGhostPlanFillArgs),
                ("fine_restrict", AdjStepRestrict), ("job_fill", AdjJobFill),
                ("phys_bc", I32 * 4), ("phys_normal", I32 * 2), ("job_class", P),
                ("uniform_c", D), ("uniform_z", D), ("job_uniform", P)]


class AdjPhysArgs(C.Structure):
    _fields_ = [("q", P), ("patches", P), ("comp_stride", I64), ("npatch", I32), ("ndim", I32),
                ("ghost", I32), ("m", I32), ("bc", I32 * 4), ("normal_comp", I32 * 2),
                ("max_ghost_cells", I32), ("pad", I32), ("stream", P)]


class AdjGhostArgs(C.Structure):
    _fields_ = [("q_dst", P), ("q_src", P), ("q_coarse_old", P), ("q_coarse_new", P),
                ("dst_patches", P), ("src_patches", P), ("coarse_patches", P), ("rects", P),
                ("dst_comp_stride", I64), ("src_comp_stride", I64), ("coarse_comp_stride", I64),
                ("nrect", I32), ("ndim", I32), ("m", I32), ("ghost_dst", I32), ("ghost_src", I32),
                ("ratio", I32), ("origin_x", D), ("origin_y", D), ("dx_f", D), ("dy_f", D),
                ("dx_c", D), ("dy_c", D), ("w_time", D), ("w_time_dev", P), ("axis_w", P), ("axis_i", P), ("time_mode", I32),
                ("max_rect_cells", I32), ("stream", P)]


class AdjRestrictArgs(C.Structure):
    _fields_ = [("q_coarse", P), ("q_fine", P), ("aux_coarse", P), ("aux_fine", P),
                ("coarse_patches", P), ("fine_patches", P), ("rects", P),
                ("coarse_comp_stride", I64), ("fine_comp_stride", I64),
                ("coarse_aux_stride", I64), ("fine_aux_stride", I64),
                ("nrect", I32), ("ndim", I32), ("m", I32), ("ratio", I32), ("swe", I32),
                ("max_rect_cells", I32), ("ghost_coarse", I32), ("ghost_fine", I32),
                ("cell_dst", P), ("cell_src", P), ("cell_meta", P), ("ncell", I32), ("pad", I32), ("stream", P)]


class AdjFlagArgs(C.Structure):
    _fields_ = [("q", P), ("aux", P), ("patches", P), ("ring", P), ("adj_wet", P),
                ("snap_index", P), ("interp_w", P), ("flag_bits", P), ("counts", P), ("best", P),
                ("best_offset", P), ("status", P), ("axis_w", P), ("axis_i", P), ("axis_dry", P),
                ("axis_off", P), ("comp_stride", I64), ("aux_stride", I64),
                ("npatch", I32), ("ndim", I32), ("m", I32), ("ghost", I32), ("swe", I32),
                ("mode", I32), ("nidx", I32), ("nxa", I32), ("nya", I32), ("max_cells", I32),
                ("layout", I32), ("max_rows", I32), ("max_cols", I32), ("variant", I32),
                ("origin_x", D), ("origin_y", D), ("dx", D), ("dy", D),
                ("a_origin_x", D), ("a_origin_y", D), ("a_dx", D), ("a_dy", D),
                ("tolerance", D), ("envelope", P), ("work", P), ("stream", P)]


ABI_VERSION = 8
FLAG_ROWS = 1        # AdjFlagArgs.layout: ADJ_FLAG_ROWS
FLAG_PAIRS = 2       # AdjFlagArgs.layout: ADJ_FLAG_PAIRS
FLAG_QUADS = 4       # AdjFlagArgs.layout: ADJ_FLAG_QUADS
FLAG_DIRECT = 8      # AdjFlagArgs.layout: ADJ_FLAG_DIRECT

class AdjFunctionalArgs(C.Structure):
    _fields_ = [("q", P), ("patches", P), ("ring", P), ("finer", P), ("covered", P), ("partial", P), ("status", P),
                ("comp_stride", I64), ("npatch", I32), ("nfiner", I32), ("ratio", I32), ("ndim", I32), ("m", I32),
                ("ghost", I32), ("nxa", I32), ("nya", I32), ("level_nx", I32), ("level_ny", I32),
                ("blocks_x", I32), ("snap", I32), ("w", D), ("origin_x", D), ("origin_y", D), ("dx", D), ("dy", D),
                ("a_origin_x", D), ("a_origin_y", D), ("a_dx", D), ("a_dy", D), ("stream", P)]


GAUGE_DTYPE = np.dtype([("base", np.int64), ("pitch", np.int32), ("i0", np.int32), ("i1", np.int32),
                        ("j0", np.int32), ("j1", np.int32), ("pad", np.int32), ("wx", np.float64),
                        ("wy", np.float64)], align=True)


class AdjGaugeArgs(C.Structure):
    _fields_ = [("q", P), ("gauges", P), ("out", P), ("comp_stride", I64), ("ngauge", I32), ("ndim", I32),
                ("m", I32), ("pad", I32), ("stream", P)]


class AdjFlagMaskArgs(C.Structure):
    _fields_ = [("flag_bits", P), ("patches", P), ("region_rows", P), ("region_cols", P),
                ("region_row_off", P), ("region_col_off", P), ("mask", P), ("occupancy", P), ("raw_count", P),
                ("npatch", I32), ("ndim", I32), ("level_nx", I32), ("level_ny", I32), ("buffer", I32),
                ("max_cells", I32), ("force_regions", C.c_uint32), ("clear_regions", C.c_uint32), ("stream", P)]


STRUCTS = [AdjGhostPlan, AdjGhostPlanBuildArgs, AdjGhostPlanFillArgs, AdjStepRestrict, AdjJobFill, AdjStepArgs,
           AdjPhysArgs, AdjGhostArgs, AdjRestrictArgs, AdjFlagArgs, AdjFunctionalArgs, AdjGaugeArgs, AdjFlagMaskArgs]

EXPORTS = {
    "adj_abi_version": ([], C.c_int),
    "adj_struct_size": ([C.c_char_p], C.c_int),
    "adj_copy2d_async": ([C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p],
                         C.c_int),
    "adj_last_error": ([], C.c_char_p),
    "adj_step_tile_shape": ([C.c_int, C.c_int, C.POINTER(I32), C.POINTER(I32)], C.c_int),
    "adj_step_level": ([C.POINTER(AdjStepArgs)], C.c_int),
    "adj_fill_physical": ([C.POINTER(AdjPhysArgs)], C.c_int),
    "adj_fill_ghost_rects": ([C.POINTER(AdjGhostArgs)], C.c_int),
    "adj_ghost_plan_build": ([C.POINTER(AdjGhostPlanBuildArgs)], C.c_int),
    "adj_fill_ghost_plan": ([C.POINTER(AdjGhostPlanFillArgs)], C.c_int),
    "adj_restrict": ([C.POINTER(AdjRestrictArgs)], C.c_int),
    "adj_flag_level_mask": ([C.POINTER(AdjFlagMaskArgs)], C.c_int),
    "adj_functional": ([C.POINTER(AdjFunctionalArgs)], C.c_int),
    "adj_gauges": ([C.POINTER(AdjGaugeArgs)], C.c_int),
    "adj_flag_adjoint": ([C.POINTER(AdjFlagArgs)], C.c_int),
    "adj_ghost_rects": ([C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                         C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.POINTER(I32), C.c_void_p],
                        C.c_int),
    "adj_box_overlaps": ([C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                          C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.POINTER(I32)], C.c_int),
    "adj_cluster": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                     C.c_int, C.POINTER(I32)], C.c_int),
}

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library (no GPU needed) and bind every exported symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailableError(
            f"{path} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (argtypes, restype) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    if lib.adj_abi_version() != ABI_VERSION:
        raise NativeUnavailableError("ABI version mismatch")
    for cls in STRUCTS:        # the ctypes layouts against the compiled ones
        if lib.adj_struct_size(cls.__name__.encode()) != C.sizeof(cls):
            raise NativeUnavailableError(f"{cls.__name__}: ctypes layout ({C.sizeof(cls)} bytes) differs from the "
                                         f"library's ({lib.adj_struct_size(cls.__name__.encode())})")
    _lib = lib
    return lib


_cuda_ok = None


def lib() -> C.CDLL:
    """The loaded library; raises when the CUDA path is unavailable."""
    global _cuda_ok
    if _cuda_ok is None:
        import torch
        _cuda_ok = bool(torch.cuda.is_available())
    if not _cuda_ok:
        raise NativeUnavailableError("no CUDA device: the adjamr B200 path has no CPU fallback")
    return load_library()


def check(rc: int, what: str):
    if rc == ADJ_OK:
        return
    msg = load_library().adj_last_error().decode(errors="replace")
    if rc == ADJ_ERR_BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed (status {rc}): {msg}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
