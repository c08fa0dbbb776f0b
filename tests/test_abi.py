"""The C-ABI library loads (no GPU needed) and exports every declared symbol;
ctypes struct layouts match the header."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "adjamr_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(adj_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for want in ("adj_step_level", "adj_fill_physical", "adj_fill_ghost_rects", "adj_restrict",
                 "adj_flag_adjoint", "adj_step_tile_shape", "adj_abi_version", "adj_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_1511_03645_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.adj_abi_version() == _lib.ABI_VERSION
    ni, nj = C.c_int32(), C.c_int32()
    assert lib.adj_step_tile_shape(1, 2, C.byref(ni), C.byref(nj)) == 0 and nj.value == 28
    assert lib.adj_step_tile_shape(7, 2, C.byref(ni), C.byref(nj)) == _lib.ADJ_ERR_BAD_ARG
    assert b"variant" in lib.adj_last_error()


def test_null_args_rejected_without_gpu():
    from paper_1511_03645_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load_library()
    a = _lib.AdjStepArgs()
    assert lib.adj_step_level(C.byref(a)) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_flag_adjoint(C.byref(_lib.AdjFlagArgs())) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_ghost_plan_build(C.byref(_lib.AdjGhostPlanBuildArgs())) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_fill_ghost_plan(C.byref(_lib.AdjGhostPlanFillArgs())) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_flag_level_mask(C.byref(_lib.AdjFlagMaskArgs())) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_functional(C.byref(_lib.AdjFunctionalArgs())) == _lib.ADJ_ERR_BAD_ARG
    assert lib.adj_gauges(C.byref(_lib.AdjGaugeArgs())) == _lib.ADJ_ERR_BAD_ARG


def _struct_fields(name):
    text = open(HEADER).read()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    typewords = {"const", "unsigned", "long", "double", "int32_t", "int64_t", "uint32_t", "uint8_t", "int8_t", "void", "char",
                 "AdjPatch", "AdjTile", "AdjRect", "AdjGhostPlan", "AdjGauge", "AdjGhostPlanFillArgs",
                 "AdjStepRestrict", "AdjJobFill"}
    for decl in body.split(";"):
        toks = decl.replace("*", " ").replace(",", " , ").split()
        if not toks:
            continue
        rest = [t for t in toks if t not in typewords]
        for n in " ".join(rest).split(","):
            n = n.strip()
            arr = re.match(r"(\w+)\[(\d+)\]", n)
            fields.append(arr.group(1) if arr else n)
    return fields


@pytest.mark.parametrize("name", ["AdjStepArgs", "AdjStepRestrict", "AdjJobFill", "AdjPhysArgs", "AdjGhostArgs", "AdjRestrictArgs", "AdjFlagArgs",
                                  "AdjGhostPlan", "AdjGhostPlanBuildArgs", "AdjGhostPlanFillArgs",
                                  "AdjFlagMaskArgs", "AdjFunctionalArgs", "AdjGaugeArgs"])
def test_ctypes_structs_mirror_header(name):
    from paper_1511_03645_b200 import _lib
    assert [f[0] for f in getattr(_lib, name)._fields_] == _struct_fields(name)


def test_table_dtypes_mirror_header():
    from paper_1511_03645_b200 import _lib
    assert list(_lib.PATCH_DTYPE.names) == _struct_fields("AdjPatch")
    assert list(_lib.TILE_DTYPE.names) == _struct_fields("AdjTile")
    assert list(_lib.RECT_DTYPE.names) == _struct_fields("AdjRect")
    assert list(_lib.GAUGE_DTYPE.names) == _struct_fields("AdjGauge")
    assert _lib.GAUGE_DTYPE.itemsize == 48


def test_product_refuses_cpu_fallback():
    import torch
    from paper_1511_03645_b200 import _lib
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailableError):
        _lib.lib()


def test_integration_stub_matches_header():
    """The ctypes binding shown in INTEGRATION.md mirrors AdjStepArgs."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text[text.index("class AdjStepArgs"):text.index("lib.adj_step_level.argtypes")]
    assert re.findall(r'\("(\w+)"', block) == _struct_fields("AdjStepArgs")
    for name in declared_functions():
        assert name in text, name


def test_struct_sizes_match_the_compiled_library():
    """sizeof of every argument struct and table row, ctypes / numpy against the library."""
    from paper_1511_03645_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load_library()
    for cls in _lib.STRUCTS:
        assert lib.adj_struct_size(cls.__name__.encode()) == C.sizeof(cls), cls.__name__
    assert lib.adj_struct_size(b"AdjPatch") == _lib.PATCH_DTYPE.itemsize
    assert lib.adj_struct_size(b"AdjTile") == _lib.TILE_DTYPE.itemsize
    assert lib.adj_struct_size(b"AdjRect") == _lib.RECT_DTYPE.itemsize
    assert lib.adj_struct_size(b"NoSuchStruct") == 0
