"""The C-ABI library loads and exports every entry point include/romap.h
declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2304_05735_b200", "libromap.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "romap.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(romap_[a-z_0-9]+)\s*\(", src)) - {"romap_alloc_fn", "romap_free_fn"})


def test_header_declares_the_survey_boundary():
    names = declared_symbols()
    for n in ["romap_ctx_create", "romap_create_object", "romap_add_observation", "romap_train_step",
              "romap_render", "romap_render_scene", "romap_query_density", "romap_get_params", "romap_set_params",
              "romap_debug_dump", "romap_sync", "romap_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_no_device_is_reported_not_crashed(lib):
    lib.romap_ctx_create.restype = ctypes.c_int32
    out = ctypes.c_void_p()
    st = lib.romap_ctx_create(0, None, None, None, None, ctypes.byref(out))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert st == -4                       # ROMAP_E_CUDA: no device
        lib.romap_last_error.restype = ctypes.c_char_p
        assert b"device" in lib.romap_last_error()


def test_binding_names_match_the_abi():
    from paper_2304_05735_b200 import romap as R
    for n in ["create_object", "add_observation", "train_step", "render", "render_scene", "query_density",
              "get_params", "set_params", "debug_dump", "forward_backward", "optimizer_step"]:
        assert hasattr(R.Context, n)
    assert R.version().startswith("romap-b200")
