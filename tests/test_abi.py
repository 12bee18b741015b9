"""The C-ABI library builds, loads and exports every symbol include/fgl.h declares (CPU only:
no compute call is made without a GPU). Also: the product package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fgl.h")).read()
    return sorted(set(re.findall(r"^FGL_API[^(]*?\b(fgl_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2509_17390_b200 import _build
    return _build.build()


def test_header_declares_the_boundary():
    syms = _header_symbols()
    for s in ("fgl_scene_create", "fgl_scene_upload_mesh", "fgl_scene_build", "fgl_cast_spinning",
              "fgl_cast_rosette", "fgl_cast_rays", "fgl_last_error", "fgl_scene_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = set(re.findall(r"\sT\s(fgl_\w+)", out))
    missing = set(_header_symbols()) - exported
    assert not missing, missing


def test_binding_covers_the_header(libpath):
    import paper_2509_17390_b200 as fgl
    assert sorted(fgl.SYMBOLS) == _header_symbols()
    L = fgl.lib()
    assert L.fgl_abi_version() == 2
    assert b"sm_100a" in L.fgl_version()


def test_library_is_sm100a(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(libpath):
    import torch
    import paper_2509_17390_b200 as fgl
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        fgl.Scene(device="cuda:0")


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2509_17390_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert all(not a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(os.path.join(dirpath, f)).read().lower().replace("(never by the oracle)", ""), f
