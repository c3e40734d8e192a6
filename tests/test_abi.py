"""CPU-side checks of the C-ABI boundary: the library builds, loads, and
exports every entry point include/synperf.h declares; struct layouts of the
ctypes binding match the header.  No compute call is made (no GPU here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "synperf.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libsp():
    from __graft_entry__ import _build_module

    build = _build_module()
    build.build()
    return C.CDLL(build.LIB)


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("sp_create", "sp_destroy", "sp_last_error", "sp_load_gpu_specs",
                     "sp_free_specs", "sp_load_model", "sp_free_model", "sp_featurize",
                     "sp_predict"):
        assert required in names


def test_library_exports_every_declared_symbol(libsp):
    missing = [n for n in declared_functions() if not hasattr(libsp, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2601_14910_b200 import _abi

    assert sorted(_abi.EXPORTED) == declared_functions()


def test_struct_layouts():
    from paper_2601_14910_b200 import _abi
    from workloads import specs

    assert C.sizeof(_abi.sp_gpu_spec) == specs.SPEC_DTYPE.itemsize == 112
    for name, _ in _abi.sp_gpu_spec._fields_:
        if name == "reserved_":
            continue
        key = name if name in specs.SPEC_DTYPE.names else "_pad"
        assert getattr(_abi.sp_gpu_spec, name).offset == specs.SPEC_DTYPE.fields[key][1], name
    assert C.sizeof(_abi.sp_config_batch) == 56
    assert C.sizeof(_abi.sp_pairing) == 40
    assert C.sizeof(_abi.sp_features) == 48
    assert C.sizeof(_abi.sp_mlp_desc) == 16 + 21 * 8 + 8


def test_version_string(libsp):
    libsp.sp_version.restype = C.c_char_p
    assert b"sm_100a" in libsp.sp_version()


def test_no_oracle_in_product_path():
    """The product package never imports, links or executes oracle/."""
    pkg = os.path.join(ROOT, "paper_2601_14910_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", "orc_", "synperf_oracle"):
                    assert pat not in txt, (f, pat)


def test_sass_is_sm100a(libsp):
    """The kernels are compiled for sm_100a (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    cuobj = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobj):
        pytest.skip("cuobjdump not available")
    from __graft_entry__ import _build_module

    build = _build_module()
    out = subprocess.run([cuobj, "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
