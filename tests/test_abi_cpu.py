"""CPU-only checks of the boundary: the C-ABI library builds/loads and exports every symbol that
include/encf.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "encf.h")).read()
    return sorted(set(re.findall(r"^(?:encf_status|const char\*|uint32_t)\s+(encf_\w+)\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("encf_keygen", "encf_encrypt_sk", "encf_decrypt", "encf_pt_ct_matmul", "encf_ct_ct_attn_score",
                 "encf_ct_ct_attn_value", "encf_rotate", "encf_rescale", "encf_export_c2m"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_09975_b200 import build as b
    so = b.build()
    lib = ctypes.CDLL(so)
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # status strings work without a device
    lib.encf_status_string.restype = ctypes.c_char_p
    assert lib.encf_status_string(3) == b"scale mismatch"


def test_binding_covers_header():
    import importlib
    try:
        E = importlib.import_module("paper_2604_09975_b200.encf")
    except ImportError as e:      # only if the .so is absent, which the previous test would catch
        raise AssertionError(e)
    assert set(declared_symbols()) <= set(E.exported_symbols())


def test_sass_is_sm100a():
    import subprocess
    from paper_2604_09975_b200 import build as b
    so = b.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
