"""The C-ABI library loads and exports every symbol include/tf.h declares (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tf.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:tf_status|const char \*|int)\s*\*?\s*(tf_\w+)\s*\(", src, re.M)))


def load_builder():
    import importlib.util
    spec = importlib.util.spec_from_file_location("tf_build", os.path.join(ROOT, "paper_2110_05997_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def lib_path():
    return load_builder().build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["tf_ctx_create", "tf_ctx_destroy", "tf_cpd_eval", "tf_cpd_eval_host", "tf_grams", "tf_hadamard",
              "tf_gn_matvec", "tf_cg_solve", "tf_status_str", "tf_last_error"]:
        assert s in syms, s


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s), f"{s} not exported by {lib_path}"
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_status_strings(lib_path):
    lib = ctypes.CDLL(lib_path)
    lib.tf_status_str.restype = ctypes.c_char_p
    assert lib.tf_status_str(0) == b"TF_OK"
    assert lib.tf_status_str(5) == b"TF_ERR_NONFINITE"
    assert lib.tf_version() >= 1


def test_binding_exports_match_header(lib_path):
    import paper_2110_05997_b200 as tf
    assert sorted(tf.EXPORTED) == declared_symbols()
    for s in declared_symbols():
        if s.startswith("tf_ctx") or s in ("tf_status_str", "tf_last_error", "tf_version"):
            continue
        assert hasattr(tf.Context, s), s


def test_no_cpu_fallback_without_gpu(lib_path):
    import torch
    import paper_2110_05997_b200 as tf
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = ctypes.CDLL(lib_path)
    h = ctypes.c_void_p()
    assert lib.tf_ctx_create(ctypes.byref(h), 0, None) == tf.TF_ERR_CUDA
