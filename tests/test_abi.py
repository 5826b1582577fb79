"""CPU: the C-ABI library loads and exports exactly what include/mtsph_b200.h
declares; without a GPU the product path refuses to run (no fallback)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mtsph_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mtsph_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2309_04010_b200 import _lib
    lib = _lib.load_library(require_device=False)
    names = declared_functions()
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the whole header, and nothing else
    assert sorted(_lib.SIGNATURES) == names
    assert lib.mtsph_abi_version() == 1


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2309_04010_b200", "libmtsph_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data


def test_no_device_fails_loudly():
    from paper_2309_04010_b200 import _lib, errors
    lib = _lib.load_library(require_device=False)
    if lib.mtsph_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(errors.BackendError, match="no CUDA device"):
        _lib.load_library(require_device=True)
    # a C-level call also refuses (status 2, message), never computes on CPU
    out = np.zeros((2, 2, 2))
    st = lib.mtsph_velocity_gradient_gather(
        2, 2, _lib.ptr(np.zeros((2, 2))), _lib.ptr(np.array([0, 0, 0], np.int64)),
        _lib.ptr(np.zeros(0, np.int64)), _lib.ptr(np.zeros((0, 2))), _lib.ptr(np.ones(2)),
        _lib.ptr(out))
    assert st == 2 and b"no CUDA device" in lib.mtsph_last_error()


def test_problem_construction_requires_gpu():
    from paper_2309_04010_b200 import _lib, errors, scenarios
    from paper_2309_04010_b200.config import resolve
    if _lib.load_library(require_device=False).mtsph_device_count() > 0:
        pytest.skip("a GPU is visible")
    p = resolve({"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
                 "n_outer": 4}).params
    with pytest.raises(errors.BackendError):
        scenarios.build(p)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2309_04010_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f


def test_select_device_without_gpu_fails_loudly():
    from paper_2309_04010_b200 import _lib, errors
    from paper_2309_04010_b200.device import select_device
    if _lib.load_library(require_device=False).mtsph_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(errors.BackendError):
        select_device(0)


def test_null_handles_are_rejected():
    """Every entry point that takes a problem / neighbourhood handle returns
    MTSPH_ERR_ARG with a message for a null handle (destroy: a no-op, like
    free(NULL)) -- no device needed, nothing is dereferenced."""
    import ctypes
    from paper_2309_04010_b200 import _lib
    lib = _lib.load_library(require_device=False)
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    names = sorted(set(re.findall(
        r"\b(mtsph_[a-z0-9_]+)\s*\(\s*(?:const\s+)?mtsph_(?:solid|porous|nbh)\s*\*", text)))
    assert len(names) >= 50
    for name in names:
        _, argtypes = _lib.SIGNATURES[name]
        args = [0.0 if t is ctypes.c_double else 0 if t in (ctypes.c_int, ctypes.c_int64)
                else None for t in argtypes]
        st = getattr(lib, name)(*args)
        if name.endswith("_destroy"):
            assert st == 0, name
        else:
            assert st == 1, name
            assert b"null handle" in lib.mtsph_last_error(), name


def test_accel_shim_has_the_reference_kernel_signatures():
    """paper_2309_04010_b200.accel is a drop-in for mtsph/_accel.py: the
    same seven public functions with the same parameter names and order.
    The signatures are pinned here; when the reference package is present
    (this container, not the GPU box) they are also compared with it."""
    import inspect
    import os
    from paper_2309_04010_b200 import accel
    want = {
        "velocity_gradient_gather": "src indptr idx grad vol out",
        "pair_tensor_divergence": "tens indptr idx grad vol out",
        "pair_tensor_divergence_mapped": "tens amap indptr idx grad vol out",
        "scalar_difference_flux": "sat coeff amap indptr idx vol grad out",
        "damping_sweep": "vel pair_i pair_j pair_damp inv_mass_i inv_mass_j group_ptr eta dt",
        "conservative_mass_rate": "flux amap pair_i pair_j pair_grad vol out",
        "porous_stress_rhs": "def_grad pressure corr indptr idx grad0 vol0 mu lam tbuf out_j out_rate",
    }
    for name, params in want.items():
        got = " ".join(inspect.signature(getattr(accel, name)).parameters)
        assert got == params, name
    src = "/root/reference/pkg/src/mtsph/_accel.py"
    if os.path.exists(src):
        import ast
        tree = ast.parse(open(src).read())
        ref = {f.name: " ".join(a.arg for a in f.args.args) for f in tree.body
               if isinstance(f, ast.FunctionDef) and not f.name.startswith("_")}
        assert ref == want
