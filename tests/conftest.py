import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

REF_SRC = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(os.path.join(REF_SRC, "hefir"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    meta = None
    jp = os.path.join(GOLDEN, name + ".json")
    if os.path.exists(jp):
        with open(jp) as fh:
            meta = json.load(fh)
    npz = os.path.join(GOLDEN, name + ".npz")
    arrs = dict(np.load(npz, allow_pickle=False)) if os.path.exists(npz) else None
    return meta, arrs


@pytest.fixture(scope="session")
def golden_small():
    return load_golden("small")


@pytest.fixture(scope="session")
def golden_n1024():
    return load_golden("n1024")


@pytest.fixture(scope="session")
def golden_cifar64():
    return load_golden("cifar64")


def import_reference():
    """The reference package (build container only), via the gmpy2 shim."""
    if not HAVE_REF:
        pytest.skip("reference tree not mounted")
    shim = os.path.join(ROOT, "tests", "_shim")
    for p in (shim, REF_SRC):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    import hefir  # noqa: F401

    return hefir


INSTALLED_REF = os.path.join(ROOT, "baseline", "_ref")


def import_installed_reference():
    """The reference package as installed (unmodified) into baseline/_ref by
    `pip install --target` (it travels to the GPU box, /root/reference does
    not), imported through the gmpy2 shim (tests/_shim: mpz = int)."""
    if not os.path.isdir(os.path.join(INSTALLED_REF, "hefir")):
        pytest.skip("baseline/_ref (installed reference) not present")
    shim = os.path.join(ROOT, "tests", "_shim")
    for p in (shim, INSTALLED_REF):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_tests")
    import hefir

    if not os.path.abspath(hefir.__file__).startswith(os.path.abspath(INSTALLED_REF)) and not HAVE_REF:
        pytest.skip("a different hefir is importable")
    return hefir
