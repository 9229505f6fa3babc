"""The C-ABI library loads on a CPU host and exports every symbol the header
declares; host-only entry points behave (no device work here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pf_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2108_11826_b200 import _native

    lib = _native.load_library()
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_native.EXPORTED_SYMBOLS)


def test_abi_version_and_kernel_names():
    from paper_2108_11826_b200 import _native

    lib = _native.load_library()
    assert lib.pf_abi_version() == 1
    names = [lib.pf_kernel_name(k).decode() for k in range(_native.PF_N_KERNELS)]
    assert "k_nms_up_win" in names and "k_parse_frames" in names


@pytest.mark.parametrize("kw,code", [({}, 0), (dict(nms_window=4), 1), (dict(n_samples=1), 1),
                                     (dict(conf_threshold=1.1), 1), (dict(min_parts=0), 1),
                                     (dict(upsample=0), 1), (dict(blur_sigma=-2.0), 1),
                                     (dict(blur_sigma=100.0), 1)])
def test_validate_params_codes(kw, code):
    import paper_2108_11826_b200 as pf
    from paper_2108_11826_b200 import _native

    lib = _native.load_library()
    p = pf.ParserParams(**kw).to_native()
    assert lib.pf_validate_params(ctypes.byref(p)) == code


def test_product_has_no_oracle_dependency():
    """The product package never imports the checker."""
    pkg = os.path.join(ROOT, "paper_2108_11826_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "pf_oracle" not in src, f


def test_no_device_means_loud_failure():
    import torch

    import paper_2108_11826_b200 as pf

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(pf.DeviceError):
        pf.PafParser(pf.load_topology("coco18"))
