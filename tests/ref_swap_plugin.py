"""pytest plugin: run the reference's own test suite with ``poseflow.paf.parse``
swapped for the B200 path (``paper_2108_11826_b200.integration.install``).

Loaded with ``-p ref_swap_plugin`` by ``tests/test_gpu_reference_dropin.py``
before the reference test modules are imported, so their
``from poseflow.paf import parse`` binds the GPU parse.  At exit it writes
the number of GPU parse calls to ``$PF_SWAP_REPORT`` (evidence the swapped
path actually ran).
"""

import json
import os

_SHIM = None


def pytest_configure(config):
    global _SHIM
    from paper_2108_11826_b200 import integration

    _SHIM = integration.install("poseflow")


def pytest_unconfigure(config):
    path = os.environ.get("PF_SWAP_REPORT")
    if path and _SHIM is not None:
        import poseflow.operators
        import poseflow.paf

        with open(path, "w") as f:
            json.dump({"gpu_parse_calls": _SHIM.calls,
                       "paf_parse_is_gpu": poseflow.paf.parse is _SHIM,
                       "operators_parse_is_gpu": poseflow.operators.parse is _SHIM}, f)
