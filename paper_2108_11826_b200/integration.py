"""Drop-in of the GPU parser into an installed ``poseflow`` (the reference).

``install()`` swaps ``poseflow.paf.parse`` (``paf.py:292-305``) — and the
module-level alias the post-processing operator calls,
``poseflow.operators.parse`` (``operators.py:25``, used at ``:153``) — for
``gpu_parse``, the B200 path behind the same signature:

* validation first, with the reference objects' own ``validate()``
  (``paf.py:295-296``), so ``ConfigError`` / ``ContractError`` are the
  reference's exception classes, raised before any device work;
* the frame parsed through ``libpf_b200.so`` (``parser.parse``);
* a new list of the reference's own ``HumanPose`` / ``Keypoint`` instances
  (``types.py:75-78``, ``:208-230``), byte-identical ``pose_record`` lines.

Nothing here imports ``poseflow`` until ``install()`` is called; the
product never depends on the reference.  INTEGRATION.md §1 shows the same
swap as the two lines a maintainer would add to ``paf.py``.
"""

from __future__ import annotations

import importlib
import threading
from typing import Callable, Optional


class GpuParse:
    """Callable ``parse(maps, topo, params)`` with the reference's contract.

    ``calls`` / ``frames`` count what went through the GPU (evidence that a
    swapped pipeline really used it)."""

    def __init__(self, ref_types=None, device: Optional[int] = None):
        self._types = ref_types
        self._device = device
        self._lock = threading.Lock()
        self.calls = 0

    def __call__(self, maps, topo, params):
        from .parser import _params_of, default_parser

        params.validate()                     # the reference's ConfigError (paf.py:295)
        maps.validate(topo)                   # the reference's ContractError (paf.py:296)
        ours = _params_of(params)
        eng = default_parser(topo, self._device)
        conf = maps.conf.array[None]
        paf = maps.paf.array[None]
        res = eng.parse_arrays(conf, paf, maps.stride, ours)
        with self._lock:
            self.calls += 1
        poses = res.poses(0)
        t = self._types
        if t is None:
            return poses
        return [t.HumanPose(keypoints=tuple(None if kp is None else t.Keypoint(kp.x, kp.y, kp.score)
                                            for kp in p.keypoints),
                            score=p.score, n_parts=p.n_parts) for p in poses]


def install(package: str = "poseflow", device: Optional[int] = None) -> GpuParse:
    """Replace ``<package>.paf.parse`` and every module-level ``parse`` alias
    of it (``<package>.operators.parse``) with a ``GpuParse``.  Returns the
    installed callable; ``uninstall()`` restores the reference."""
    paf = importlib.import_module(f"{package}.paf")
    types = importlib.import_module(f"{package}.types")
    original = getattr(paf, "_pf_b200_original_parse", paf.parse)
    shim = GpuParse(types, device)
    paf._pf_b200_original_parse = original
    paf.parse = shim
    for name in ("operators", "pipeline", "cli", "selftest"):
        try:
            mod = importlib.import_module(f"{package}.{name}")
        except Exception:          # noqa: BLE001 - optional modules of the reference
            continue
        if getattr(mod, "parse", None) is original or isinstance(getattr(mod, "parse", None), GpuParse):
            mod.parse = shim
    return shim


def uninstall(package: str = "poseflow") -> None:
    paf = importlib.import_module(f"{package}.paf")
    original: Optional[Callable] = getattr(paf, "_pf_b200_original_parse", None)
    if original is None:
        return
    for name in ("paf", "operators", "pipeline", "cli", "selftest"):
        try:
            mod = importlib.import_module(f"{package}.{name}")
        except Exception:          # noqa: BLE001
            continue
        if isinstance(getattr(mod, "parse", None), GpuParse):
            mod.parse = original
