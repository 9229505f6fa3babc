"""GPU overlay rasteriser against the reference's visualize
(poseflow/operators.py:249-290), via tests/golden/overlay_golden.npz (made by
tests/golden/make_overlay_golden.py from the reference itself).

CPU: the host half (keypoint placement, draw-order primitive list, label
glyph expansion) rastered by a plain-Python checker equals the golden images.
GPU: pf_overlay / visualize_batch / visualize equal them byte for byte."""

import os

import numpy as np
import pytest

import paper_2108_11826_b200 as pf
from paper_2108_11826_b200.overlay import _primitives

GOLD = os.path.join(os.path.dirname(__file__), "golden", "overlay_golden.npz")


def load():
    g = np.load(GOLD)
    n, h, w = (int(x) for x in g["shape"])
    images = np.random.default_rng(2108).random((n, h, w, 3)).astype(np.float32)   # as the generator
    poses = []
    for f in range(n):
        fp = []
        for i in range(int(g["n_humans"][f])):
            kps = tuple(pf.Keypoint(float(x), float(y), float(s)) if pres else None
                        for x, y, s, pres in g["kp"][f, i])
            fp.append(pf.HumanPose(keypoints=kps, score=float(g["score"][f, i]),
                                   n_parts=sum(k is not None for k in kps)))
        poses.append(fp)
    expected = []
    for si in range(len(g["styles"])):
        out = images.copy().reshape(-1, 3)
        lo, hi = int(g["style_first"][si]), int(g["style_first"][si + 1])
        out[g["changed"][lo:hi]] = g["changed_rgb"][lo:hi]
        expected.append(out.reshape(images.shape))
    styles = [pf.OverlayStyle(int(r), int(t), bool(lab)) for r, t, lab in g["styles"]]
    return images, poses, styles, expected, [int(x) for x in g["input_wh"]]


def py_raster(image, prims):
    """Checker: the primitives drawn in order with the reference's integer rules."""
    img = image.copy()
    h, w = img.shape[:2]

    def put(x, y, c):
        if 0 <= y < h and 0 <= x < w:
            img[y, x] = c

    def disc(cx, cy, r, c):
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                if dx * dx + dy * dy <= r * r:
                    put(cx + dx, cy + dy, c)

    for _, kind, x0, y0, x1, y1, r, rgb in prims:
        c = np.array(rgb, np.float32)
        if kind == 1:
            disc(x0, y0, r, c)
            continue
        dx, dy = abs(x1 - x0), -abs(y1 - y0)
        sx, sy = (1 if x0 < x1 else -1), (1 if y0 < y1 else -1)
        err, x, y = dx + dy, x0, y0
        while True:
            if r == 0:
                put(x, y, c)
            else:
                disc(x, y, r, c)
            if x == x1 and y == y1:
                break
            e2 = 2 * err
            if e2 >= dy:
                err += dy
                x += sx
            if e2 <= dx:
                err += dx
                y += sy
    return img


def test_host_primitives_reproduce_reference():
    images, poses, styles, expected, (iw, ih) = load()
    topo = pf.load_topology("coco18")
    h, w = images.shape[1:3]
    for si, style in enumerate(styles):
        for f in range(len(images)):
            prims = _primitives(f, poses[f], style, topo, h, w, iw, ih)
            assert np.array_equal(py_raster(images[f], prims), expected[si][f]), (si, f)


@pytest.mark.gpu
def test_gpu_overlay_matches_reference():
    images, poses, styles, expected, (iw, ih) = load()
    topo = pf.load_topology("coco18")
    for si, style in enumerate(styles):
        got = pf.visualize_batch(images, poses, style, topo, iw, ih)
        assert np.array_equal(got, expected[si]), si
        one = pf.visualize(pf.Frame(seq_id=0, image=pf.TensorF32(images[2].copy()), ingest_ns=0), poses[2],
                           style, topo, iw, ih)
        assert np.array_equal(one.array, expected[si][2])
    empty = pf.visualize(pf.Frame(seq_id=0, image=pf.TensorF32(images[0].copy()), ingest_ns=0), [], styles[0],
                         topo, iw, ih)
    assert np.array_equal(empty.array, images[0])
    with pytest.raises(pf.ContractError):
        pf.OverlayStyle(keypoint_radius=0).validate()
