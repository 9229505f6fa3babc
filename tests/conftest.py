import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpf_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def topo():
    import paper_2108_11826_b200 as pf

    return pf.load_topology("coco18")


@pytest.fixture(scope="session")
def golden_frames():
    data = np.load(os.path.join(GOLDEN, "frames_golden.npz"))
    with open(os.path.join(GOLDEN, "frames_records.json")) as f:
        recs = json.load(f)
    return data, recs


def golden_path(name):
    return os.path.join(GOLDEN, name)


def record_of(humans, topo, seq=0):
    """pose_record of oracle humans ((score, n, kps) tuples) — operators.py:293-310."""
    import paper_2108_11826_b200 as pf

    poses = [pf.HumanPose(keypoints=tuple(None if k is None else pf.Keypoint(*k) for k in kps),
                          score=s, n_parts=n) for s, n, kps in humans]
    return pf.pose_record(seq, poses, topo)
