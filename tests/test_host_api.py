"""Host-side API mirror (no GPU): params, topology, maps contracts, formats,
pose_record, synthetic generator vs the reference's own outputs."""

import io
import json
import warnings

import numpy as np
import pytest

import paper_2108_11826_b200 as pf
from support import synth
from conftest import golden_path


class TestParserParams:                       # paf.py:44-54, test_paf.py:317-328
    def test_defaults(self):
        p = pf.ParserParams()
        assert (p.conf_threshold, p.nms_window, p.n_samples, p.sample_dot_threshold,
                p.good_fraction_min, p.min_parts, p.min_human_score) == (0.1, 3, 10, 0.05, 0.8, 4, 0.2)
        assert (p.upsample, p.blur_sigma) == (1, 0.0)
        p.validate()

    @pytest.mark.parametrize("kw", [dict(nms_window=4), dict(nms_window=1), dict(n_samples=1),
                                    dict(conf_threshold=1.5), dict(conf_threshold=-0.1),
                                    dict(sample_dot_threshold=2.0), dict(good_fraction_min=-1.0),
                                    dict(conf_threshold=float("nan")), dict(min_parts=0),
                                    dict(upsample=0), dict(blur_sigma=-1.0)])
    def test_invalid(self, kw):
        with pytest.raises(pf.ConfigError):
            pf.ParserParams(**kw).validate()


class TestTopology:
    def test_coco18(self, topo):                # test_topology.py:8-16
        assert topo.n_keypoints == 18 and topo.n_limbs == 19
        chans = [c for pair in topo.paf_channels for c in pair]
        assert sorted(chans) == list(range(38))
        assert topo.limbs[12] == (1, 0) and topo.limbs[17] == (2, 16) and topo.limbs[18] == (5, 17)
        assert topo.keypoint_names[0] == "nose" and topo.part_index("left_ear") == 17

    def test_same_tables_as_reference_data_file(self, topo):
        ref = json.load(open(golden_path("frames_records.json")))
        assert ref["names"]                       # fixtures exist
        # the keypoint names appear in the reference records in part order
        names = {kp["part"] for line in ref["R"].values() for h in json.loads(line)["humans"]
                 for kp in h["keypoints"]}
        assert names <= set(topo.keypoint_names)

    @pytest.mark.parametrize("limbs,chans", [([[0, 0]], None), ([[0, 5]], None),
                                              ([[0, 1]], [[0, 0]]), ([[0, 1]], [[0, 3]]),
                                              ([[0, 1], [1, 2]], [[0, 1], [1, 2]])])
    def test_invalid(self, limbs, chans):
        with pytest.raises(pf.ContractError):
            pf.SkeletonTopology.create(["a", "b", "c"], limbs, chans)

    def test_duplicate_names(self):
        with pytest.raises(pf.ContractError):
            pf.SkeletonTopology.create(["a", "a"], [[0, 1]])

    def test_disconnected_warns(self):
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            pf.SkeletonTopology.create(["a", "b", "c", "d"], [[0, 1], [2, 3]])
        assert any("disconnected" in str(x.message) for x in w)

    def test_load_errors(self, tmp_path):
        with pytest.raises(pf.FormatError):
            pf.load_topology(tmp_path / "missing.toml")
        bad = tmp_path / "bad.toml"
        bad.write_text("keypoints = [")
        with pytest.raises(pf.FormatError):
            pf.load_topology(bad)
        ok = tmp_path / "ok.toml"
        ok.write_text('keypoints = ["a", "b"]\nlimbs = [[0, 1]]\n')
        assert pf.load_topology(ok).paf_channels == ((0, 1),)


class TestFeatureMaps:
    def test_dims(self, topo):
        good = pf.FeatureMaps(pf.TensorF32.from_array(np.zeros((19, 4, 5))),
                              pf.TensorF32.from_array(np.zeros((38, 4, 5))), 8, 0)
        good.validate(topo, input_w=40, input_h=32)
        for conf, paf in [((18, 4, 5), (38, 4, 5)), ((19, 4, 5), (36, 4, 5)), ((19, 4, 5), (38, 4, 6))]:
            m = pf.FeatureMaps(pf.TensorF32.from_array(np.zeros(conf)),
                               pf.TensorF32.from_array(np.zeros(paf)), 8, 0)
            with pytest.raises(pf.ContractError):
                m.validate(topo)
        with pytest.raises(pf.ContractError):
            good.validate(topo, input_w=41)

    def test_cell_to_pixel(self):
        assert pf.cell_to_pixel(3, 4, 8) == (4 * 8 + 3.5, 3 * 8 + 3.5)
        assert pf.cell_to_pixel(3, 4, 1) == (4.0, 3.0)
        assert pf.pixel_to_cell(*pf.cell_to_pixel(2, 7, 8), 8) == (2.0, 7.0)

    def test_human_pose_validate(self):
        kps = [None] * 18
        kps[0] = pf.Keypoint(1.0, 2.0, 0.5)
        pf.HumanPose(tuple(kps), 0.5, 1).validate(input_w=8, input_h=8)
        with pytest.raises(pf.ContractError):
            pf.HumanPose(tuple(kps), 0.5, 2).validate()


class TestFormats:
    def test_hpt_round_trip(self):
        t = pf.TensorF32.from_array(np.random.default_rng(0).random((2, 3, 4)))
        buf = io.BytesIO()
        n = pf.write_tensor(t, buf)
        assert n == 4 + 1 + 12 + 96
        buf.seek(0)
        assert np.array_equal(pf.read_tensor(buf).array, t.array)

    def test_hpt_errors(self):
        with pytest.raises(pf.FormatError):
            pf.read_tensor(io.BytesIO(b"HPT2\x01"))
        with pytest.raises(pf.FormatError):
            pf.read_tensor(io.BytesIO(b"HPT1\x01\x04\x00\x00\x00abc"))

    def test_ppm(self):
        img = np.random.default_rng(1).random((3, 5, 3)).astype(np.float32)
        buf = io.BytesIO()
        pf.write_ppm(pf.TensorF32.from_array(img), buf)
        buf.seek(0)
        back = pf.read_ppm(buf).array
        q = np.floor(img * 255 + 0.5).astype(np.uint8)
        assert np.array_equal(back, q.astype(np.float32) / np.float32(255.0))  # formats.py:116-117


class TestPoseRecord:
    def test_known_answers(self, topo):
        want = json.load(open(golden_path("records_golden.json")))
        kps = [None] * 18
        kps[0] = pf.Keypoint(x=1.5, y=2.5, score=0.75)
        kps[2] = pf.Keypoint(x=3.0, y=4.0, score=0.5)
        pose = pf.HumanPose(keypoints=tuple(kps), score=1.25, n_parts=2)
        kps2 = [None] * 18
        kps2[5] = pf.Keypoint(x=655.0, y=0.0, score=float(np.float32(0.1)))
        pose2 = pf.HumanPose(keypoints=tuple(kps2), score=0.30000000000000004, n_parts=1)
        assert pf.pose_record(7, [pose], topo) == want["one"]
        assert pf.pose_record(8, [pose, pose2], topo) == want["two"]
        assert pf.pose_record(3, [], topo) == want["empty"]


class TestSynthPort:
    """The input generator reproduces the reference renderer bit for bit."""

    def test_procedural_scenes(self):
        want = json.load(open(golden_path("scenes_golden.json")))
        sp = synth.SynthParams()
        for key, humans in want.items():
            seed, seq = (int(x) for x in key.split("_"))
            got = synth.procedural_scene(seed, seq, 656, 368, sp)
            assert [[list(k) for k in h.keypoints] for h in got.humans] == humans

    def test_render_matches_reference(self, topo, golden_frames):
        data, recs = golden_frames
        sp = synth.SynthParams()
        for name in recs["names"]:
            kps = data[f"{name}.kps"]
            humans = tuple(synth.GroundTruthHuman(tuple(None if np.isnan(k[0]) else (float(k[0]), float(k[1]))
                                                     for k in h)) for h in kps)
            m = synth.render_feature_maps(synth.GroundTruthScene(humans, 656, 368), topo, sp)
            assert np.array_equal(m.conf.array, data[f"{name}.conf"]), name
            assert np.array_equal(m.paf.array, data[f"{name}.paf"]), name

    def test_crowd_scene(self):
        s = synth.crowd_scene(3, 0)
        assert len(s.humans) == 40
        s.validate(18)
