"""The drop-in, proven with the reference's own code.

* The reference's own test suite (installed with it in ``baseline/_ref`` by
  ``tools/install_reference.sh``) runs with ``poseflow.paf.parse`` swapped for
  the GPU path (``integration.install``, the INTEGRATION.md §1 swap): the
  parse tests (``test_paf.py``), the operator / pipeline tests
  (``test_operators.py``, byte-identical ``poses.jsonl`` across runs), the
  scheduler and dataflow tests, the CLI, and acceptance criteria 4-7
  (round-trip accuracy, oracle equivalence, 5x1000-frame determinism and
  batch invariance, ordering) — all through the GPU parse.
* ``make_batched_postprocess`` runs as the post-processing stage of the
  reference's own pipeline (``build_pose_pipeline`` + ``run_pipeline``,
  dataflow.py:383-499) with ``linger_us``; its ``poses.jsonl`` bytes equal
  the reference pipeline's, its batches show up in the reference's
  ``PipelineStats.batch_hist`` and its parse time in the stage's busy time.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "poseflow_tests")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                 reason="reference not installed (tools/install_reference.sh)")]

HOT_PATH_TESTS = [
    "test_paf.py", "test_operators.py", "test_scheduler.py", "test_dataflow.py",
    "test_cli.py",
    "test_acceptance.py::test_criterion_4_round_trip_accuracy",
    "test_acceptance.py::test_criterion_5_parser_oracle_equivalence",
    "test_acceptance.py::test_criterion_6_determinism_batch_invariance",
    "test_acceptance.py::test_criterion_7_ordering_and_conservation",
]


def _ref_env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    return env


def test_reference_suite_with_gpu_parse(tmp_path):
    report = tmp_path / "swap.json"
    env = _ref_env()
    env["PF_SWAP_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_swap_plugin",
           "--deselect", "test_cli.py::TestBench::test_tiny_profile",    # needs matplotlib (report plot)
           *HOT_PATH_TESTS]
    proc = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1200)
    tail = proc.stdout[-3000:] + proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    assert " passed" in proc.stdout and " failed" not in proc.stdout, tail
    rep = json.loads(report.read_text())
    assert rep["paf_parse_is_gpu"] and rep["operators_parse_is_gpu"], rep
    assert rep["gpu_parse_calls"] > 5000, rep         # criterion 6 alone parses 5 x 1000 frames


def _ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from poseflow import config, dataflow, pipeline, synth as ref_synth   # noqa: F401

    return config, dataflow, pipeline, ref_synth


@pytest.mark.parametrize("linger_us,batch_max", [(0, 64), (3000, 16)])
def test_batched_operator_in_reference_pipeline(tmp_path, linger_us, batch_max):
    import paper_2108_11826_b200 as pf

    config, dataflow, pipeline, ref_synth = _ref_modules()
    from poseflow.paf import ParserParams as RefParams
    from poseflow.topology import load_topology as ref_topology

    def cfg():
        # a bursty backend (1 ms per batch + 0.1 ms per item) so frames queue up
        return config.PipelineConfig(input_w=640, input_h=368, frames=300, seed=23, batch_max=8,
                                     synth=ref_synth.SynthParams(batch_overhead_us=1000, per_item_us=100))

    # the reference pipeline as shipped (CPU parse)
    ref_stats = pipeline.run_pose_pipeline(cfg(), tmp_path / "ref", watchdog_s=120)
    want = (tmp_path / "ref" / "poses.jsonl").read_bytes()

    # the same graph with the GPU batched stage in the post-processing slot
    graph, sink = pipeline.build_pose_pipeline(cfg(), tmp_path / "gpu")
    topo = ref_topology("coco18")
    idx = [op.name for op in graph.operators].index("postprocess")
    graph.operators[idx] = pf.make_batched_postprocess(topo, RefParams(), batch_max=batch_max, linger_us=linger_us)
    try:
        stats = dataflow.run_pipeline(graph, watchdog_s=120)
    finally:
        sink.close()
    got = (tmp_path / "gpu" / "poses.jsonl").read_bytes()
    assert got == want
    assert stats.ordered and stats.frames_out == 300
    post = stats.ops[idx]
    assert post.items_in == post.items_out == 300
    assert post.busy_ns > 0                                   # ctx.timed charged the GPU parse
    # batch_hist sums every runner's batches: the inference stage's and ours
    assert sum(k * v for k, v in stats.batch_hist.items()) == 600
    assert sum(k * v for k, v in ref_stats.batch_hist.items()) == 300
    if linger_us:
        assert max(stats.batch_hist) > 1                      # the linger window formed real batches
