"""Test and benchmark support (not part of the product package).

``support.synth`` restates the reference's synthetic scene generator
(``poseflow/synth.py``) so that the GPU box, where the reference is absent,
can regenerate the same inputs.  Only ``tests/``, ``bench.py``,
``__graft_entry__.smoke()`` and ``tools/`` import it.
"""
