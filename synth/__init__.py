"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the SART method (no attention, no sampler,
no scheduler).  It only draws random inputs: model shapes, random-init weights,
prompts, scripted branch lengths / labels / reward trajectories, and arrival
times.  Both sides of every parity test (``oracle/`` and the CUDA path through
``paper_2505_13326_b200``) consume the same arrays produced here.
"""
from .workload import *  # noqa: F401,F403
