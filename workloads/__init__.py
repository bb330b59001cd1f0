"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This package holds NO arithmetic of the method (no waiting-time scan, no
violation probability, no objective): it only draws the raw problem
description -- request groups, virtual queues, per-(device, model) profile
constants and output-length tables -- that both the CUDA path and the oracle
consume.  See DESIGN.md "Input recipe".
"""
from .synth import Problem, make_config, make_problem, balanced_row, CONFIGS  # noqa: F401
