"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no cost, no collision test of
edges, no heuristic, no search).  It only produces input arrays: Halton samples
(the harness side of ``SampleFree``, PAPER.md P:188 / P:335), box obstacles
(P:338), feature points, MLP weights (synthetic), and the
per-config constants of ``configs/*.json``.  Both implementations consume the
identical float64 bytes it returns.
"""
from .halton import halton, halton_points  # noqa: F401
from .envs import Problem, make_problem, load_config, CONFIG_DIR  # noqa: F401
from .mc import DEFAULT_MC, mc_params, line_problem  # noqa: F401
