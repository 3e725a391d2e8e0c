"""Seeded synthetic inputs shared by the product path, the oracle tests and bench.py.

This module holds NO arithmetic of the method (no basis, quadrature, assembly,
smoothing or solving).  It only defines *what* each workload is (grid size,
order, geometry recipe, solver constants) and draws the seeded random geometry
and random vectors.  Both the CUDA path (via ``paper_2010_00881_b200``) and the
CPU oracle (``oracle/``) consume these inputs; neither imports the other.

Geometry recipe: DESIGN.md "Input recipe" / SURVEY.md §8(c) reading R12.
"""
from .configs import CONFIGS, Config, get_config, hp_plate, small_config  # noqa: F401
from .voids import sample_voids, config_voids  # noqa: F401
