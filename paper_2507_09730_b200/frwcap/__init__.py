"""Floating random walk capacitance extraction -- B200 device build.

Drop-in for the reference package `frwcap` (proj/python/frwcap/__init__.py):
the same eight names, backed by the pybind11 module `_core` built from
paper_2507_09730_b200/csrc/host over the CUDA library lib/libfrwgpu.so.
"""
from .._core import (  # noqa: F401
    __version__,
    analytic_plate_capacitance,
    expected_steps_uniform,
    extract_file,
    extract_json,
    reference_capacitance_file,
    run_cli,
    transit_tv,
)
from .._core import run_walks_json, sgf_cache_clear, sgf_cache_load, sgf_cache_save  # noqa: F401
from .._core import sgf_cache_stats  # noqa: F401
# single-transit API (microwalk.hpp:70-100, geometry.hpp:151-182) -- B200 extras
from .._core import build_grid, neighbor_weights, transits_grid, transits_structure  # noqa: F401
from .._core import transitions_json, walks_by_transitions  # noqa: F401
from .._core import SgfCache  # noqa: F401
from .._core import direct_sgf, exact_absorption_row  # noqa: F401  (host direct solves)

__all__ = [
    "analytic_plate_capacitance",
    "expected_steps_uniform",
    "extract_file",
    "extract_json",
    "reference_capacitance_file",
    "run_cli",
    "transit_tv",
    "__version__",
]
