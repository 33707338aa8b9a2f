"""Seeded synthetic workloads (cfg0..cfg4 of BASELINE.json) shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic: only the problem statement (grid, parameters,
boundary types, forcing tables) and the seeded input rasters. Both sides read identical bits.
"""
from .configs import SwofConfig, GreenAmpt, Inflow, make, CONFIG_NAMES  # noqa: F401
