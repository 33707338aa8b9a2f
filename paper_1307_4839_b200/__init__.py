"""B200-native FullSWOF_2D explicit time step (arXiv 1307.4839): C-ABI library + thin binding.

    from paper_1307_4839_b200 import Solver, params_from_config
The product path is libswof.so (csrc/, include/swof.h); this package never imports the oracle.
"""
from .swof import (  # noqa: F401
    EXPORTS, SwofDiag, SwofError, SwofParams, Solver, flow_direction, lib, params_from_config,
)
