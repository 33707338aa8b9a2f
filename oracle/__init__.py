"""CPU oracle for the FullSWOF_2D explicit time step -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  It shares no code with the CUDA path (paper_1307_4839_b200/), and the product path
never imports it.  See oracle/swof_oracle.h for the method, citations and parity-unpinned readings.
"""
from .oracle import (  # noqa: F401
    build, lib, params_from_config, minmod, icbrt, muscl_cell, face, centered_source, green_ampt, friction,
    friction_gcf, rain_rate, hydrograph, cfl_dt, stage, heun_step, run, pairwise_sum, Counters,
    face_rusanov, cfl_dt_face, flow_direction,
)
