"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no Exp/Log, Jacobians, assembly,
factorisation or optimiser step).  It only draws random poses / measurements with
numpy and composes 4x4 / 3x3 homogeneous matrices.  See DESIGN.md "Input recipe".
"""
from .cube import (  # noqa: F401
    CubeTopology,
    cube_topology,
    cube_batch,
    quat_to_rot,
    rot2,
)
