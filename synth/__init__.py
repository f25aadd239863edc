"""Seeded synthetic workloads for the MOREA hot path (input generation only).

This package is shared by the oracle tests and the CUDA path, so it holds NONE
of the method's arithmetic: no ownership, no signed volumes / fold tests, no
transform, no interpolation, no objective.  It only draws inputs with the shapes,
sizes and value distributions of the paper's workloads.
"""
from .workloads import (CONFIGS, Workload, make_workload, kuhn_lattice_mesh,
                        fos_plan, partial_request, random_tiny_mesh)

__all__ = ["CONFIGS", "Workload", "make_workload", "kuhn_lattice_mesh",
           "fos_plan", "partial_request", "random_tiny_mesh"]
