"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds ONLY input generation: mesh topology and coordinates, the
seeded jitter, the box partition into subdomains, the per-cell viscosity field
and the parameters of the analytic problem data.  It contains none of the
method's arithmetic (no VEM projector, no quadrature, no BDDC step); both
`oracle/` and `paper_2304_09770_b200/` import it, and neither imports the other.
"""
from .mesh import PolyMesh, hex_mesh, box_partition, cvt_mesh, centroid_partition
from .configs import CONFIGS, make_problem, make_cvt_problem, make_octa_problem, poly_problem, Problem

__all__ = ["PolyMesh", "hex_mesh", "box_partition", "cvt_mesh", "centroid_partition", "CONFIGS", "make_problem",
           "make_cvt_problem", "make_octa_problem", "poly_problem", "Problem"]
