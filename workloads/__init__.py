"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic: it only builds the
triangle meshes of the five BASELINE.json cube-array configurations, the RWG
edge table (mesh topology), and the seeded N(0,1) complex vectors.  Both
`oracle/` and `paper_1712_02443_b200/` consume what it returns; neither
imports the other.  Conventions follow SURVEY.md §8(c)-D13.
"""
from .meshes import cube_surface, cube_array, rwg_edges_from_triangles, Mesh  # noqa: F401
from .configs import CONFIGS, get_config, make_mesh, make_vectors  # noqa: F401
