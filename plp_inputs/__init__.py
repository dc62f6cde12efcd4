"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no F_p, gradient, Hessian, k-means, RCut):
only graph construction and random draws, so that the oracle (`oracle/`) and the CUDA path
(`paper_2605_26975_b200/`) can be fed identical inputs without sharing any code.
Recipes follow BASELINE.json `configs` and the conventions in SURVEY.md §8(d); every reading
is listed in DESIGN.md §3.
"""
from .graphs import (  # noqa: F401
    Graph, CONFIGS, make_config, knn_graph, csr_from_undirected, grid3d_longrange, delaunay_graph,
    blobs_2d, two_moons, gmm, uniform_square, path_graph, cycle_graph, single_edge,
    four_cycle, two_triangles, random_graph, draw_U, draw_eta, draw_uniforms, streams,
    validate_graph, permute_graph,
)
