"""paper_2008_07799_b200: B200-native DRGraph layout path (arxiv 2008.07799).

Drop-in for the reference package ``drgraph`` on its hot path: the same public
names, signatures, result types and exceptions, computed by hand-written sm_100a
kernels in ``libdrgraph_b200.so`` (C ABI: include/drgraph_b200.h) -- no CPU path.
"""

from .graph import (DeviceGraph, DeviceNeighborDistances, Graph, NeighborDistances, ParseError,
                    all_k_neighborhoods, bfs_k_neighborhood, connected_components,
                    device_from_edges,
                    device_k_neighborhoods, from_edges, parse_edge_list, parse_matrix_market,
                    read_graph)
from .multilevel import (DeviceHierarchy, Hierarchy, build_hierarchy, coarsen_once,
                         coarsen_with_order, compose_maps, device_build_hierarchy, prolong)
from .output import SvgStyle, format_edge_list, read_coords, write_coords, write_svg
from .optimizer import (AliasTable, Layout, LayoutPlan, OptimizerParams, PositiveSampler,
                        Samplers, attractive_gradient, build_alias_table,
                        build_negative_sampler, build_positive_sampler, build_samplers,
                        layout_device, layout_graph, prepare_layout, repulsive_gradient,
                        sgd_epoch)
from .quality import neighborhood_preservation
from .similarity import (DeviceSimilarity, SimilarityParams, SparseSimilarity,
                         build_sparse_similarity, conditional_similarity_row, device_similarity,
                         precompute_gaussian_table, search_sigma)

__version__ = "0.1.0"

__all__ = [
    "Graph", "NeighborDistances", "ParseError", "from_edges", "parse_edge_list",
    "parse_matrix_market", "read_graph", "format_edge_list", "write_coords", "read_coords",
    "write_svg", "SvgStyle", "all_k_neighborhoods", "bfs_k_neighborhood",
    "connected_components", "SimilarityParams", "SparseSimilarity", "build_sparse_similarity",
    "conditional_similarity_row", "search_sigma", "precompute_gaussian_table",
    "Hierarchy", "coarsen_once", "coarsen_with_order", "build_hierarchy", "compose_maps",
    "prolong", "OptimizerParams", "Layout", "AliasTable", "build_alias_table",
    "build_negative_sampler", "build_positive_sampler", "PositiveSampler",
    "attractive_gradient", "repulsive_gradient",
    "build_samplers", "Samplers", "sgd_epoch", "layout_graph",
    # metrics.py:114-145 (the one metric on the path: the parity instrument)
    "neighborhood_preservation",
    # device-resident API
    "DeviceGraph", "DeviceNeighborDistances", "DeviceSimilarity", "DeviceHierarchy",
    "LayoutPlan", "device_from_edges", "device_k_neighborhoods", "device_similarity",
    "device_build_hierarchy", "prepare_layout", "layout_device",
    "__version__",
]
