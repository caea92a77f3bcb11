"""B200-native (sm_100a) H0 persistent-homology barcode pipeline — drop-in for the
reference ph0 library's hot path (pairwise_distances -> build_filtration ->
build_boundary_matrix -> reduce -> extract_barcode).  See include/ph0b.h and DESIGN.md."""
from .ph0b import (  # noqa: F401
    Barcode, Context, InvalidArgument, PinnedArray, Ph0bError, build_filtration, claimed_lows, reduced_supports,
    config_cloud, generate_cloud, h0_barcode, kruskal_barcode, last_launch_count, lib,
    pairwise_distances,
    CONFIGS,
)
