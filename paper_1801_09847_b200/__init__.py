"""B200-native point-to-plane ICP (the hot path of arXiv 1801.09847's
registration workflow) behind the C ABI of include/o3g.h."""
from .o3g import (Context, O3GError, InvalidArgument, RegistrationResult,  # noqa: F401
                  icp_point_to_plane, icp_point_to_point, nccl_unique_id, loopback_run, loopback_peer_connect, lib, LIB_PATH,
                  FLAG_DEGENERATE, FLAG_NO_CORRESPONDENCES, NTERMS,
                  OPT_SEARCH, OPT_GRID, OPT_TIMING, OPT_BLOCKS_PER_SM, OPT_NBR_MASK, OPT_COOP_MIN,
                  OPT_ESTIMATION, OPT_SOURCE_ORDER, OPT_TARGET_SORT, OPT_PRUNE_MIN, OPT_INTERLEAVE,
                  OPT_XSORT, OPT_CERT, OPT_TRACE_PASS, OPT_CERT_SWEEP)
