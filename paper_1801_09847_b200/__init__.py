"""B200-native point-to-plane ICP (the hot path of arXiv 1801.09847's
registration workflow) behind the C ABI of include/o3g.h."""
from .o3g import (Context, O3GError, InvalidArgument, RegistrationResult,  # noqa: F401
                  icp_point_to_plane, icp_point_to_point, nccl_unique_id, lib, LIB_PATH,
                  FLAG_DEGENERATE, FLAG_NO_CORRESPONDENCES, NTERMS)
