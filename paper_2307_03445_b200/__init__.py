"""B200-native clump-DEM hot path (arXiv 2307.03445): CUDA library + thin ctypes binding.

The product is `libdem_b200.so` (hand-written sm_100a CUDA behind the C-ABI in
include/dem.h); `binding` marshals arguments and provides PyTorch's allocator and stream.
"""
from .binding import (DEM_STATUS, EXPORTS, LIB_PATH, STAGES, TRANSPORT_LOOPBACK, TRANSPORT_LOOPBACK_PEER,  # noqa: F401
                      TRANSPORT_NCCL, TRANSPORT_PEER,
                      DemError, System, halo_width, load_library, migrate_group, migration_plan, nccl_unique_id,
                      partition_plan, set_state_local_group, slab_bounds, step_group, system_from_scene)
