"""B200-native MulMent hot path (arXiv 1506.04383): C-ABI library
libmm_b200.so (include/mm.h) with hand-written sm_100a CUDA kernels, and this
thin ctypes binding.  See DESIGN.md."""
from .mulment import (DeviceGraph, DeviceSSet, Hierarchy, MMError, build_hierarchy, coords_from_device,  # noqa: F401
                      coords_layout, coords_to_device, energy, exact_kernel_variant, full_stress, graph_to_device, launch_count, layout, layout_schedule, load,
                      paper_schedule, prolong, sweeps,
                      profile_enable, profile_last, profile_read, profile_reset, sset_to_device, sweep, sweep_workspace, validate_sset, EXPORTS,
                      LIB_PATH)
