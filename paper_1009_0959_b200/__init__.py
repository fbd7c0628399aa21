"""B200-native minimax order-statistics vector filtering (arXiv 1009.0959).

Public API (all calls run CUDA kernels of libvf.so; no CPU fallback):
    filter, fidelity, vf_filter, vf_filter_batch, vf_filter_batch_algo,
    vf_filter_rows, vf_filter_host, vf_host_workspace_bytes, vf_image_stats, vf_image_stats_multi,
    vf_plan_create / Plan (CUDA-graph executor), vf_status_string, vf_last_error, vf_version
Multi-GPU partitioner: paper_1009_0959_b200.parallel
"""
from .vf import (ALGOS, CRITERIA, VARIANTS, Plan, VFError, fidelity, filter, load_library, vf_filter,  # noqa: F401
                 vf_filter_batch, vf_filter_batch_algo, vf_filter_host, vf_filter_rows, vf_host_workspace_bytes,
                 vf_image_stats, vf_image_stats_multi, vf_kernel_info, vf_last_error, vf_plan_create, vf_status_string, vf_version)

__version__ = "0.2.0"
