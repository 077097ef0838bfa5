"""paper_1611_06565_b200 -- B200-native N-D Winograd convolution layer.

Budden et al., "Deep Tensor Convolution on Multicores" (arXiv 1611.06565):
one N-dimensional ConvNet layer computed by the fast algorithm F(m^N, r^N)
(Eq. (4)-(5)), with exact-rational Toom-Cook synthesis on the host
and hand-written sm_100a kernels behind the C ABI of include/wino.h.

    from paper_1611_06565_b200 import Plan
    plan = Plan(N=3, dims=(8, 28, 28), m=4, r=3, C=256, K=256, batch=32, padding=(1, 1, 1))
    plan.filter_transform(g)          # g: cuda fp32 [K][C][3][3][3]
    y = plan.forward(x)               # x: cuda fp32 [B][C][8][28][28]
"""
from .net import Net
from .wino import (Plan, WinoError, wino_filter_buffer, wino_filter_mark_ready, wino_filter_transform,
                   wino_forward, wino_forward_ex, wino_forward_host, wino_get_transforms, wino_last_error, wino_plan_create,
                   wino_plan_create_ex, wino_plan_create_nd, wino_plan_destroy, wino_plan_info, wino_plan_out_dims,
                   wino_plan_sizes, wino_profile_enable, wino_profile_read, wino_synthesize, wino_version,
                   wino_workspace, WINO_GEMM_AUTO, WINO_GEMM_FFMA, WINO_GEMM_1XTF32, WINO_GEMM_3XTF32,
                   WINO_ACT_NONE, WINO_ACT_RELU)

__all__ = ["Plan", "Net", "WinoError", "wino_plan_create", "wino_plan_create_ex", "wino_plan_create_nd", "wino_plan_destroy",
           "wino_filter_transform", "wino_forward", "wino_forward_ex", "wino_forward_host", "wino_plan_out_dims",
           "wino_plan_sizes", "wino_plan_info", "wino_filter_buffer", "wino_filter_mark_ready",
           "wino_workspace", "wino_profile_enable", "wino_profile_read", "wino_synthesize",
           "wino_get_transforms", "wino_last_error", "wino_version", "WINO_GEMM_AUTO", "WINO_GEMM_FFMA",
           "WINO_GEMM_1XTF32", "WINO_GEMM_3XTF32"]
