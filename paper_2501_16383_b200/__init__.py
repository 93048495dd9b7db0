"""B200-native RotateKV KV-cache hot path (arxiv 2501.16383).

The product is the sm_100a C-ABI library built from csrc/ into
_lib/librotatekv_b200.so (include/rotatekv/rotatekv.h); rotatekv.py is the
Python host layer mirroring the reference's C++ API.
"""
from .rotatekv import (  # noqa: F401
    ROWS_F16,
    ROWS_F32,
    SCALE_E4M3_CEIL,
    SCALE_FP16_CEIL,
    STAT_MEAN_ABS,
    STAT_SUM,
    WIRE_FP16_SCALE,
    WIRE_REFERENCE,
    LayerConfig,
    RotateKVLayer,
    apply_reorder,
    calibrate_reorder,
    calibrate_reorder_device,
    detect_massive_activations,
    detect_massive_activations_device,
    layer_plan_build,
    lib,
    rotate_keys,
    set_debug_option, decode_plan_info,
)
