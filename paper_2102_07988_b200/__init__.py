"""B200-native TeraPipe hot path (arXiv 2102.07988): token-sliced pipelined GPT fwd+bwd.

The product is libtp.so (include/tp.h, built from csrc/ for sm_100a); this package is its thin
ctypes binding. Importing it without the built library raises ImportError — no CPU fallback.
"""
from ._tp import (  # noqa: F401
    Context, Slicing, BatchPlan, TpError, plan, plan_joint, schedule_oplist, stage_layers, TP_PARTITION_UNIFORM, TP_PARTITION_BALANCED, stage_param_count, nccl_unique_id, lib, EXPORTED, KEXPORTED, LIB_PATH, k_gemm, k_attention_fwd, k_attention_bwd, k_layernorm_fwd, k_layernorm_bwd,
    TP_BF16, TP_FP32, TP_FLAG_KEEP_LOGITS, TP_FLAG_KERNEL_STATS, TP_FLAG_FORCE_SIMT, TP_FLAG_NCCL_LOOPBACK, TP_FLAG_DEVICE_P2P, TP_FLAG_SCHEDULE_1F1B,
    TP_OK, TP_EINVAL, TP_EINFEASIBLE, TP_ECUDA, TP_ESTATE,
)
