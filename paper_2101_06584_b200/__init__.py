"""B200-native DD/TD/QD GEMM (arXiv 2101.06584's hot path, re-designed for
sm_100a).  The compute lives in libmpfk.so (csrc/); this package is the
Python mirror of the reference's mpfkit::linalg API over its C ABI."""
from .linalg import (  # noqa: F401
    EwOp,
    KernelVariant,
    MPMatrix,
    OpCounts,
    binop_batch,
    bits_equal,
    device_count,
    ew_add,
    ew_add_merge,
    ew_apply_into,
    ew_device,
    ew_mul,
    fill_baseline,
    format_eps,
    fp64_peak,
    gemm_device,
    gemm_device_acc,
    last_stats,
    load_matrix_binary,
    mpfm_info,
    mpfm_load_device,
    mpfm_save_device,
    save_matrix_binary,
    matmul_block,
    matmul_block_into,
    matmul_block_parallel,
    matmul_block_parallel_into,
    matmul_naive,
    matmul_naive_into,
    op_counters_read,
    op_counters_reset,
    pad_columns,
)

OPS_PER_MAC = {2: 20, 3: 132, 4: 218}  # reference sequence, renorm5 path A
