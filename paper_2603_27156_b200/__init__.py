"""B200-native GSR-GNN training step (arxiv 2603.27156).

The package is the host mirror of the reference's operator interface for the
one hot path this build accelerates: the GSR-GNN training step
(grouped reversible residual blocks, CSR neighbour aggregation, group-wise
top-k sparse operator, fused transform GEMM), run by hand-written sm_100a
kernels behind the C-ABI in include/gsr_cuda.h.

    from paper_2603_27156_b200 import Context, synth
    g, data = synth.generate_synthetic(synth.config_graph("c1"))
    ctx = Context(0)
    ctx.graph_upload(g.row_ptr, g.col_idx, norm=NORM_ROW_MEAN)
    ctx.model_init(MODE_GSRC, layers=8, hidden=64, groups=2, k=8, d_in=8)
    ...
"""
from ._capi import (  # noqa: F401
    EPI_ADD, EPI_NONE, EPI_SCATTER_ADD, EPI_SCATTER_SUB, EPI_SUB, GEMM_FP32, GEMM_TF32, MODE_ALG12, MODE_GSRC, MODE_REV,
    NORM_NONE, NORM_ROW_MEAN, NORM_SYM_DEGREE, ConfigError, Context, GsrError, ResourceError, SequencingError, version,
)
from . import synth  # noqa: F401
from .model import init_params, param_layout  # noqa: F401
