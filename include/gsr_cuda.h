/*
 * gsr_cuda.h — C-ABI of the B200-native GSR-GNN training step.
 *
 * The reference (arxiv 2603.27156, /root/reference) is a C++20 in-process
 * API (namespace gsr, typed exceptions, proj/include/gsr/common.hpp) whose
 * numeric operations are specified in SPEC.md; it ships no FFI. This header is
 * the thin C boundary a host binding (C++ wrapper include/gsr/cuda_api.hpp,
 * Python ctypes paper_2603_27156_b200/_capi.py, or any cgo/JNI stub — see
 * INTEGRATION.md) calls to run that path on a B200. Plain pointers and sizes
 * only; every function returns a gsrc_status and never throws.
 *
 * Each entry point names the reference interface it replaces (SPEC.md:line).
 * Host arrays are borrowed for the call and copied; nothing is retained.
 * Activations are exchanged as row-major n × D (SPEC DenseMatrix);
 * SparseActivation values / indices as row-major n × k.
 */
#ifndef GSR_CUDA_H
#define GSR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes map 1:1 onto proj/include/gsr/common.hpp:13-35. */
typedef enum {
    GSRC_OK = 0,
    GSRC_ERR_CONFIG = 1,     /* ConfigError / ShapeError / FormatError (CLI exit 1)   */
    GSRC_ERR_INTERNAL = 2,   /* unexpected CUDA error                                   */
    GSRC_ERR_RESOURCE = 3,   /* ResourceError: allocation / NCCL / device (CLI exit 3) */
    GSRC_ERR_SEQUENCING = 4  /* SequencingError: backward without forward, etc.        */
} gsrc_status;

typedef enum { GSRC_NORM_NONE = 0, GSRC_NORM_ROW_MEAN = 1, GSRC_NORM_SYM_DEGREE = 2 } gsrc_norm;
typedef enum { GSRC_MODE_ALG12 = 0, GSRC_MODE_GSRC = 1, GSRC_MODE_REV = 2 } gsrc_mode;
typedef enum { GSRC_GEMM_FP32 = 0, GSRC_GEMM_TF32 = 1 } gsrc_gemm;
typedef enum {
    GSRC_EPI_NONE = 0, GSRC_EPI_ADD = 1, GSRC_EPI_SUB = 2, GSRC_EPI_SCATTER_ADD = 3, GSRC_EPI_SCATTER_SUB = 4
} gsrc_epilogue;

typedef struct gsrc_ctx gsrc_ctx;

/* RunConfig subset for the network (GsrNet :380-383; RevNet :310-313). */
typedef struct {
    int mode;          /* gsrc_mode: ALG12 = Alg. 1/2 (C = 2), GSRC = Eq. 6-7 with GS blocks, REV = dense baseline */
    int layers;        /* L */
    int hidden;        /* D */
    int groups;        /* C (ALG12 forces 2) */
    int k;             /* GS top-k per group (ignored by REV) */
    int d_in;          /* encoder input width */
    int use_weight;    /* BlockParams flags */
    int use_bias;
    int index_source;  /* Alg. 2 backward-block indices: 0 = Alg.-2-local, 1 = forward cache */
    int gemm;          /* gsrc_gemm */
} gsrc_model_cfg;

/* optimizer_step. */
typedef struct {
    int optimizer;     /* 0 = Adam (bias-corrected), 1 = SGD (+momentum) */
    float lr, beta1, beta2, eps, weight_decay, momentum;
} gsrc_optim_cfg;

/* MemoryReport for the device arena. */
typedef struct {
    uint64_t reserved_bytes, active_bytes, peak_reserved_bytes, peak_active_bytes;
    uint64_t alloc_count, reuse_count, release_count;
    double utilization;  /* peak_active / peak_reserved; 1.0 for an empty arena */
} gsrc_mem_report;

/* Phase timing (TimingBreakdown SPEC.md:525-532), CUDA-event based, seconds. */
typedef struct { double t_forward, t_backward, t_copy, t_optimizer, t_total; } gsrc_timing;

/* ---- lifecycle ----------------------------------------------------------- */
int gsrc_create(int device, gsrc_ctx** out);
void gsrc_destroy(gsrc_ctx* ctx);
const char* gsrc_last_error(gsrc_ctx* ctx);
/* Bind the context to a caller's cudaStream_t. NULL selects the context-owned
   non-blocking stream (the default) — NOT the legacy default stream: a caller
   that must order its own work with the context's uses gsrc_get_stream. */
int gsrc_set_stream(gsrc_ctx* ctx, void* cuda_stream);
int gsrc_get_stream(gsrc_ctx* ctx, void** cuda_stream_out);  /* the stream every call enqueues on */
int gsrc_synchronize(gsrc_ctx* ctx);
int gsrc_version(char* buf, size_t len);                    /* kArtifactVersion common.hpp:9 */

/* ---- graph-store (CsrGraph SPEC.md:142-148, cached transpose :211) -------- */
int gsrc_graph_upload(gsrc_ctx* ctx, int64_t n, int64_t e, const int64_t* row_ptr, const int32_t* col_idx, int norm);

/* ---- model / params / data --------------------------------------------------- */
int gsrc_model_init(gsrc_ctx* ctx, const gsrc_model_cfg* cfg);
int gsrc_num_params(gsrc_ctx* ctx, int64_t* out);
/* Flat parameter order (GSRP block order): encoder W (d_in×D), b (D);
   for each layer, for each block: W (w×w), b (w); head w (D), b (1). */
int gsrc_params_set(gsrc_ctx* ctx, const float* host, int64_t n);
int gsrc_params_get(gsrc_ctx* ctx, float* host, int64_t n);
int gsrc_grads_get(gsrc_ctx* ctx, float* host, int64_t n);
int gsrc_zero_grads(gsrc_ctx* ctx);
int gsrc_grads_device(gsrc_ctx* ctx, float** dptr, int64_t* n);   /* for an external (NCCL) all-reduce */
int gsrc_params_device(gsrc_ctx* ctx, float** dptr, int64_t* n);
int gsrc_data_upload(gsrc_ctx* ctx, const float* x0, const float* y, const uint8_t* train_mask);  /* NodeData SPEC.md:149-152 */

/* ---- training step (cmd_train epoch body SPEC.md:597-605) ------------------- */
int gsrc_forward(gsrc_ctx* ctx, float* yhat_out);                          /* net_forward SPEC.md:404-412 */
int gsrc_forward_backward(gsrc_ctx* ctx, double* loss_out);               /* + mse_loss :422-430 + net_backward :413-421 */
int gsrc_optimizer_step(gsrc_ctx* ctx, const gsrc_optim_cfg* opt);        /* optimizer_step :626-630 */
int gsrc_train_step(gsrc_ctx* ctx, const gsrc_optim_cfg* opt, double* loss_out);
int gsrc_activation_get(gsrc_ctx* ctx, float* host_nD);                   /* current X (row-major n×D) */
int gsrc_activation_set(gsrc_ctx* ctx, const float* host_nD);
int gsrc_gradient_get(gsrc_ctx* ctx, float* host_nD);                     /* current dL/dX (row-major n×D) */
int gsrc_gradient_set(gsrc_ctx* ctx, const float* host_nD);
int gsrc_set_graph_capture(gsrc_ctx* ctx, int enable);                    /* capture the step in a CUDA graph */
int gsrc_last_timing(gsrc_ctx* ctx, gsrc_timing* out);
int gsrc_mem_stats(gsrc_ctx* ctx, gsrc_mem_report* out);                  /* Arena::stats SPEC.md:486-490 */
int gsrc_high_water_reset(gsrc_ctx* ctx);
int gsrc_kernel_launches(gsrc_ctx* ctx, int64_t* out);                    /* kernels enqueued since create */
/* WorkCounter: scalar multiply-adds and rows touched of the
   SPEC operations executed since create / the last reset, with the oracle's
   accounting — gsr_forward_block e·k + n·w² with W (also each
   block of gsrc_layer_forward / gsrc_layer_inverse and of the steps),
   gsr_backward_block e·k + n·w² + e·w with W (Alg. 2 layers), spmm e·cols and
   spmm_sparse e·k (+ n rows). Counted per call, so CUDA graph
   replays count; the rev-baseline's dense blocks and the grouped-reversible
   exact-chain-rule backward have no SPEC work formula and add 0. */
int gsrc_work_counter(gsrc_ctx* ctx, uint64_t* scalar_mul_adds, uint64_t* rows_touched);
int gsrc_work_reset(gsrc_ctx* ctx);
/* Live per-kernel timing for the roofline report. out must hold 16 + 3·C
   doubles: out[0..15] = 4 kernel classes × {ms per launch (mean over the C
   blocks), algorithmic bytes per launch, launches per step, flops per launch},
   then out[16 + c·C + i] = ms per launch of block i for classes c = 0..2.
   The activation arena is snapshotted and restored: no device state changes. */
int gsrc_profile_kernels(gsrc_ctx* ctx, int reps, double* out);

/* Exactly invertible residual stream (GSRC / REV modes; default shift 20). Each
   block output h is rounded to the grid 2^-shift before the Eq. 6 add
   (y = x + q(h)) and the Eq. 7 subtract, and the encoder output is put on the
   same grid, so every residual add is exact for |x| < 2^(24-shift) and the
   backward's inverse recompute reproduces each layer input
   bit for bit at any depth: no reconstruction drift, no GS-mask flips. The
   gradient treats q as the identity. shift 0 = plain fp32 adds (drifting). */
int gsrc_set_residual_quant(gsrc_ctx* ctx, int shift);
int gsrc_get_residual_quant(gsrc_ctx* ctx, int* shift);

/* Optimizer state for exact resume (the GSRP checkpoint holds parameters
   only): Adam first/second moments and the step count. */
int gsrc_optim_state_get(gsrc_ctx* ctx, float* m, float* v, int64_t* step, int64_t n);
int gsrc_optim_state_set(gsrc_ctx* ctx, const float* m, const float* v, int64_t step, int64_t n);

/* ---- data parallelism (one process or thread per GPU) ----------
   Each rank trains on its own subgraph; gsrc_train_step then averages the flat
   gradient buffer over the ranks with one NCCL all-reduce on the context stream,
   between backward and optimizer. NCCL is loaded at run time (libnccl.so.2);
   without it these return GSRC_ERR_RESOURCE. */
int gsrc_comm_unique_id(void* out, size_t len);                         /* rank 0: len ≥ 128 (ncclUniqueId) */
int gsrc_comm_init(gsrc_ctx* ctx, const void* unique_id, int nranks, int rank);
int gsrc_comm_allreduce_grads(gsrc_ctx* ctx);                           /* for the split forward_backward / optimizer_step path */
int gsrc_comm_destroy(gsrc_ctx* ctx);

/* ---- reconstruction diagnostics (GSRC) ------------------------------------------
   With diagnostics on, the forward stores the GS mask (index bytes) of every
   row_stride-th row for each (layer, block), and the backward counts the sampled
   rows whose mask recomputed from the reconstructed activations differs.
   flips must hold layers × groups counts (layer-major). */
int gsrc_diag_masks(gsrc_ctx* ctx, int enable, int row_stride);
int gsrc_diag_mask_flips(gsrc_ctx* ctx, int64_t* flips, int64_t* sampled_rows);

/* ---- layer-level entry points (device activation = gsrc_activation_*) ----- */
int gsrc_layer_forward(gsrc_ctx* ctx, int layer);    /* gsr_forward_layer SPEC.md:386 / rev_forward_layer :316 */
int gsrc_layer_inverse(gsrc_ctx* ctx, int layer);    /* rev_inverse_layer SPEC.md:325 (GSRC / REV) */
int gsrc_layer_backward(gsrc_ctx* ctx, int layer);   /* gsr_backward_layer SPEC.md:395 / rev_backward :334 */

/* ---- op-level parity entry points (host pointers; graph = uploaded graph) -- */
int gsrc_set_op_precision(gsrc_ctx* ctx, int gemm);   /* transform precision of the gsrc_op_* blocks (gsrc_gemm) */
int gsrc_op_gs_topk(gsrc_ctx* ctx, int64_t n, int w, int k, const float* x, float* vals, int32_t* idx);
int gsrc_op_spmm(gsrc_ctx* ctx, int transpose, int cols, const float* x, float* y);
int gsrc_op_spmm_sparse(gsrc_ctx* ctx, int transpose, int w, int k, const float* vals, const int32_t* idx, float* y);
int gsrc_op_block_forward(gsrc_ctx* ctx, int w, int k, const float* vals, const int32_t* idx, const float* W, const float* b,
                          int use_weight, int use_bias, int epilogue, const float* R, const float* rvals, const int32_t* ridx,
                          float* out, int gs_k, float* gs_vals, int32_t* gs_idx);
int gsrc_op_dense_block(gsrc_ctx* ctx, int w, const float* x, const float* W, const float* b, int use_weight, int use_bias,
                        float* out);
int gsrc_op_block_backward(gsrc_ctx* ctx, int w, int k, const float* m, const int32_t* isrc, const float* fvals,
                           const int32_t* fidx, const float* W, int use_weight, int use_bias, float* out, float* dW,
                           float* db);

#ifdef __cplusplus
}
#endif

#endif /* GSR_CUDA_H */
