// C-ABI implementation (include/gsr_cuda.h): context, device arena, graph /
// model / data upload, and the host-side orchestration of the GSR-GNN
// training step on one stream (optionally replayed from a CUDA graph).
//
// Layer orchestration follows the reference spec:
//   GSRC  — Eq. 6-7 grouped reversible layer (PAPER.md:275-276,
//           SPEC.md:316-342) with GS-sparse blocks f_i(u) = Â·scatter(GS_k(u))·W_i
//           + b_i (gsr_forward_block SPEC.md:253-256): forward keeps only the
//           final activation; backward reconstructs each layer input by
//           inverse recomputation and back-propagates the exact gradient.
//   ALG12 — Algorithms 1-2 verbatim
//           with the per-layer index/value caches the paper keeps (O(LNk)).
//   REV   — rev-baseline dense blocks.
// Every kernel launch goes through launch_tile / launch_gs / the small
// kernels in kernels.cu; there is no host or CPU fallback for any of them.
#include "../../include/gsr_cuda.h"
#include "kernels.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

using namespace gsrk;

namespace {

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, int line) {
    const int code = (e == cudaErrorMemoryAllocation) ? GSRC_ERR_RESOURCE : GSRC_ERR_INTERNAL;
    throw Fail(code, std::string("CUDA error '") + cudaGetErrorString(e) + "' at capi.cu:" + std::to_string(line) + " (" + what + ")");
}
#define CK(x)                                                 \
    do {                                                      \
        cudaError_t e_ = (x);                                 \
        if (e_ != cudaSuccess) throw_cuda(e_, #x, __LINE__);  \
    } while (0)

[[noreturn]] void cfg_err(const std::string& m) { throw Fail(GSRC_ERR_CONFIG, m); }
[[noreturn]] void seq_err(const std::string& m) { throw Fail(GSRC_ERR_SEQUENCING, m); }

// Single contiguous device arena (SPEC mem-arena; north_star
// "one contiguous activation arena"). Buffers are carved at plan time; the
// steady-state step performs zero allocations.
struct Arena {
    char* base = nullptr;
    size_t reserved = 0, used = 0, peak_active = 0, peak_reserved = 0;
    uint64_t alloc_count = 0, reuse_count = 0, release_count = 0;
    int leases = 0;

    void plan(size_t bytes) {
        release_all();
        if (bytes > reserved) {
            if (base) { cudaFree(base); base = nullptr; reserved = 0; }
            cudaError_t e = cudaMalloc(&base, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw Fail(GSRC_ERR_RESOURCE, "arena: cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e) +
                                                  " [reserved=" + std::to_string(reserved) + " active=" + std::to_string(used) + "]");
            }
            reserved = bytes;
            ++alloc_count;
        } else {
            ++reuse_count;
        }
        peak_reserved = std::max(peak_reserved, reserved);
    }
    template <typename T>
    T* lease(size_t count) {
        const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
        if (used + bytes > reserved) throw Fail(GSRC_ERR_RESOURCE, "arena exhausted");
        T* p = reinterpret_cast<T*>(base + used);
        used += bytes;
        ++leases;
        peak_active = std::max(peak_active, used);
        return p;
    }
    void release_all() {
        release_count += leases;
        leases = 0;
        used = 0;
    }
    ~Arena() { if (base) cudaFree(base); }
};

size_t bytes_rounded(size_t b) { return (b + 255) & ~size_t(255); }

struct DevBuf {  // scratch for op-level parity entry points
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        CK(cudaMalloc(&p, bytes ? bytes : 16));
        CK(cudaMemset(p, 0, bytes ? bytes : 16));
        CK(cudaDeviceSynchronize());
    }
    ~DevBuf() { if (p) cudaFree(p); }
    template <typename T> T* as() { return static_cast<T*>(p); }
};

// NCCL, resolved at run time (dlopen) so the library loads on hosts without
// it; inside a torch process the already-loaded libnccl.so.2 is reused. Only
// the data-parallel entry points (gsrc_comm_*) need it (one
// gradient all-reduce per step).
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
    bool ok() const { return get_unique_id && comm_init_rank && all_reduce && comm_destroy && error_string; }
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { a.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return a; }
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!a.ok()) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}
const NcclApi& nccl_or_throw() {
    const NcclApi& a = nccl_api();
    if (!a.ok()) throw Fail(GSRC_ERR_RESOURCE, "NCCL unavailable: " + a.why);
    return a;
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Fail(GSRC_ERR_RESOURCE, std::string(what) + ": " + nccl_api().error_string(r));
}

}  // namespace

struct gsrc_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own = nullptr;
    std::string err;
    int64_t launches = 0;
    // WorkCounter: the scalar multiply-adds and rows touched of
    // the SPEC operations executed, counted per call of an entry point (CUDA
    // graph replays included), with the oracle's accounting (oracle/
    // gsr_oracle.hpp): gsr_forward_block e·k + n·w² with W,
    // gsr_backward_block e·k + (n·w² + e·w with W), spmm e·cols and
    // spmm_sparse e·k (+ n rows each). The rev-baseline's
    // dense blocks and the exact-chain-rule backward of the grouped-reversible
    // modes are composite operations without a SPEC work formula: not counted.
    uint64_t work_ma = 0, work_rows = 0;

    // persistent: graph
    int64_t n = 0, e = 0;
    int norm = 0;
    int *rp = nullptr, *ci = nullptr, *trp = nullptr, *tci = nullptr;
    float *row_f = nullptr, *col_f = nullptr;
    int2 *ell_f = nullptr, *ell_b = nullptr;  // Dir::ell per direction
    int nhub_f = 0, nhub_b = 0;  // rows with > kSeg edges (fwd CSR / transpose), fast path
    // their kSeg-edge segments (edge ranges) and each hub row's segment range
    int4* item_f = nullptr;  // sparse hub work items (launch_hub_rows)
    int* hcnt_f = nullptr;   // per hub: chunks finished (self-resetting)
    int2* seg_b = nullptr;   // dense hub segments {lo, hi} (launch_hub_dense)
    int *hub_b = nullptr, *segoff_b = nullptr;
    int2* seg_fd = nullptr;  // forward-direction dense hub segments (rev-baseline FWD / INV)
    int *hub_fd = nullptr, *segoff_fd = nullptr;
    int nseg_f = 0, nseg_b = 0, nitem_f = 0, nseg_fd = 0;
    size_t graph_bytes = 0;

    // persistent: model state
    bool model = false;
    gsrc_model_cfg cfg{};
    int C = 0, nb = 0, w = 0, ld = 0, k = 0;
    int64_t P = 0;
    float *params = nullptr, *grads = nullptr, *opt_m = nullptr, *opt_v = nullptr, *bc = nullptr;
    long long* d_step = nullptr;
    size_t model_bytes = 0;

    // persistent: node data
    float *X0 = nullptr, *y = nullptr;
    uint8_t* mask = nullptr;
    float cnt = 0.f, captured_cnt = -1.f;
    int64_t data_n = 0;
    bool data = false;
    size_t data_bytes = 0;

    // activation arena
    Arena arena;
    float *X = nullptr, *G = nullptr, *M1 = nullptr, *M2 = nullptr, *U = nullptr, *Zh = nullptr;
    float* Zh2 = nullptr;     // dense (transpose) hub-row aggregates: BIN's, built on the side stream
    float* Pseg2 = nullptr;   // their segment partials
    std::vector<CUtensorMap> xmaps, gmaps;  // TMA maps of the X and G planes (fast path)
    uint8_t *recA = nullptr, *recB = nullptr, *t1 = nullptr, *t2 = nullptr, *vg = nullptr;
    std::vector<uint8_t*> rblk;  // fast backward sweep: records of block i's input (rblk[0] = recA, rblk[1] = recB)
    std::vector<uint8_t*> c1, c2;
    std::vector<char> filled;
    double* part = nullptr;
    int nparts = 0, nparts_small = 0;
    float *yhat = nullptr, *gy = nullptr;
    double *loss_part = nullptr, *loss_dev = nullptr;
    int loss_nparts = 0;
    double* loss_host = nullptr;  // pinned

    // graph replay
    bool use_graph = false;
    // the step replays as three graphs (forward, backward, optimizer) so the
    // Eq. 9 phase events sit between graph launches
    cudaGraphExec_t g_fwd = nullptr, g_bwd = nullptr, g_opt = nullptr;
    int64_t g_fwd_launches = 0, g_bwd_launches = 0, g_opt_launches = 0;
    gsrc_optim_cfg g_step_opt{};

    cudaEvent_t ev[4] = {};
    cudaStream_t side = nullptr;                 // backward sweep: dense hub pre-pass beside the INV
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // backward sweep: the fixed-order dW partial reduction of block i runs on
    // side2 beside the next block's work; BIN partials alternate between two
    // buffers, each reused only once its reduction has finished
    cudaStream_t side2 = nullptr;
    cudaEvent_t ev_bin[2] = {}, ev_red[2] = {};
    double* part_bin[2] = {};
    bool red_pending[2] = {false, false};
    int part_sel = 0;
    cudaEvent_t tev[4] = {};  // phase marks inside the step (Eq. 9): after forward, after backward, after optimizer, after the all-reduce
    gsrc_timing timing{};

    // data parallelism: one NCCL communicator, the gradient all-reduce (average)
    // between backward and optimizer on the context stream (gsrc_comm_init)
    ncclComm_t comm = nullptr;
    int comm_ranks = 1, comm_rank = 0;

    // mask-flip diagnostic (gsrc_diag_masks): forward GS index bytes of every
    // stride-th row per (layer, block), compared with the backward's recomputed masks
    bool diag = false;
    int diag_stride = 1;
    int64_t diag_rows = 0;
    uint4* diag_store = nullptr;
    unsigned long long* diag_cnt = nullptr;

    ~gsrc_ctx() {
        for (cudaGraphExec_t g : {g_fwd, g_bwd, g_opt}) if (g) cudaGraphExecDestroy(g);
        for (void* p : {(void*)rp, (void*)ci, (void*)trp, (void*)tci, (void*)row_f, (void*)col_f, (void*)ell_f, (void*)ell_b, (void*)item_f, (void*)seg_b, (void*)hub_b, (void*)segoff_b,
                        (void*)seg_fd, (void*)hub_fd, (void*)segoff_fd,
                        (void*)hcnt_f, (void*)params, (void*)grads,
                        (void*)opt_m, (void*)opt_v, (void*)bc, (void*)d_step, (void*)X0, (void*)y, (void*)mask})
            if (p) cudaFree(p);
        if (loss_host) cudaFreeHost(loss_host);
        for (auto& e_ : ev) if (e_) cudaEventDestroy(e_);
        for (auto& e_ : tev) if (e_) cudaEventDestroy(e_);
        for (cudaEvent_t e_ : {fork_ev, join_ev, ev_bin[0], ev_bin[1], ev_red[0], ev_red[1]}) if (e_) cudaEventDestroy(e_);
        if (diag_store) cudaFree(diag_store);
        if (diag_cnt) cudaFree(diag_cnt);
        if (comm) nccl_api().comm_destroy(comm);
        if (side) cudaStreamDestroy(side);
        if (side2) cudaStreamDestroy(side2);
        if (own) cudaStreamDestroy(own);
    }

    // ---- helpers -----------------------------------------------------------
    float* plane(float* base, int p) const { return base + static_cast<size_t>(p) * n * ld; }
    int64_t off_block(int l, int i) const {
        return static_cast<int64_t>(cfg.d_in) * cfg.hidden + cfg.hidden + (static_cast<int64_t>(l) * nb + i) * (static_cast<int64_t>(w) * w + w);
    }
    const float* Wb(int l, int i) const { return params + off_block(l, i); }
    const float* Bb(int l, int i) const { return cfg.use_bias ? params + off_block(l, i) + static_cast<int64_t>(w) * w : nullptr; }
    // col_f ≡ 1 unless sym_degree; row_f ≡ 1 only for norm none
    Dir fwd() const { return Dir{rp, ci, row_f, col_f, norm != GSRC_NORM_SYM_DEGREE, ell_f}; }
    Dir bwd() const { return Dir{trp, tci, col_f, row_f, norm == GSRC_NORM_NONE, ell_b}; }

    // exactly invertible residual stream (GSRC / REV): grid 2^-qshift, 0 = off
    int qshift = 20;
    float q_scale() const { return cfg.mode != GSRC_MODE_ALG12 && qshift > 0 ? std::ldexp(1.f, qshift) : 0.f; }
    float q_inv() const { return cfg.mode != GSRC_MODE_ALG12 && qshift > 0 ? std::ldexp(1.f, -qshift) : 0.f; }
    TileArgs tile_base() const {
        TileArgs a;
        a.n = static_cast<int>(n);
        a.w = w;
        a.ld = ld;
        a.tc = cfg.gemm == GSRC_GEMM_TF32;
        a.qs = q_scale();
        a.qi = q_inv();
        return a;
    }
    int last_grid = 0;
    int op_tc = 0;  // transform precision of the op-level parity entry points
    void run_tile(const TileArgs& a) {
        CK(launch_tile(a, stream, &last_grid));
        ++launches;
    }
    // TMA map of an activation / gradient plane (fast path), nullptr otherwise
    const CUtensorMap* map_of(const float* p) const {
        for (int q = 0; q < C && q < static_cast<int>(xmaps.size()); ++q) {
            if (p == plane(X, q)) return &xmaps[static_cast<size_t>(q)];
            if (p == plane(G, q)) return &gmaps[static_cast<size_t>(q)];
        }
        return nullptr;
    }
    void launch_gs_any(GsArgs& g) {
        bool tma = fast();
        for (int i = 0; i < g.nplanes && tma; ++i) {
            const CUtensorMap* m = map_of(g.planes[i]);
            if (m) g.maps[i] = *m; else tma = false;
        }
        CK(tma ? launch_gs_tma(g, stream) : launch_gs(g, stream));
        ++launches;
    }
    void run_gs(std::initializer_list<const float*> planes, uint8_t* rec) {
        GsArgs g;
        g.n = static_cast<int>(n);
        g.w = w;
        g.ld = ld;
        g.k = k;
        int i = 0;
        for (const float* p : planes) g.planes[i++] = p;
        g.nplanes = i;
        g.rec = rec;
        launch_gs_any(g);
    }
    void run_gs_groupsum(const float* base, uint8_t* rec) {  // GS(Σ_{j≥2} x_j), planes 1..C-1
        GsArgs g;
        g.n = static_cast<int>(n);
        g.w = w;
        g.ld = ld;
        g.k = k;
        for (int p = 1; p < C; ++p) g.planes[p - 1] = plane(const_cast<float*>(base), p);
        g.nplanes = C - 1;
        g.rec = rec;
        launch_gs_any(g);
    }
    void run_sum_planes(const float* base, float* out) {
        GsArgs g;
        g.n = static_cast<int>(n);
        g.w = w;
        g.ld = ld;
        for (int p = 1; p < C; ++p) g.planes[p - 1] = plane(const_cast<float*>(base), p);
        g.nplanes = C - 1;
        CK(launch_sum_planes(g, out, stream));
        ++launches;
    }
    void reduce_block_grads(int l, int i, const double* src = nullptr, cudaStream_t s_ = nullptr) {
        const int plen = w * w + w;
        float* dst = grads + off_block(l, i);
        const double* pp = src ? src : part;
        cudaStream_t st = s_ ? s_ : stream;
        if (cfg.use_weight) CK(launch_reduce_parts(pp, last_grid, plen, plen, dst, 1, st));
        else CK(launch_reduce_parts(pp + static_cast<size_t>(w) * w, last_grid, plen, w, dst + static_cast<size_t>(w) * w, 1, st));
        ++launches;
    }
    // join side2: every pending dW reduction of the sweep is complete on `stream`
    void join_reductions() {
        for (int b = 0; b < 2; ++b)
            if (red_pending[b]) {
                CK(cudaStreamWaitEvent(stream, ev_red[b], 0));
                red_pending[b] = false;
            }
    }

    // mask-flip diagnostic: mode 0 stores the forward masks of block i of layer
    // l, mode 1 counts the sampled rows whose backward recompute differs
    void diag_rec(int l, int i, const uint8_t* rec, int mode) {
        if (!diag || cfg.mode != GSRC_MODE_GSRC) return;
        const size_t slot = static_cast<size_t>(l) * C + static_cast<size_t>(i);
        CK(launch_diag_masks(rec, static_cast<int>(n), diag_stride, rec_bytes(k), diag_store + slot * static_cast<size_t>(diag_rows), mode,
                             diag_cnt + slot, stream));
        ++launches;
    }

    // ---- thread-per-row tcgen05 fast path (fast.cu): GSR-C in TF32 mode ------
    bool no_fast = std::getenv("GSRC_NO_FAST") != nullptr;  // A/B switch: generic k_tile for every block
    bool fast() const { return !no_fast && cfg.mode == GSRC_MODE_GSRC && cfg.gemm == GSRC_GEMM_TF32 && fast_supported(w, k); }
    // rev-baseline (dense blocks) on the same tcgen05 kernels: dense aggregation of relu(u)
    bool fast_rev() const { return !no_fast && cfg.mode == GSRC_MODE_REV && cfg.gemm == GSRC_GEMM_TF32 && cfg.use_weight && w <= 64; }
    bool fastpath() const { return fast() || fast_rev(); }
    FastArgs fast_base(bool transpose) const {
        FastArgs f;
        f.n = static_cast<int>(n);
        f.w = w;
        f.ld = ld;
        f.k = k;
        f.dir = transpose ? bwd() : fwd();
        f.Zh = Zh;
        f.qs = q_scale();
        f.qi = q_inv();
        return f;
    }
    float* Pseg = nullptr;  // hub segment partials (arena)
    void run_hub(bool sparse, const FastArgs& f, bool transpose, cudaStream_t s_ = nullptr) {
        cudaStream_t st = s_ ? s_ : stream;
        const int nh = transpose ? nhub_b : nhub_f;
        if (!nh) return;
        if (sparse && !transpose) {
            CK(launch_hub_rows(f, item_f, nitem_f, hcnt_f, Pseg, st));
            ++launches;
        } else if (!sparse && transpose) {
            CK(launch_hub_dense(f, seg_b, nseg_b, hub_b, segoff_b, nhub_b, Pseg2, st));
            launches += 2;
        } else if (!sparse && !transpose) {  // rev-baseline: Â·relu(u) of the forward hub rows into f.Zh
            CK(launch_hub_dense(f, seg_fd, nseg_fd, hub_fd, segoff_fd, nhub_f, Pseg, st));
            launches += 2;
        } else {
            throw Fail(GSRC_ERR_CONFIG, "hub pre-pass: unsupported direction");
        }
    }
    void run_fast(int kind, const FastArgs& f) {
        CK(launch_fast(kind, f, stream, &last_grid));
        ++launches;
    }
    // f_i with Eq. 6 add (+ GS of the output for the next block)
    void fast_block_forward(int l, int i, const uint8_t* rec, uint8_t* gs_out) {
        FastArgs f = fast_base(false);
        f.rec_in = rec;
        run_hub(true, f, false);
        f.Wm = Wb(l, i);
        f.bias = Bb(l, i);
        f.R = plane(X, i);
        f.out = plane(X, i);
        f.tm_x = xmaps[static_cast<size_t>(i)];
        f.gs_out = gs_out;
        f.k_gs = k;
        run_fast(0, f);
    }
    // Eq. 7 inverse of block i + dW/db, then the masked input gradient
    void fast_block_backward(int l, int i, const uint8_t* rec) {
        fast_inverse(l, i, rec);
        fast_input_grad(l, i, rec);
        reduce_block_grads(l, i);  // dW = Sᵀ·(Âᵀ·G_i) partials from BIN
        if (cfg.use_bias) {        // db = colsum(G_i)
            CK(launch_colsum(plane(G, i), static_cast<int>(n), w, ld, part, &last_grid, stream));
            ++launches;
            CK(launch_reduce_parts(part, last_grid, w, w, grads + off_block(l, i) + static_cast<size_t>(w) * w, 1, stream));
            ++launches;
        }
    }
    // gs_out: GS_k of the reconstructed rows (the lower layer's records)
    void fast_inverse(int l, int i, const uint8_t* rec, uint8_t* gs_out = nullptr) {
        FastArgs f = fast_base(false);
        f.rec_in = rec;
        run_hub(true, f, false);
        f.Wm = Wb(l, i);
        f.bias = Bb(l, i);
        f.R = plane(X, i);
        f.out = plane(X, i);
        f.tm_x = xmaps[static_cast<size_t>(i)];
        f.gs_out = gs_out;
        f.k_gs = k;
        run_fast(1, f);
    }
    // GSR-C backward of layer l on the fast path. Block i ≥ 1 reads rblk[i] =
    // GS(y_{i-1}); block 0 reads rblk[0] = GS(Σ_{p≥1} x_p), computed by k_gs
    // once x_1..x_{C-1} are reconstructed. With `produce`, the INV of block
    // i ≤ C-2 also writes the GS of its reconstructed rows x_i = the lower
    // layer's y_i, i.e. rblk[i+1] of layer l-1 (free again: block i+1 of this
    // layer is done), so the sweep needs no per-block GS recompute. Without
    // `have` (the first layer of the sweep, or a single-layer call) the
    // records come from the planes.
    void fast_layer_backward(int l, bool have, bool produce) {
        if (!have)
            for (int i = 1; i < C; ++i) run_gs({plane(X, i - 1)}, rblk[static_cast<size_t>(i)]);
        for (int i = C - 1; i >= 0; --i) {
            uint8_t* rec = rblk[static_cast<size_t>(i)];
            uint8_t* own = produce && i <= C - 2 ? rblk[static_cast<size_t>(i) + 1] : nullptr;
            // the dense hub rows of block i need only G_i (final since block
            // i + 1's BIN): on the side stream, beside the sparse hub pass and INV
            const bool side_hub = nhub_b > 0;
            if (side_hub) {
                CK(cudaEventRecord(fork_ev, stream));
                CK(cudaStreamWaitEvent(side, fork_ev, 0));
                FastArgs hb = fast_base(true);
                hb.x_in = plane(G, i);
                hb.Zh = Zh2;
                run_hub(false, hb, true, side);
                CK(cudaEventRecord(join_ev, side));
            }
            if (i == 0) run_gs_groupsum(X, rec);
            diag_rec(l, i, rec, 1);
            fast_inverse(l, i, rec, own);
            if (side_hub) CK(cudaStreamWaitEvent(stream, join_ev, 0));
            // BIN into part_bin[b] once that buffer's previous reduction is done;
            // its own reduction then runs on side2 beside the next block
            const int b = part_sel;
            part_sel ^= 1;
            if (red_pending[b]) CK(cudaStreamWaitEvent(stream, ev_red[b], 0));
            fast_input_grad(l, i, rec, side_hub, part_bin[b]);
            CK(cudaEventRecord(ev_bin[b], stream));
            CK(cudaStreamWaitEvent(side2, ev_bin[b], 0));
            reduce_block_grads(l, i, part_bin[b], side2);
            CK(cudaEventRecord(ev_red[b], side2));
            red_pending[b] = true;
            if (cfg.use_bias) {
                CK(launch_colsum(plane(G, i), static_cast<int>(n), w, ld, part, &last_grid, stream));
                ++launches;
                CK(launch_reduce_parts(part, last_grid, w, w, grads + off_block(l, i) + static_cast<size_t>(w) * w, 1, stream));
                ++launches;
            }
        }
    }
    bool fast_sweep() const { return fast() && cfg.use_weight && cfg.mode == GSRC_MODE_GSRC && C >= 2; }
    // hub_done: the dense hub pre-pass into Zh2 was already enqueued (side stream)
    void fast_input_grad(int l, int i, const uint8_t* rec, bool hub_done = false, double* bin_part = nullptr) {
        FastArgs b = fast_base(true);
        b.x_in = plane(G, i);
        b.Zh = Zh2;
        if (!hub_done) run_hub(false, b, true);
        b.Wm = Wb(l, i);
        b.gemm_t = 1;
        b.mrec = rec;
        b.k_m = k;
        b.part = bin_part ? bin_part : part;
        if (i > 0) { b.dst[0] = plane(G, i - 1); b.tm_dst[0] = gmaps[static_cast<size_t>(i - 1)]; b.ndst = 1; }
        else {
            for (int p = 1; p < C; ++p) { b.dst[p - 1] = plane(G, p); b.tm_dst[p - 1] = gmaps[static_cast<size_t>(p)]; }
            b.ndst = C - 1;
        }
        run_fast(2, b);
    }
    // ---- rev-baseline on the fast path ----------------------------------------
    // f_i(u) = (Â·relu(u))·W_i + b_i with the Eq. 6 add (kind 0) or the Eq. 7
    // subtract (kind 1): the forward hub rows come from the dense hub pre-pass.
    void rev_fast_block(int l, int i, const float* u, int kind) {
        FastArgs f = fast_base(false);
        f.dense = 1;
        f.relu = 1;
        f.x_in = u;
        run_hub(false, f, false);
        f.Wm = Wb(l, i);
        f.bias = Bb(l, i);
        f.R = plane(X, i);
        f.out = plane(X, i);
        f.tm_x = xmaps[static_cast<size_t>(i)];
        run_fast(kind, f);
    }
    // du = (u > 0) ⊙ ((Âᵀ·G_i)·W_iᵀ) into G_{i-1} or every G_j, j ≥ 1; dW_i += relu(u)ᵀ·(Âᵀ·G_i)
    void rev_fast_input_grad(int l, int i, const float* u, bool hub_done) {
        FastArgs b = fast_base(true);
        b.x_in = plane(G, i);
        b.Zh = Zh2;
        if (!hub_done) run_hub(false, b, true);
        b.Wm = Wb(l, i);
        b.gemm_t = 1;
        b.mplane = u;
        b.part = part;
        if (i > 0) { b.dst[0] = plane(G, i - 1); b.tm_dst[0] = gmaps[static_cast<size_t>(i - 1)]; b.ndst = 1; }
        else {
            for (int p = 1; p < C; ++p) { b.dst[p - 1] = plane(G, p); b.tm_dst[p - 1] = gmaps[static_cast<size_t>(p)]; }
            b.ndst = C - 1;
        }
        run_fast(2, b);
    }
    // one block of the rev backward sweep: inverse, dW/db and the input gradient
    void rev_fast_block_backward(int l, int i, const float* u) {
        const bool side_hub = nhub_b > 0;  // the dense transpose hub rows of G_i beside the forward hub pass and INV
        if (side_hub) {
            CK(cudaEventRecord(fork_ev, stream));
            CK(cudaStreamWaitEvent(side, fork_ev, 0));
            FastArgs hb = fast_base(true);
            hb.x_in = plane(G, i);
            hb.Zh = Zh2;
            run_hub(false, hb, true, side);
            CK(cudaEventRecord(join_ev, side));
        }
        rev_fast_block(l, i, u, 1);
        if (side_hub) CK(cudaStreamWaitEvent(stream, join_ev, 0));
        rev_fast_input_grad(l, i, u, side_hub);
        reduce_block_grads(l, i);
        if (cfg.use_bias) {
            CK(launch_colsum(plane(G, i), static_cast<int>(n), w, ld, part, &last_grid, stream));
            ++launches;
            CK(launch_reduce_parts(part, last_grid, w, w, grads + off_block(l, i) + static_cast<size_t>(w) * w, 1, stream));
            ++launches;
        }
    }

    // ---- GSR-C / REV layers ---------------------------------------------------
    void rev_layer_forward(int l) {
        const bool sparse = cfg.mode == GSRC_MODE_GSRC;
        uint8_t* cur = recA;
        uint8_t* nxt = recB;
        if (sparse) run_gs_groupsum(X, cur);
        else run_sum_planes(X, U);
        if (fast_rev()) {
            for (int i = 0; i < C; ++i) rev_fast_block(l, i, i == 0 ? U : plane(X, i - 1), 0);
            return;
        }
        if (fast() && cfg.use_weight) {
            for (int i = 0; i < C; ++i) {
                diag_rec(l, i, cur, 0);
                fast_block_forward(l, i, cur, i + 1 < C ? nxt : nullptr);
                std::swap(cur, nxt);
            }
            return;
        }
        for (int i = 0; i < C; ++i) {
            if (sparse) diag_rec(l, i, cur, 0);
            TileArgs a = tile_base();
            a.dir = fwd();
            if (sparse) {
                a.agg = AGG_SPARSE;
                a.rec_in = cur;
                a.k_in = k;
                if (i + 1 < C) { a.gs_out = nxt; a.k_gs = k; }
            } else {
                a.agg = AGG_DENSE_RELU;
                a.x_in = (i == 0) ? U : plane(X, i - 1);
            }
            a.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE;
            a.Wm = Wb(l, i);
            a.bias = Bb(l, i);
            a.epi = EPI_ADD;
            a.R = plane(X, i);
            a.out = plane(X, i);
            run_tile(a);
            std::swap(cur, nxt);
        }
    }
    // inverse of one block: x_i = y'_i − f_i(u)
    void rev_block_inverse(int l, int i, bool with_grads) {
        const bool sparse = cfg.mode == GSRC_MODE_GSRC;
        const float* u = nullptr;
        if (sparse) {
            if (i > 0) run_gs({plane(X, i - 1)}, recA);
            else run_gs_groupsum(X, recA);
            if (with_grads) diag_rec(l, i, recA, 1);
        } else {
            if (i > 0) u = plane(X, i - 1);
            else { run_sum_planes(X, U); u = U; }
        }
        if (fast_rev()) {
            if (with_grads) rev_fast_block_backward(l, i, u);
            else rev_fast_block(l, i, u, 1);
            return;
        }
        if (fast() && cfg.use_weight) {  // the same tensor-core kernels as the forward: an exact inverse on the residual grid
            if (with_grads) fast_block_backward(l, i, recA);
            else fast_inverse(l, i, recA);
            return;
        }
        TileArgs a = tile_base();
        a.dir = fwd();
        if (sparse) { a.agg = AGG_SPARSE; a.rec_in = recA; a.k_in = k; }
        else { a.agg = AGG_DENSE_RELU; a.x_in = u; }
        a.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE;
        a.Wm = Wb(l, i);
        a.bias = Bb(l, i);
        a.epi = EPI_SUB;
        a.R = plane(X, i);
        a.out = plane(X, i);
        if (with_grads) {
            a.G = plane(G, i);
            a.want_db = cfg.use_bias;
            a.part = part;
        }
        run_tile(a);
        if (!with_grads) return;
        reduce_block_grads(l, i);
        // input gradient: du = act'(u) ⊙ ((Âᵀ G_i)·W_iᵀ) into G_{i-1} or every G_j, j ≥ 2
        TileArgs b = tile_base();
        b.agg = AGG_DENSE;
        b.dir = bwd();
        b.x_in = plane(G, i);
        b.gemm = cfg.use_weight ? GEMM_WT : GEMM_NONE;
        b.Wm = Wb(l, i);
        if (sparse) { b.epi = EPI_MASKED_ADD; b.rrec = recA; b.k_r = k; }
        else { b.epi = EPI_MASKED_ADD_RELU; b.mask_plane = u; }
        if (i > 0) { b.dst[0] = plane(G, i - 1); b.ndst = 1; }
        else { for (int p = 1; p < C; ++p) b.dst[p - 1] = plane(G, p); b.ndst = C - 1; }
        run_tile(b);
    }
    void rev_layer_inverse(int l) { for (int i = C - 1; i >= 0; --i) rev_block_inverse(l, i, false); }
    void rev_layer_backward(int l) {
        if (fast_sweep()) {
            fast_layer_backward(l, false, false);
            join_reductions();
            return;
        }
        for (int i = C - 1; i >= 0; --i) rev_block_inverse(l, i, true);
    }

    // ---- Algorithms 1-2 --------------------------------------------------------
    void alg12_layer_forward(int l) {
        if (filled[l]) seq_err("gsr_forward_layer: cache already occupied for layer " + std::to_string(l));
        float* X1 = plane(X, 0);
        float* X2 = plane(X, 1);
        run_gs({X1}, c1[l]);                                 // line 5
        TileArgs a = tile_base();                            // lines 6-8: x2' = x2 + A(GS(x1)); GS(x2')
        a.agg = AGG_SPARSE; a.dir = fwd(); a.rec_in = c1[l]; a.k_in = k;
        a.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE; a.Wm = Wb(l, 0); a.bias = Bb(l, 0);
        a.epi = EPI_ADD; a.R = X2; a.out = X2; a.gs_out = c2[l]; a.k_gs = k;
        run_tile(a);
        TileArgs b = tile_base();                            // lines 9-10: x1' = scatter(s1) + B(GS(x2'))
        b.agg = AGG_SPARSE; b.dir = fwd(); b.rec_in = c2[l]; b.k_in = k;
        b.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE; b.Wm = Wb(l, 1); b.bias = Bb(l, 1);
        b.epi = EPI_SCATTER_ADD; b.rrec = c1[l]; b.k_r = k; b.out = X1;
        run_tile(b);
        filled[l] = 1;
    }
    // gsr_backward_block for block i with upstream m:
    //   out = Âᵀ·scatter(gather(m·Wᵀ, I_src)); dW += (Â·S_fwd)ᵀ·m; db += colsum(m)
    void alg12_block_backward(int l, int i, const float* m, const uint8_t* isrc, const uint8_t* fwd_rec, float* out) {
        TileArgs a = tile_base();
        a.agg = AGG_NONE; a.x_in = m;
        a.gemm = cfg.use_weight ? GEMM_WT : GEMM_NONE; a.Wm = Wb(l, i);
        a.epi = EPI_GATHER_REC; a.rrec = isrc; a.k_r = k; a.out_rec = vg;
        run_tile(a);
        TileArgs b = tile_base();
        b.agg = AGG_SPARSE; b.dir = bwd(); b.rec_in = vg; b.k_in = k; b.gemm = GEMM_NONE;
        b.epi = EPI_NONE; b.out = out;
        run_tile(b);
        TileArgs c = tile_base();
        c.agg = AGG_SPARSE; c.dir = fwd(); c.rec_in = fwd_rec; c.k_in = k; c.gemm = GEMM_NONE;
        c.epi = EPI_DISCARD; c.G = m; c.want_db = cfg.use_bias; c.part = part;
        run_tile(c);
        reduce_block_grads(l, i);
    }
    void alg12_layer_backward(int l) {
        if (!filled[l]) seq_err("gsr_backward_layer: missing forward cache for layer " + std::to_string(l));
        float* g1 = plane(G, 0);
        float* g2 = plane(G, 1);
        run_gs({g2}, t2);                                    // line 4
        TileArgs a = tile_base();                            // line 5-6: M1 = g1 − B(GS(g2)); GS(M1)
        a.agg = AGG_SPARSE; a.dir = fwd(); a.rec_in = t2; a.k_in = k;
        a.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE; a.Wm = Wb(l, 1); a.bias = Bb(l, 1);
        a.epi = EPI_SUB; a.R = g1; a.out = M1; a.gs_out = t1; a.k_gs = k;
        run_tile(a);
        TileArgs b = tile_base();                            // lines 6-7: M2 = scatter(GS(g2)) − A(GS(M1))
        b.agg = AGG_SPARSE; b.dir = fwd(); b.rec_in = t1; b.k_in = k;
        b.gemm = cfg.use_weight ? GEMM_W : GEMM_NONE; b.Wm = Wb(l, 0); b.bias = Bb(l, 0);
        b.epi = EPI_SCATTER_SUB; b.rrec = t2; b.k_r = k; b.out = M2;
        run_tile(b);
        const bool local = cfg.index_source == 0;            // line 8
        alg12_block_backward(l, 0, M1, local ? t1 : c1[l], c1[l], g1);
        alg12_block_backward(l, 1, M2, local ? t2 : c2[l], c2[l], g2);
        filled[l] = 0;
    }

    // ---- WorkCounter formulas (per layer, this model) ------------------------------
    uint64_t work_block_fwd(int w_, int k_, bool uw) const {
        return static_cast<uint64_t>(e) * k_ + (uw ? static_cast<uint64_t>(n) * w_ * w_ : 0);
    }
    uint64_t work_block_bwd(int w_, int k_, bool uw) const {
        return static_cast<uint64_t>(e) * k_ + (uw ? static_cast<uint64_t>(n) * w_ * w_ + static_cast<uint64_t>(e) * w_ : 0);
    }
    uint64_t work_layer_fwd() const {
        if (cfg.mode == GSRC_MODE_REV) return 0;
        return static_cast<uint64_t>(cfg.mode == GSRC_MODE_ALG12 ? 2 : C) * work_block_fwd(w, k, cfg.use_weight != 0);
    }
    uint64_t work_layer_bwd() const {  // Alg. 2: two recomputed forward blocks (lines 5-7) and two backward blocks
        if (cfg.mode != GSRC_MODE_ALG12) return 0;
        return 2 * work_block_fwd(w, k, cfg.use_weight != 0) + 2 * work_block_bwd(w, k, cfg.use_weight != 0);
    }

    // ---- network ---------------------------------------------------------------
    void layer_forward(int l) { if (cfg.mode == GSRC_MODE_ALG12) alg12_layer_forward(l); else rev_layer_forward(l); }
    void layer_backward(int l) { if (cfg.mode == GSRC_MODE_ALG12) alg12_layer_backward(l); else rev_layer_backward(l); }

    void enqueue_forward() {
        if (diag) CK(cudaMemsetAsync(diag_cnt, 0, sizeof(unsigned long long) * static_cast<size_t>(cfg.layers) * C, stream));
        CK(launch_encoder(X0, static_cast<int>(n), cfg.d_in, params, params + static_cast<size_t>(cfg.d_in) * cfg.hidden, cfg.hidden,
                          C, w, ld, X, q_scale(), q_inv(), stream));
        ++launches;
        if (cfg.mode == GSRC_MODE_ALG12) std::fill(filled.begin(), filled.end(), 0);
        for (int l = 0; l < cfg.layers; ++l) layer_forward(l);
        const float* wh = params + off_block(cfg.layers, 0);
        CK(launch_head_loss(X, static_cast<int>(n), cfg.hidden, C, w, ld, wh, wh + cfg.hidden, y, mask, 0.f, cnt, yhat, gy, loss_part,
                            loss_nparts, stream));
        ++launches;
        CK(launch_sum_double(loss_part, loss_nparts, 1.0 / static_cast<double>(cnt), loss_dev, stream));
        ++launches;
    }
    void enqueue_backward() {
        const float* wh = params + off_block(cfg.layers, 0);
        CK(launch_head_bwd(X, gy, static_cast<int>(n), cfg.hidden, C, w, ld, wh, G, part, nparts_small, stream));
        ++launches;
        CK(launch_reduce_parts(part, nparts_small, cfg.hidden + 1, cfg.hidden + 1, grads + off_block(cfg.layers, 0), 0, stream));
        ++launches;
        for (int l = cfg.layers - 1; l >= 0; --l) {
            if (fast_sweep()) fast_layer_backward(l, l < cfg.layers - 1, l > 0);
            else layer_backward(l);
        }
        join_reductions();
        const int elen = cfg.d_in * cfg.hidden + cfg.hidden;
        CK(launch_encoder_bwd(X0, G, static_cast<int>(n), cfg.d_in, cfg.hidden, C, w, ld, part, nparts_small, stream));
        ++launches;
        CK(launch_reduce_parts(part, nparts_small, elen, elen, grads, 0, stream));
        ++launches;
    }
    void enqueue_zero_grads() { CK(cudaMemsetAsync(grads, 0, sizeof(float) * P, stream)); }
    // one in-place NCCL all-reduce (average) of the flat gradient buffer on the
    // context stream: ordered after the backward and before the optimizer by
    // the stream itself
    void enqueue_allreduce() {
        if (!comm) return;  // a 1-rank communicator still runs the call (AVG over one rank is the identity)
        nccl_check(nccl_api().all_reduce(grads, grads, static_cast<size_t>(P), ncclFloat32, ncclAvg, comm, stream), "ncclAllReduce");
    }
    void enqueue_optimizer(const gsrc_optim_cfg& o) {
        if (o.optimizer == 0) {
            CK(launch_adam_prep(d_step, static_cast<double>(o.beta1), static_cast<double>(o.beta2), bc, stream));
            CK(launch_adam(params, grads, opt_m, opt_v, P, o.lr, o.beta1, o.beta2, o.eps, o.weight_decay, bc, stream));
            launches += 2;
        } else {
            CK(launch_sgd(params, grads, opt_m, P, o.lr, o.momentum, stream));
            ++launches;
        }
    }

    void require_model() const {
        if (!model) seq_err("model not initialised (gsrc_model_init)");
    }
    void require_data() const {
        require_model();
        if (!data) seq_err("node data not uploaded (gsrc_data_upload)");
    }
    void drop_graphs() {
        for (cudaGraphExec_t* g : {&g_fwd, &g_bwd, &g_opt})
            if (*g) { cudaGraphExecDestroy(*g); *g = nullptr; }
    }

    // Activation arena plan (bytes independent of L except the ALG12 caches,
    // which Alg. 1 retains by design: O(L·n·k)).
    void plan_arena() {
        const size_t pl = static_cast<size_t>(n) * ld;
        const size_t rb = static_cast<size_t>(n) * rec_bytes(k > 0 ? k : 1);
        nparts = tile_grid_max(static_cast<int>(n));
        nparts_small = 148 * 8;
        loss_nparts = static_cast<int>((n + kThreads - 1) / kThreads);
        const size_t plen = static_cast<size_t>(w) * w + w;
        size_t part_len = std::max(static_cast<size_t>(nparts) * plen, static_cast<size_t>(nparts_small) * (cfg.d_in * cfg.hidden + cfg.hidden));
        part_len = std::max(part_len, static_cast<size_t>(nparts_small) * (cfg.hidden + 1));
        const bool alg12 = cfg.mode == GSRC_MODE_ALG12;
        size_t total = 0;
        total += 2 * bytes_rounded(pl * C * sizeof(float));               // X, G
        total += 2 * bytes_rounded(rb);                                    // recA, recB
        if (fast() && C > 2) total += static_cast<size_t>(C - 2) * bytes_rounded(rb);  // rblk[2..C-1]
        total += bytes_rounded(part_len * sizeof(double));
        const size_t bin_part_len = static_cast<size_t>(fast_bin_grid_max()) * plen;
        if (fast_sweep()) total += 2 * bytes_rounded(bin_part_len * sizeof(double));  // part_bin[0..1]
        total += 2 * bytes_rounded(static_cast<size_t>(n) * sizeof(float));  // yhat, gy
        total += bytes_rounded(static_cast<size_t>(loss_nparts) * sizeof(double)) + 256;
        if (cfg.mode == GSRC_MODE_REV) total += bytes_rounded(pl * sizeof(float));
        if (fastpath()) total += 2 * bytes_rounded(pl * sizeof(float));    // Zh, Zh2 (hub-row aggregates)
        const size_t nsegmax = static_cast<size_t>(std::max(nseg_f, nseg_b));
        if (fastpath()) total += 2 * bytes_rounded(std::max<size_t>(nsegmax, 1) * ld * sizeof(float));  // Pseg, Pseg2
        if (alg12) total += 2 * bytes_rounded(pl * sizeof(float)) + 3 * bytes_rounded(rb) + 2 * static_cast<size_t>(cfg.layers) * bytes_rounded(rb);
        arena.plan(total);
        X = arena.lease<float>(pl * C);
        G = arena.lease<float>(pl * C);
        recA = arena.lease<uint8_t>(rb);
        recB = arena.lease<uint8_t>(rb);
        rblk.assign({recA, recB});
        if (fast())
            for (int i = 2; i < C; ++i) rblk.push_back(arena.lease<uint8_t>(rb));
        part = arena.lease<double>(part_len);
        part_bin[0] = part_bin[1] = nullptr;
        if (fast_sweep())
            for (auto& pb_ : part_bin) pb_ = arena.lease<double>(bin_part_len);
        yhat = arena.lease<float>(static_cast<size_t>(n));
        gy = arena.lease<float>(static_cast<size_t>(n));
        loss_part = arena.lease<double>(static_cast<size_t>(loss_nparts));
        loss_dev = arena.lease<double>(1);
        U = nullptr;
        if (cfg.mode == GSRC_MODE_REV) U = arena.lease<float>(pl);
        Zh = fastpath() ? arena.lease<float>(pl) : nullptr;
        Pseg = fastpath() ? arena.lease<float>(std::max<size_t>(nsegmax, 1) * ld) : nullptr;
        Zh2 = fastpath() ? arena.lease<float>(pl) : nullptr;
        Pseg2 = fastpath() ? arena.lease<float>(std::max<size_t>(nsegmax, 1) * ld) : nullptr;
        xmaps.assign(static_cast<size_t>(C), CUtensorMap{});
        gmaps.assign(static_cast<size_t>(C), CUtensorMap{});
        if (fastpath())
            for (int p = 0; p < C; ++p) {
                CK(encode_plane_map(&xmaps[static_cast<size_t>(p)], plane(X, p), static_cast<int>(n), ld));
                CK(encode_plane_map(&gmaps[static_cast<size_t>(p)], plane(G, p), static_cast<int>(n), ld));
            }
        c1.clear();
        c2.clear();
        if (alg12) {
            M1 = arena.lease<float>(pl);
            M2 = arena.lease<float>(pl);
            t1 = arena.lease<uint8_t>(rb);
            t2 = arena.lease<uint8_t>(rb);
            vg = arena.lease<uint8_t>(rb);
            for (int l = 0; l < cfg.layers; ++l) { c1.push_back(arena.lease<uint8_t>(rb)); c2.push_back(arena.lease<uint8_t>(rb)); }
        }
        filled.assign(static_cast<size_t>(cfg.layers), 0);
        // zero planes once so padding columns are 0
        CK(cudaMemsetAsync(arena.base, 0, arena.used, stream));
        CK(cudaStreamSynchronize(stream));
    }
};

namespace {

template <typename F>
int guarded(gsrc_ctx* ctx, F&& f) {
    if (!ctx) return GSRC_ERR_CONFIG;
    try {
        int dev = -1;
        cudaGetDevice(&dev);
        if (dev != ctx->device) CK(cudaSetDevice(ctx->device));
        f();
        return GSRC_OK;
    } catch (const Fail& e) {
        ctx->err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failure";
        return GSRC_ERR_RESOURCE;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return GSRC_ERR_INTERNAL;
    }
}

template <typename T>
T* dmalloc(size_t count, size_t* acct = nullptr) {
    T* p = nullptr;
    const size_t bytes = count * sizeof(T) ? count * sizeof(T) : 16;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); throw Fail(GSRC_ERR_RESOURCE, std::string("cudaMalloc failed: ") + cudaGetErrorString(e)); }
    if (acct) *acct += bytes;
    return p;
}

void h2d_rows(float* dplane_base, int64_t n, int C, int w, int ld, const float* host, int D, cudaStream_t s) {
    for (int p = 0; p < C; ++p)
        CK(cudaMemcpy2DAsync(dplane_base + static_cast<size_t>(p) * n * ld, ld * sizeof(float), host + static_cast<size_t>(p) * w,
                             D * sizeof(float), w * sizeof(float), n, cudaMemcpyHostToDevice, s));
}
void d2h_rows(float* host, const float* dplane_base, int64_t n, int C, int w, int ld, int D, cudaStream_t s) {
    for (int p = 0; p < C; ++p)
        CK(cudaMemcpy2DAsync(host + static_cast<size_t>(p) * w, D * sizeof(float), dplane_base + static_cast<size_t>(p) * n * ld,
                             ld * sizeof(float), w * sizeof(float), n, cudaMemcpyDeviceToHost, s));
}

// Pack host (vals, idx) n×k into device records.
void upload_records(const float* vals, const int32_t* idx, int64_t n, int k, uint8_t* rec, cudaStream_t s) {
    DevBuf dv(static_cast<size_t>(n) * k * sizeof(float)), di(static_cast<size_t>(n) * k * sizeof(int));
    CK(cudaMemcpyAsync(dv.p, vals, static_cast<size_t>(n) * k * sizeof(float), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(di.p, idx, static_cast<size_t>(n) * k * sizeof(int), cudaMemcpyHostToDevice, s));
    CK(launch_rec_pack(dv.as<float>(), di.as<int>(), static_cast<int>(n), k, rec, s));
    CK(cudaStreamSynchronize(s));
}
void download_records(const uint8_t* rec, int64_t n, int k, float* vals, int32_t* idx, cudaStream_t s) {
    DevBuf dv(static_cast<size_t>(n) * k * sizeof(float)), di(static_cast<size_t>(n) * k * sizeof(int));
    CK(launch_rec_unpack(rec, static_cast<int>(n), k, dv.as<float>(), di.as<int>(), s));
    CK(cudaMemcpyAsync(vals, dv.p, static_cast<size_t>(n) * k * sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(idx, di.p, static_cast<size_t>(n) * k * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

void check_rec_idx(const int32_t* idx, int64_t n, int k, int w) {
    for (int64_t r = 0; r < n; ++r)
        for (int j = 0; j < k; ++j) {
            const int32_t c = idx[r * k + j];
            if (c < 0 || c >= w) cfg_err("SparseActivation index out of range at row " + std::to_string(r));
            if (j > 0 && c <= idx[r * k + j - 1]) cfg_err("SparseActivation indices not strictly ascending at row " + std::to_string(r));
        }
}

}  // namespace

extern "C" {

int gsrc_version(char* buf, size_t len) {
    const char* v = "gsrnet 0.1.0 (b200 sm_100a)";
    if (buf && len) { std::strncpy(buf, v, len - 1); buf[len - 1] = 0; }
    return GSRC_OK;
}

int gsrc_create(int device, gsrc_ctx** out) {
    if (!out) return GSRC_ERR_CONFIG;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return GSRC_ERR_RESOURCE; }
    if (device < 0 || device >= ndev) return GSRC_ERR_CONFIG;
    if (cudaSetDevice(device) != cudaSuccess) return GSRC_ERR_RESOURCE;
    auto* ctx = new (std::nothrow) gsrc_ctx();
    if (!ctx) return GSRC_ERR_RESOURCE;
    ctx->device = device;
    if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return GSRC_ERR_RESOURCE; }
    ctx->stream = ctx->own;
    for (auto& e : ctx->ev) cudaEventCreate(&e);
    for (auto& e : ctx->tev) cudaEventCreate(&e);
    if (cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return GSRC_ERR_RESOURCE; }
    cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming);
    if (cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return GSRC_ERR_RESOURCE; }
    for (int b = 0; b < 2; ++b) {
        cudaEventCreateWithFlags(&ctx->ev_bin[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ctx->ev_red[b], cudaEventDisableTiming);
    }
    if (init_kernel_attributes() != cudaSuccess) { delete ctx; return GSRC_ERR_RESOURCE; }
    if (cudaMallocHost(&ctx->loss_host, sizeof(double)) != cudaSuccess) { delete ctx; return GSRC_ERR_RESOURCE; }
    *out = ctx;
    return GSRC_OK;
}

void gsrc_destroy(gsrc_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    delete ctx;
}

const char* gsrc_last_error(gsrc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gsrc_set_stream(gsrc_ctx* ctx, void* s) {
    return guarded(ctx, [&] {
        ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
        ctx->drop_graphs();
    });
}

int gsrc_synchronize(gsrc_ctx* ctx) { return guarded(ctx, [&] { CK(cudaStreamSynchronize(ctx->stream)); }); }

int gsrc_graph_upload(gsrc_ctx* ctx, int64_t n, int64_t e, const int64_t* row_ptr, const int32_t* col_idx, int norm) {
    return guarded(ctx, [&] {
        if (n <= 0) cfg_err("graph: n must be > 0");
        if (e < 0 || e > 0x7fffffffLL) cfg_err("graph: e out of range for int32 CSR");
        if (norm < 0 || norm > 2) cfg_err("graph: bad norm_mode");
        if (!row_ptr || (e > 0 && !col_idx)) cfg_err("graph: null arrays");
        if (row_ptr[0] != 0 || row_ptr[n] != e) throw Fail(GSRC_ERR_CONFIG, "graph: row_ptr endpoints (FormatError)");
        std::vector<int> rp(static_cast<size_t>(n + 1)), trp(static_cast<size_t>(n + 1), 0), tci(static_cast<size_t>(e));
        std::vector<float> rf(static_cast<size_t>(n)), cf(static_cast<size_t>(n));
        for (int64_t r = 0; r < n; ++r) {
            if (row_ptr[r + 1] < row_ptr[r]) cfg_err("graph: row_ptr decreasing at row " + std::to_string(r));
            rp[r] = static_cast<int>(row_ptr[r]);
            for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
                const int32_t c = col_idx[q];
                if (c < 0 || c >= n) cfg_err("graph: col_idx out of range at edge " + std::to_string(q));
                if (q > row_ptr[r] && c <= col_idx[q - 1]) cfg_err("graph: col_idx not strictly ascending in row " + std::to_string(r));
                trp[static_cast<size_t>(c) + 1]++;
            }
            const int64_t deg = row_ptr[r + 1] - row_ptr[r];
            // same double-then-round expressions as the oracle (oracle/gsr_oracle.hpp norm_*_factor)
            if (norm == GSRC_NORM_NONE) { rf[r] = 1.f; cf[r] = 1.f; }
            else if (deg <= 0) { rf[r] = 0.f; cf[r] = norm == GSRC_NORM_SYM_DEGREE ? 0.f : 1.f; }
            else if (norm == GSRC_NORM_ROW_MEAN) { rf[r] = static_cast<float>(1.0 / static_cast<double>(deg)); cf[r] = 1.f; }
            else { rf[r] = cf[r] = static_cast<float>(1.0 / std::sqrt(static_cast<double>(deg))); }
        }
        rp[n] = static_cast<int>(e);
        for (int64_t r = 0; r < n; ++r) trp[r + 1] += trp[r];
        {
            std::vector<int> fill(trp.begin(), trp.end() - 1);
            for (int64_t r = 0; r < n; ++r)
                for (int64_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) tci[static_cast<size_t>(fill[col_idx[q]]++)] = static_cast<int>(r);
        }
        CK(cudaStreamSynchronize(ctx->stream));
        for (void* p : {(void*)ctx->rp, (void*)ctx->ci, (void*)ctx->trp, (void*)ctx->tci, (void*)ctx->row_f, (void*)ctx->col_f}) if (p) cudaFree(p);
        ctx->rp = ctx->ci = ctx->trp = ctx->tci = nullptr;
        ctx->graph_bytes = 0;
        ctx->rp = dmalloc<int>(n + 1, &ctx->graph_bytes);
        ctx->ci = dmalloc<int>(e, &ctx->graph_bytes);
        ctx->trp = dmalloc<int>(n + 1, &ctx->graph_bytes);
        ctx->tci = dmalloc<int>(e, &ctx->graph_bytes);
        ctx->row_f = dmalloc<float>(n, &ctx->graph_bytes);
        ctx->col_f = dmalloc<float>(n, &ctx->graph_bytes);
        CK(cudaMemcpy(ctx->rp, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
        if (e) CK(cudaMemcpy(ctx->ci, col_idx, sizeof(int) * e, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->trp, trp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
        if (e) CK(cudaMemcpy(ctx->tci, tci.data(), sizeof(int) * e, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->row_f, rf.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->col_f, cf.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
        // rows longer than one aggregation segment, per direction (fast path hubs)
        std::vector<int> hf, hb;
        for (int64_t r = 0; r < n; ++r) {
            if (row_ptr[r + 1] - row_ptr[r] > kAggSeg) hf.push_back(static_cast<int>(r));
            if (trp[r + 1] - trp[r] > kAggSeg) hb.push_back(static_cast<int>(r));
        }
        for (void* p : {(void*)ctx->item_f, (void*)ctx->hcnt_f, (void*)ctx->seg_b, (void*)ctx->hub_b, (void*)ctx->segoff_b,
                        (void*)ctx->seg_fd, (void*)ctx->hub_fd, (void*)ctx->segoff_fd, (void*)ctx->ell_f, (void*)ctx->ell_b})
            if (p) cudaFree(p);
        // per-row neighbour slots (Dir::ell): edge scale = the direction's edge_f of the neighbour
        auto ell_table = [&](const std::vector<int>& ptr, const int* idx, const std::vector<float>& ef) {
            std::vector<int2> t(static_cast<size_t>(n) * kAggSeg, make_int2(-1, 0));
            for (int64_t r = 0; r < n; ++r) {
                int2* s = t.data() + static_cast<size_t>(r) * kAggSeg;
                const int e0 = ptr[static_cast<size_t>(r)], e1 = ptr[static_cast<size_t>(r) + 1];
                if (e1 - e0 > kAggSeg) { s[0].x = -2; continue; }
                for (int q = e0; q < e1; ++q) {
                    float f = ef[static_cast<size_t>(idx[q])];
                    int bits;
                    std::memcpy(&bits, &f, sizeof bits);
                    s[q - e0] = make_int2(idx[q], bits);
                }
            }
            int2* d = dmalloc<int2>(t.size(), &ctx->graph_bytes);
            CK(cudaMemcpy(d, t.data(), sizeof(int2) * t.size(), cudaMemcpyHostToDevice));
            return d;
        };
        ctx->ell_f = ell_table(rp, col_idx, cf);
        ctx->ell_b = ell_table(trp, tci.data(), rf);
        ctx->nhub_f = static_cast<int>(hf.size());
        ctx->nhub_b = static_cast<int>(hb.size());
        auto hub_table = [&](const std::vector<int>& hubs, const std::vector<int>& ptr, int chunk, int4*& items, int& nitem, int*& cnt, int& nseg) {
            std::vector<int4> iv;
            int total = 0;
            for (size_t h = 0; h < hubs.size(); ++h) {
                const int r = hubs[h], e0 = ptr[static_cast<size_t>(r)], e1 = ptr[static_cast<size_t>(r) + 1];
                const int ns = (e1 - e0 + kAggSeg - 1) / kAggSeg;
                for (int c0 = 0; c0 < ns; c0 += chunk) {
                    iv.push_back(make_int4(r, e0, e1, c0));
                    iv.push_back(make_int4(static_cast<int>(h), total, 0, 0));
                }
                total += ns;
            }
            nseg = total;
            nitem = static_cast<int>(iv.size() / 2);
            items = dmalloc<int4>(iv.size(), &ctx->graph_bytes);
            cnt = dmalloc<int>(hubs.size(), &ctx->graph_bytes);
            if (!iv.empty()) CK(cudaMemcpy(items, iv.data(), sizeof(int4) * iv.size(), cudaMemcpyHostToDevice));
            if (!hubs.empty()) CK(cudaMemset(cnt, 0, sizeof(int) * hubs.size()));
        };
        hub_table(hf, rp, kHubChunk, ctx->item_f, ctx->nitem_f, ctx->hcnt_f, ctx->nseg_f);
        // dense: flattened segments, per-hub first segment (transpose for BIN; forward for the rev-baseline)
        auto dense_table = [&](const std::vector<int>& hubs, const std::vector<int>& ptr, int2*& seg, int*& segoff, int*& hubrows, int& nseg) {
            std::vector<int2> sv;
            std::vector<int> ov(hubs.size() + 1, 0);
            for (size_t h = 0; h < hubs.size(); ++h) {
                ov[h] = static_cast<int>(sv.size());
                const int e0 = ptr[static_cast<size_t>(hubs[h])], e1 = ptr[static_cast<size_t>(hubs[h]) + 1];
                for (int lo = e0; lo < e1; lo += kAggSeg) sv.push_back(make_int2(lo, std::min(e1, lo + kAggSeg)));
            }
            ov[hubs.size()] = static_cast<int>(sv.size());
            nseg = static_cast<int>(sv.size());
            seg = dmalloc<int2>(sv.size(), &ctx->graph_bytes);
            segoff = dmalloc<int>(ov.size(), &ctx->graph_bytes);
            hubrows = dmalloc<int>(hubs.size(), &ctx->graph_bytes);
            if (!sv.empty()) CK(cudaMemcpy(seg, sv.data(), sizeof(int2) * sv.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(segoff, ov.data(), sizeof(int) * ov.size(), cudaMemcpyHostToDevice));
            if (!hubs.empty()) CK(cudaMemcpy(hubrows, hubs.data(), sizeof(int) * hubs.size(), cudaMemcpyHostToDevice));
        };
        dense_table(hb, trp, ctx->seg_b, ctx->segoff_b, ctx->hub_b, ctx->nseg_b);
        dense_table(hf, rp, ctx->seg_fd, ctx->segoff_fd, ctx->hub_fd, ctx->nseg_fd);
        CK(cudaDeviceSynchronize());  // pageable copies may still be in flight when cudaMemcpy returns
        const bool resize = ctx->n != n;
        ctx->n = n;
        ctx->e = e;
        ctx->norm = norm;
        ctx->drop_graphs();
        if (resize) {
            ctx->data = false;
            if (ctx->diag_store) { cudaFree(ctx->diag_store); ctx->diag_store = nullptr; }
            if (ctx->diag_cnt) { cudaFree(ctx->diag_cnt); ctx->diag_cnt = nullptr; }
            ctx->diag = false;
        }
        if (ctx->model) ctx->plan_arena();  // node count / hub segments changed: re-plan activations
    });
}

int gsrc_model_init(gsrc_ctx* ctx, const gsrc_model_cfg* cfg) {
    return guarded(ctx, [&] {
        if (!cfg) cfg_err("null cfg");
        if (ctx->n <= 0) seq_err("upload a graph before gsrc_model_init");
        gsrc_model_cfg c = *cfg;
        if (c.mode < 0 || c.mode > 2) cfg_err("mode");
        if (c.layers < 0) cfg_err("layers < 0");
        if (c.mode == GSRC_MODE_ALG12) c.groups = 2;
        if (c.groups < 2 || c.hidden <= 0 || c.hidden % c.groups) cfg_err("hidden must be divisible by groups >= 2");
        const int w = c.hidden / c.groups;
        if (w > 128) cfg_err("group width > 128 not supported by the sm_100a kernels");
        if (c.groups > kMaxDst + 1) cfg_err("groups > 9 not supported");
        if (c.mode != GSRC_MODE_REV && (c.k < 1 || c.k > w)) cfg_err("k out of [1, width]");
        if (c.d_in < 1 || c.d_in > 16) cfg_err("d_in must be in [1, 16]");
        if (c.gemm != GSRC_GEMM_FP32 && c.gemm != GSRC_GEMM_TF32) cfg_err("gemm precision");
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->cfg = c;
        ctx->C = c.groups;
        ctx->nb = c.groups;
        ctx->w = w;
        ctx->ld = pad_ld(w);
        ctx->k = c.mode == GSRC_MODE_REV ? 1 : c.k;
        ctx->P = static_cast<int64_t>(c.d_in) * c.hidden + c.hidden + static_cast<int64_t>(c.layers) * ctx->nb * (static_cast<int64_t>(w) * w + w) +
                 c.hidden + 1;
        for (void* p : {(void*)ctx->params, (void*)ctx->grads, (void*)ctx->opt_m, (void*)ctx->opt_v, (void*)ctx->bc, (void*)ctx->d_step}) if (p) cudaFree(p);
        ctx->model_bytes = 0;
        ctx->params = dmalloc<float>(ctx->P, &ctx->model_bytes);
        ctx->grads = dmalloc<float>(ctx->P, &ctx->model_bytes);
        ctx->opt_m = dmalloc<float>(ctx->P, &ctx->model_bytes);
        ctx->opt_v = dmalloc<float>(ctx->P, &ctx->model_bytes);
        ctx->bc = dmalloc<float>(2, &ctx->model_bytes);
        ctx->d_step = dmalloc<long long>(1, &ctx->model_bytes);
        CK(cudaMemset(ctx->params, 0, sizeof(float) * ctx->P));
        CK(cudaMemset(ctx->grads, 0, sizeof(float) * ctx->P));
        CK(cudaMemset(ctx->opt_m, 0, sizeof(float) * ctx->P));
        CK(cudaMemset(ctx->opt_v, 0, sizeof(float) * ctx->P));
        CK(cudaMemset(ctx->d_step, 0, sizeof(long long)));
        CK(cudaDeviceSynchronize());
        if (ctx->diag_store) { cudaFree(ctx->diag_store); ctx->diag_store = nullptr; }
        if (ctx->diag_cnt) { cudaFree(ctx->diag_cnt); ctx->diag_cnt = nullptr; }
        ctx->diag = false;
        ctx->model = true;
        ctx->drop_graphs();
        ctx->plan_arena();
    });
}

int gsrc_num_params(gsrc_ctx* ctx, int64_t* out) {
    return guarded(ctx, [&] { ctx->require_model(); *out = ctx->P; });
}

int gsrc_params_set(gsrc_ctx* ctx, const float* host, int64_t n) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (n != ctx->P) cfg_err("params_set: expected " + std::to_string(ctx->P) + " values");
        CK(cudaMemcpyAsync(ctx->params, host, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(ctx->opt_m, 0, sizeof(float) * n, ctx->stream));
        CK(cudaMemsetAsync(ctx->opt_v, 0, sizeof(float) * n, ctx->stream));
        CK(cudaMemsetAsync(ctx->d_step, 0, sizeof(long long), ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_params_get(gsrc_ctx* ctx, float* host, int64_t n) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (n != ctx->P) cfg_err("params_get: size mismatch");
        CK(cudaMemcpyAsync(host, ctx->params, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_grads_get(gsrc_ctx* ctx, float* host, int64_t n) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (n != ctx->P) cfg_err("grads_get: size mismatch");
        CK(cudaMemcpyAsync(host, ctx->grads, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_zero_grads(gsrc_ctx* ctx) {
    return guarded(ctx, [&] { ctx->require_model(); ctx->enqueue_zero_grads(); CK(cudaStreamSynchronize(ctx->stream)); });
}

int gsrc_grads_device(gsrc_ctx* ctx, float** dptr, int64_t* n) {
    return guarded(ctx, [&] { ctx->require_model(); *dptr = ctx->grads; *n = ctx->P; });
}

int gsrc_params_device(gsrc_ctx* ctx, float** dptr, int64_t* n) {
    return guarded(ctx, [&] { ctx->require_model(); *dptr = ctx->params; *n = ctx->P; });
}

int gsrc_data_upload(gsrc_ctx* ctx, const float* x0, const float* y, const uint8_t* train_mask) {
    return guarded(ctx, [&] {
        ctx->require_model();
        const int64_t n = ctx->n;
        if (!ctx->X0 || ctx->data_n != n) {
            for (void* p : {(void*)ctx->X0, (void*)ctx->y, (void*)ctx->mask}) if (p) cudaFree(p);
            ctx->data_n = n;
            ctx->data_bytes = 0;
            ctx->X0 = dmalloc<float>(static_cast<size_t>(n) * 16, &ctx->data_bytes);
            ctx->y = dmalloc<float>(n, &ctx->data_bytes);
            ctx->mask = dmalloc<uint8_t>(n, &ctx->data_bytes);
        }
        int64_t cnt = 0;
        for (int64_t r = 0; r < n; ++r) cnt += train_mask[r] ? 1 : 0;
        if (cnt == 0) cfg_err("mse_loss: empty mask");
        ctx->cnt = static_cast<float>(cnt);
        CK(cudaMemcpyAsync(ctx->X0, x0, sizeof(float) * n * ctx->cfg.d_in, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->y, y, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->mask, train_mask, n, cudaMemcpyHostToDevice, ctx->stream));
        // the mask count is a kernel argument of the captured step: re-capture on change
        if (!ctx->data || ctx->captured_cnt != ctx->cnt) ctx->drop_graphs();
        ctx->captured_cnt = ctx->cnt;
        ctx->data = true;
    });
}

int gsrc_forward(gsrc_ctx* ctx, float* yhat_out) {
    return guarded(ctx, [&] {
        ctx->require_data();
        ctx->enqueue_forward();
        ctx->work_ma += static_cast<uint64_t>(ctx->cfg.layers) * ctx->work_layer_fwd();
        if (yhat_out) CK(cudaMemcpyAsync(yhat_out, ctx->yhat, sizeof(float) * ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

static void run_maybe_graph(gsrc_ctx* ctx, cudaGraphExec_t& exec, int64_t& nl, const std::function<void()>& body) {
    if (!ctx->use_graph) { body(); return; }
    if (!exec) {
        const int64_t before = ctx->launches;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        try { body(); } catch (...) { cudaStreamEndCapture(ctx->stream, &g); if (g) cudaGraphDestroy(g); throw; }
        CK(cudaStreamEndCapture(ctx->stream, &g));
        cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) throw_cuda(e, "cudaGraphInstantiate", __LINE__);
        nl = ctx->launches - before;
        ctx->launches = before;
    }
    CK(cudaGraphLaunch(exec, ctx->stream));
    ctx->launches += nl;
}

// TimingBreakdown (Eq. 9) from events recorded around and
// inside the (possibly graph-replayed) step: forward (encoder, layers, head,
// loss), backward (head, layers with inverse recomputation, encoder),
// optimizer, and the loss copy-out (the host-analogue of Table 3's cudaMemcpy).
static gsrc_timing phase_timing(gsrc_ctx* ctx, bool with_opt) {
    float t_all = 0.f, t_f = 0.f, t_b = 0.f, t_o = 0.f;
    cudaEventElapsedTime(&t_all, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&t_f, ctx->ev[0], ctx->tev[0]);
    cudaEventElapsedTime(&t_b, ctx->tev[0], ctx->tev[1]);
    // the gradient all-reduce (tev[1] → tev[3]) and the loss read-back count as "copy"
    if (with_opt) cudaEventElapsedTime(&t_o, ctx->tev[3], ctx->tev[2]);
    const float t_c = t_all - t_f - t_b - t_o;
    return gsrc_timing{t_f * 1e-3, t_b * 1e-3, (t_c > 0.f ? t_c : 0.f) * 1e-3, t_o * 1e-3, t_all * 1e-3};
}

int gsrc_forward_backward(gsrc_ctx* ctx, double* loss_out) {
    return guarded(ctx, [&] {
        ctx->require_data();
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_maybe_graph(ctx, ctx->g_fwd, ctx->g_fwd_launches, [&] {
            ctx->enqueue_zero_grads();
            ctx->enqueue_forward();
        });
        CK(cudaEventRecord(ctx->tev[0], ctx->stream));
        run_maybe_graph(ctx, ctx->g_bwd, ctx->g_bwd_launches, [&] { ctx->enqueue_backward(); });
        CK(cudaEventRecord(ctx->tev[1], ctx->stream));
        CK(cudaMemcpyAsync(ctx->loss_host, ctx->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += static_cast<uint64_t>(ctx->cfg.layers) * (ctx->work_layer_fwd() + ctx->work_layer_bwd());
        ctx->timing = phase_timing(ctx, false);
        if (loss_out) *loss_out = *ctx->loss_host;
    });
}

int gsrc_optimizer_step(gsrc_ctx* ctx, const gsrc_optim_cfg* opt) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (!opt) cfg_err("null optimizer cfg");
        ctx->enqueue_optimizer(*opt);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_train_step(gsrc_ctx* ctx, const gsrc_optim_cfg* opt, double* loss_out) {
    return guarded(ctx, [&] {
        ctx->require_data();
        if (!opt) cfg_err("null optimizer cfg");
        if (ctx->g_opt && std::memcmp(&ctx->g_step_opt, opt, sizeof(gsrc_optim_cfg)) != 0) {
            cudaGraphExecDestroy(ctx->g_opt);
            ctx->g_opt = nullptr;
        }
        ctx->g_step_opt = *opt;
        CK(cudaEventRecord(ctx->ev[0], ctx->stream));
        run_maybe_graph(ctx, ctx->g_fwd, ctx->g_fwd_launches, [&] {
            ctx->enqueue_zero_grads();
            ctx->enqueue_forward();
        });
        CK(cudaEventRecord(ctx->tev[0], ctx->stream));
        run_maybe_graph(ctx, ctx->g_bwd, ctx->g_bwd_launches, [&] { ctx->enqueue_backward(); });
        CK(cudaEventRecord(ctx->tev[1], ctx->stream));
        ctx->enqueue_allreduce();  // data parallel: average the gradients over the ranks (no-op without a communicator)
        CK(cudaEventRecord(ctx->tev[3], ctx->stream));
        run_maybe_graph(ctx, ctx->g_opt, ctx->g_opt_launches, [&] { ctx->enqueue_optimizer(*opt); });
        CK(cudaEventRecord(ctx->tev[2], ctx->stream));
        CK(cudaMemcpyAsync(ctx->loss_host, ctx->loss_dev, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaEventRecord(ctx->ev[1], ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += static_cast<uint64_t>(ctx->cfg.layers) * (ctx->work_layer_fwd() + ctx->work_layer_bwd());
        ctx->timing = phase_timing(ctx, true);
        if (loss_out) *loss_out = *ctx->loss_host;
    });
}

int gsrc_activation_get(gsrc_ctx* ctx, float* host) {
    return guarded(ctx, [&] {
        ctx->require_model();
        d2h_rows(host, ctx->X, ctx->n, ctx->C, ctx->w, ctx->ld, ctx->cfg.hidden, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}
int gsrc_activation_set(gsrc_ctx* ctx, const float* host) {
    return guarded(ctx, [&] {
        ctx->require_model();
        h2d_rows(ctx->X, ctx->n, ctx->C, ctx->w, ctx->ld, host, ctx->cfg.hidden, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}
int gsrc_gradient_get(gsrc_ctx* ctx, float* host) {
    return guarded(ctx, [&] {
        ctx->require_model();
        d2h_rows(host, ctx->G, ctx->n, ctx->C, ctx->w, ctx->ld, ctx->cfg.hidden, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}
int gsrc_gradient_set(gsrc_ctx* ctx, const float* host) {
    return guarded(ctx, [&] {
        ctx->require_model();
        h2d_rows(ctx->G, ctx->n, ctx->C, ctx->w, ctx->ld, host, ctx->cfg.hidden, ctx->stream);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_set_op_precision(gsrc_ctx* ctx, int gemm) {
    return guarded(ctx, [&] {
        if (gemm != GSRC_GEMM_FP32 && gemm != GSRC_GEMM_TF32) cfg_err("gemm precision");
        ctx->op_tc = gemm == GSRC_GEMM_TF32;
    });
}

int gsrc_set_graph_capture(gsrc_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        ctx->use_graph = enable != 0;
        if (!ctx->use_graph) ctx->drop_graphs();
    });
}

int gsrc_last_timing(gsrc_ctx* ctx, gsrc_timing* out) { return guarded(ctx, [&] { *out = ctx->timing; }); }

int gsrc_mem_stats(gsrc_ctx* ctx, gsrc_mem_report* out) {
    return guarded(ctx, [&] {
        const uint64_t persist = ctx->graph_bytes + ctx->model_bytes + ctx->data_bytes;
        out->reserved_bytes = ctx->arena.reserved + persist;
        out->active_bytes = ctx->arena.used + persist;
        out->peak_reserved_bytes = ctx->arena.peak_reserved + persist;
        out->peak_active_bytes = ctx->arena.peak_active + persist;
        out->alloc_count = ctx->arena.alloc_count;
        out->reuse_count = ctx->arena.reuse_count;
        out->release_count = ctx->arena.release_count;
        out->utilization = out->peak_reserved_bytes ? static_cast<double>(out->peak_active_bytes) / out->peak_reserved_bytes : 1.0;
    });
}

int gsrc_high_water_reset(gsrc_ctx* ctx) {
    return guarded(ctx, [&] {
        ctx->arena.peak_active = ctx->arena.used;
        ctx->arena.peak_reserved = ctx->arena.reserved;
    });
}

int gsrc_kernel_launches(gsrc_ctx* ctx, int64_t* out) { return guarded(ctx, [&] { *out = ctx->launches; }); }
int gsrc_work_counter(gsrc_ctx* ctx, uint64_t* scalar_mul_adds, uint64_t* rows_touched) {
    return guarded(ctx, [&] {
        if (scalar_mul_adds) *scalar_mul_adds = ctx->work_ma;
        if (rows_touched) *rows_touched = ctx->work_rows;
    });
}
int gsrc_work_reset(gsrc_ctx* ctx) { return guarded(ctx, [&] { ctx->work_ma = ctx->work_rows = 0; }); }

int gsrc_layer_forward(gsrc_ctx* ctx, int layer) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (layer < 0 || layer >= ctx->cfg.layers) cfg_err("layer out of range");
        ctx->layer_forward(layer);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += ctx->work_layer_fwd();
    });
}
int gsrc_layer_inverse(gsrc_ctx* ctx, int layer) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (layer < 0 || layer >= ctx->cfg.layers) cfg_err("layer out of range");
        if (ctx->cfg.mode == GSRC_MODE_ALG12) cfg_err("Alg. 1 layers are not invertible (use GSRC or REV)");
        ctx->rev_layer_inverse(layer);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += ctx->work_layer_fwd();  // the inverse re-applies every block
    });
}
int gsrc_layer_backward(gsrc_ctx* ctx, int layer) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (layer < 0 || layer >= ctx->cfg.layers) cfg_err("layer out of range");
        ctx->layer_backward(layer);
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += ctx->work_layer_bwd();
    });
}

// ---- op-level parity entry points ----------------------------------------------
int gsrc_op_gs_topk(gsrc_ctx* ctx, int64_t n, int w, int k, const float* x, float* vals, int32_t* idx) {
    return guarded(ctx, [&] {
        if (w < 1 || w > 128) cfg_err("gs_topk: width must be in [1, 128]");
        if (k < 1 || k > w) cfg_err("gs_topk: k=" + std::to_string(k) + " out of [1," + std::to_string(w) + "]");
        if (n <= 0) return;
        const int ld = pad_ld(w);
        DevBuf dx(static_cast<size_t>(n) * ld * sizeof(float)), drec(static_cast<size_t>(n) * rec_bytes(k));
        CK(cudaMemcpy2DAsync(dx.p, ld * sizeof(float), x, w * sizeof(float), w * sizeof(float), n, cudaMemcpyHostToDevice, ctx->stream));
        GsArgs g;
        g.n = static_cast<int>(n); g.w = w; g.ld = ld; g.k = k; g.planes[0] = dx.as<float>(); g.nplanes = 1; g.rec = drec.as<uint8_t>();
        // the fast path's GS (thread-per-row selection over TMA tiles) serves every
        // shape it supports, so the SPEC tie / zero / padding cases pin it bit-exactly
        if (w <= 64 && k <= 16) {
            CK(encode_plane_map(&g.maps[0], g.planes[0], static_cast<int>(n), ld));
            CK(launch_gs_tma(g, ctx->stream));
        } else {
            CK(launch_gs(g, ctx->stream));
        }
        ++ctx->launches;
        download_records(drec.as<uint8_t>(), n, k, vals, idx, ctx->stream);
    });
}

int gsrc_op_spmm(gsrc_ctx* ctx, int transpose, int cols, const float* x, float* y) {
    return guarded(ctx, [&] {
        if (ctx->n <= 0) seq_err("no graph uploaded");
        if (cols < 1 || cols > 128) cfg_err("spmm: cols must be in [1, 128]");
        const int64_t n = ctx->n;
        const int ld = pad_ld(cols);
        DevBuf dx(static_cast<size_t>(n) * ld * 4), dy(static_cast<size_t>(n) * ld * 4);
        CK(cudaMemcpy2DAsync(dx.p, ld * 4, x, cols * 4, cols * 4, n, cudaMemcpyHostToDevice, ctx->stream));
        TileArgs a;
        a.n = static_cast<int>(n); a.w = cols; a.ld = ld;
        a.agg = AGG_DENSE; a.dir = transpose ? ctx->bwd() : ctx->fwd(); a.x_in = dx.as<float>();
        a.gemm = GEMM_NONE; a.epi = EPI_NONE; a.out = dy.as<float>();
        ctx->run_tile(a);
        CK(cudaMemcpy2DAsync(y, cols * 4, dy.p, ld * 4, cols * 4, n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += static_cast<uint64_t>(ctx->e) * cols;
        ctx->work_rows += static_cast<uint64_t>(n);
    });
}

int gsrc_op_spmm_sparse(gsrc_ctx* ctx, int transpose, int w, int k, const float* vals, const int32_t* idx, float* y) {
    return guarded(ctx, [&] {
        if (ctx->n <= 0) seq_err("no graph uploaded");
        if (w < 1 || w > 128 || k < 1 || k > w) cfg_err("spmm_sparse: bad width / k");
        const int64_t n = ctx->n;
        check_rec_idx(idx, n, k, w);
        const int ld = pad_ld(w);
        DevBuf drec(static_cast<size_t>(n) * rec_bytes(k)), dy(static_cast<size_t>(n) * ld * 4);
        upload_records(vals, idx, n, k, drec.as<uint8_t>(), ctx->stream);
        TileArgs a;
        a.n = static_cast<int>(n); a.w = w; a.ld = ld;
        a.agg = AGG_SPARSE; a.dir = transpose ? ctx->bwd() : ctx->fwd(); a.rec_in = drec.as<uint8_t>(); a.k_in = k;
        a.gemm = GEMM_NONE; a.epi = EPI_NONE; a.out = dy.as<float>();
        ctx->run_tile(a);
        CK(cudaMemcpy2DAsync(y, w * 4, dy.p, ld * 4, w * 4, n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->work_ma += static_cast<uint64_t>(ctx->e) * k;
        ctx->work_rows += static_cast<uint64_t>(n);
    });
}

int gsrc_op_block_forward(gsrc_ctx* ctx, int w, int k, const float* vals, const int32_t* idx, const float* W, const float* b,
                          int use_weight, int use_bias, int epilogue, const float* R, const float* rvals, const int32_t* ridx,
                          float* out, int gs_k, float* gs_vals, int32_t* gs_idx) {
    return guarded(ctx, [&] {
        if (ctx->n <= 0) seq_err("no graph uploaded");
        if (w < 1 || w > 128 || k < 1 || k > w) cfg_err("block_forward: bad width / k");
        if (epilogue < 0 || epilogue > EPI_SCATTER_SUB) cfg_err("block_forward: bad epilogue");
        if (gs_k < 0 || gs_k > w) cfg_err("block_forward: bad gs_k");
        const int64_t n = ctx->n;
        check_rec_idx(idx, n, k, w);
        const int ld = pad_ld(w);
        DevBuf drec(static_cast<size_t>(n) * rec_bytes(k)), dout(static_cast<size_t>(n) * ld * 4), dR(static_cast<size_t>(n) * ld * 4);
        DevBuf dW(static_cast<size_t>(w) * w * 4), db(static_cast<size_t>(w) * 4), drr(static_cast<size_t>(n) * rec_bytes(k));
        DevBuf dgs(static_cast<size_t>(n) * rec_bytes(gs_k > 0 ? gs_k : 1));
        upload_records(vals, idx, n, k, drec.as<uint8_t>(), ctx->stream);
        if (use_weight) CK(cudaMemcpyAsync(dW.p, W, static_cast<size_t>(w) * w * 4, cudaMemcpyHostToDevice, ctx->stream));
        if (use_bias) CK(cudaMemcpyAsync(db.p, b, static_cast<size_t>(w) * 4, cudaMemcpyHostToDevice, ctx->stream));
        TileArgs a;
        a.n = static_cast<int>(n); a.w = w; a.ld = ld; a.tc = ctx->op_tc;
        a.agg = AGG_SPARSE; a.dir = ctx->fwd(); a.rec_in = drec.as<uint8_t>(); a.k_in = k;
        a.gemm = use_weight ? GEMM_W : GEMM_NONE; a.Wm = dW.as<float>(); a.bias = use_bias ? db.as<float>() : nullptr;
        a.epi = epilogue; a.out = dout.as<float>();
        if (epilogue == EPI_ADD || epilogue == EPI_SUB) {
            if (!R) cfg_err("block_forward: residual required");
            CK(cudaMemcpy2DAsync(dR.p, ld * 4, R, w * 4, w * 4, n, cudaMemcpyHostToDevice, ctx->stream));
            a.R = dR.as<float>();
        }
        if (epilogue == EPI_SCATTER_ADD || epilogue == EPI_SCATTER_SUB) {
            if (!rvals || !ridx) cfg_err("block_forward: scatter residual required");
            check_rec_idx(ridx, n, k, w);
            upload_records(rvals, ridx, n, k, drr.as<uint8_t>(), ctx->stream);
            a.rrec = drr.as<uint8_t>(); a.k_r = k;
        }
        if (gs_k > 0) { a.gs_out = dgs.as<uint8_t>(); a.k_gs = gs_k; }
        ctx->run_tile(a);
        CK(cudaMemcpy2DAsync(out, w * 4, dout.p, ld * 4, w * 4, n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (gs_k > 0) download_records(dgs.as<uint8_t>(), n, gs_k, gs_vals, gs_idx, ctx->stream);
        ctx->work_ma += ctx->work_block_fwd(w, k, use_weight != 0);
    });
}

int gsrc_op_dense_block(gsrc_ctx* ctx, int w, const float* x, const float* W, const float* b, int use_weight, int use_bias, float* out) {
    return guarded(ctx, [&] {
        if (ctx->n <= 0) seq_err("no graph uploaded");
        if (w < 1 || w > 128) cfg_err("dense_block: bad width");
        const int64_t n = ctx->n;
        const int ld = pad_ld(w);
        DevBuf dx(static_cast<size_t>(n) * ld * 4), dout(static_cast<size_t>(n) * ld * 4), dW(static_cast<size_t>(w) * w * 4), db(static_cast<size_t>(w) * 4);
        CK(cudaMemcpy2DAsync(dx.p, ld * 4, x, w * 4, w * 4, n, cudaMemcpyHostToDevice, ctx->stream));
        if (use_weight) CK(cudaMemcpyAsync(dW.p, W, static_cast<size_t>(w) * w * 4, cudaMemcpyHostToDevice, ctx->stream));
        if (use_bias) CK(cudaMemcpyAsync(db.p, b, static_cast<size_t>(w) * 4, cudaMemcpyHostToDevice, ctx->stream));
        TileArgs a;
        a.n = static_cast<int>(n); a.w = w; a.ld = ld; a.tc = ctx->op_tc;
        a.agg = AGG_DENSE_RELU; a.dir = ctx->fwd(); a.x_in = dx.as<float>();
        a.gemm = use_weight ? GEMM_W : GEMM_NONE; a.Wm = dW.as<float>(); a.bias = use_bias ? db.as<float>() : nullptr;
        a.epi = EPI_NONE; a.out = dout.as<float>();
        ctx->run_tile(a);
        CK(cudaMemcpy2DAsync(out, w * 4, dout.p, ld * 4, w * 4, n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_op_block_backward(gsrc_ctx* ctx, int w, int k, const float* m, const int32_t* isrc, const float* fvals, const int32_t* fidx,
                           const float* W, int use_weight, int use_bias, float* out, float* dW, float* db) {
    return guarded(ctx, [&] {
        if (ctx->n <= 0) seq_err("no graph uploaded");
        if (w < 1 || w > 128 || k < 1 || k > w) cfg_err("block_backward: bad width / k");
        const int64_t n = ctx->n;
        check_rec_idx(isrc, n, k, w);
        check_rec_idx(fidx, n, k, w);
        const int ld = pad_ld(w);
        const int grid = tile_grid_max(static_cast<int>(n));
        const size_t plen = static_cast<size_t>(w) * w + w;
        DevBuf dm(static_cast<size_t>(n) * ld * 4), dout(static_cast<size_t>(n) * ld * 4), dWm(static_cast<size_t>(w) * w * 4);
        DevBuf rsrc(static_cast<size_t>(n) * rec_bytes(k)), rfwd(static_cast<size_t>(n) * rec_bytes(k)), rvg(static_cast<size_t>(n) * rec_bytes(k));
        DevBuf part(grid * plen * sizeof(double)), dgrad(plen * 4);
        std::vector<float> zeros(static_cast<size_t>(n) * k, 0.f);
        CK(cudaMemcpy2DAsync(dm.p, ld * 4, m, w * 4, w * 4, n, cudaMemcpyHostToDevice, ctx->stream));
        if (use_weight) CK(cudaMemcpyAsync(dWm.p, W, static_cast<size_t>(w) * w * 4, cudaMemcpyHostToDevice, ctx->stream));
        upload_records(zeros.data(), isrc, n, k, rsrc.as<uint8_t>(), ctx->stream);
        upload_records(fvals, fidx, n, k, rfwd.as<uint8_t>(), ctx->stream);
        TileArgs a;
        a.n = static_cast<int>(n); a.w = w; a.ld = ld;
        a.agg = AGG_NONE; a.x_in = dm.as<float>(); a.gemm = use_weight ? GEMM_WT : GEMM_NONE; a.Wm = dWm.as<float>();
        a.epi = EPI_GATHER_REC; a.rrec = rsrc.as<uint8_t>(); a.k_r = k; a.out_rec = rvg.as<uint8_t>();
        ctx->run_tile(a);
        TileArgs b;
        b.n = static_cast<int>(n); b.w = w; b.ld = ld;
        b.agg = AGG_SPARSE; b.dir = ctx->bwd(); b.rec_in = rvg.as<uint8_t>(); b.k_in = k; b.gemm = GEMM_NONE;
        b.epi = EPI_NONE; b.out = dout.as<float>();
        ctx->run_tile(b);
        TileArgs c;
        c.n = static_cast<int>(n); c.w = w; c.ld = ld;
        c.agg = AGG_SPARSE; c.dir = ctx->fwd(); c.rec_in = rfwd.as<uint8_t>(); c.k_in = k; c.gemm = GEMM_NONE;
        c.epi = EPI_DISCARD; c.G = dm.as<float>(); c.want_db = use_bias; c.part = part.as<double>();
        ctx->run_tile(c);
        CK(launch_reduce_parts(part.as<double>(), ctx->last_grid, static_cast<int>(plen), static_cast<int>(plen), dgrad.as<float>(), 0, ctx->stream));
        CK(cudaMemcpy2DAsync(out, w * 4, dout.p, ld * 4, w * 4, n, cudaMemcpyDeviceToHost, ctx->stream));
        std::vector<float> g(plen);
        CK(cudaMemcpyAsync(g.data(), dgrad.p, plen * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (dW) for (size_t i = 0; i < static_cast<size_t>(w) * w; ++i) dW[i] = use_weight ? g[i] : 0.f;
        if (db) for (int j = 0; j < w; ++j) db[j] = use_bias ? g[static_cast<size_t>(w) * w + j] : 0.f;
        ctx->work_ma += ctx->work_block_bwd(w, k, use_weight != 0);
    });
}

// Live per-kernel timing for the roofline report (bench.py): each GSR-C kernel
// class is launched `reps` times per block on the context stream between CUDA
// events with the real step's arguments (layer 0, every block i = 0..C-1).
// out[c*4 + 0..3] = ms per launch (mean over the blocks), algorithmic bytes per
// launch, launches per training step, flops per launch; out[16 + c*C + i] = ms
// per launch of block i (classes 0..2). Classes: 0 fused forward block, 1
// backward recompute block (fast sweep: with its GS epilogue for blocks
// 0..C-2), 2 backward input-gradient block (+dW; block 0 adds into C-1
// planes), 3 GS of the group sum. The activation arena is snapshotted first and
// restored afterwards, so the call leaves every device buffer as it found it.
int gsrc_profile_kernels(gsrc_ctx* ctx, int reps, double* out) {
    return guarded(ctx, [&] {
        ctx->require_data();
        if (ctx->cfg.mode != GSRC_MODE_GSRC) cfg_err("profile: GSRC mode only");
        if (reps < 1) cfg_err("profile: reps < 1");
        const double n = static_cast<double>(ctx->n), e = static_cast<double>(ctx->e), w = ctx->w, k = ctx->k, L = ctx->cfg.layers, C = ctx->C;
        const double rb = rec_bytes(ctx->k), csr = 4.0 * (n + 1) + 4.0 * e;
        const int l = 0, nC = ctx->C;
        // snapshot of the arena (activations, gradients, records, partials)
        void* snap = nullptr;
        const size_t used = ctx->arena.used;
        CK(cudaStreamSynchronize(ctx->stream));
        if (cudaMalloc(&snap, used) != cudaSuccess) {
            cudaGetLastError();
            throw Fail(GSRC_ERR_RESOURCE, "profile: no device memory for the arena snapshot (" + std::to_string(used) + " bytes)");
        }
        struct Restore {
            gsrc_ctx* c; void* p; size_t b;
            ~Restore() {
                cudaMemcpyAsync(c->arena.base, p, b, cudaMemcpyDeviceToDevice, c->stream);
                cudaStreamSynchronize(c->stream);
                cudaFree(p);
            }
        } restore{ctx, snap, used};
        CK(cudaMemcpyAsync(snap, ctx->arena.base, used, cudaMemcpyDeviceToDevice, ctx->stream));
        for (int q = 0; q < 16 + 3 * nC; ++q) out[q] = 0.0;
        ctx->run_gs({ctx->plane(ctx->X, 0)}, ctx->recA);
        auto time_it = [&](const std::function<void()>& f) {
            f();  // warm
            CK(cudaEventRecord(ctx->ev[2], ctx->stream));
            for (int r = 0; r < reps; ++r) f();
            CK(cudaEventRecord(ctx->ev[3], ctx->stream));
            CK(cudaEventSynchronize(ctx->ev[3]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]));
            return static_cast<double>(ms) / reps;
        };
        auto per_block = [&](int cls, const std::function<void(int)>& f) {
            double sum = 0.0;
            for (int i = 0; i < nC; ++i) {
                const double ms = time_it([&] { f(i); });
                out[16 + cls * nC + i] = ms;
                sum += ms;
            }
            out[cls * 4] = sum / nC;
        };
        const bool fp = ctx->fast() && ctx->cfg.use_weight;
        if (fp) {
            // the three fast-path block kernels, each with its hub-row pre-pass
            per_block(0, [&](int i) { ctx->fast_block_forward(l, i, ctx->recA, i + 1 < nC ? ctx->recB : nullptr); });
            // INV as the backward sweep runs it: blocks 0..C-2 write the lower layer's records
            per_block(1, [&](int i) { ctx->fast_inverse(l, i, ctx->recA, i <= nC - 2 ? ctx->recB : nullptr); });
            per_block(2, [&](int i) { ctx->fast_input_grad(l, i, ctx->recA); });
        } else {
            per_block(0, [&](int i) {
                TileArgs fa = ctx->tile_base();
                fa.agg = AGG_SPARSE; fa.dir = ctx->fwd(); fa.rec_in = ctx->recA; fa.k_in = ctx->k;
                fa.gemm = ctx->cfg.use_weight ? GEMM_W : GEMM_NONE; fa.Wm = ctx->Wb(l, i); fa.bias = ctx->Bb(l, i);
                fa.epi = EPI_ADD; fa.R = ctx->plane(ctx->X, i); fa.out = ctx->plane(ctx->X, i);
                if (i + 1 < nC) { fa.gs_out = ctx->recB; fa.k_gs = ctx->k; }
                ctx->run_tile(fa);
            });
            per_block(1, [&](int i) {
                TileArgs ra = ctx->tile_base();
                ra.agg = AGG_SPARSE; ra.dir = ctx->fwd(); ra.rec_in = ctx->recA; ra.k_in = ctx->k;
                ra.gemm = ctx->cfg.use_weight ? GEMM_W : GEMM_NONE; ra.Wm = ctx->Wb(l, i); ra.bias = ctx->Bb(l, i);
                ra.epi = EPI_SUB; ra.R = ctx->plane(ctx->X, i); ra.out = ctx->plane(ctx->X, i);
                ra.G = ctx->plane(ctx->G, i); ra.want_db = ctx->cfg.use_bias; ra.part = ctx->part;
                ctx->run_tile(ra);
            });
            per_block(2, [&](int i) {
                TileArgs ba = ctx->tile_base();
                ba.agg = AGG_DENSE; ba.dir = ctx->bwd(); ba.x_in = ctx->plane(ctx->G, i);
                ba.gemm = ctx->cfg.use_weight ? GEMM_WT : GEMM_NONE; ba.Wm = ctx->Wb(l, i);
                ba.epi = EPI_MASKED_ADD; ba.rrec = ctx->recA; ba.k_r = ctx->k;
                if (i > 0) { ba.dst[0] = ctx->plane(ctx->G, i - 1); ba.ndst = 1; }
                else { for (int p = 1; p < nC; ++p) ba.dst[p - 1] = ctx->plane(ctx->G, p); ba.ndst = nC - 1; }
                ctx->run_tile(ba);
            });
        }
        // algorithmic bytes per launch; BIN's block 0 updates C-1 planes
        out[1] = csr + 2 * n * rb + 8 * n * w;
        out[2] = L * C;
        out[3] = 2 * n * w * w;
        out[5] = fp ? csr + 2 * n * rb + 8 * n * w   // fast path: dW rides on BIN; records out
                    : csr + n * rb + 12 * n * w;
        out[6] = L * C;
        out[7] = 4 * n * w * w;
        out[9] = csr + 4 * n * w + n * rb + 8 * n * k * (1.0 + (C - 2) / C);  // block 0 writes C-1 planes: mean over blocks
        out[10] = L * C;
        out[11] = 2 * n * w * w;
        out[12] = time_it([&] { ctx->run_gs_groupsum(ctx->X, ctx->recB); });
        out[13] = (C - 1) * 4 * n * w + n * rb;
        out[14] = ctx->fast_sweep() ? 2 * L : L * (C + 1);  // fast sweep: the group sums only (+ C-1 single planes once)
        out[15] = 0;
    });
}

int gsrc_set_residual_quant(gsrc_ctx* ctx, int shift) {
    return guarded(ctx, [&] {
        if (shift < 0 || shift > 30) cfg_err("residual quant: shift must be in [0, 30] (0 = off)");
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->qshift = shift;
        ctx->drop_graphs();
    });
}

int gsrc_get_residual_quant(gsrc_ctx* ctx, int* shift) { return guarded(ctx, [&] { *shift = ctx->qshift; }); }

int gsrc_get_stream(gsrc_ctx* ctx, void** out) {
    return guarded(ctx, [&] {
        if (!out) cfg_err("get_stream: null out");
        *out = static_cast<void*>(ctx->stream);
    });
}

// ---- optimizer state (exact resume: Adam m, v and the step count) -------------
int gsrc_optim_state_get(gsrc_ctx* ctx, float* m, float* v, int64_t* step, int64_t n) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (n != ctx->P) cfg_err("optim_state_get: expected " + std::to_string(ctx->P) + " values");
        long long t = 0;
        if (m) CK(cudaMemcpyAsync(m, ctx->opt_m, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
        if (v) CK(cudaMemcpyAsync(v, ctx->opt_v, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&t, ctx->d_step, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (step) *step = t;
    });
}

int gsrc_optim_state_set(gsrc_ctx* ctx, const float* m, const float* v, int64_t step, int64_t n) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (n != ctx->P) cfg_err("optim_state_set: expected " + std::to_string(ctx->P) + " values");
        if (step < 0) cfg_err("optim_state_set: step < 0");
        const long long t = step;
        if (m) CK(cudaMemcpyAsync(ctx->opt_m, m, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        if (v) CK(cudaMemcpyAsync(ctx->opt_v, v, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->d_step, &t, sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

// ---- data parallelism (SURVEY.md §8b "DP", §8e) --------------------------------
int gsrc_comm_unique_id(void* out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return GSRC_ERR_CONFIG;
    const NcclApi& a = nccl_api();
    if (!a.ok()) return GSRC_ERR_RESOURCE;
    ncclUniqueId id;
    if (a.get_unique_id(&id) != ncclSuccess) return GSRC_ERR_RESOURCE;
    std::memcpy(out, &id, sizeof id);
    return GSRC_OK;
}

int gsrc_comm_init(gsrc_ctx* ctx, const void* unique_id, int nranks, int rank) {
    return guarded(ctx, [&] {
        if (!unique_id) cfg_err("comm_init: null unique id");
        if (nranks < 1 || rank < 0 || rank >= nranks) cfg_err("comm_init: bad nranks / rank");
        const NcclApi& a = nccl_or_throw();
        if (ctx->comm) { a.comm_destroy(ctx->comm); ctx->comm = nullptr; }
        ncclUniqueId id;
        std::memcpy(&id, unique_id, sizeof id);
        CK(cudaStreamSynchronize(ctx->stream));
        nccl_check(a.comm_init_rank(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
        ctx->comm_ranks = nranks;
        ctx->comm_rank = rank;
    });
}

int gsrc_comm_allreduce_grads(gsrc_ctx* ctx) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (!ctx->comm) seq_err("comm_allreduce_grads: no communicator (gsrc_comm_init)");
        ctx->enqueue_allreduce();
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int gsrc_comm_destroy(gsrc_ctx* ctx) {
    return guarded(ctx, [&] {
        if (ctx->comm) {
            CK(cudaStreamSynchronize(ctx->stream));
            nccl_api().comm_destroy(ctx->comm);
            ctx->comm = nullptr;
        }
        ctx->comm_ranks = 1;
        ctx->comm_rank = 0;
    });
}

// ---- reconstruction diagnostics -------------------------------------------------
int gsrc_diag_masks(gsrc_ctx* ctx, int enable, int row_stride) {
    return guarded(ctx, [&] {
        ctx->require_model();
        if (enable && ctx->cfg.mode != GSRC_MODE_GSRC) cfg_err("diag_masks: GSRC mode only");
        if (enable && row_stride < 1) cfg_err("diag_masks: row_stride < 1");
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->diag_store) { cudaFree(ctx->diag_store); ctx->diag_store = nullptr; }
        if (ctx->diag_cnt) { cudaFree(ctx->diag_cnt); ctx->diag_cnt = nullptr; }
        ctx->diag = false;
        ctx->drop_graphs();
        if (!enable) return;
        ctx->diag_stride = row_stride;
        ctx->diag_rows = (ctx->n + row_stride - 1) / row_stride;
        const size_t slots = static_cast<size_t>(ctx->cfg.layers) * ctx->C;
        ctx->diag_store = dmalloc<uint4>(slots * static_cast<size_t>(ctx->diag_rows));
        ctx->diag_cnt = dmalloc<unsigned long long>(slots);
        CK(cudaMemset(ctx->diag_cnt, 0, sizeof(unsigned long long) * slots));
        ctx->diag = true;
    });
}

int gsrc_diag_mask_flips(gsrc_ctx* ctx, int64_t* flips, int64_t* sampled_rows) {
    return guarded(ctx, [&] {
        if (!ctx->diag) seq_err("diag_mask_flips: diagnostics not enabled (gsrc_diag_masks)");
        const size_t slots = static_cast<size_t>(ctx->cfg.layers) * ctx->C;
        std::vector<unsigned long long> h(slots);
        CK(cudaMemcpyAsync(h.data(), ctx->diag_cnt, sizeof(unsigned long long) * slots, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (size_t q = 0; q < slots; ++q) flips[q] = static_cast<int64_t>(h[q]);
        if (sampled_rows) *sampled_rows = ctx->diag_rows;
    });
}

}  // extern "C"
