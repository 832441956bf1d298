// GSR-GNN B200 kernels — shared declarations between kernels.cu and capi.cu.
//
// Device data layout:
//   * activations / gradients: C planes, each n × ld floats (ld = w rounded
//     up to 4; padding columns are kept at 0), plane p = group p. split /
//     concat are zero-cost.
//   * compressed embeddings ("CBSR" SparseActivation): one
//     packed record per node: k u8 column indices (ascending) padded to 16 B,
//     then k f32 values; record stride rec_bytes(k) (16 B multiple) so a
//     neighbour gather is one contiguous ≤ 80 B read at k = 16.
//   * graph: int32 CSR and its transpose (CSR of Aᵀ, sources ascending), and
//     per-node row/column normalisation factors (Â = diag(row_f)·A·diag(col_f)).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace gsrk {

constexpr int kThreads = 256;
constexpr int kTileRows = 128;
constexpr int kAggSeg = 8;  // canonical aggregation segment (== oracle kAggSeg, tile::kSeg)

__host__ __device__ inline int rec_kh(int k) { return (k + 15) & ~15; }
__host__ __device__ inline int rec_bytes(int k) { return (rec_kh(k) + 4 * k + 15) & ~15; }
__host__ __device__ inline int pad_ld(int w) { return (w + 3) & ~3; }

// One aggregation direction.
//   forward:   y[r] = row_f[r] · Σ_{c∈CSR(r)}  col_f[c] · x[c]
//   transpose: y[r] = col_f[r] · Σ_{c: r∈CSR(c)} row_f[c] · x[c]
struct Dir {
    const int* ptr = nullptr;
    const int* idx = nullptr;
    const float* out_f = nullptr;
    const float* edge_f = nullptr;
    int unit_edge = 0;   // edge_f ≡ 1 (multiplication by 1 is exact: skipped)
    // fast path: kAggSeg {neighbour, edge scale bits} slots per row in CSR order,
    // −1 padding after the last edge; a row with > kAggSeg edges (hub) has −2 in
    // slot 0. Row-addressed, so a tile's neighbour ids need no row_ptr → col_idx →
    // edge_f chain of dependent loads.
    const int2* ell = nullptr;
};

enum Agg : int { AGG_SPARSE = 0, AGG_DENSE = 1, AGG_DENSE_RELU = 2, AGG_NONE = 3 };
enum Gemm : int { GEMM_NONE = 0, GEMM_W = 1, GEMM_WT = 2 };
enum Epi : int {
    EPI_NONE = 0,          // out = h
    EPI_ADD = 1,           // out = R + h
    EPI_SUB = 2,           // out = R - h
    EPI_SCATTER_ADD = 3,   // out = scatter(rrec) + h
    EPI_SCATTER_SUB = 4,   // out = scatter(rrec) - h
    EPI_MASKED_ADD = 5,    // dst_p[c] += h[c] for c in mask(rrec)        (p over ndst planes)
    EPI_MASKED_ADD_RELU = 6,  // dst_p[c] += h[c] where mask_plane[c] > 0
    EPI_GATHER_REC = 7,    // out_rec = (idx of rrec, h at those idx)
    EPI_DISCARD = 8,       // no output (dW/db side-products only)
};

constexpr int kMaxDst = 8;

// One fused tile kernel launch: aggregation → transform → epilogue
// (→ GS of the output) (→ dW/db partials). See kernels.cu.
struct TileArgs {
    int n = 0, w = 0, ld = 0;
    int agg = AGG_SPARSE;
    Dir dir;
    const std::uint8_t* rec_in = nullptr;  // AGG_SPARSE input records
    int k_in = 0;
    const float* x_in = nullptr;           // AGG_DENSE* / AGG_NONE input plane
    int gemm = GEMM_W;
    const float* Wm = nullptr;             // w×w row-major
    const float* bias = nullptr;           // nullptr → no bias
    int epi = EPI_NONE;
    const float* R = nullptr;              // residual plane (EPI_ADD/SUB)
    const std::uint8_t* rrec = nullptr;    // records for scatter / mask / gather epilogues
    int k_r = 0;
    const float* mask_plane = nullptr;     // EPI_MASKED_ADD_RELU
    float* out = nullptr;                  // output plane (may alias R)
    float* dst[kMaxDst] = {};              // EPI_MASKED_ADD destinations
    int ndst = 0;
    std::uint8_t* out_rec = nullptr;       // EPI_GATHER_REC output records
    std::uint8_t* gs_out = nullptr;        // GS(out) records (k_gs)
    int k_gs = 0;
    const float* G = nullptr;              // dW partial: dW += Zᵀ G, db += colsum(G)
    int want_db = 0;
    double* part = nullptr;                // [gridDim.x][w*w + w]
    int tc = 0;                            // 1: transform on tcgen05 (TF32), 0: FP32-strict FFMA
    float qs = 0.f, qi = 0.f;              // EPI_ADD / EPI_SUB: residual-stream grid 2^-s (dev::quant); 0 = off
};

// Thread-per-row tcgen05 fast path (fast.cu) for the GSR-C step in TF32 mode.
// kind: 0 FWD (out = R + h, GS(out) → gs_out), 1 INV (out = R − h),
// 2 BIN (dst_p[r, I_m[r]] += h[r, I_m[r]], h = (Âᵀ·x_in)·Wᵀ; dW partials
// += scatter(mrec)ᵀ·(Âᵀ·x_in)).
struct FastArgs {
    int n = 0, w = 0, ld = 0, k = 0;       // k: records of rec_in
    Dir dir;
    const std::uint8_t* rec_in = nullptr;  // FWD / INV aggregation input
    const float* x_in = nullptr;           // BIN aggregation input (dense plane)
    float* Zh = nullptr;                   // hub-row aggregates (n × ld), written by k_hub
    const float* Wm = nullptr;
    const float* bias = nullptr;
    int gemm_t = 0;                        // 0: h = Z·W, 1: h = Z·Wᵀ
    const float* R = nullptr;
    float* out = nullptr;                  // FWD / INV: out aliases R (in place), moved by TMA through tm_x
    std::uint8_t* gs_out = nullptr;        // FWD / INV: GS_k of the output rows (the next block's, or the lower layer's, records)
    int k_gs = 0;
    double* part = nullptr;                // BIN: dW partials [grid][w*w + w]
    const std::uint8_t* mrec = nullptr;    // BIN: mask records
    int k_m = 0;
    float* dst[kMaxDst] = {};
    int ndst = 0;
    CUtensorMap tm_x;                      // FWD / INV: 2-D tiled map of the R/out plane (128 rows × 32 cols, SWIZZLE_128B)
    CUtensorMap tm_dst[kMaxDst];           // BIN: maps of the dst planes (TMA reduce-add of the masked gradient tile)
    float qs = 0.f, qi = 0.f;              // FWD / INV: residual-stream grid 2^-s (dev::quant); 0 = off
    // rev-baseline (dense_block SPEC.md:244-252): FWD / INV aggregate Â·relu(x_in)
    // (dense rows, ld) instead of records; BIN takes S = relu(u) and the mask
    // u > 0 from the dense rows of mplane instead of mrec; the dense hub
    // pre-pass applies relu to its input rows when relu is set
    int dense = 0;
    int relu = 0;
    const float* mplane = nullptr;
};

bool fast_supported(int w, int k);
int fast_bin_grid_max();  // largest BIN grid (dW partial slots) of the fast path
// TMA map of an n × ld fp32 plane in 128-row × 32-column boxes, SWIZZLE_128B
// (the boxes land in exactly the UMMA K-major SW128 tile layout of fast.cu).
cudaError_t encode_plane_map(CUtensorMap* m, const float* base, int n, int ld);
cudaError_t init_fast_attributes();
cudaError_t launch_fast(int kind, const FastArgs& a, cudaStream_t s, int* grid_out);
// hub rows of the fast path. Sparse (forward direction): work items of two
// int4 each, {row, first edge, end edge, first segment of the chunk}, {hub
// index, the row's first partial in Pseg}; chunks of kHubChunk segments;
// cnt[nhub] zeroed (left zeroed by every launch). Dense (transpose): the
// flattened segment list {lo, hi} of all hub rows, then a fold per hub row.
constexpr int kHubChunk = 64;
cudaError_t launch_hub_rows(const FastArgs& a, const int4* items, int nitem, int* cnt, float* Pseg, cudaStream_t s);
cudaError_t launch_hub_dense(const FastArgs& a, const int2* segs, int nseg, const int* rows, const int* seg_off, int nhub, float* Pseg,
                             cudaStream_t s);
cudaError_t launch_colsum(const float* G, int n, int w, int ld, double* part, int* grid_out, cudaStream_t s);

// GS top-k of (sum of) planes: u = p0 + p1 + ... (left to right), records out.
struct GsArgs {
    int n = 0, w = 0, ld = 0, k = 0;
    const float* planes[kMaxDst] = {};
    int nplanes = 1;
    std::uint8_t* rec = nullptr;
    CUtensorMap maps[kMaxDst];  // launch_gs_tma: TMA maps of the planes
};

// GS top-k of (a left-to-right sum of) planes, thread per row over TMA-loaded
// tiles (fast.cu; w ≤ 64, k ≤ 16)
cudaError_t launch_gs_tma(const GsArgs& a, cudaStream_t s);


// Host launchers (kernels.cu). All enqueue on `s` and return cudaError_t.
cudaError_t launch_tile(const TileArgs& a, cudaStream_t s, int* grid_out);  // grid = SMs × occupancy
cudaError_t launch_gs(const GsArgs& a, cudaStream_t s);
int tile_grid_max(int n);      // upper bound of any tile launch's grid (partial-buffer sizing)
cudaError_t init_kernel_attributes();  // opt-in dynamic smem for every k_tile instantiation
cudaError_t launch_reduce_parts(const double* part, int nparts, int stride, int len, float* out, int accumulate, cudaStream_t s);
cudaError_t launch_sum_double(const double* in, int n, double scale, double* out, cudaStream_t s);
cudaError_t launch_sum_planes(const GsArgs& a, float* out, cudaStream_t s);
cudaError_t launch_adam_prep(long long* t, double b1, double b2, float* bc, cudaStream_t s);

// mask-flip diagnostic: store (mode 0) or compare-and-count (mode 1) the index
// bytes of the GS records of rows r = j·stride
cudaError_t launch_diag_masks(const std::uint8_t* rec, int n, int stride, int rb, uint4* store, int mode, unsigned long long* counter,
                              cudaStream_t s);

// records <-> host-layout helpers (parity entry points)
cudaError_t launch_rec_unpack(const std::uint8_t* rec, int n, int k, float* vals, int* idx, cudaStream_t s);
cudaError_t launch_rec_pack(const float* vals, const int* idx, int n, int k, std::uint8_t* rec, cudaStream_t s);

// encoder / head / loss / optimizer
cudaError_t launch_encoder(const float* X0, int n, int d_in, const float* We, const float* be, int D, int C, int w, int ld,
                           float* X, float qs, float qi, cudaStream_t s);
cudaError_t launch_head_loss(const float* X, int n, int D, int C, int w, int ld, const float* wh, const float* bh,
                             const float* y, const std::uint8_t* mask, float inv_cnt_unused, float cnt, float* yhat, float* gy,
                             double* loss_part, int nparts, cudaStream_t s);
cudaError_t launch_head_bwd(const float* X, const float* gy, int n, int D, int C, int w, int ld, const float* wh, float* G,
                            double* part, int nparts, cudaStream_t s);
cudaError_t launch_encoder_bwd(const float* X0, const float* G, int n, int d_in, int D, int C, int w, int ld, double* part,
                               int nparts, cudaStream_t s);
cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2, float eps,
                        float wd, const float* bc, cudaStream_t s);
cudaError_t launch_sgd(float* p, const float* g, float* mom, long long n, float lr, float momentum, cudaStream_t s);
cudaError_t launch_scale(float* p, long long n, float s_, cudaStream_t s);

}  // namespace gsrk
