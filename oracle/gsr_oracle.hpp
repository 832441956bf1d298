// =============================================================================
// GSR-GNN CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// This is a from-scratch CPU restatement of the reference's behavioural spec
// and the paper's Algorithms 1-2
// and Eq. 6-7.
// The reference ships no implementation, so this oracle is the
// parity anchor. It is pinned against every golden vector the SPEC holds
// (tests/golden/spec_vectors.json, tests/test_oracle_golden.py).
//
// It is the CHECKER, never the thing measured or shipped: only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it. The product (paper_2603_27156_b200/csrc) never links it.
//
// Arithmetic contract ("FP32 strict mode", shared with the CUDA kernels so
// that top-k masks and CSR indexing match bit-exactly):
//   * aggregation: a row's edge list (CSR order forward,
//     ascending source order for the transpose) is cut into consecutive
//     segments of kAggSeg = 8 edges; each segment sums acc_s = acc_s +
//     (edge_scale * x) from +0 in list order; the row total folds the
//     segment sums left to right (acc = acc_0, acc = acc + acc_s), then
//     y = row_scale * acc. Rows of degree ≤ 8 are plain sequential sums. The
//     segmentation is the deterministic merge order SPEC.md:128 allows; it lets
//     the GPU split hub rows (">8000 neighbours") over many lanes
//     while staying bit-identical to this oracle;
//   * dense transform: out = fma-chain over the contraction index ascending,
//     starting from +0, then + bias;
//   * residual epilogues are one IEEE add/sub each in the order written in
//     Eq. 6-7 / Alg. 1-2;
//   * reductions over rows (dW, db, losses) accumulate in double in fixed
//     row-chunk order; they are compared within tolerance, never bit-exactly.
// Built with -ffp-contract=off so the compiler cannot fuse mul+add.
// =============================================================================
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "threads.hpp"

namespace gsro {

// Error hierarchy restated from /root/reference/proj/include/gsr/common.hpp:13-35.
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : ConfigError { using ConfigError::ConfigError; };
struct FormatError : ConfigError { using ConfigError::ConfigError; };
struct SequencingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ResourceError : std::runtime_error { using std::runtime_error::runtime_error; };

// WorkCounter: scalar multiply-adds, rows touched.
struct WorkCounter {
    std::atomic<std::uint64_t> scalar_mul_adds{0};
    std::atomic<std::uint64_t> rows_touched{0};
};
inline WorkCounter& work() { static WorkCounter w; return w; }

inline ThreadPool*& pool_ref() { static ThreadPool* p = nullptr; return p; }
inline void pfor(index_t n, const std::function<void(index_t, index_t)>& fn) { parallel_for(pool_ref(), n, fn); }

enum Norm : int { NORM_NONE = 0, NORM_ROW_MEAN = 1, NORM_SYM_DEGREE = 2 };

// Per-node scale factors: Â[r][c] = row_f[r] * A[r][c] * col_f[c].
//   none:       1, 1
//   row_mean:   1/deg(r), 1               (mean aggregation)
//   sym_degree: deg(r)^-1/2, deg(c)^-1/2
// deg = CSR out-degree; isolated rows get scale 0. The same double-then-round
// expression is used by the device upload path (csrc/capi.cu).
template <typename T>
inline T norm_row_factor(int norm, index_t deg) {
    if (norm == NORM_NONE) return T(1);
    if (deg <= 0) return T(0);
    if (norm == NORM_ROW_MEAN) return static_cast<T>(1.0 / static_cast<double>(deg));
    return static_cast<T>(1.0 / std::sqrt(static_cast<double>(deg)));
}
template <typename T>
inline T norm_col_factor(int norm, index_t deg) {
    if (norm != NORM_SYM_DEGREE) return T(1);
    if (deg <= 0) return T(0);
    return static_cast<T>(1.0 / std::sqrt(static_cast<double>(deg)));
}

// CsrGraph with the cached transpose.
struct Graph {
    index_t n = 0, e = 0;
    int norm = NORM_NONE;
    std::vector<index_t> row_ptr;
    std::vector<std::int32_t> col_idx;
    std::vector<index_t> trow_ptr;      // CSR of Aᵀ: sources ascending per row
    std::vector<std::int32_t> tcol_idx;

    void validate() const {
        if (static_cast<index_t>(row_ptr.size()) != n + 1) throw ShapeError("row_ptr length != n+1");
        if (row_ptr[0] != 0 || row_ptr[static_cast<size_t>(n)] != e) throw FormatError("row_ptr endpoints");
        for (index_t r = 0; r < n; ++r) {
            if (row_ptr[r + 1] < row_ptr[r]) throw FormatError("row_ptr decreasing");
            for (index_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) {
                if (col_idx[q] < 0 || col_idx[q] >= n) throw FormatError("col_idx out of range");
                if (q > row_ptr[r] && col_idx[q] <= col_idx[q - 1]) throw FormatError("col_idx not strictly ascending");
            }
        }
    }
    void build_transpose() {
        trow_ptr.assign(static_cast<size_t>(n + 1), 0);
        tcol_idx.assign(static_cast<size_t>(e), 0);
        for (index_t q = 0; q < e; ++q) trow_ptr[static_cast<size_t>(col_idx[q]) + 1]++;
        for (index_t r = 0; r < n; ++r) trow_ptr[r + 1] += trow_ptr[r];
        std::vector<index_t> fill(trow_ptr.begin(), trow_ptr.end() - 1);
        for (index_t r = 0; r < n; ++r)
            for (index_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q)
                tcol_idx[static_cast<size_t>(fill[static_cast<size_t>(col_idx[q])]++)] = static_cast<std::int32_t>(r);
    }
    index_t deg(index_t r) const { return row_ptr[r + 1] - row_ptr[r]; }
};

// from_edge_list: deduplicated, row-sorted CSR.
inline Graph from_edge_list(index_t n, index_t m, const std::int64_t* uv, int norm) {
    std::vector<std::int64_t> codes;
    codes.reserve(static_cast<size_t>(m));
    for (index_t i = 0; i < m; ++i) {
        std::int64_t u = uv[2 * i], v = uv[2 * i + 1];
        if (u < 0 || u >= n || v < 0 || v >= n) throw FormatError("edge endpoint out of range at pair " + std::to_string(i));
        codes.push_back(u * n + v);
    }
    std::sort(codes.begin(), codes.end());
    codes.erase(std::unique(codes.begin(), codes.end()), codes.end());
    Graph g;
    g.n = n;
    g.e = static_cast<index_t>(codes.size());
    g.norm = norm;
    g.row_ptr.assign(static_cast<size_t>(n + 1), 0);
    g.col_idx.resize(codes.size());
    for (size_t i = 0; i < codes.size(); ++i) {
        g.row_ptr[static_cast<size_t>(codes[i] / n) + 1]++;
        g.col_idx[i] = static_cast<std::int32_t>(codes[i] % n);
    }
    for (index_t r = 0; r < n; ++r) g.row_ptr[r + 1] += g.row_ptr[r];
    g.build_transpose();
    return g;
}

// ---------------------------------------------------------------------------
// tensor-core module. Matrices are row-major with an explicit
// leading dimension so that split() views are zero-copy.
// SparseActivation: vals n×k, idx n×k, ascending per row.
// ---------------------------------------------------------------------------

template <typename T>
inline bool mag_before(T a, int ia, T b, int ib) {  // |a| ranks before |b|
    const T fa = std::fabs(a), fb = std::fabs(b);
    return fa > fb || (fa == fb && ia < ib);
}

// gs_topk: per row, the k largest |x|, sign kept, ties to the
// smallest column, indices ascending.
template <typename T>
void gs_topk_row(const T* x, int w, int k, T* vals, std::int32_t* idx) {
    int order[1024];
    for (int j = 0; j < w; ++j) order[j] = j;
    std::partial_sort(order, order + k, order + w, [&](int a, int b) { return mag_before(x[a], a, x[b], b); });
    std::sort(order, order + k);
    for (int j = 0; j < k; ++j) {
        idx[j] = order[j];
        vals[j] = x[order[j]];
    }
}

template <typename T>
void gs_topk(index_t n, int w, int k, const T* x, index_t ldx, T* vals, std::int32_t* idx) {
    if (k < 1 || k > w) throw ConfigError("gs_topk: k=" + std::to_string(k) + " out of [1," + std::to_string(w) + "]");
    if (w > 1024) throw ConfigError("gs_topk: width > 1024");
    pfor(n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) gs_topk_row(x + r * ldx, w, k, vals + r * k, idx + r * k);
    });
}

// scatter
template <typename T>
void scatter(index_t n, int w, int k, const T* vals, const std::int32_t* idx, T* out, index_t ldo) {
    pfor(n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) {
            T* o = out + r * ldo;
            for (int m = 0; m < w; ++m) o[m] = T(0);
            for (int j = 0; j < k; ++j) o[idx[r * k + j]] = vals[r * k + j];
        }
    });
}

// gather
template <typename T>
void gather(index_t n, int w, int k, const T* x, index_t ldx, const std::int32_t* idx, T* vals) {
    pfor(n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r)
            for (int j = 0; j < k; ++j) {
                const int c = idx[r * k + j];
                if (c < 0 || c >= w) throw ShapeError("gather: index out of bounds");
                vals[r * k + j] = x[r * ldx + c];
            }
    });
}

template <typename T>
struct Scales {
    std::vector<T> row_f, col_f;
    explicit Scales(const Graph& g) : row_f(static_cast<size_t>(g.n)), col_f(static_cast<size_t>(g.n)) {
        for (index_t r = 0; r < g.n; ++r) {
            row_f[r] = norm_row_factor<T>(g.norm, g.deg(r));
            col_f[r] = norm_col_factor<T>(g.norm, g.deg(r));
        }
    }
};

// Edge list and scales for one direction.
//   forward:   y[r] = row_f[r] * Σ_{c∈CSR(r)} col_f[c] * x[c]
//   transpose: y[r] = col_f[r] * Σ_{c: r∈CSR(c)} row_f[c] * x[c]
template <typename T>
struct Dir {
    const index_t* ptr;
    const std::int32_t* idx;
    const T* out_f;
    const T* edge_f;
};
template <typename T>
Dir<T> direction(const Graph& g, const Scales<T>& s, bool transpose) {
    if (!transpose) return {g.row_ptr.data(), g.col_idx.data(), s.row_f.data(), s.col_f.data()};
    return {g.trow_ptr.data(), g.tcol_idx.data(), s.col_f.data(), s.row_f.data()};
}

// Canonical segment length of the aggregation order (see header).
constexpr index_t kAggSeg = 8;

// spmm: dense Â·x or Âᵀ·x; WorkCounter += e × cols.
template <typename T>
void spmm_row(const Dir<T>& d, index_t r, int cols, const T* x, index_t ldx, T* y) {
    T acc[1024], part[1024];
    for (int m = 0; m < cols; ++m) acc[m] = T(0);
    const index_t q0 = d.ptr[r], q1 = d.ptr[r + 1];
    for (index_t s0 = q0; s0 < q1; s0 += kAggSeg) {
        for (int m = 0; m < cols; ++m) part[m] = T(0);
        for (index_t q = s0; q < std::min(q1, s0 + kAggSeg); ++q) {
            const index_t c = d.idx[q];
            const T sc = d.edge_f[c];
            const T* xr = x + c * ldx;
            for (int m = 0; m < cols; ++m) part[m] = part[m] + sc * xr[m];
        }
        if (s0 == q0) for (int m = 0; m < cols; ++m) acc[m] = part[m];
        else for (int m = 0; m < cols; ++m) acc[m] = acc[m] + part[m];
    }
    const T rf = d.out_f[r];
    for (int m = 0; m < cols; ++m) y[m] = rf * acc[m];
}

template <typename T>
void spmm(const Graph& g, bool transpose, int cols, const T* x, index_t ldx, T* y, index_t ldy) {
    if (cols > 1024) throw ConfigError("spmm: cols > 1024");
    Scales<T> s(g);
    auto d = direction(g, s, transpose);
    pfor(g.n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) spmm_row(d, r, cols, x, ldx, y + r * ldy);
    });
    work().scalar_mul_adds += static_cast<std::uint64_t>(g.e) * static_cast<std::uint64_t>(cols);
    work().rows_touched += static_cast<std::uint64_t>(g.n);
}

// spmm_sparse: == spmm(g, scatter(s)) computed in O(e·k).
template <typename T>
void spmm_sparse_row(const Dir<T>& d, index_t r, int w, int k, const T* vals, const std::int32_t* idx, T* y) {
    T acc[1024], part[1024];
    for (int m = 0; m < w; ++m) acc[m] = T(0);
    const index_t q0 = d.ptr[r], q1 = d.ptr[r + 1];
    for (index_t s0 = q0; s0 < q1; s0 += kAggSeg) {
        for (int m = 0; m < w; ++m) part[m] = T(0);
        for (index_t q = s0; q < std::min(q1, s0 + kAggSeg); ++q) {
            const index_t c = d.idx[q];
            const T sc = d.edge_f[c];
            for (int j = 0; j < k; ++j) {
                const int m = idx[c * k + j];
                part[m] = part[m] + sc * vals[c * k + j];
            }
        }
        if (s0 == q0) for (int m = 0; m < w; ++m) acc[m] = part[m];
        else for (int m = 0; m < w; ++m) acc[m] = acc[m] + part[m];
    }
    const T rf = d.out_f[r];
    for (int m = 0; m < w; ++m) y[m] = rf * acc[m];
}

template <typename T>
void spmm_sparse(const Graph& g, bool transpose, int w, int k, const T* vals, const std::int32_t* idx, T* y, index_t ldy) {
    Scales<T> s(g);
    auto d = direction(g, s, transpose);
    pfor(g.n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) spmm_sparse_row(d, r, w, k, vals, idx, y + r * ldy);
    });
    work().scalar_mul_adds += static_cast<std::uint64_t>(g.e) * static_cast<std::uint64_t>(k);
    work().rows_touched += static_cast<std::uint64_t>(g.n);
}

// TF32 transform mode (the device's tcgen05 kind::tf32 path, GSRC_GEMM_TF32):
// both operands of every block transform are read as TF32, i.e. the low 13
// mantissa bits truncated — what the tensor core does with fp32 operands
// (measured on the B200: scratch/tf32_probe.cu, 128/128 truncation). Products
// of two TF32 values are exact in FP32, so this oracle and the tensor core
// then differ only by the accumulation order of w exact products.
inline bool& tf32_transform() { static bool v = false; return v; }
inline float tf32_op(float x) {
    std::uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u &= 0xffffe000u;
    std::memcpy(&x, &u, 4);
    return x;
}
inline double tf32_op(double x) { return static_cast<double>(tf32_op(static_cast<float>(x))); }

// Exactly invertible residual stream (the device's gsrc_set_residual_quant;
// a B200-build extension): a block output h is rounded to
// the grid 2^-s, half to even, before the Eq. 6 add / Eq. 7 subtract, and the
// encoder output is put on the same grid. x + q(h) is then exact for
// |x| < 2^(24-s) (f32), so rev_inverse_layer reproduces the forward input bit
// for bit at any depth (SPEC.md:332-333,353 reversibility). s = 0: off.
template <typename T>
inline T quant(T h, int s) {
    if (s <= 0) return h;
    const T qs = std::ldexp(T(1), s), qi = std::ldexp(T(1), -s);
    return std::nearbyint(h * qs) * qi;
}

// One row of a dense transform: out[j] = fma-chain_m a[m]*B(m,j) (+0 start).
// B(m,j) = b[m*ldb + j] (plain) or b[j*ldb + m] (transposed operand).
// rnd: TF32 operand rounding (see tf32_transform).
template <typename T>
inline void gemm_row(const T* a, int K, int N, const T* b, index_t ldb, bool bt, T* out, bool rnd = false) {
    T acc[1024];
    for (int j = 0; j < N; ++j) acc[j] = T(0);
    auto B = [&](T v) { return rnd ? static_cast<T>(tf32_op(v)) : v; };
    if (!bt) {
        for (int m = 0; m < K; ++m) {
            const T am = B(a[m]);
            const T* brow = b + m * ldb;
            for (int j = 0; j < N; ++j) acc[j] = std::fma(am, B(brow[j]), acc[j]);
        }
    } else {
        for (int m = 0; m < K; ++m) {
            const T am = B(a[m]);
            for (int j = 0; j < N; ++j) acc[j] = std::fma(am, B(b[j * ldb + m]), acc[j]);
        }
    }
    for (int j = 0; j < N; ++j) out[j] = acc[j];
}

// gemm: out = a·b (+= when accumulate); WorkCounter += M·K·N.
template <typename T>
void gemm(index_t M, int K, int N, const T* a, index_t lda, const T* b, index_t ldb, bool bt, bool accumulate, T* out, index_t ldo,
          bool rnd = false) {
    pfor(M, [&](index_t bg, index_t en) {
        T tmp[1024];
        for (index_t r = bg; r < en; ++r) {
            gemm_row(a + r * lda, K, N, b, ldb, bt, tmp, rnd);
            T* o = out + r * ldo;
            for (int j = 0; j < N; ++j) o[j] = accumulate ? o[j] + tmp[j] : tmp[j];
        }
    });
    work().scalar_mul_adds += static_cast<std::uint64_t>(M) * K * N;
}

// ---------------------------------------------------------------------------
// gnn-blocks
// ---------------------------------------------------------------------------
struct BlockFlags {
    bool use_weight = true;
    bool use_bias = false;  // "Bias default: off"
};

enum Epi : int {
    EPI_NONE = 0,         // out = h
    EPI_ADD = 1,          // out = R + h
    EPI_SUB = 2,          // out = R - h
    EPI_SCATTER_ADD = 3,  // out = scatter(s_res) + h
    EPI_SCATTER_SUB = 4,  // out = scatter(s_res) - h
};

// h = Z·W + b for one row given its aggregated row Z (the transform half of
// gsr_forward_block / dense_block, aggregate-then-transform SPEC.md:286).
template <typename T>
inline void transform_row(const T* z, int w, const T* W, const T* bias, BlockFlags f, T* h) {
    if (f.use_weight) gemm_row(z, w, w, W, w, false, h, tf32_transform());
    else for (int j = 0; j < w; ++j) h[j] = z[j];
    if (f.use_bias) for (int j = 0; j < w; ++j) h[j] = h[j] + bias[j];
}

template <typename T>
inline void epilogue_row(int epi, const T* h, const T* R, const T* svals, const std::int32_t* sidx, int w, int k, T* out, int qshift = 0) {
    switch (epi) {
        case EPI_NONE: for (int j = 0; j < w; ++j) out[j] = h[j]; break;
        case EPI_ADD: for (int j = 0; j < w; ++j) out[j] = R[j] + quant(h[j], qshift); break;
        case EPI_SUB: for (int j = 0; j < w; ++j) out[j] = R[j] - quant(h[j], qshift); break;
        case EPI_SCATTER_ADD:
        case EPI_SCATTER_SUB: {
            T sc[1024];
            for (int j = 0; j < w; ++j) sc[j] = T(0);
            for (int j = 0; j < k; ++j) sc[sidx[j]] = svals[j];
            if (epi == EPI_SCATTER_ADD) for (int j = 0; j < w; ++j) out[j] = sc[j] + h[j];
            else for (int j = 0; j < w; ++j) out[j] = sc[j] - h[j];
        } break;
        default: throw ConfigError("bad epilogue");
    }
}

// gsr_forward_block, fused with a residual epilogue.
// out may alias R (in-place residual update is row-local).
template <typename T>
void gsr_block_apply(const Graph& g, int w, int k, const T* vals, const std::int32_t* idx, const T* W, const T* bias, BlockFlags f,
                     int epi, const T* R, index_t ldr, const T* rvals, const std::int32_t* ridx, T* out, index_t ldo, int qshift = 0) {
    Scales<T> s(g);
    auto d = direction(g, s, false);
    pfor(g.n, [&](index_t b, index_t e) {
        T z[1024], h[1024];
        for (index_t r = b; r < e; ++r) {
            spmm_sparse_row(d, r, w, k, vals, idx, z);
            transform_row(z, w, W, bias, f, h);
            epilogue_row(epi, h, R ? R + r * ldr : nullptr, rvals ? rvals + r * k : nullptr, ridx ? ridx + r * k : nullptr, w, k, out + r * ldo,
                         qshift);
        }
    });
    work().scalar_mul_adds += static_cast<std::uint64_t>(g.e) * k + (f.use_weight ? static_cast<std::uint64_t>(g.n) * w * w : 0);
}

// dense_block: f(x) = spmm(g, relu(x))·W + b (ReLU input-side).
template <typename T>
void dense_block_apply(const Graph& g, int w, const T* x, index_t ldx, const T* W, const T* bias, BlockFlags f,
                       int epi, const T* R, index_t ldr, T* out, index_t ldo, int qshift = 0) {
    Scales<T> s(g);
    auto d = direction(g, s, false);
    std::vector<T> rx(static_cast<size_t>(g.n) * w);
    pfor(g.n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r)
            for (int m = 0; m < w; ++m) { const T v = x[r * ldx + m]; rx[r * w + m] = v > T(0) ? v : T(0); }
    });
    pfor(g.n, [&](index_t b, index_t e) {
        T z[1024], h[1024];
        for (index_t r = b; r < e; ++r) {
            spmm_row(d, r, w, rx.data(), w, z);
            transform_row(z, w, W, bias, f, h);
            epilogue_row<T>(epi, h, R ? R + r * ldr : nullptr, nullptr, nullptr, w, 0, out + r * ldo, qshift);
        }
    });
}

// Fixed-order reduction over rows: Σ_r a[r][m] * b[r][n] into out (double).
// Chunks of kRedChunk rows are reduced separately and combined in chunk
// order, so results do not depend on the worker count.
constexpr index_t kRedChunk = 512;
template <typename T, typename RowA, typename RowB>
void reduce_outer(index_t n, int wa, int wb, RowA rowa, RowB rowb, std::vector<double>& out) {
    const index_t nch = (n + kRedChunk - 1) / kRedChunk;
    std::vector<double> part(static_cast<size_t>(nch) * wa * wb, 0.0);
    pfor(nch, [&](index_t b, index_t e) {
        std::vector<T> ta(static_cast<size_t>(wa)), tb(static_cast<size_t>(wb));
        for (index_t ch = b; ch < e; ++ch) {
            double* p = part.data() + ch * wa * wb;
            for (index_t r = ch * kRedChunk; r < std::min(n, (ch + 1) * kRedChunk); ++r) {
                rowa(r, ta.data());
                rowb(r, tb.data());
                for (int m = 0; m < wa; ++m) {
                    const double am = ta[m];
                    if (am == 0.0) continue;
                    for (int j = 0; j < wb; ++j) p[m * wb + j] += am * static_cast<double>(tb[j]);
                }
            }
        }
    });
    out.assign(static_cast<size_t>(wa) * wb, 0.0);
    for (index_t ch = 0; ch < nch; ++ch)
        for (size_t i = 0; i < out.size(); ++i) out[i] += part[ch * wa * wb + i];
}

template <typename T>
void colsum(index_t n, int w, const T* x, index_t ldx, std::vector<double>& out) {
    reduce_outer<T>(n, 1, w, [](index_t, T* a) { a[0] = T(1); }, [&](index_t r, T* b) { for (int j = 0; j < w; ++j) b[j] = x[r * ldx + j]; }, out);
}

// gsr_backward_block, literal form:
//   v_g = gather(m·Wᵀ, I_src); out = spmm_sparse(g, (v_g, I_src), transpose)
//   dW += scatter(s_fwd)ᵀ · spmm(g, m, transpose); db += colsum(m)
template <typename T>
void gsr_backward_block(const Graph& g, int w, int k, const T* m, index_t ldm, const std::int32_t* isrc, const T* fvals,
                        const std::int32_t* fidx, const T* W, BlockFlags f, T* out, index_t ldo, T* dW, T* db) {
    const index_t n = g.n;
    std::vector<T> tm(static_cast<size_t>(n) * w), vg(static_cast<size_t>(n) * k);
    if (f.use_weight) gemm<T>(n, w, w, m, ldm, W, w, true, false, tm.data(), w, tf32_transform());
    else pfor(n, [&](index_t b, index_t e) { for (index_t r = b; r < e; ++r) for (int j = 0; j < w; ++j) tm[r * w + j] = m[r * ldm + j]; });
    gather<T>(n, w, k, tm.data(), w, isrc, vg.data());
    spmm_sparse<T>(g, true, w, k, vg.data(), isrc, out, ldo);
    if (f.use_weight && dW) {
        std::vector<T> am(static_cast<size_t>(n) * w);
        spmm<T>(g, true, w, m, ldm, am.data(), w);
        std::vector<double> acc;
        reduce_outer<T>(n, w, w,
            [&](index_t r, T* a) { for (int j = 0; j < w; ++j) a[j] = T(0); for (int j = 0; j < k; ++j) a[fidx[r * k + j]] = fvals[r * k + j]; },
            [&](index_t r, T* b) { for (int j = 0; j < w; ++j) b[j] = am[r * w + j]; }, acc);
        for (int i = 0; i < w * w; ++i) dW[i] = static_cast<T>(static_cast<double>(dW[i]) + acc[i]);
    }
    if (f.use_bias && db) {
        std::vector<double> acc;
        colsum<T>(n, w, m, ldm, acc);
        for (int j = 0; j < w; ++j) db[j] = static_cast<T>(static_cast<double>(db[j]) + acc[j]);
    }
}

// ---------------------------------------------------------------------------
// networks: rev-baseline, gsr-net and the
// GSR-C extension (SURVEY.md §7 hard part 1: Eq. 6-7 with GS-sparse blocks).
// ---------------------------------------------------------------------------
enum Mode : int { MODE_ALG12 = 0, MODE_GSRC = 1, MODE_REV = 2 };
enum IndexSource : int { IDX_ALG2_LOCAL = 0, IDX_FORWARD_CACHE = 1 };

struct NetCfg {
    int mode = MODE_GSRC;
    int L = 0, D = 0, C = 2, k = 1, d_in = 1;
    BlockFlags flags{};
    int index_source = IDX_ALG2_LOCAL;
    int qshift = 0;  // residual-stream grid 2^-qshift in the grouped-reversible modes (quant), 0 = off

    int groups() const { return mode == MODE_ALG12 ? 2 : C; }
    int width() const { return D / groups(); }
    int blocks() const { return groups(); }
    index_t block_params() const { return static_cast<index_t>(width()) * width() + width(); }
    index_t off_enc_w() const { return 0; }
    index_t off_enc_b() const { return static_cast<index_t>(d_in) * D; }
    index_t off_block(int l, int i) const { return off_enc_b() + D + (static_cast<index_t>(l) * blocks() + i) * block_params(); }
    index_t off_head_w() const { return off_block(L, 0); }
    index_t off_head_b() const { return off_head_w() + D; }
    index_t num_params() const { return off_head_b() + 1; }

    void validate() const {
        if (mode < 0 || mode > 2) throw ConfigError("mode");
        if (L < 0) throw ConfigError("L < 0");
        if (mode == MODE_ALG12 && D % 2) throw ConfigError("gsr requires even D");
        if (mode != MODE_ALG12 && (C < 2 || D % C)) throw ConfigError("D must be divisible by C >= 2");
        if (width() > 1024) throw ConfigError("group width > 1024");
        if (mode != MODE_REV && (k < 1 || k > width())) throw ConfigError("k out of [1, width]");
        if (mode == MODE_ALG12 && k > D / 2) throw ConfigError("k > D/2");
        if (d_in < 1) throw ConfigError("d_in");
    }
};

// Alg. 1 forward cache of one layer: GS outputs (values + indices) of both
// groups ("selective save-for-backward", §4.2).
template <typename T>
struct LayerCache {
    bool filled = false;
    std::vector<T> v1, v2;
    std::vector<std::int32_t> i1, i2;
};

template <typename T>
struct Net {
    NetCfg cfg;
    const Graph* g = nullptr;
    std::vector<T> params, grads;
    std::vector<LayerCache<T>> cache;

    const T* W(int l, int i) const { return params.data() + cfg.off_block(l, i); }
    const T* B(int l, int i) const { return W(l, i) + static_cast<index_t>(cfg.width()) * cfg.width(); }
    T* dW(int l, int i) { return grads.data() + cfg.off_block(l, i); }
    T* dB(int l, int i) { return dW(l, i) + static_cast<index_t>(cfg.width()) * cfg.width(); }
};

// y'_0 = Σ_{j=2..C} x_j, summed left to right (Eq. 6).
template <typename T>
void group_sum(index_t n, int C, int w, const T* X, index_t ld, T* u) {
    pfor(n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r)
            for (int m = 0; m < w; ++m) {
                T s = X[r * ld + 1 * w + m];
                for (int j = 2; j < C; ++j) s = s + X[r * ld + j * w + m];
                u[r * w + m] = s;
            }
    });
}

// Sparse activation of a block input: GS top-k (gsr modes) or ReLU (rev).
template <typename T>
struct Act {
    std::vector<T> vals;
    std::vector<std::int32_t> idx;
    std::vector<T> dense;  // rev: relu(u)
};

template <typename T>
void make_act(const Net<T>& net, const T* u, index_t ldu, Act<T>& a) {
    const index_t n = net.g->n;
    const int w = net.cfg.width(), k = net.cfg.k;
    if (net.cfg.mode == MODE_REV) {
        a.dense.resize(static_cast<size_t>(n) * w);
        pfor(n, [&](index_t b, index_t e) {
            for (index_t r = b; r < e; ++r) for (int m = 0; m < w; ++m) { const T v = u[r * ldu + m]; a.dense[r * w + m] = v > T(0) ? v : T(0); }
        });
    } else {
        a.vals.resize(static_cast<size_t>(n) * k);
        a.idx.resize(static_cast<size_t>(n) * k);
        gs_topk<T>(n, w, k, u, ldu, a.vals.data(), a.idx.data());
    }
}

// f_i applied with an epilogue (grouped-reversible modes).
template <typename T>
void apply_block(const Net<T>& net, int l, int i, const Act<T>& a, int epi, const T* R, index_t ldr, T* out, index_t ldo) {
    const int w = net.cfg.width();
    if (net.cfg.mode == MODE_REV)
        dense_block_apply<T>(*net.g, w, a.dense.data(), w, net.W(l, i), net.B(l, i), net.cfg.flags, epi, R, ldr, out, ldo, net.cfg.qshift);
    else
        gsr_block_apply<T>(*net.g, w, net.cfg.k, a.vals.data(), a.idx.data(), net.W(l, i), net.B(l, i), net.cfg.flags, epi, R, ldr, nullptr, nullptr, out,
                           ldo, net.cfg.qshift);
}

// Grouped reversible forward (Eq. 6; SPEC rev_forward_layer :316-324), in place.
template <typename T>
void rev_forward_layer(const Net<T>& net, int l, T* X) {
    const index_t n = net.g->n;
    const int C = net.cfg.C, w = net.cfg.width(), D = net.cfg.D;
    std::vector<T> u(static_cast<size_t>(n) * w);
    Act<T> a;
    group_sum<T>(n, C, w, X, D, u.data());
    make_act(net, u.data(), w, a);
    apply_block(net, l, 0, a, EPI_ADD, X, D, X, D);
    for (int i = 1; i < C; ++i) {
        make_act(net, X + (i - 1) * w, D, a);
        apply_block(net, l, i, a, EPI_ADD, X + i * w, D, X + i * w, D);
    }
}

// Grouped reversible inverse (Eq. 7; SPEC rev_inverse_layer :325-333), in place.
template <typename T>
void rev_inverse_layer(const Net<T>& net, int l, T* Y) {
    const index_t n = net.g->n;
    const int C = net.cfg.C, w = net.cfg.width(), D = net.cfg.D;
    Act<T> a;
    for (int i = C - 1; i >= 1; --i) {
        make_act(net, Y + (i - 1) * w, D, a);
        apply_block(net, l, i, a, EPI_SUB, Y + i * w, D, Y + i * w, D);
    }
    std::vector<T> u(static_cast<size_t>(n) * w);
    group_sum<T>(n, C, w, Y, D, u.data());
    make_act(net, u.data(), w, a);
    apply_block(net, l, 0, a, EPI_SUB, Y, D, Y, D);
}

// Exact backward of one grouped-reversible layer with inverse recomputation
// (SPEC rev_backward :334-342). On entry Y = layer output, G = dL/dY; on exit
// Y = reconstructed layer input, G = dL/dX. Parameter grads are accumulated.
// For block i with input u (u = y'_{i-1}, or y'_0 for i = 1), activation
// s = act(u), Z = Â·s, G_i = dL/dy'_i (complete once blocks > i are done):
//   x_i = y'_i − (Z·W_i + b_i)                      (Eq. 7)
//   dW_i += Zᵀ·G_i ; db_i += colsum(G_i)
//   du = act'(u) ⊙ ((Âᵀ·G_i)·W_iᵀ)   added to G_{i-1}, or to every G_j, j≥2
template <typename T>
void rev_backward_layer(Net<T>& net, int l, T* Y, T* G) {
    const Graph& g = *net.g;
    const index_t n = g.n;
    const int C = net.cfg.C, w = net.cfg.width(), D = net.cfg.D, k = net.cfg.k;
    const bool rev = net.cfg.mode == MODE_REV;
    const BlockFlags f = net.cfg.flags;
    Scales<T> s(g);
    auto fwd = direction(g, s, false);
    auto bwd = direction(g, s, true);
    std::vector<T> u(static_cast<size_t>(n) * w), Z(static_cast<size_t>(n) * w);
    Act<T> a;
    for (int i = C - 1; i >= 0; --i) {
        const T* up;
        index_t ldu;
        if (i > 0) { up = Y + (i - 1) * w; ldu = D; }
        else { group_sum<T>(n, C, w, Y, D, u.data()); up = u.data(); ldu = w; }
        make_act(net, up, ldu, a);
        // recompute Z, h and reconstruct x_i in place
        pfor(n, [&](index_t b, index_t e) {
            T h[1024];
            for (index_t r = b; r < e; ++r) {
                T* z = Z.data() + r * w;
                if (rev) spmm_row(fwd, r, w, a.dense.data(), w, z);
                else spmm_sparse_row(fwd, r, w, k, a.vals.data(), a.idx.data(), z);
                transform_row(z, w, net.W(l, i), net.B(l, i), f, h);
                T* yr = Y + r * D + i * w;
                for (int j = 0; j < w; ++j) yr[j] = yr[j] - quant(h[j], net.cfg.qshift);
            }
        });
        T* Gi = G + i * w;
        // dW_i = Zᵀ·G_i = (Â·S)ᵀ·G_i. FP32 mode evaluates Zᵀ·G_i.
        // TF32 GSR-C mode evaluates the same product as Sᵀ·(Âᵀ·G_i) from the
        // tensor-core operands the device uses (its BIN kernel: S = the
        // block's GS records, Âᵀ·G_i = the aggregation it already holds for the
        // input gradient), both read as TF32 (tf32_op) — see below.
        // (rev-baseline in TF32 likewise, with S = relu(u): the device's BIN in
        // its dense-mask mode.)
        const bool tf32_sy = tf32_transform() && f.use_weight;
        if (f.use_weight && !tf32_sy) {
            std::vector<double> acc;
            const bool rz = tf32_transform();
            reduce_outer<T>(n, w, w, [&](index_t r, T* x) { for (int j = 0; j < w; ++j) x[j] = rz ? static_cast<T>(tf32_op(Z[r * w + j])) : Z[r * w + j]; },
                            [&](index_t r, T* x) { for (int j = 0; j < w; ++j) x[j] = rz ? static_cast<T>(tf32_op(Gi[r * D + j])) : Gi[r * D + j]; }, acc);
            T* dw = net.dW(l, i);
            for (int q = 0; q < w * w; ++q) dw[q] = static_cast<T>(static_cast<double>(dw[q]) + acc[q]);
        }
        std::vector<T> Yb(tf32_sy ? static_cast<size_t>(n) * w : 0);
        if (f.use_bias) {
            std::vector<double> acc;
            colsum<T>(n, w, Gi, D, acc);
            T* db = net.dB(l, i);
            for (int q = 0; q < w; ++q) db[q] = static_cast<T>(static_cast<double>(db[q]) + acc[q]);
        }
        // input gradient through the block, masked by the activation
        pfor(n, [&](index_t b, index_t e) {
            T yt[1024], t[1024];
            for (index_t r = b; r < e; ++r) {
                spmm_row(bwd, r, w, Gi, D, yt);
                if (tf32_sy) std::memcpy(Yb.data() + r * w, yt, sizeof(T) * w);
                if (f.use_weight) gemm_row(yt, w, w, net.W(l, i), w, true, t, tf32_transform());
                else for (int j = 0; j < w; ++j) t[j] = yt[j];
                auto add_to = [&](T* dst) {
                    if (rev) {
                        for (int j = 0; j < w; ++j) if (up[r * ldu + j] > T(0)) dst[j] = dst[j] + t[j];
                    } else {
                        for (int j = 0; j < k; ++j) { const int c = a.idx[r * k + j]; dst[c] = dst[c] + t[c]; }
                    }
                };
                if (i > 0) add_to(G + r * D + (i - 1) * w);
                else for (int j = 1; j < C; ++j) add_to(G + r * D + j * w);
            }
        });
        if (tf32_sy) {
            std::vector<double> acc;
            reduce_outer<T>(n, w, w,
                [&](index_t r, T* x) {
                    if (rev) {
                        for (int j = 0; j < w; ++j) x[j] = static_cast<T>(tf32_op(a.dense[r * w + j]));
                        return;
                    }
                    for (int j = 0; j < w; ++j) x[j] = T(0);
                    for (int j = 0; j < k; ++j) x[a.idx[r * k + j]] = static_cast<T>(tf32_op(a.vals[r * k + j]));
                },
                [&](index_t r, T* x) { for (int j = 0; j < w; ++j) x[j] = static_cast<T>(tf32_op(Yb[r * w + j])); }, acc);
            T* dw = net.dW(l, i);
            for (int q = 0; q < w * w; ++q) dw[q] = static_cast<T>(static_cast<double>(dw[q]) + acc[q]);
        }
    }
}

// gsr_forward_layer = Algorithm 1 lines 4-11, modular form.
template <typename T>
void gsr_forward_layer(Net<T>& net, int l, T* X) {
    const Graph& g = *net.g;
    const index_t n = g.n;
    const int w = net.cfg.width(), D = net.cfg.D, k = net.cfg.k;
    LayerCache<T>& c = net.cache[static_cast<size_t>(l)];
    if (c.filled) throw SequencingError("gsr_forward_layer: cache already occupied for layer " + std::to_string(l));
    c.v1.resize(static_cast<size_t>(n) * k); c.i1.resize(static_cast<size_t>(n) * k);
    c.v2.resize(static_cast<size_t>(n) * k); c.i2.resize(static_cast<size_t>(n) * k);
    T* X1 = X;
    T* X2 = X + w;
    gs_topk<T>(n, w, k, X1, D, c.v1.data(), c.i1.data());                        // line 5
    gsr_block_apply<T>(g, w, k, c.v1.data(), c.i1.data(), net.W(l, 0), net.B(l, 0), net.cfg.flags,
                       EPI_ADD, X2, D, nullptr, nullptr, X2, D);                    // lines 6-7
    gs_topk<T>(n, w, k, X2, D, c.v2.data(), c.i2.data());                        // line 8
    gsr_block_apply<T>(g, w, k, c.v2.data(), c.i2.data(), net.W(l, 1), net.B(l, 1), net.cfg.flags,
                       EPI_SCATTER_ADD, nullptr, 0, c.v1.data(), c.i1.data(), X1, D);  // lines 9-10
    c.filled = true;
}

// gsr_backward_layer = Algorithm 2 lines 4-9, modular form.
// Block roles: GSRBlock(V2,I2) uses block B's parameters (B consumes group-2
// GS in Alg. 1), GSRBlock(V1,I1) uses block A's.
template <typename T>
void gsr_backward_layer(Net<T>& net, int l, T* Gm) {
    const Graph& g = *net.g;
    const index_t n = g.n;
    const int w = net.cfg.width(), D = net.cfg.D, k = net.cfg.k;
    LayerCache<T>& c = net.cache[static_cast<size_t>(l)];
    if (!c.filled) throw SequencingError("gsr_backward_layer: missing forward cache for layer " + std::to_string(l));
    std::vector<T> V2(static_cast<size_t>(n) * k), V1(static_cast<size_t>(n) * k), M1(static_cast<size_t>(n) * w), M2(static_cast<size_t>(n) * w);
    std::vector<std::int32_t> I2(static_cast<size_t>(n) * k), I1(static_cast<size_t>(n) * k);
    T* g1 = Gm;
    T* g2 = Gm + w;
    gs_topk<T>(n, w, k, g2, D, V2.data(), I2.data());                                          // line 4
    gsr_block_apply<T>(g, w, k, V2.data(), I2.data(), net.W(l, 1), net.B(l, 1), net.cfg.flags,
                       EPI_SUB, g1, D, nullptr, nullptr, M1.data(), w);                            // line 5
    gs_topk<T>(n, w, k, M1.data(), w, V1.data(), I1.data());                                   // line 6
    gsr_block_apply<T>(g, w, k, V1.data(), I1.data(), net.W(l, 0), net.B(l, 0), net.cfg.flags,
                       EPI_SCATTER_SUB, nullptr, 0, V2.data(), I2.data(), M2.data(), w);          // lines 6-7
    const bool local = net.cfg.index_source == IDX_ALG2_LOCAL;
    gsr_backward_block<T>(g, w, k, M1.data(), w, local ? I1.data() : c.i1.data(), c.v1.data(), c.i1.data(),
                          net.W(l, 0), net.cfg.flags, g1, D, net.dW(l, 0), net.dB(l, 0));        // line 8
    gsr_backward_block<T>(g, w, k, M2.data(), w, local ? I2.data() : c.i2.data(), c.v2.data(), c.i2.data(),
                          net.W(l, 1), net.cfg.flags, g2, D, net.dW(l, 1), net.dB(l, 1));
    c = LayerCache<T>{};                                                                           // cache consumed
}

// Encoder: X = X0·We + be (affine d_in→D).
template <typename T>
void encoder_forward(const Net<T>& net, const T* X0, T* X) {
    const int D = net.cfg.D, din = net.cfg.d_in;
    const T* We = net.params.data() + net.cfg.off_enc_w();
    const T* be = net.params.data() + net.cfg.off_enc_b();
    pfor(net.g->n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) {
            gemm_row(X0 + r * din, din, D, We, D, false, X + r * D);
            const int qs = net.cfg.mode == MODE_ALG12 ? 0 : net.cfg.qshift;  // grouped-reversible modes: on the residual grid
            for (int j = 0; j < D; ++j) X[r * D + j] = quant(X[r * D + j] + be[j], qs);
        }
    });
}

// Head: ŷ = X·wh + bh (affine D→1).
template <typename T>
void head_forward(const Net<T>& net, const T* X, T* yhat) {
    const int D = net.cfg.D;
    const T* wh = net.params.data() + net.cfg.off_head_w();
    const T bh = net.params[static_cast<size_t>(net.cfg.off_head_b())];
    pfor(net.g->n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) {
            T acc = T(0);
            for (int j = 0; j < D; ++j) acc = std::fma(X[r * D + j], wh[j], acc);
            yhat[r] = acc + bh;
        }
    });
}

// net_forward: encoder → L layers → head.
template <typename T>
void net_forward(Net<T>& net, const T* X0, T* X, T* yhat) {
    encoder_forward(net, X0, X);
    if (net.cfg.mode == MODE_ALG12) {
        net.cache.assign(static_cast<size_t>(net.cfg.L), LayerCache<T>{});
        for (int l = 0; l < net.cfg.L; ++l) gsr_forward_layer(net, l, X);
    } else {
        for (int l = 0; l < net.cfg.L; ++l) rev_forward_layer(net, l, X);
    }
    head_forward(net, X, yhat);
}

// mse_loss: mean over masked nodes; grad 2(ŷ−y)/|mask|.
template <typename T>
double mse_loss(index_t n, const T* yhat, const T* y, const std::uint8_t* mask, T* gy) {
    index_t cnt = 0;
    for (index_t r = 0; r < n; ++r) cnt += mask[r] ? 1 : 0;
    if (cnt == 0) throw ConfigError("mse_loss: empty mask");
    const T fc = static_cast<T>(cnt);
    double loss = 0.0;
    for (index_t r = 0; r < n; ++r) {
        if (mask[r]) {
            const T d = yhat[r] - y[r];
            loss += static_cast<double>(d) * static_cast<double>(d);
            gy[r] = (T(2) * d) / fc;
        } else {
            gy[r] = T(0);
        }
    }
    return loss / static_cast<double>(cnt);
}

// net_backward. X holds the final activation on entry (it is
// consumed: grouped-reversible modes reconstruct the encoder output in place).
template <typename T>
void net_backward(Net<T>& net, const T* X0, T* X, const T* gy) {
    const index_t n = net.g->n;
    const int D = net.cfg.D, din = net.cfg.d_in;
    std::fill(net.grads.begin(), net.grads.end(), T(0));
    const T* wh = net.params.data() + net.cfg.off_head_w();
    std::vector<T> G(static_cast<size_t>(n) * D);
    pfor(n, [&](index_t b, index_t e) {
        for (index_t r = b; r < e; ++r) for (int j = 0; j < D; ++j) G[r * D + j] = gy[r] * wh[j];
    });
    {
        std::vector<double> acc;
        reduce_outer<T>(n, 1, D, [&](index_t r, T* a) { a[0] = gy[r]; }, [&](index_t r, T* b) { std::memcpy(b, X + r * D, sizeof(T) * D); }, acc);
        for (int j = 0; j < D; ++j) net.grads[net.cfg.off_head_w() + j] = static_cast<T>(acc[j]);
        double s = 0.0;
        for (index_t r = 0; r < n; ++r) s += gy[r];
        net.grads[net.cfg.off_head_b()] = static_cast<T>(s);
    }
    for (int l = net.cfg.L - 1; l >= 0; --l) {
        if (net.cfg.mode == MODE_ALG12) gsr_backward_layer(net, l, G.data());
        else rev_backward_layer(net, l, X, G.data());
    }
    std::vector<double> acc;
    reduce_outer<T>(n, din, D, [&](index_t r, T* a) { std::memcpy(a, X0 + r * din, sizeof(T) * din); },
                    [&](index_t r, T* b) { std::memcpy(b, G.data() + r * D, sizeof(T) * D); }, acc);
    for (int q = 0; q < din * D; ++q) net.grads[net.cfg.off_enc_w() + q] = static_cast<T>(acc[q]);
    colsum<T>(n, D, G.data(), D, acc);
    for (int j = 0; j < D; ++j) net.grads[net.cfg.off_enc_b() + j] = static_cast<T>(acc[j]);
}

// optimizer_step: bias-corrected Adam (L2 weight decay
// folded into the gradient), or SGD with optional momentum.
template <typename T>
void adam_step(index_t n, T* p, const T* g, T* m, T* v, T lr, T b1, T b2, T eps, T wd, T bc1, T bc2) {
    for (index_t i = 0; i < n; ++i) {
        T gi = g[i];
        if (wd != T(0)) gi = gi + wd * p[i];
        m[i] = b1 * m[i] + (T(1) - b1) * gi;
        v[i] = b2 * v[i] + (T(1) - b2) * (gi * gi);
        const T mh = m[i] / bc1;
        const T vh = v[i] / bc2;
        p[i] = p[i] - lr * (mh / (std::sqrt(vh) + eps));
    }
}

template <typename T>
void sgd_step(index_t n, T* p, const T* g, T* mom, T lr, T momentum) {
    for (index_t i = 0; i < n; ++i) {
        if (momentum != T(0)) {
            mom[i] = momentum * mom[i] + g[i];
            p[i] = p[i] - lr * mom[i];
        } else {
            p[i] = p[i] - lr * g[i];
        }
    }
}

}  // namespace gsro
