// TEST INFRASTRUCTURE ONLY — extern "C" surface of the CPU oracle, loaded by
// tests/ (ctypes) and by bench.py's cpu_baseline / --impl reference legs.
// Status codes follow the product's C-ABI (include/gsr_cuda.h), which mirrors
// /root/reference/proj/include/gsr/common.hpp:13-35.
#include <cstdio>
#include <memory>
#include <new>
#include <string>

#include "gsr_oracle.hpp"

using namespace gsro;

namespace {
thread_local std::string g_err;
std::unique_ptr<ThreadPool> g_pool;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const SequencingError& e) { g_err = e.what(); return 4; }
    catch (const ConfigError& e) { g_err = e.what(); return 1; }
    catch (const ResourceError& e) { g_err = e.what(); return 3; }
    catch (const std::bad_alloc& e) { g_err = "allocation failure"; return 3; }
    catch (const std::exception& e) { g_err = e.what(); return 2; }
}

struct NetBox {
    int is64;
    void* net;
};

// ---- Algorithms 1-2, straight-line transcriptions.
// Deliberately naive: no calls into the block/op layer, every loop inline.
template <typename T>
void transcribe_alg1(Net<T>& net, int l, T* X) {
    const Graph& g = *net.g;
    const index_t n = g.n;
    const int w = net.cfg.width(), D = net.cfg.D, k = net.cfg.k;
    const BlockFlags f = net.cfg.flags;
    Scales<T> sc(g);
    LayerCache<T>& c = net.cache[static_cast<size_t>(l)];
    c.v1.assign(static_cast<size_t>(n) * k, T(0)); c.i1.assign(static_cast<size_t>(n) * k, 0);
    c.v2.assign(static_cast<size_t>(n) * k, T(0)); c.i2.assign(static_cast<size_t>(n) * k, 0);
    auto topk = [&](const T* row, T* v, std::int32_t* ix) {
        std::vector<int> ord(static_cast<size_t>(w));
        for (int j = 0; j < w; ++j) ord[j] = j;
        std::sort(ord.begin(), ord.end(), [&](int a, int b) {
            return std::fabs(row[a]) > std::fabs(row[b]) || (std::fabs(row[a]) == std::fabs(row[b]) && a < b);
        });
        std::sort(ord.begin(), ord.begin() + k);
        for (int j = 0; j < k; ++j) { ix[j] = ord[j]; v[j] = row[ord[j]]; }
    };
    auto block = [&](const T* V, const std::int32_t* I, const T* W, const T* b, std::vector<T>& M) {
        M.assign(static_cast<size_t>(n) * w, T(0));
        for (index_t r = 0; r < n; ++r) {
            std::vector<T> acc(static_cast<size_t>(w), T(0)), part(static_cast<size_t>(w));
            for (index_t s0 = g.row_ptr[r]; s0 < g.row_ptr[r + 1]; s0 += kAggSeg) {
                std::fill(part.begin(), part.end(), T(0));
                for (index_t q = s0; q < std::min<index_t>(s0 + kAggSeg, g.row_ptr[r + 1]); ++q) {
                    const index_t cc = g.col_idx[q];
                    for (int j = 0; j < k; ++j) part[I[cc * k + j]] = part[I[cc * k + j]] + sc.col_f[cc] * V[cc * k + j];
                }
                for (int j = 0; j < w; ++j) acc[j] = (s0 == g.row_ptr[r]) ? part[j] : acc[j] + part[j];
            }
            for (int j = 0; j < w; ++j) acc[j] = sc.row_f[r] * acc[j];
            for (int j = 0; j < w; ++j) {
                T h = T(0);
                if (f.use_weight) { for (int m = 0; m < w; ++m) h = std::fma(acc[m], W[m * w + j], h); }
                else h = acc[j];
                if (f.use_bias) h = h + b[j];
                M[r * w + j] = h;
            }
        }
    };
    // line 4: split
    std::vector<T> X1(static_cast<size_t>(n) * w), X2(static_cast<size_t>(n) * w), M1, M2;
    for (index_t r = 0; r < n; ++r) for (int j = 0; j < w; ++j) { X1[r * w + j] = X[r * D + j]; X2[r * w + j] = X[r * D + w + j]; }
    for (index_t r = 0; r < n; ++r) topk(&X1[r * w], &c.v1[r * k], &c.i1[r * k]);              // line 5
    block(c.v1.data(), c.i1.data(), net.W(l, 0), net.B(l, 0), M1);                               // line 6
    for (index_t q = 0; q < n * w; ++q) X2[q] = X2[q] + M1[q];                                    // line 7
    for (index_t r = 0; r < n; ++r) topk(&X2[r * w], &c.v2[r * k], &c.i2[r * k]);              // line 8
    block(c.v2.data(), c.i2.data(), net.W(l, 1), net.B(l, 1), M2);                               // line 9
    for (index_t r = 0; r < n; ++r) {                                                              // line 10
        std::vector<T> s(static_cast<size_t>(w), T(0));
        for (int j = 0; j < k; ++j) s[c.i1[r * k + j]] = c.v1[r * k + j];
        for (int j = 0; j < w; ++j) X1[r * w + j] = s[j] + M2[r * w + j];
    }
    for (index_t r = 0; r < n; ++r) for (int j = 0; j < w; ++j) { X[r * D + j] = X1[r * w + j]; X[r * D + w + j] = X2[r * w + j]; }  // line 11
    c.filled = true;
}

template <typename T>
void transcribe_alg2(Net<T>& net, int l, T* Gm) {
    const Graph& g = *net.g;
    const index_t n = g.n;
    const int w = net.cfg.width(), D = net.cfg.D, k = net.cfg.k;
    const BlockFlags f = net.cfg.flags;
    Scales<T> sc(g);
    LayerCache<T>& c = net.cache[static_cast<size_t>(l)];
    if (!c.filled) throw SequencingError("transcription: missing cache");
    auto topk = [&](const T* row, T* v, std::int32_t* ix) {
        std::vector<int> ord(static_cast<size_t>(w));
        for (int j = 0; j < w; ++j) ord[j] = j;
        std::sort(ord.begin(), ord.end(), [&](int a, int b) {
            return std::fabs(row[a]) > std::fabs(row[b]) || (std::fabs(row[a]) == std::fabs(row[b]) && a < b);
        });
        std::sort(ord.begin(), ord.begin() + k);
        for (int j = 0; j < k; ++j) { ix[j] = ord[j]; v[j] = row[ord[j]]; }
    };
    auto block = [&](const std::vector<T>& V, const std::vector<std::int32_t>& I, const T* W, const T* b, std::vector<T>& M) {
        M.assign(static_cast<size_t>(n) * w, T(0));
        for (index_t r = 0; r < n; ++r) {
            std::vector<T> acc(static_cast<size_t>(w), T(0)), part(static_cast<size_t>(w));
            for (index_t s0 = g.row_ptr[r]; s0 < g.row_ptr[r + 1]; s0 += kAggSeg) {
                std::fill(part.begin(), part.end(), T(0));
                for (index_t q = s0; q < std::min<index_t>(s0 + kAggSeg, g.row_ptr[r + 1]); ++q) {
                    const index_t cc = g.col_idx[q];
                    for (int j = 0; j < k; ++j) part[I[cc * k + j]] = part[I[cc * k + j]] + sc.col_f[cc] * V[cc * k + j];
                }
                for (int j = 0; j < w; ++j) acc[j] = (s0 == g.row_ptr[r]) ? part[j] : acc[j] + part[j];
            }
            for (int j = 0; j < w; ++j) acc[j] = sc.row_f[r] * acc[j];
            for (int j = 0; j < w; ++j) {
                T h = T(0);
                if (f.use_weight) { for (int m = 0; m < w; ++m) h = std::fma(acc[m], W[m * w + j], h); }
                else h = acc[j];
                if (f.use_bias) h = h + b[j];
                M[r * w + j] = h;
            }
        }
    };
    // backward block output only (parameter grads are checked by the modular path)
    auto bwd_out = [&](const std::vector<T>& M, const std::vector<std::int32_t>& I, const T* W, T* out) {
        std::vector<T> vg(static_cast<size_t>(n) * k);
        for (index_t r = 0; r < n; ++r)
            for (int j = 0; j < k; ++j) {
                const int col = I[r * k + j];
                T t = T(0);
                if (f.use_weight) { for (int m = 0; m < w; ++m) t = std::fma(M[r * w + m], W[col * w + m], t); }
                else t = M[r * w + col];
                vg[r * k + j] = t;
            }
        for (index_t r = 0; r < n; ++r) {
            std::vector<T> acc(static_cast<size_t>(w), T(0)), part(static_cast<size_t>(w));
            for (index_t s0 = g.trow_ptr[r]; s0 < g.trow_ptr[r + 1]; s0 += kAggSeg) {
                std::fill(part.begin(), part.end(), T(0));
                for (index_t q = s0; q < std::min<index_t>(s0 + kAggSeg, g.trow_ptr[r + 1]); ++q) {
                    const index_t cc = g.tcol_idx[q];
                    for (int j = 0; j < k; ++j) part[I[cc * k + j]] = part[I[cc * k + j]] + sc.row_f[cc] * vg[cc * k + j];
                }
                for (int j = 0; j < w; ++j) acc[j] = (s0 == g.trow_ptr[r]) ? part[j] : acc[j] + part[j];
            }
            for (int j = 0; j < w; ++j) out[r * D + j] = sc.col_f[r] * acc[j];
        }
    };
    std::vector<T> g1(static_cast<size_t>(n) * w), g2(static_cast<size_t>(n) * w), V2(static_cast<size_t>(n) * k), V1(static_cast<size_t>(n) * k), M1, Z1, M2(static_cast<size_t>(n) * w), B2;
    std::vector<std::int32_t> I2(static_cast<size_t>(n) * k), I1(static_cast<size_t>(n) * k);
    for (index_t r = 0; r < n; ++r) for (int j = 0; j < w; ++j) { g1[r * w + j] = Gm[r * D + j]; g2[r * w + j] = Gm[r * D + w + j]; }
    for (index_t r = 0; r < n; ++r) topk(&g2[r * w], &V2[r * k], &I2[r * k]);                  // line 4
    block(V2, I2, net.W(l, 1), net.B(l, 1), B2);                                                 // line 5
    M1.resize(static_cast<size_t>(n) * w);
    for (index_t q = 0; q < n * w; ++q) M1[q] = g1[q] - B2[q];
    for (index_t r = 0; r < n; ++r) topk(&M1[r * w], &V1[r * k], &I1[r * k]);                  // line 6
    block(V1, I1, net.W(l, 0), net.B(l, 0), Z1);
    for (index_t r = 0; r < n; ++r) {                                                             // line 7
        std::vector<T> s(static_cast<size_t>(w), T(0));
        for (int j = 0; j < k; ++j) s[I2[r * k + j]] = V2[r * k + j];
        for (int j = 0; j < w; ++j) M2[r * w + j] = s[j] - Z1[r * w + j];
    }
    const bool local = net.cfg.index_source == IDX_ALG2_LOCAL;
    bwd_out(M1, local ? I1 : c.i1, net.W(l, 0), Gm);                                             // line 8
    bwd_out(M2, local ? I2 : c.i2, net.W(l, 1), Gm + w);
    c = LayerCache<T>{};                                                                          // line 9
}
}  // namespace

extern "C" {

const char* gsro_last_error() { return g_err.c_str(); }

int gsro_set_tf32(int on) {
    gsro::tf32_transform() = on != 0;
    return 0;
}

int gsro_set_threads(int n) {
    return guarded([&] {
        pool_ref() = nullptr;
        g_pool.reset();
        if (n > 1) {
            g_pool = std::make_unique<ThreadPool>(n);
            pool_ref() = g_pool.get();
        }
    });
}

unsigned long long gsro_work_muladds() { return work().scalar_mul_adds.load(); }
void gsro_work_reset() { work().scalar_mul_adds = 0; work().rows_touched = 0; }

void* gsro_graph_create(long long n, long long e, const long long* row_ptr, const int* col_idx, int norm) {
    Graph* g = nullptr;
    int st = guarded([&] {
        auto gg = std::make_unique<Graph>();
        gg->n = n; gg->e = e; gg->norm = norm;
        if (norm < 0 || norm > 2) throw ConfigError("norm_mode");
        gg->row_ptr.assign(row_ptr, row_ptr + n + 1);
        gg->col_idx.assign(col_idx, col_idx + e);
        gg->validate();
        gg->build_transpose();
        g = gg.release();
    });
    return st == 0 ? g : nullptr;
}

void* gsro_graph_from_edges(long long n, long long m, const long long* uv, int norm) {
    Graph* g = nullptr;
    int st = guarded([&] { g = new Graph(from_edge_list(n, m, reinterpret_cast<const std::int64_t*>(uv), norm)); });
    return st == 0 ? g : nullptr;
}

long long gsro_graph_e(void* h) { return static_cast<Graph*>(h)->e; }
void gsro_graph_csr(void* h, long long* row_ptr, int* col_idx) {
    auto* g = static_cast<Graph*>(h);
    std::copy(g->row_ptr.begin(), g->row_ptr.end(), row_ptr);
    std::copy(g->col_idx.begin(), g->col_idx.end(), col_idx);
}
void gsro_graph_csc(void* h, long long* trow_ptr, int* tcol_idx) {
    auto* g = static_cast<Graph*>(h);
    std::copy(g->trow_ptr.begin(), g->trow_ptr.end(), trow_ptr);
    std::copy(g->tcol_idx.begin(), g->tcol_idx.end(), tcol_idx);
}
void gsro_graph_destroy(void* h) { delete static_cast<Graph*>(h); }

#define GSRO_OPS(T, S)                                                                                          \
    int gsro_gs_topk_##S(long long n, int w, int k, const T* x, long long ldx, T* vals, int* idx) {                \
        return guarded([&] { gs_topk<T>(n, w, k, x, ldx, vals, idx); });                                        \
    }                                                                                                           \
    int gsro_scatter_##S(long long n, int w, int k, const T* vals, const int* idx, T* out, long long ldo) {       \
        return guarded([&] { scatter<T>(n, w, k, vals, idx, out, ldo); });                                      \
    }                                                                                                           \
    int gsro_gather_##S(long long n, int w, int k, const T* x, long long ldx, const int* idx, T* vals) {           \
        return guarded([&] { gather<T>(n, w, k, x, ldx, idx, vals); });                                         \
    }                                                                                                           \
    int gsro_spmm_##S(void* g, int tr, int cols, const T* x, long long ldx, T* y, long long ldy) {                 \
        return guarded([&] { spmm<T>(*static_cast<Graph*>(g), tr != 0, cols, x, ldx, y, ldy); });               \
    }                                                                                                           \
    int gsro_spmm_sparse_##S(void* g, int tr, int w, int k, const T* vals, const int* idx, T* y, long long ldy) {   \
        return guarded([&] { spmm_sparse<T>(*static_cast<Graph*>(g), tr != 0, w, k, vals, idx, y, ldy); });    \
    }                                                                                                           \
    int gsro_gemm_##S(long long M, int K, int N, const T* a, long long lda, const T* b, long long ldb, int bt,    \
                      int acc, T* out, long long ldo) {                                                         \
        return guarded([&] { gemm<T>(M, K, N, a, lda, b, ldb, bt != 0, acc != 0, out, ldo); });                \
    }                                                                                                           \
    int gsro_block_fwd_##S(void* g, int w, int k, const T* vals, const int* idx, const T* W, const T* b, int uw,   \
                           int ub, int epi, const T* R, long long ldr, const T* rv, const int* ri, T* out,       \
                           long long ldo) {                                                                     \
        return guarded([&] {                                                                                    \
            gsr_block_apply<T>(*static_cast<Graph*>(g), w, k, vals, idx, W, b, BlockFlags{uw != 0, ub != 0}, epi, \
                               R, ldr, rv, ri, out, ldo);                                                       \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_dense_block_##S(void* g, int w, const T* x, long long ldx, const T* W, const T* b, int uw, int ub,    \
                             T* out, long long ldo) {                                                           \
        return guarded([&] {                                                                                    \
            dense_block_apply<T>(*static_cast<Graph*>(g), w, x, ldx, W, b, BlockFlags{uw != 0, ub != 0}, EPI_NONE, \
                                 nullptr, 0, out, ldo);                                                         \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_block_bwd_##S(void* g, int w, int k, const T* m, long long ldm, const int* isrc, const T* fv,         \
                           const int* fi, const T* W, int uw, int ub, T* out, long long ldo, T* dW, T* db) {     \
        return guarded([&] {                                                                                    \
            gsr_backward_block<T>(*static_cast<Graph*>(g), w, k, m, ldm, isrc, fv, fi, W, BlockFlags{uw != 0, ub != 0}, \
                                  out, ldo, dW, db);                                                            \
        });                                                                                                     \
    }                                                                                                           \
    void* gsro_net_create_##S(void* g, int mode, int L, int D, int C, int k, int d_in, int uw, int ub, int isrc) { \
        NetBox* box = nullptr;                                                                                  \
        int st = guarded([&] {                                                                                  \
            auto net = std::make_unique<Net<T>>();                                                              \
            net->cfg.mode = mode; net->cfg.L = L; net->cfg.D = D; net->cfg.C = C; net->cfg.k = k;               \
            net->cfg.d_in = d_in; net->cfg.flags = BlockFlags{uw != 0, ub != 0}; net->cfg.index_source = isrc;  \
            net->cfg.validate();                                                                                \
            net->g = static_cast<Graph*>(g);                                                                    \
            net->params.assign(static_cast<size_t>(net->cfg.num_params()), T(0));                              \
            net->grads.assign(static_cast<size_t>(net->cfg.num_params()), T(0));                                \
            net->cache.assign(static_cast<size_t>(L), LayerCache<T>{});                                         \
            box = new NetBox{sizeof(T) == 8, net.release()};                                                    \
        });                                                                                                     \
        return st == 0 ? box : nullptr;                                                                         \
    }                                                                                                           \
    int gsro_net_set_params_##S(void* h, const T* p) {                                                          \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        std::copy(p, p + net->params.size(), net->params.begin());                                              \
        return 0;                                                                                               \
    }                                                                                                           \
    int gsro_net_get_params_##S(void* h, T* p) {                                                                \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        std::copy(net->params.begin(), net->params.end(), p);                                                   \
        return 0;                                                                                               \
    }                                                                                                           \
    int gsro_net_get_grads_##S(void* h, T* p) {                                                                 \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        std::copy(net->grads.begin(), net->grads.end(), p);                                                     \
        return 0;                                                                                               \
    }                                                                                                           \
    int gsro_net_zero_grads_##S(void* h) {                                                                      \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        std::fill(net->grads.begin(), net->grads.end(), T(0));                                                  \
        return 0;                                                                                               \
    }                                                                                                           \
    int gsro_net_forward_##S(void* h, const T* X0, T* X, T* yhat) {                                             \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] { net_forward<T>(*net, X0, X, yhat); });                                             \
    }                                                                                                           \
    int gsro_net_loss_grads_##S(void* h, const T* X0, const T* y, const unsigned char* mask, double* loss,        \
                                T* yhat, T* X) {                                                                \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            const index_t n = net->g->n;                                                                        \
            std::vector<T> gy(static_cast<size_t>(n));                                                          \
            net_forward<T>(*net, X0, X, yhat);                                                                  \
            *loss = mse_loss<T>(n, yhat, y, mask, gy.data());                                                   \
            net_backward<T>(*net, X0, X, gy.data());                                                            \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_net_layer_forward_##S(void* h, int l, T* X) {                                                      \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            if (net->cfg.mode == MODE_ALG12) gsr_forward_layer<T>(*net, l, X);                                  \
            else rev_forward_layer<T>(*net, l, X);                                                              \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_net_layer_inverse_##S(void* h, int l, T* X) {                                                      \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            if (net->cfg.mode == MODE_ALG12) throw ConfigError("alg12 layers are not invertible");              \
            rev_inverse_layer<T>(*net, l, X);                                                                   \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_net_layer_backward_##S(void* h, int l, T* Y, T* G) {                                               \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            if (net->cfg.mode == MODE_ALG12) gsr_backward_layer<T>(*net, l, G);                                 \
            else rev_backward_layer<T>(*net, l, Y, G);                                                          \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_net_transcribe_forward_##S(void* h, int l, T* X) {                                                 \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            if (net->cfg.mode != MODE_ALG12) throw ConfigError("transcription is Alg. 1 only");                  \
            transcribe_alg1<T>(*net, l, X);                                                                     \
        });                                                                                                     \
    }                                                                                                           \
    int gsro_net_transcribe_backward_##S(void* h, int l, T* G) {                                                \
        auto* net = static_cast<Net<T>*>(static_cast<NetBox*>(h)->net);                                         \
        return guarded([&] {                                                                                    \
            if (net->cfg.mode != MODE_ALG12) throw ConfigError("transcription is Alg. 2 only");                  \
            transcribe_alg2<T>(*net, l, G);                                                                     \
        });                                                                                                     \
    }                                                                                                           \
    double gsro_mse_##S(long long n, const T* yhat, const T* y, const unsigned char* mask, T* gy) {            \
        double out = -1.0;                                                                                      \
        int st = guarded([&] { out = mse_loss<T>(n, yhat, y, mask, gy); });                                     \
        return st == 0 ? out : -1.0;                                                                            \
    }                                                                                                           \
    void gsro_adam_##S(long long n, T* p, const T* g, T* m, T* v, T lr, T b1, T b2, T eps, T wd, T bc1, T bc2) { \
        adam_step<T>(n, p, g, m, v, lr, b1, b2, eps, wd, bc1, bc2);                                             \
    }                                                                                                           \
    void gsro_sgd_##S(long long n, T* p, const T* g, T* mom, T lr, T momentum) {                                \
        sgd_step<T>(n, p, g, mom, lr, momentum);                                                                \
    }

GSRO_OPS(float, f32)
GSRO_OPS(double, f64)

long long gsro_net_num_params(void* h) {
    auto* box = static_cast<NetBox*>(h);
    if (box->is64) return static_cast<Net<double>*>(box->net)->cfg.num_params();
    return static_cast<Net<float>*>(box->net)->cfg.num_params();
}

int gsro_net_set_quant(void* h, int shift) {
    auto* box = static_cast<NetBox*>(h);
    if (shift < 0 || shift > 60) return 1;
    if (box->is64) static_cast<Net<double>*>(box->net)->cfg.qshift = shift;
    else static_cast<Net<float>*>(box->net)->cfg.qshift = shift;
    return 0;
}

void gsro_net_destroy(void* h) {
    auto* box = static_cast<NetBox*>(h);
    if (!box) return;
    if (box->is64) delete static_cast<Net<double>*>(box->net);
    else delete static_cast<Net<float>*>(box->net);
    delete box;
}

}  // extern "C"
