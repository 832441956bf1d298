// GSR-GNN training-step kernels for sm_100a (FP32-strict path).
//
// The hot path of the reference maps onto three kernel
// families, each bit-compatible with the CPU oracle's per-row arithmetic
// (oracle/gsr_oracle.hpp header comment) so that top-k masks and CSR indexing
// match the reference restatement exactly:
//
//   k_tile  — one persistent kernel for every "block" shape of the path:
//             neighbour aggregation (sparse CBSR records: spmm_sparse
//             SPEC.md:177-185; dense rows: spmm SPEC.md:168-176) into a
//             64-row shared-memory tile → dense transform (·W or ·Wᵀ,
//             SPEC.md:95-103) → bias → residual epilogue (Eq. 6-7 /
//             Alg. 1-2 add/sub/scatter) → optional GS top-k of the output
//             (emits the next block's compressed records) → optional dW/db
//             partial sums (deterministic per-CTA slots, double accumulators).
//             Fusion removes every intermediate HBM round-trip between
//             aggregation, sparse nonlinearity and transform (north_star).
//   k_gs    — GS top-k of one plane or of a left-to-right sum
//             of planes (Eq. 6's y'_0 = Σ_{j≥2} x_j never materialised).
//   small   — encoder / head / masked-MSE / Adam.
//
// Aggregation keeps the reference's row-ownership determinism contract
// (/root/reference/proj/include/gsr/threads.hpp:14-16): one half-warp (sparse)
// or one warp (dense) owns an output row and walks its edges in CSR order.
#include "kernels.cuh"
#include "common.cuh"

#include <cstdio>

namespace gsrk {

namespace {

using dev::kFull;
using dev::ld4;

// ---------------------------------------------------------------------------
// k_gs: GS of a plane or of a left-to-right sum of planes.
// ---------------------------------------------------------------------------
template <int W, int TPR>
__global__ void __launch_bounds__(kThreads) k_gs(GsArgs a) {
    constexpr int P = W / TPR;
    constexpr int ROWS = kThreads / TPR;
    const int g = threadIdx.x / TPR, q = threadIdx.x % TPR;
    const int row = blockIdx.x * ROWS + g;
    const bool valid = row < a.n;
    float x[P];
#pragma unroll
    for (int i = 0; i < P; ++i) x[i] = 0.f;
    if (valid) {
        for (int p = 0; p < a.nplanes; ++p) {
            const float* src = a.planes[p] + static_cast<size_t>(row) * a.ld + q * P;
#pragma unroll
            for (int i = 0; i < P; i += 4) {
                if (q * P + i < a.ld) {
                    const float4 v = ld4(src + i);
                    if (p == 0) { x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w; }
                    else {
                        x[i] = __fadd_rn(x[i], v.x); x[i + 1] = __fadd_rn(x[i + 1], v.y);
                        x[i + 2] = __fadd_rn(x[i + 2], v.z); x[i + 3] = __fadd_rn(x[i + 3], v.w);
                    }
                }
            }
        }
    }
    dev::gs_select<P, TPR>(x, q, a.w, a.k, valid, a.rec + static_cast<size_t>(valid ? row : 0) * rec_bytes(a.k));
}

// Fixed-order reduction of per-CTA partials (double) into a float gradient.
// 32 outputs per block, each summed by 8 warps over contiguous partial
// ranges in fixed order, the 8 range sums then added in order: deterministic,
// coalesced across the 32 outputs, and 8× the parallelism of a thread per output.
__global__ void __launch_bounds__(256) k_reduce_parts(const double* __restrict__ part, int nparts, int stride, int len, float* __restrict__ out,
                                                      int accumulate) {
    __shared__ double red[8][32];
    const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
    const int i = blockIdx.x * 32 + lane;
    const int per = (nparts + 7) / 8, p0 = c * per, p1 = min(nparts, p0 + per);
    double s = 0.0;
    dev::pdl_wait();
    if (i < len) {
#pragma unroll 8
        for (int p = p0; p < p1; ++p) s += part[static_cast<size_t>(p) * stride + i];
    }
    red[c][lane] = s;
    __syncthreads();
    if (c == 0 && i < len) {
        double t = red[0][lane];
        for (int q = 1; q < 8; ++q) t += red[q][lane];
        if (accumulate) t += static_cast<double>(out[i]);
        out[i] = static_cast<float>(t);
    }
}

// Single-CTA fixed-order sum of n doubles (loss partials), scaled.
__global__ void k_sum_double(const double* __restrict__ in, int n, double scale, double* __restrict__ out) {
    __shared__ double red[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) s += in[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0] * scale;
}

// u = p0 + p1 + ... (left to right), whole planes.
__global__ void k_sum_planes(GsArgs a, float* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(a.n) * a.ld) return;
    float s = a.planes[0][i];
    for (int p = 1; p < a.nplanes; ++p) s = __fadd_rn(s, a.planes[p][i]);
    out[i] = s;
}

// Adam bias corrections for step t (t incremented on device so the whole
// step can be replayed from a CUDA graph).
__global__ void k_adam_prep(long long* t, double b1, double b2, float* bc) {
    const long long s = ++(*t);
    bc[0] = static_cast<float>(1.0 - pow(b1, static_cast<double>(s)));
    bc[1] = static_cast<float>(1.0 - pow(b2, static_cast<double>(s)));
}

__global__ void k_rec_unpack(const uint8_t* __restrict__ rec, int n, int k, float* vals, int* idx) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    const int r = i / k, j = i % k;
    const uint8_t* rc = rec + static_cast<size_t>(r) * rec_bytes(k);
    idx[i] = rc[j];
    vals[i] = reinterpret_cast<const float*>(rc + rec_kh(k))[j];
}

__global__ void k_rec_pack(const float* __restrict__ vals, const int* __restrict__ idx, int n, int k, uint8_t* rec) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * k) return;
    const int r = i / k, j = i % k;
    uint8_t* rc = rec + static_cast<size_t>(r) * rec_bytes(k);
    rc[j] = static_cast<uint8_t>(idx[i]);
    reinterpret_cast<float*>(rc + rec_kh(k))[j] = vals[i];
}

// ---------------------------------------------------------------------------
// encoder / head / loss / optimizer
// ---------------------------------------------------------------------------
// The node-wise kernels move the n × D activation once (≈ 1 GB at c3): their
// layouts are chosen for whole 16 B accesses. A "quad" is 4 consecutive
// columns m..m+3 of one plane (ld is a multiple of 4); NQ = C·ld/4 quads per
// row; padding columns m ≥ w are written as 0.
constexpr int kEncRows = 64;  // k_encoder rows per CTA

// X[p][r][m] = fma-chain_a X0[r][a]·We[a][p·w+m] + be[p·w+m] (oracle
// encoder_forward: gemm_row, then + be, then the residual grid). Thread →
// one quad (its DIN × 4 weights and 4 biases in registers) and the CTA's rows
// ≡ its lane group (mod RL = 256 / NQ); one float4 store per row.
template <int DIN, bool EXACT>
__global__ void __launch_bounds__(256) k_encoder(const float* __restrict__ X0, int n, int d_in_rt, const float* __restrict__ We,
                                                 const float* __restrict__ be, int D, int C, int w, int ld, float* __restrict__ X, float qs,
                                                 float qi) {
    const int d_in = EXACT ? DIN : d_in_rt;  // EXACT: d_in is DIN, every input-width check folds away
    const int L4 = ld >> 2, NQ = C * L4;
    const int RL = NQ >= 256 ? 1 : 256 / NQ;
    const int r0 = blockIdx.x * kEncRows, r1 = min(n, r0 + kEncRows);
    for (int qb = 0; qb < NQ; qb += 256) {
        const int q = NQ >= 256 ? qb + static_cast<int>(threadIdx.x) : static_cast<int>(threadIdx.x) % NQ;
        const int g = NQ >= 256 ? 0 : static_cast<int>(threadIdx.x) / NQ;
        if (g >= RL || q >= NQ) continue;
        const int p = q / L4, m = 4 * (q - p * L4);
        float wv[DIN][4], bv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool ok = m + j < w;
#pragma unroll
            for (int t = 0; t < DIN; ++t) wv[t][j] = (ok && t < d_in) ? __ldg(We + static_cast<size_t>(t) * D + p * w + m + j) : 0.f;
            bv[j] = ok ? __ldg(be + p * w + m + j) : 0.f;
        }
#pragma unroll 4
        for (int r = r0 + g; r < r1; r += RL) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const float* xr = X0 + static_cast<size_t>(r) * d_in;
            float xv[DIN];
            if (d_in == DIN) {  // whole 16 B loads of the input row
#pragma unroll
                for (int t = 0; t < DIN; t += 4) {
                    const float4 v = dev::ld4(xr + t);
                    xv[t] = v.x; xv[t + 1] = v.y; xv[t + 2] = v.z; xv[t + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int t = 0; t < DIN; ++t) xv[t] = t < d_in ? __ldg(xr + t) : 0.f;
            }
#pragma unroll
            for (int t = 0; t < DIN; ++t) {
                if (t < d_in) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[j] = fmaf(xv[t], wv[t][j], acc[j]);
                }
            }
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = m + j < w ? dev::quant(__fadd_rn(acc[j], bv[j]), qs, qi) : 0.f;
            *reinterpret_cast<float4*>(X + (static_cast<size_t>(p) * n + r) * ld + m) = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
}

// ŷ[r] = fma-chain over col = p·w + m of X[p][r][m]·wh[col], + bh (oracle
// head_forward); masked MSE gradient and per-CTA loss partials (mse_loss).
// Thread t owns row r0 + t. The CTA stages 32-column slices of its rows
// through shared memory with coalesced 16 B loads; the row stride of 33 makes
// both the staging stores and the thread-per-row chain conflict-free.
__global__ void __launch_bounds__(kThreads) k_head_loss(const float* __restrict__ X, int n, int C, int w, int ld, const float* __restrict__ wh,
                                                        const float* __restrict__ bh, const float* __restrict__ y,
                                                        const uint8_t* __restrict__ mask, float cnt, float* __restrict__ yhat,
                                                        float* __restrict__ gy, double* __restrict__ loss_part) {
    constexpr int SP = 33;
    __shared__ float sm[kThreads * SP];
    __shared__ double red[kThreads / 32];
    const int t = threadIdx.x, r0 = blockIdx.x * kThreads, r = r0 + t;
    float acc = 0.f;
    for (int p = 0; p < C; ++p) {
        const float* Xp = X + (static_cast<size_t>(p) * n + r0) * ld;
        for (int c0 = 0; c0 < w; c0 += 32) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int e = t + j * kThreads, rr = e >> 3, q = e & 7;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (r0 + rr < n && c0 + 4 * q < ld) v = dev::ld4(Xp + static_cast<size_t>(rr) * ld + c0 + 4 * q);
                float* s = sm + rr * SP + 4 * q;
                s[0] = v.x; s[1] = v.y; s[2] = v.z; s[3] = v.w;
            }
            __syncthreads();
            const int nm = w - c0 < 32 ? w - c0 : 32;
            const float* wp = wh + p * w + c0;
            for (int m = 0; m < nm; ++m) acc = fmaf(sm[t * SP + m], __ldg(wp + m), acc);
            __syncthreads();
        }
    }
    double l = 0.0;
    if (r < n) {
        const float yh = __fadd_rn(acc, __ldg(bh));
        yhat[r] = yh;
        if (mask[r]) {
            const float d = __fsub_rn(yh, y[r]);
            l = static_cast<double>(d) * static_cast<double>(d);
            gy[r] = __fdiv_rn(__fmul_rn(2.f, d), cnt);
        } else {
            gy[r] = 0.f;
        }
    }
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(kFull, l, o);
    if ((t & 31) == 0) red[t >> 5] = l;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int i = 0; i < kThreads / 32; ++i) s += red[i];
        loss_part[blockIdx.x] = s;
    }
}

// Ordered combine of the CTA's RL row-lane partials into pp (deterministic):
// lane group 0 stores, groups 1..RL−1 add in turn.
__device__ __forceinline__ void combine_lanes(double* pp, int idx, double v, int g, int RL, bool act) {
    for (int gg = 0; gg < RL; ++gg) {
        if (act && g == gg) pp[idx] = gg == 0 ? v : pp[idx] + v;
        __syncthreads();
    }
}

// Fixed-order double sum of gy over [r0, r1) by warp 0 → *out.
__device__ __forceinline__ void warp_sum_rows(const float* __restrict__ v, int r0, int r1, double* out) {
    if (threadIdx.x >= 32) return;
    double s = 0.0;
    for (int r = r0 + static_cast<int>(threadIdx.x); r < r1; r += 32) s += static_cast<double>(__ldg(v + r));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (threadIdx.x == 0) *out = s;
}

// G[p][r][m] = gy[r]·wh[p·w+m]; per-CTA partials of dwh = Σ_r X·gy and
// dbh = Σ_r gy over the CTA's contiguous row range (part layout [cta][D + 1]).
// Thread → one quad and the rows ≡ its lane group (mod RL = 256 / NQ);
// 32-row float FMA chunks flushed into double accumulators.
__global__ void __launch_bounds__(256) k_head_bwd(const float* __restrict__ X, const float* __restrict__ gy, int n, int D, int C, int w, int ld,
                                                  const float* __restrict__ wh, float* __restrict__ G, double* __restrict__ part,
                                                  int rows_per_cta) {
    const int L4 = ld >> 2, NQ = C * L4, RL = 256 / NQ;
    const int tid = threadIdx.x, q = tid % NQ, g = tid / NQ;
    const bool act = g < RL;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    const int p = q / L4, m = 4 * (q - p * L4);
    float whv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) whv[j] = m + j < w ? __ldg(wh + p * w + m + j) : 0.f;
    double sd[4] = {0.0, 0.0, 0.0, 0.0};
    if (act) {
        const size_t pbase = static_cast<size_t>(p) * n;
        for (int rc = r0 + g; rc < r1; rc += 32 * RL) {  // 32-row float chunks
            float sf[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
            for (int rb = rc; rb < rc + 32 * RL && rb < r1; rb += 8 * RL) {  // eight rows of loads in flight
                float4 x[8];
                float gr[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = rb + u * RL;
                    const bool ok = r < r1;
                    gr[u] = ok ? __ldg(gy + r) : 0.f;
                    x[u] = ok ? dev::ld4(X + (pbase + r) * ld + m) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = rb + u * RL;
                    if (r < r1) {
                        sf[0] = fmaf(x[u].x, gr[u], sf[0]); sf[1] = fmaf(x[u].y, gr[u], sf[1]);
                        sf[2] = fmaf(x[u].z, gr[u], sf[2]); sf[3] = fmaf(x[u].w, gr[u], sf[3]);
                        *reinterpret_cast<float4*>(G + (pbase + r) * ld + m) =
                            make_float4(m < w ? __fmul_rn(gr[u], whv[0]) : 0.f, m + 1 < w ? __fmul_rn(gr[u], whv[1]) : 0.f,
                                        m + 2 < w ? __fmul_rn(gr[u], whv[2]) : 0.f, m + 3 < w ? __fmul_rn(gr[u], whv[3]) : 0.f);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) sd[j] += static_cast<double>(sf[j]);
        }
    }
    double* pp = part + static_cast<size_t>(blockIdx.x) * (D + 1);
#pragma unroll
    for (int j = 0; j < 4; ++j) combine_lanes(pp, p * w + (m + j < w ? m + j : 0), sd[j], g, RL, act && m + j < w);
    warp_sum_rows(gy, r0, r1, pp + D);
}

// dWe[t][col] = Σ_r X0[r][t]·G[r][col]; dbe[col] = Σ_r G[r][col]
// (part layout [cta][d_in·D + D]). Thread → V consecutive columns of a plane
// (NV = C·ld/V per row) and the CTA's rows ≡ its lane group (mod RL = 256/NV);
// 32-row float FMA chunks flushed into double accumulators (V = 2 keeps the
// (DIN + 1)·V doubles in registers); lane groups combined in fixed order.
template <int DIN, int V, bool EXACT>
__global__ void __launch_bounds__(256, 2) k_encoder_bwd(const float* __restrict__ X0, const float* __restrict__ G, int n, int d_in_rt, int D, int C,
                                                        int w, int ld, double* __restrict__ part, int rows_per_cta) {
    const int d_in = EXACT ? DIN : d_in_rt;  // EXACT: d_in is DIN, every input-width check folds away
    const int LV = ld / V, NV = C * LV, RL = 256 / NV;
    const int tid = threadIdx.x, q = tid % NV, g = tid / NV;
    const bool act = g < RL;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    const int p = q / LV, m = V * (q - p * LV);
    double sd[DIN + 1][V];
#pragma unroll
    for (int t = 0; t <= DIN; ++t)
#pragma unroll
        for (int j = 0; j < V; ++j) sd[t][j] = 0.0;
    auto ldv = [&](const float* ptr, float (&o)[V]) {
        if constexpr (V == 4) {
            const float4 v = dev::ld4(ptr);
            o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
        } else {
            const float2 v = __ldg(reinterpret_cast<const float2*>(ptr));
            o[0] = v.x; o[1] = v.y;
        }
    };
    if (act) {
        const size_t pbase = static_cast<size_t>(p) * n;
        for (int rc = r0 + g; rc < r1; rc += 32 * RL) {
            float sf[DIN + 1][V];
#pragma unroll
            for (int t = 0; t <= DIN; ++t)
#pragma unroll
                for (int j = 0; j < V; ++j) sf[t][j] = 0.f;
#pragma unroll 1
            for (int rb = rc; rb < rc + 32 * RL && rb < r1; rb += 4 * RL) {  // four rows of loads in flight
                float gv[4][V];
                float xv[4][DIN];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = rb + u * RL;
                    const bool ok = r < r1;
#pragma unroll
                    for (int j = 0; j < V; ++j) gv[u][j] = 0.f;
#pragma unroll
                    for (int t = 0; t < DIN; ++t) xv[u][t] = 0.f;
                    if (ok) {
                        ldv(G + (pbase + r) * ld + m, gv[u]);
                        const float* xr = X0 + static_cast<size_t>(r) * d_in;
                        if (d_in == DIN) {
#pragma unroll
                            for (int t = 0; t < DIN; t += 4) {
                                const float4 v = dev::ld4(xr + t);
                                xv[u][t] = v.x; xv[u][t + 1] = v.y; xv[u][t + 2] = v.z; xv[u][t + 3] = v.w;
                            }
                        } else {
#pragma unroll
                            for (int t = 0; t < DIN; ++t) xv[u][t] = t < d_in ? __ldg(xr + t) : 0.f;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (rb + u * RL < r1) {
#pragma unroll
                        for (int t = 0; t < DIN; ++t)
#pragma unroll
                            for (int j = 0; j < V; ++j) sf[t][j] = fmaf(xv[u][t], gv[u][j], sf[t][j]);
#pragma unroll
                        for (int j = 0; j < V; ++j) sf[DIN][j] = __fadd_rn(sf[DIN][j], gv[u][j]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t <= DIN; ++t)
#pragma unroll
                for (int j = 0; j < V; ++j) sd[t][j] += static_cast<double>(sf[t][j]);
        }
    }
    double* pp = part + static_cast<size_t>(blockIdx.x) * (d_in * D + D);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const bool ok = act && m + j < w;
        const int col = p * w + (m + j < w ? m + j : 0);
#pragma unroll
        for (int t = 0; t < DIN; ++t)
            if (t < d_in) combine_lanes(pp, t * D + col, sd[t][j], g, RL, ok);
        combine_lanes(pp, d_in * D + col, sd[DIN][j], g, RL, ok);
    }
}

__global__ void k_adam(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m, float* __restrict__ v, long long n,
                       float lr, float b1, float b2, float eps, float wd, const float* __restrict__ bc) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float bc1 = bc[0], bc2 = bc[1];
    float gi = g[i];
    if (wd != 0.f) gi = __fadd_rn(gi, __fmul_rn(wd, p[i]));
    const float mi = __fadd_rn(__fmul_rn(b1, m[i]), __fmul_rn(__fsub_rn(1.f, b1), gi));
    const float vi = __fadd_rn(__fmul_rn(b2, v[i]), __fmul_rn(__fsub_rn(1.f, b2), __fmul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const float mh = __fdiv_rn(mi, bc1);
    const float vh = __fdiv_rn(vi, bc2);
    p[i] = __fsub_rn(p[i], __fmul_rn(lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), eps))));
}

__global__ void k_sgd(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ mom, long long n, float lr, float momentum) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (momentum != 0.f) {
        mom[i] = __fadd_rn(__fmul_rn(momentum, mom[i]), g[i]);
        p[i] = __fsub_rn(p[i], __fmul_rn(lr, mom[i]));
    } else {
        p[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
    }
}

__global__ void k_scale(float* __restrict__ p, long long n, float s) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = __fmul_rn(p[i], s);
}

int sm_count();

template <int W, int TPR>


cudaError_t launch_gs_t(const GsArgs& a, cudaStream_t s) {
    constexpr int ROWS = kThreads / TPR;
    const int grid = (a.n + ROWS - 1) / ROWS;
    if (grid == 0) return cudaSuccess;
    k_gs<W, TPR><<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int W>
cudaError_t launch_gs_w(const GsArgs& a, cudaStream_t s) {
    if (a.k <= W / 4) return launch_gs_t<W, 4>(a, s);
    if (a.k <= W / 2) return launch_gs_t<W, 2>(a, s);
    return launch_gs_t<W, 1>(a, s);
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

// Mask-flip diagnostic (gsrc_diag_masks): the index bytes of sampled rows'
// GS records (rows r = j·stride). mode 0 stores them (forward); mode 1 counts
// the sampled rows whose recomputed mask differs (backward reconstruction).
__global__ void k_diag_masks(const uint8_t* __restrict__ rec, int n, int stride, int rb, uint4* __restrict__ store, int mode,
                             unsigned long long* __restrict__ counter) {
    const long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long r = j * stride;
    int diff = 0;
    if (r < n) {
        const uint4 v = *reinterpret_cast<const uint4*>(rec + r * rb);
        if (mode == 0) store[j] = v;
        else {
            const uint4 o = store[j];
            diff = (v.x != o.x) | (v.y != o.y) | (v.z != o.z) | (v.w != o.w);
        }
    }
    if (mode == 1) {
        const int c = __syncthreads_count(diff);
        if (threadIdx.x == 0 && c) atomicAdd(counter, static_cast<unsigned long long>(c));
    }
}

inline int blocks_for(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

namespace tile {
int sm_count_host() { return sm_count(); }
}  // namespace tile

cudaError_t launch_tile_w32(const TileArgs& a, cudaStream_t s, int* g);
cudaError_t launch_tile_w64(const TileArgs& a, cudaStream_t s, int* g);
cudaError_t launch_tile_w128(const TileArgs& a, cudaStream_t s, int* g);
cudaError_t init_tile_w32();
cudaError_t init_tile_w64();
cudaError_t init_tile_w128();

cudaError_t init_kernel_attributes() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {init_tile_w32(), init_tile_w64(), init_tile_w128(), init_fast_attributes()})
        if (r != cudaSuccess) e = r;
    return e;
}

int tile_grid_max(int n) {
    const int tiles = (n + kTileRows - 1) / kTileRows;
    const int cap = sm_count() * 8;
    return tiles < cap ? (tiles > 0 ? tiles : 1) : cap;
}

cudaError_t launch_tile(const TileArgs& a, cudaStream_t s, int* grid_out) {
    if (grid_out) *grid_out = 0;
    if (a.n == 0) return cudaSuccess;
    // Gs aliases the epilogue tile: dW partials cannot share a launch with row epilogues
    if (a.G && (a.gs_out || a.epi == EPI_SCATTER_ADD || a.epi == EPI_SCATTER_SUB || a.epi == EPI_MASKED_ADD || a.epi == EPI_GATHER_REC))
        return cudaErrorInvalidValue;
    if (a.w <= 32) return launch_tile_w32(a, s, grid_out);
    if (a.w <= 64) return launch_tile_w64(a, s, grid_out);
    if (a.w <= 128) return launch_tile_w128(a, s, grid_out);
    return cudaErrorInvalidValue;
}

cudaError_t launch_gs(const GsArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.k < 1 || a.k > a.w) return cudaErrorInvalidValue;
    if (a.w <= 32) return launch_gs_w<32>(a, s);
    if (a.w <= 64) return launch_gs_w<64>(a, s);
    if (a.w <= 128) return launch_gs_w<128>(a, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_reduce_parts(const double* part, int nparts, int stride, int len, float* out, int accumulate, cudaStream_t s) {
    if (len <= 0) return cudaSuccess;
    return launch_pdl(k_reduce_parts, dim3(blocks_for(len, 32)), dim3(256), 0, s, static_cast<const double*>(part), nparts, stride, len, out, accumulate);
}

cudaError_t launch_sum_double(const double* in, int n, double scale, double* out, cudaStream_t s) {
    k_sum_double<<<1, 256, 0, s>>>(in, n, scale, out);
    return cudaGetLastError();
}

cudaError_t launch_sum_planes(const GsArgs& a, float* out, cudaStream_t s) {
    const long long tot = static_cast<long long>(a.n) * a.ld;
    if (!tot) return cudaSuccess;
    k_sum_planes<<<blocks_for(tot, 256), 256, 0, s>>>(a, out);
    return cudaGetLastError();
}

cudaError_t launch_adam_prep(long long* t, double b1, double b2, float* bc, cudaStream_t s) {
    k_adam_prep<<<1, 1, 0, s>>>(t, b1, b2, bc);
    return cudaGetLastError();
}

cudaError_t launch_rec_unpack(const uint8_t* rec, int n, int k, float* vals, int* idx, cudaStream_t s) {
    if (n * k == 0) return cudaSuccess;
    k_rec_unpack<<<blocks_for(static_cast<long long>(n) * k, 256), 256, 0, s>>>(rec, n, k, vals, idx);
    return cudaGetLastError();
}

cudaError_t launch_rec_pack(const float* vals, const int* idx, int n, int k, uint8_t* rec, cudaStream_t s) {
    if (n * k == 0) return cudaSuccess;
    k_rec_pack<<<blocks_for(static_cast<long long>(n) * k, 256), 256, 0, s>>>(vals, idx, n, k, rec);
    return cudaGetLastError();
}

cudaError_t launch_encoder(const float* X0, int n, int d_in, const float* We, const float* be, int D, int C, int w, int ld, float* X,
                           float qs, float qi, cudaStream_t s) {
    if (!n) return cudaSuccess;
    if (d_in > 16) return cudaErrorInvalidValue;
    const int g = blocks_for(n, kEncRows);
    if (d_in == 8) k_encoder<8, true><<<g, 256, 0, s>>>(X0, n, d_in, We, be, D, C, w, ld, X, qs, qi);
    else if (d_in < 8) k_encoder<8, false><<<g, 256, 0, s>>>(X0, n, d_in, We, be, D, C, w, ld, X, qs, qi);
    else k_encoder<16, false><<<g, 256, 0, s>>>(X0, n, d_in, We, be, D, C, w, ld, X, qs, qi);
    return cudaGetLastError();
}

cudaError_t launch_head_loss(const float* X, int n, int D, int C, int w, int ld, const float* wh, const float* bh, const float* y,
                             const uint8_t* mask, float, float cnt, float* yhat, float* gy, double* loss_part, int nparts, cudaStream_t s) {
    (void)D;
    (void)nparts;
    k_head_loss<<<blocks_for(n, kThreads), kThreads, 0, s>>>(X, n, C, w, ld, wh, bh, y, mask, cnt, yhat, gy, loss_part);
    return cudaGetLastError();
}

cudaError_t launch_head_bwd(const float* X, const float* gy, int n, int D, int C, int w, int ld, const float* wh, float* G, double* part,
                            int nparts, cudaStream_t s) {
    if (C * (ld / 4) > 256) return cudaErrorInvalidValue;
    const int rows = (n + nparts - 1) / nparts;
    k_head_bwd<<<nparts, 256, 0, s>>>(X, gy, n, D, C, w, ld, wh, G, part, rows);
    return cudaGetLastError();
}

cudaError_t launch_encoder_bwd(const float* X0, const float* G, int n, int d_in, int D, int C, int w, int ld, double* part, int nparts,
                               cudaStream_t s) {
    if (d_in > 16 || C * (ld / 4) > 256) return cudaErrorInvalidValue;
    const int rows = (n + nparts - 1) / nparts;
    const bool pairs = C * (ld / 2) <= 256;  // two columns per thread when a row's pairs fit one CTA
    if (d_in == 8 && pairs) k_encoder_bwd<8, 2, true><<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, C, w, ld, part, rows);
    else if (d_in <= 8) {
        if (pairs) k_encoder_bwd<8, 2, false><<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, C, w, ld, part, rows);
        else k_encoder_bwd<8, 4, false><<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, C, w, ld, part, rows);
    } else {
        if (pairs) k_encoder_bwd<16, 2, false><<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, C, w, ld, part, rows);
        else k_encoder_bwd<16, 4, false><<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, C, w, ld, part, rows);
    }
    return cudaGetLastError();
}

cudaError_t launch_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1, float b2, float eps, float wd,
                        const float* bc, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_adam<<<blocks_for(n, 256), 256, 0, s>>>(p, g, m, v, n, lr, b1, b2, eps, wd, bc);
    return cudaGetLastError();
}

cudaError_t launch_sgd(float* p, const float* g, float* mom, long long n, float lr, float momentum, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_sgd<<<blocks_for(n, 256), 256, 0, s>>>(p, g, mom, n, lr, momentum);
    return cudaGetLastError();
}

cudaError_t launch_scale(float* p, long long n, float sc, cudaStream_t s) {
    if (!n) return cudaSuccess;
    k_scale<<<blocks_for(n, 256), 256, 0, s>>>(p, n, sc);
    return cudaGetLastError();
}

cudaError_t launch_diag_masks(const uint8_t* rec, int n, int stride, int rb, uint4* store, int mode, unsigned long long* counter,
                              cudaStream_t s) {
    const long long m = (static_cast<long long>(n) + stride - 1) / stride;
    if (!m) return cudaSuccess;
    k_diag_masks<<<blocks_for(m, 256), 256, 0, s>>>(rec, n, stride, rb, store, mode, counter);
    return cudaGetLastError();
}

}  // namespace gsrk
