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

#include <cstdio>

namespace gsrk {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int TR = kTileRows;

template <int W>
struct Cfg {
    static constexpr int ZLD = W + 4;          // smem row stride (floats)
    static constexpr int TPRC = W / 4;         // GEMM threads per row (4 columns each)
    static constexpr int RG = kThreads / TPRC; // GEMM row groups
    static constexpr int RPT = TR / RG;        // GEMM rows per thread
    static constexpr int DWE = W * W / kThreads;  // dW entries per thread
    static constexpr int DMB = DWE / 4;        // dW m-rows per thread (4 n-cols each)
    static constexpr int DNB = W / 4;          // dW n-blocks
    static constexpr bool kRegAcc = (W <= 64);
};

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// ---------------------------------------------------------------------------
// GS top-k selection (ledger :121-126)
// A row of W (padded) columns is owned by TPR consecutive lanes; lane q holds
// columns [q·P, q·P+P). Keys are |x| bit patterns + 1 (padding = 0), so
// unsigned order == magnitude order and padding is never selected. Each lane
// bitonic-sorts its keys, pairs of lanes merge with the half-cleaner
// max(a_i, b_{P-1-i}) (top-P of the union) + bitonic merge, so after log2(TPR)
// rounds every lane holds the row's top-P keys, sorted. T = the k-th largest
// key; ties at T are taken lowest column first, exactly as the oracle's
// (|x| desc, index asc) order.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void bitonic_sort_desc(uint32_t (&s)[P]) {
#pragma unroll
    for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
        for (int stride = size / 2; stride > 0; stride >>= 1) {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const uint32_t a = s[i], b = s[j];
                    const uint32_t hi = max(a, b), lo = min(a, b);
                    if ((i & size) == 0) { s[i] = hi; s[j] = lo; }
                    else { s[i] = lo; s[j] = hi; }
                }
            }
        }
    }
}

template <int P>
__device__ __forceinline__ void bitonic_merge_desc(uint32_t (&s)[P]) {
#pragma unroll
    for (int stride = P / 2; stride > 0; stride >>= 1) {
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int j = i ^ stride;
            if (j > i) {
                const uint32_t a = s[i], b = s[j];
                s[i] = max(a, b);
                s[j] = min(a, b);
            }
        }
    }
}

// All 32 lanes must call this (shuffles); `valid` gates the record write.
template <int P, int TPR>
__device__ __forceinline__ void gs_select(const float (&x)[P], int q, int w, int k, bool valid, uint8_t* rec) {
    uint32_t key[P], s[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const int col = q * P + i;
        key[i] = (col < w) ? ((__float_as_uint(x[i]) & 0x7fffffffu) + 1u) : 0u;
        s[i] = key[i];
    }
    bitonic_sort_desc<P>(s);
#pragma unroll
    for (int lvl = 1; lvl < TPR; lvl <<= 1) {
        uint32_t o[P];
#pragma unroll
        for (int i = 0; i < P; ++i) o[i] = __shfl_xor_sync(kFull, s[P - 1 - i], lvl);
#pragma unroll
        for (int i = 0; i < P; ++i) s[i] = max(s[i], o[i]);
        bitonic_merge_desc<P>(s);
    }
    uint32_t T = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) if (i == k - 1) T = s[i];
    int gt = 0, eq = 0;
#pragma unroll
    for (int i = 0; i < P; ++i) { gt += key[i] > T; eq += key[i] == T; }
    int gt_tot = gt, eq_incl = eq;
#pragma unroll
    for (int d = 1; d < TPR; d <<= 1) {
        gt_tot += __shfl_xor_sync(kFull, gt_tot, d);
        const int v = __shfl_up_sync(kFull, eq_incl, d, TPR);
        if (q >= d) eq_incl += v;
    }
    const int need = k - gt_tot;
    const int take = min(max(need - (eq_incl - eq), 0), eq);
    const int sel = gt + take;
    int sel_incl = sel;
#pragma unroll
    for (int d = 1; d < TPR; d <<= 1) {
        const int v = __shfl_up_sync(kFull, sel_incl, d, TPR);
        if (q >= d) sel_incl += v;
    }
    if (!valid) return;
    int slot = sel_incl - sel;
    int eq_seen = 0;
    float* rv = reinterpret_cast<float*>(rec + rec_kh(k));
#pragma unroll
    for (int i = 0; i < P; ++i) {
        const bool is_eq = key[i] == T;
        const bool pick = key[i] > T || (is_eq && eq_seen < take);
        eq_seen += is_eq;
        if (pick) {
            rec[slot] = static_cast<uint8_t>(q * P + i);
            rv[slot] = x[i];
            ++slot;
        }
    }
}

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
    gs_select<P, TPR>(x, q, a.w, a.k, valid, a.rec + static_cast<size_t>(valid ? row : 0) * rec_bytes(a.k));
}

// ---------------------------------------------------------------------------
// Aggregation (spmm / spmm_sparse) in the canonical segmented
// order of the oracle: each row's edge list is cut into kSeg-edge segments;
// a segment is summed in CSR order from +0 and the row total folds its
// segments left to right. A tile's segments are "items" (≤ kSeg edges each),
// so a hub row of 700 (or 20 000) neighbours is spread over many lanes instead
// of serialising one half-warp (load balance), while every column sum keeps
// the exact oracle order (bit-identical). Items are processed in rounds of
// ≤ kRMax: the round's neighbour ids are staged in smem with coalesced loads,
// each item accumulates into its own smem slot (sparse: half-warp, one value
// slot per lane, 8 neighbour records in flight; dense: warp, W/32 columns per
// lane, 8 neighbour rows in flight), then slots fold into the tile in order.
// ---------------------------------------------------------------------------
constexpr int kSeg = 32;    // == oracle kAggSeg
constexpr int kRMax = 64;   // items per round
constexpr int kPF = 8;      // neighbour prefetch depth

template <int W>
struct Smem {
    static constexpr int ZLD = Cfg<W>::ZLD;
    static constexpr size_t ws = static_cast<size_t>(W) * W;
    static constexpr size_t zs = static_cast<size_t>(TR) * ZLD;
    static constexpr size_t epi = 2 * zs;                                   // Es + Gs
    static constexpr size_t agg = static_cast<size_t>(kRMax) * W + kRMax * kSeg;  // P slots + staged ids
    static constexpr size_t un = epi > agg ? epi : agg;
    static constexpr size_t meta_ints = 2 * (TR + 1) + kRMax + 4;
    static constexpr size_t floats = ws + zs + un + meta_ints;
    static constexpr size_t bytes = floats * sizeof(float);
};

__device__ __forceinline__ int nseg_of(int deg) { return (deg + kSeg - 1) / kSeg; }

template <int W, int AGG>
__device__ __forceinline__ void aggregate_tile(const TileArgs& a, int row0, float* Zs, float* U, int* meta) {
    constexpr int ZLD = Cfg<W>::ZLD;
    constexpr bool SPARSE = AGG == AGG_SPARSE;
    constexpr bool RELU = AGG == AGG_DENSE_RELU;
    float* P = U;                                            // kRMax × W slots (segments of multi-segment rows)
    int* cid = reinterpret_cast<int*>(U + kRMax * W);        // kRMax × kSeg staged neighbour ids
    int* rp = meta;                                          // TR + 1 row pointers
    int* soff = rp + TR + 1;                                 // TR + 1 segment offsets
    int* irow = soff + TR + 1;                               // kRMax item rows
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rows = min(TR, a.n - row0);

    for (int i = tid; i <= rows; i += kThreads) rp[i] = __ldg(a.dir.ptr + row0 + i);
    __syncthreads();
    if (wid == 0) {
        const int r0 = 2 * lane, r1 = 2 * lane + 1;
        const int c0 = r0 < rows ? nseg_of(rp[r0 + 1] - rp[r0]) : 0;
        const int c1 = r1 < rows ? nseg_of(rp[r1 + 1] - rp[r1]) : 0;
        int incl = c0 + c1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += v;
        }
        const int excl = incl - c0 - c1;
        soff[r0] = excl;
        soff[r1] = excl + c0;
        if (lane == 31) soff[TR] = incl;
    }
    __syncthreads();
    const int total = soff[TR];
    const bool unit = a.dir.unit_edge != 0;

    for (int i0 = 0; i0 < total; i0 += kRMax) {
        const int ni = min(kRMax, total - i0);
        for (int s = tid; s < ni; s += kThreads) {
            const int item = i0 + s;
            int lo = 0, hi = rows - 1;  // last row with soff[row] <= item
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (soff[mid] <= item) lo = mid; else hi = mid - 1;
            }
            irow[s] = lo;
        }
        __syncthreads();
        const int rf = irow[0], rl = irow[ni - 1];
        const int Ea = rp[rf] + (i0 - soff[rf]) * kSeg;
        const int Eb = min(rp[rl + 1], rp[rl] + (i0 + ni - soff[rl]) * kSeg);
        for (int e = Ea + tid; e < Eb; e += kThreads) cid[e - Ea] = __ldg(a.dir.idx + e);
        bool any_multi = false;
        if constexpr (SPARSE) {
            // only segments of multi-segment rows go through a slot (zeroed here);
            // single-segment rows accumulate straight into their (zeroed) tile row
            for (int i = tid; i < ni * (W / 4); i += kThreads) {
                const int sl = i / (W / 4);
                const int r = irow[sl];
                if (rp[r + 1] - rp[r] > kSeg) *reinterpret_cast<float4*>(P + sl * W + (i % (W / 4)) * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        __syncthreads();
        if constexpr (SPARSE) {
            const int k = a.k_in, KH = rec_kh(k), RB = rec_bytes(k);
            const int l16 = tid & 15, hw = tid >> 4;
            const unsigned hmask = 0xffffu << (tid & 16);
            for (int s = hw; s < ni; s += kThreads / 16) {
                const int r = irow[s];
                const int e_lo = rp[r] + (i0 + s - soff[r]) * kSeg;
                const int e_hi = min(rp[r + 1], e_lo + kSeg);
                float* pr = (rp[r + 1] - rp[r] > kSeg) ? P + s * W : Zs + r * ZLD;
                if (k <= 16) {
                    const bool act = l16 < k;
                    for (int e = e_lo; e < e_hi; e += kPF) {
                        const int cnt = min(kPF, e_hi - e);
                        int ii[kPF];
                        float vv[kPF];
#pragma unroll
                        for (int u = 0; u < kPF; ++u) {
                            ii[u] = 0;
                            vv[u] = 0.f;
                            if (act && u < cnt) {
                                const int c = cid[e + u - Ea];
                                const uint8_t* rc = a.rec_in + static_cast<size_t>(c) * RB;
                                ii[u] = __ldg(rc + l16);
                                const float v = __ldg(reinterpret_cast<const float*>(rc + KH) + l16);
                                vv[u] = unit ? v : __fmul_rn(__ldg(a.dir.edge_f + c), v);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kPF; ++u) {
                            if (u < cnt) {
                                if (act) pr[ii[u]] = __fadd_rn(pr[ii[u]], vv[u]);
                                __syncwarp(hmask);
                            }
                        }
                    }
                } else {
                    for (int e = e_lo; e < e_hi; ++e) {
                        const int c = cid[e - Ea];
                        const float sc = unit ? 1.f : __ldg(a.dir.edge_f + c);
                        const uint8_t* rc = a.rec_in + static_cast<size_t>(c) * RB;
                        for (int j = l16; j < k; j += 16) {
                            const int m = __ldg(rc + j);
                            const float v = __ldg(reinterpret_cast<const float*>(rc + KH) + j);
                            pr[m] = __fadd_rn(pr[m], unit ? v : __fmul_rn(sc, v));
                        }
                        __syncwarp(hmask);
                    }
                }
                any_multi |= (rp[r + 1] - rp[r] > kSeg);
            }
        } else {
            constexpr int VEC = W / 32;
            const int col = lane * VEC;
            const bool cok = col < a.ld;
            for (int s = wid; s < ni; s += kThreads / 32) {
                const int r = irow[s];
                const int e_lo = rp[r] + (i0 + s - soff[r]) * kSeg;
                const int e_hi = min(rp[r + 1], e_lo + kSeg);
                float acc[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = 0.f;
                for (int e = e_lo; e < e_hi; e += kPF) {
                    const int cnt = min(kPF, e_hi - e);
                    float v[kPF][VEC];
                    float sc[kPF];
#pragma unroll
                    for (int u = 0; u < kPF; ++u) {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) v[u][q] = 0.f;
                        sc[u] = 1.f;
                        if (u < cnt) {
                            const int c = cid[e + u - Ea];
                            if (!unit) sc[u] = __ldg(a.dir.edge_f + c);
                            if (cok) {
                                const float* src = a.x_in + static_cast<size_t>(c) * a.ld + col;
                                if constexpr (VEC == 4) { const float4 f = ld4(src); v[u][0] = f.x; v[u][1] = f.y; v[u][2] = f.z; v[u][3] = f.w; }
                                else if constexpr (VEC == 2) { const float2 f = __ldg(reinterpret_cast<const float2*>(src)); v[u][0] = f.x; v[u][1] = f.y; }
                                else v[u][0] = __ldg(src);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kPF; ++u) {
                        if (u < cnt) {
#pragma unroll
                            for (int q = 0; q < VEC; ++q) {
                                float xv = v[u][q];
                                if (RELU) xv = xv > 0.f ? xv : 0.f;
                                acc[q] = __fadd_rn(acc[q], unit ? xv : __fmul_rn(sc[u], xv));
                            }
                        }
                    }
                }
                const bool multi = rp[r + 1] - rp[r] > kSeg;
                float* dst = multi ? P + s * W : Zs + r * ZLD;
                if (cok) {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) dst[col + q] = acc[q];
                }
                any_multi |= multi;
            }
        }
        // fold segment slots of multi-segment rows into their tile rows, in order
        if (__syncthreads_or(any_multi)) {
            constexpr int TPG = W / 4;
            constexpr int NG = kThreads / TPG;
            const int g = tid / TPG, c4 = (tid % TPG) * 4;
            for (int r = g; r < rows; r += NG) {
                if (rp[r + 1] - rp[r] <= kSeg) continue;
                const int s_lo = max(soff[r], i0), s_hi = min(soff[r + 1], i0 + ni);
                for (int it = s_lo; it < s_hi; ++it) {
                    const float4 pv = *reinterpret_cast<const float4*>(P + (it - i0) * W + c4);
                    float4* z = reinterpret_cast<float4*>(Zs + r * ZLD + c4);
                    if (it == soff[r]) *z = pv;
                    else {
                        float4 zv = *z;
                        zv.x = __fadd_rn(zv.x, pv.x); zv.y = __fadd_rn(zv.y, pv.y);
                        zv.z = __fadd_rn(zv.z, pv.z); zv.w = __fadd_rn(zv.w, pv.w);
                        *z = zv;
                    }
                }
            }
            __syncthreads();
        }
    }
    // row normalisation y = row_scale · acc (rows of this tile)
    {
        constexpr int TPG = W / 4;
        for (int i = tid; i < rows * TPG; i += kThreads) {
            const int r = i / TPG, c4 = (i % TPG) * 4;
            const float f = __ldg(a.dir.out_f + row0 + r);
            float4* z = reinterpret_cast<float4*>(Zs + r * ZLD + c4);
            float4 zv = *z;
            zv.x = __fmul_rn(f, zv.x); zv.y = __fmul_rn(f, zv.y); zv.z = __fmul_rn(f, zv.z); zv.w = __fmul_rn(f, zv.w);
            *z = zv;
        }
    }
}

// ---------------------------------------------------------------------------
// k_tile — persistent fused block kernel. TPR > 0 selects the GS-of-output
// lane grouping (0: no GS epilogue compiled in).
// ---------------------------------------------------------------------------
template <int W, int AGG, int TPR>
__global__ void __launch_bounds__(kThreads) k_tile(TileArgs a) {
    using C = Cfg<W>;
    constexpr int ZLD = C::ZLD;
    using S = Smem<W>;
    extern __shared__ __align__(16) float smem[];
    float* Ws = smem;                    // W×W transform (padded with zeros)
    float* Zs = Ws + S::ws;              // aggregated tile
    float* U = Zs + S::zs;               // union: aggregation slots | epilogue tiles
    float* Es = U;                       // epilogue tile (scatter source / outputs)
    float* Gs = Es + TR * ZLD;           // upstream-gradient tile (dW)
    int* meta = reinterpret_cast<int*>(U + S::un);

    const int tid = threadIdx.x;
    const int n_tiles = (a.n + TR - 1) / TR;
    const bool do_dw = a.G != nullptr;
    const bool do_gemm = a.gemm != GEMM_NONE;

    // transform matrix once per CTA (zero padded to W×W)
    if (do_gemm) {
        for (int i = tid; i < W * W; i += kThreads) {
            const int r = i / W, c = i % W;
            float v = 0.f;
            if (r < a.w && c < a.w) v = (a.gemm == GEMM_W) ? a.Wm[r * a.w + c] : a.Wm[c * a.w + r];
            Ws[i] = v;
        }
    }

    // GEMM / epilogue mapping
    const int tc = tid % C::TPRC, tr = tid / C::TPRC;
    const int c0 = tc * 4;
    // dW mapping
    const int dnb = tid % C::DNB, dmb = tid / C::DNB;
    const int dn0 = dnb * 4, dm0 = dmb * C::DMB;
    double dacc[C::kRegAcc ? C::DMB : 1][4];
#pragma unroll
    for (int i = 0; i < (C::kRegAcc ? C::DMB : 1); ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dacc[i][j] = 0.0;
    double dbacc = 0.0;
    const int plen = a.w * a.w + a.w;
    if (do_dw && !C::kRegAcc) {
        for (int i = tid; i < plen; i += kThreads) a.part[static_cast<size_t>(blockIdx.x) * plen + i] = 0.0;
    }

    const bool scatter_epi = a.epi == EPI_SCATTER_ADD || a.epi == EPI_SCATTER_SUB;
    const int kr = a.k_r, KHr = rec_kh(kr), RBr = rec_bytes(kr);

    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int row0 = tile * TR;
        // ---- phase 0: clear the tile
        for (int i = tid; i < TR * ZLD; i += kThreads) Zs[i] = 0.f;
        __syncthreads();
        // ---- phase A: aggregation
        if constexpr (AGG != AGG_NONE) aggregate_tile<W, AGG>(a, row0, Zs, U, meta);
        else {
            for (int i = tid; i < TR * (W / 4); i += kThreads) {
                const int r = i / (W / 4), c = (i % (W / 4)) * 4;
                if (row0 + r < a.n && c < a.ld) {
                    const float4 v = ld4(a.x_in + static_cast<size_t>(row0 + r) * a.ld + c);
                    *reinterpret_cast<float4*>(Zs + r * ZLD + c) = v;
                }
            }
        }
        __syncthreads();
        // ---- phase A2: scatter source for the Alg. 1/2 epilogues
        if (scatter_epi) {
            for (int i = tid; i < TR * ZLD; i += kThreads) Es[i] = 0.f;
            __syncthreads();
            for (int i = tid; i < TR * 16; i += kThreads) {
                const int r = i / 16, l = i % 16;
                const int row = row0 + r;
                if (row >= a.n) continue;
                const uint8_t* rc = a.rrec + static_cast<size_t>(row) * RBr;
                for (int j = l; j < kr; j += 16) Es[r * ZLD + rc[j]] = reinterpret_cast<const float*>(rc + KHr)[j];
            }
        }
        __syncthreads();
        // ---- phase B: transform + bias + epilogue
        {
            // residual rows issued before the transform so their latency hides under it
            const bool res_epi = a.epi == EPI_ADD || a.epi == EPI_SUB;
            float4 Rpre[C::RPT];
#pragma unroll
            for (int i = 0; i < C::RPT; ++i) {
                const int row = row0 + tr * C::RPT + i;
                Rpre[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (res_epi && row < a.n && c0 < a.ld) Rpre[i] = *reinterpret_cast<const float4*>(a.R + static_cast<size_t>(row) * a.ld + c0);
            }
            float acc[C::RPT][4];
            if (do_gemm) {
#pragma unroll
                for (int i = 0; i < C::RPT; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#pragma unroll 4
                for (int m = 0; m < W; ++m) {
                    const float4 wv = *reinterpret_cast<const float4*>(Ws + m * W + c0);
#pragma unroll
                    for (int i = 0; i < C::RPT; ++i) {
                        const float z = Zs[(tr * C::RPT + i) * ZLD + m];
                        acc[i][0] = fmaf(z, wv.x, acc[i][0]);
                        acc[i][1] = fmaf(z, wv.y, acc[i][1]);
                        acc[i][2] = fmaf(z, wv.z, acc[i][2]);
                        acc[i][3] = fmaf(z, wv.w, acc[i][3]);
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < C::RPT; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = Zs[(tr * C::RPT + i) * ZLD + c0 + j];
            }
            float bv[4] = {0.f, 0.f, 0.f, 0.f};
            if (a.bias) {
#pragma unroll
                for (int j = 0; j < 4; ++j) bv[j] = (c0 + j < a.w) ? __ldg(a.bias + c0 + j) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < C::RPT; ++i) {
                const int r = tr * C::RPT + i;
                const int row = row0 + r;
                const bool rv = row < a.n && c0 < a.ld;
                float h[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) h[j] = a.bias ? __fadd_rn(acc[i][j], bv[j]) : acc[i][j];
                const size_t off = static_cast<size_t>(row) * a.ld + c0;
                float o[4] = {h[0], h[1], h[2], h[3]};
                switch (a.epi) {
                    case EPI_ADD:
                    case EPI_SUB:
                        if (rv) {
                            const float4 R = Rpre[i];
                            const float Rv[4] = {R.x, R.y, R.z, R.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) o[j] = a.epi == EPI_ADD ? __fadd_rn(Rv[j], h[j]) : __fsub_rn(Rv[j], h[j]);
                        }
                        break;
                    case EPI_SCATTER_ADD:
#pragma unroll
                        for (int j = 0; j < 4; ++j) o[j] = __fadd_rn(Es[r * ZLD + c0 + j], h[j]);
                        break;
                    case EPI_SCATTER_SUB:
#pragma unroll
                        for (int j = 0; j < 4; ++j) o[j] = __fsub_rn(Es[r * ZLD + c0 + j], h[j]);
                        break;
                    case EPI_MASKED_ADD_RELU:
                        if (rv) {
                            const float4 M = *reinterpret_cast<const float4*>(a.mask_plane + off);
                            const float Mv[4] = {M.x, M.y, M.z, M.w};
                            for (int p = 0; p < a.ndst; ++p) {
                                float4* d = reinterpret_cast<float4*>(a.dst[p] + off);
                                float4 dv = *d;
                                if (Mv[0] > 0.f) dv.x = __fadd_rn(dv.x, h[0]);
                                if (Mv[1] > 0.f) dv.y = __fadd_rn(dv.y, h[1]);
                                if (Mv[2] > 0.f) dv.z = __fadd_rn(dv.z, h[2]);
                                if (Mv[3] > 0.f) dv.w = __fadd_rn(dv.w, h[3]);
                                *d = dv;
                            }
                        }
                        break;
                    default: break;
                }
                const bool write_out = a.epi <= EPI_SCATTER_SUB;
                if (write_out && rv) *reinterpret_cast<float4*>(a.out + off) = make_float4(o[0], o[1], o[2], o[3]);
                // tile copy for the row phases (GS / masked add / gather)
                *reinterpret_cast<float4*>(Es + r * ZLD + c0) = make_float4(o[0], o[1], o[2], o[3]);
                if (do_dw) {
                    float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (rv) gv = ld4(a.G + off);
                    *reinterpret_cast<float4*>(Gs + r * ZLD + c0) = gv;
                }
            }
        }
        __syncthreads();
        // ---- phase C: row epilogues on the tile
        if (a.epi == EPI_MASKED_ADD || a.epi == EPI_GATHER_REC) {
            for (int i = tid; i < TR * 16; i += kThreads) {
                const int r = i / 16, l = i % 16;
                const int row = row0 + r;
                if (row >= a.n) continue;
                const uint8_t* rc = a.rrec + static_cast<size_t>(row) * RBr;
                for (int j = l; j < kr; j += 16) {
                    const int col = rc[j];
                    const float v = Es[r * ZLD + col];
                    if (a.epi == EPI_MASKED_ADD) {
                        for (int p = 0; p < a.ndst; ++p) {
                            float* d = a.dst[p] + static_cast<size_t>(row) * a.ld + col;
                            *d = __fadd_rn(*d, v);
                        }
                    } else {
                        uint8_t* orc = a.out_rec + static_cast<size_t>(row) * RBr;
                        orc[j] = static_cast<uint8_t>(col);
                        reinterpret_cast<float*>(orc + KHr)[j] = v;
                    }
                }
            }
        }
        if constexpr (TPR > 0) {
            if (a.gs_out) {
                constexpr int P = W / TPR;
                constexpr int ROWS = kThreads / TPR;
                const int g = tid / TPR, q = tid % TPR;
                const int RBg = rec_bytes(a.k_gs);
                for (int base = 0; base < TR; base += ROWS) {
                    const int r = base + g;
                    const bool valid = r < TR && row0 + r < a.n;
                    float x[P];
#pragma unroll
                    for (int i = 0; i < P; ++i) x[i] = valid ? Es[r * ZLD + q * P + i] : 0.f;
                    gs_select<P, TPR>(x, q, a.w, a.k_gs, valid, a.gs_out + static_cast<size_t>(valid ? row0 + r : 0) * RBg);
                }
            }
        }
        // ---- phase D: dW / db partials
        if (do_dw) {
            if (dmb * C::DMB < W) {
                float t[C::DMB][4];
#pragma unroll
                for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) t[i][j] = 0.f;
                for (int r = 0; r < TR; ++r) {
                    const float4 g = *reinterpret_cast<const float4*>(Gs + r * ZLD + dn0);
#pragma unroll
                    for (int i = 0; i < C::DMB; ++i) {
                        const float z = Zs[r * ZLD + dm0 + i];
                        t[i][0] = fmaf(z, g.x, t[i][0]);
                        t[i][1] = fmaf(z, g.y, t[i][1]);
                        t[i][2] = fmaf(z, g.z, t[i][2]);
                        t[i][3] = fmaf(z, g.w, t[i][3]);
                    }
                }
                if constexpr (C::kRegAcc) {
#pragma unroll
                    for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) dacc[i][j] += static_cast<double>(t[i][j]);
                } else {
                    double* pp = a.part + static_cast<size_t>(blockIdx.x) * plen;
#pragma unroll
                    for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int m = dm0 + i, nn = dn0 + j;
                            if (m < a.w && nn < a.w) pp[m * a.w + nn] += static_cast<double>(t[i][j]);
                        }
                }
            }
            if (a.want_db && tid < a.w) {
                float s = 0.f;
                for (int r = 0; r < TR; ++r) s = __fadd_rn(s, Gs[r * ZLD + tid]);
                dbacc += static_cast<double>(s);
            }
        }
        __syncthreads();
    }
    if (do_dw) {
        double* pp = a.part + static_cast<size_t>(blockIdx.x) * plen;
        if constexpr (C::kRegAcc) {
#pragma unroll
            for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int m = dm0 + i, nn = dn0 + j;
                    if (m < a.w && nn < a.w) pp[m * a.w + nn] = dacc[i][j];
                }
        }
        if (tid < a.w) pp[a.w * a.w + tid] = a.want_db ? dbacc : 0.0;
    }
}

// Fixed-order reduction of per-CTA partials (double) into a float gradient.
__global__ void k_reduce_parts(const double* __restrict__ part, int nparts, int stride, int len, float* __restrict__ out, int accumulate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s = 0.0;
    for (int p = 0; p < nparts; ++p) s += part[static_cast<size_t>(p) * stride + i];
    if (accumulate) s += static_cast<double>(out[i]);
    out[i] = static_cast<float>(s);
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
// X[p][r][m] = fma-chain_a X0[r][a]·We[a][p·w+m] + be[p·w+m]
__global__ void k_encoder(const float* __restrict__ X0, int n, int d_in, const float* __restrict__ We, const float* __restrict__ be,
                          int D, int w, int ld, float* __restrict__ X) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(n) * D) return;
    const int r = static_cast<int>(i / D), col = static_cast<int>(i % D);
    const int p = col / w, m = col % w;
    float acc = 0.f;
    for (int t = 0; t < d_in; ++t) acc = fmaf(__ldg(X0 + static_cast<size_t>(r) * d_in + t), __ldg(We + static_cast<size_t>(t) * D + col), acc);
    X[(static_cast<size_t>(p) * n + r) * ld + m] = __fadd_rn(acc, __ldg(be + col));
}

// ŷ[r] = fma-chain_n X[r][n]·wh[n] + bh; masked MSE gradient and loss partials.
__global__ void k_head_loss(const float* __restrict__ X, int n, int D, int w, int ld, const float* __restrict__ wh,
                            const float* __restrict__ bh, const float* __restrict__ y, const uint8_t* __restrict__ mask, float cnt,
                            float* __restrict__ yhat, float* __restrict__ gy, double* __restrict__ loss_part) {
    __shared__ double red[kThreads / 32];
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    double l = 0.0;
    if (r < n) {
        float acc = 0.f;
        for (int col = 0; col < D; ++col) {
            const int p = col / w, m = col % w;
            acc = fmaf(X[(static_cast<size_t>(p) * n + r) * ld + m], __ldg(wh + col), acc);
        }
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
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = l;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kThreads / 32; ++i) s += red[i];
        loss_part[blockIdx.x] = s;
    }
}

// G[p][r][m] = gy[r]·wh[p·w+m]; per-CTA partials of dwh = Σ_r X·gy and dbh = Σ_r gy.
// part layout: [cta][D + 1]. Each CTA owns a contiguous row range.
__global__ void k_head_bwd(const float* __restrict__ X, const float* __restrict__ gy, int n, int D, int w, int ld,
                           const float* __restrict__ wh, float* __restrict__ G, double* __restrict__ part, int rows_per_cta) {
    const int r0 = blockIdx.x * rows_per_cta;
    const int r1 = min(n, r0 + rows_per_cta);
    double* pp = part + static_cast<size_t>(blockIdx.x) * (D + 1);
    for (int col = threadIdx.x; col < D; col += blockDim.x) {
        const int p = col / w, m = col % w;
        const float whc = __ldg(wh + col);
        double s = 0.0;
        for (int r = r0; r < r1; ++r) {
            const size_t off = (static_cast<size_t>(p) * n + r) * ld + m;
            const float g = __ldg(gy + r);
            s += static_cast<double>(X[off]) * static_cast<double>(g);
            G[off] = __fmul_rn(g, whc);
        }
        pp[col] = s;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int r = r0; r < r1; ++r) s += static_cast<double>(gy[r]);
        pp[D] = s;
    }
}

// dWe[t][col] = Σ_r X0[r][t]·G[r][col]; dbe[col] = Σ_r G[r][col]. part: [cta][d_in·D + D].
__global__ void k_encoder_bwd(const float* __restrict__ X0, const float* __restrict__ G, int n, int d_in, int D, int w, int ld,
                              double* __restrict__ part, int rows_per_cta) {
    const int r0 = blockIdx.x * rows_per_cta;
    const int r1 = min(n, r0 + rows_per_cta);
    const int len = d_in * D + D;
    double* pp = part + static_cast<size_t>(blockIdx.x) * len;
    for (int col = threadIdx.x; col < D; col += blockDim.x) {
        const int p = col / w, m = col % w;
        double acc[16];
        for (int t = 0; t < 16; ++t) acc[t] = 0.0;
        double sb = 0.0;
        for (int r = r0; r < r1; ++r) {
            const double g = G[(static_cast<size_t>(p) * n + r) * ld + m];
            sb += g;
            for (int t = 0; t < d_in && t < 16; ++t) acc[t] += static_cast<double>(__ldg(X0 + static_cast<size_t>(r) * d_in + t)) * g;
        }
        for (int t = 0; t < d_in && t < 16; ++t) pp[t * D + col] = acc[t];
        pp[d_in * D + col] = sb;
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

template <int W, int AGG, int TPR>
cudaError_t set_attr_t() {
    const size_t smem = Smem<W>::bytes;
    return cudaFuncSetAttribute(k_tile<W, AGG, TPR>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}

template <int W>
cudaError_t set_attr_w() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {set_attr_t<W, AGG_SPARSE, 0>(), set_attr_t<W, AGG_SPARSE, 1>(), set_attr_t<W, AGG_SPARSE, 2>(),
                          set_attr_t<W, AGG_SPARSE, 4>(), set_attr_t<W, AGG_DENSE, 0>(), set_attr_t<W, AGG_DENSE_RELU, 0>(),
                          set_attr_t<W, AGG_NONE, 0>()})
        if (r != cudaSuccess) e = r;
    return e;
}

int sm_count();

template <int W, int AGG, int TPR>
int occupancy_t() {
    static int occ = 0;
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile<W, AGG, TPR>, kThreads, Smem<W>::bytes) != cudaSuccess) {
            cudaGetLastError();
            occ = 1;
        }
        if (occ < 1) occ = 1;
    }
    return occ;
}

// Persistent grid = SMs × resident CTAs of this instantiation (one wave).
template <int W, int AGG, int TPR>
cudaError_t launch_tile_t(const TileArgs& a, cudaStream_t s, int* grid_out) {
    const int tiles = (a.n + TR - 1) / TR;
    const int cap = sm_count() * occupancy_t<W, AGG, TPR>();
    const int grid = tiles < cap ? tiles : cap;
    if (grid_out) *grid_out = grid;
    k_tile<W, AGG, TPR><<<grid, kThreads, Smem<W>::bytes, s>>>(a);
    return cudaGetLastError();
}

template <int W>
cudaError_t launch_tile_w(const TileArgs& a, cudaStream_t s, int* g) {
    const int k = a.k_gs;
    const int tpr = (a.gs_out == nullptr) ? 0 : (k <= W / 4 ? 4 : (k <= W / 2 ? 2 : 1));
    switch (a.agg) {
        case AGG_SPARSE:
            if (tpr == 0) return launch_tile_t<W, AGG_SPARSE, 0>(a, s, g);
            if (tpr == 4) return launch_tile_t<W, AGG_SPARSE, 4>(a, s, g);
            if (tpr == 2) return launch_tile_t<W, AGG_SPARSE, 2>(a, s, g);
            return launch_tile_t<W, AGG_SPARSE, 1>(a, s, g);
        case AGG_DENSE: return launch_tile_t<W, AGG_DENSE, 0>(a, s, g);
        case AGG_DENSE_RELU: return launch_tile_t<W, AGG_DENSE_RELU, 0>(a, s, g);
        default: return launch_tile_t<W, AGG_NONE, 0>(a, s, g);
    }
}

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

inline int blocks_for(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

cudaError_t init_kernel_attributes() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {set_attr_w<32>(), set_attr_w<64>(), set_attr_w<128>()})
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
    if (a.w <= 32) return launch_tile_w<32>(a, s, grid_out);
    if (a.w <= 64) return launch_tile_w<64>(a, s, grid_out);
    if (a.w <= 128) return launch_tile_w<128>(a, s, grid_out);
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
    k_reduce_parts<<<blocks_for(len, 256), 256, 0, s>>>(part, nparts, stride, len, out, accumulate);
    return cudaGetLastError();
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
                           cudaStream_t s) {
    (void)C;
    const long long tot = static_cast<long long>(n) * D;
    if (!tot) return cudaSuccess;
    k_encoder<<<blocks_for(tot, 256), 256, 0, s>>>(X0, n, d_in, We, be, D, w, ld, X);
    return cudaGetLastError();
}

cudaError_t launch_head_loss(const float* X, int n, int D, int C, int w, int ld, const float* wh, const float* bh, const float* y,
                             const uint8_t* mask, float, float cnt, float* yhat, float* gy, double* loss_part, int nparts, cudaStream_t s) {
    (void)C;
    (void)nparts;
    k_head_loss<<<blocks_for(n, kThreads), kThreads, 0, s>>>(X, n, D, w, ld, wh, bh, y, mask, cnt, yhat, gy, loss_part);
    return cudaGetLastError();
}

cudaError_t launch_head_bwd(const float* X, const float* gy, int n, int D, int C, int w, int ld, const float* wh, float* G, double* part,
                            int nparts, cudaStream_t s) {
    (void)C;
    const int rows = (n + nparts - 1) / nparts;
    k_head_bwd<<<nparts, 256, 0, s>>>(X, gy, n, D, w, ld, wh, G, part, rows);
    return cudaGetLastError();
}

cudaError_t launch_encoder_bwd(const float* X0, const float* G, int n, int d_in, int D, int C, int w, int ld, double* part, int nparts,
                               cudaStream_t s) {
    (void)C;
    if (d_in > 16) return cudaErrorInvalidValue;
    const int rows = (n + nparts - 1) / nparts;
    k_encoder_bwd<<<nparts, 256, 0, s>>>(X0, G, n, d_in, D, w, ld, part, rows);
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

}  // namespace gsrk
