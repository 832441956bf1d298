// k_tile — the fused GSR block kernel (included by tile_w{32,64,128}.cu).
//
// One persistent CTA (256 threads, 8 warps) walks 128-row tiles of the node
// range. Per tile:
//   A  aggregation (spmm_sparse SPEC.md:177-185 over compressed CBSR records,
//      or spmm SPEC.md:168-176 over dense rows, optionally ReLU'd) into a
//      128 × W fp32 tile in shared memory, in the oracle's canonical
//      segmented edge order (bit-identical, see aggregate_tile);
//   B  dense transform h = Z·W (or Z·Wᵀ) + b:
//        TC = 1: tcgen05.mma kind::tf32 (M=128, N=W, K=8 per instruction)
//                from the smem tile (UMMA K-major SWIZZLE_128B layout) into a
//                TMEM accumulator, issued by one thread, completion signalled
//                through tcgen05.commit → mbarrier, read back with tcgen05.ld;
//        TC = 0: FP32-strict FFMA chain over the contraction index (bit-exact
//                with the oracle's std::fma chain);
//   C  epilogue on the accumulator rows: bias, residual add/sub (Eq. 6-7),
//      scatter residual (Alg. 1 line 10 / Alg. 2 line 7), masked input-gradient
//      scatter-add, index gather (Alg. 2 backward block);
//   D  GS top-k of the output tile → next block's compressed records, and
//      dW/db partial sums (deterministic per-CTA slots, double accumulators).
// Thread ↔ row mapping in B/C: warp w owns TMEM lane quadrant (w & 3) — rows
// 32·(w&3) .. +31 — and column half (w >> 2): one thread = one row × W/2 cols.
#pragma once

#include "common.cuh"

namespace gsrk {
namespace tile {

using dev::kFull;
using dev::ld4;

constexpr int TR = 128;
constexpr int kSeg = 8;     // == oracle kAggSeg
constexpr int kRMax = 64;   // aggregation items per round
constexpr int kPF = 4;      // neighbour prefetch depth per lane group (one batch covers a typical row)

// 128 × W fp32 tiles use the UMMA K-major SWIZZLE_128B canonical layout:
// W/32 regions of 128 rows × 128 B; the 16-B chunk j of row r lives at chunk
// j ^ (r & 7). The same bytes are a K-major A operand (K = column) for h = Z·W
// and conflict-free for row-wise smem RMW (a row's 32 columns hit 32 banks).
__device__ __forceinline__ int zoff(int r, int m) {
    return (m >> 5) * (TR * 32) + r * 32 + ((((m >> 2) & 7) ^ (r & 7)) << 2) + (m & 3);
}
// Bᵀ operand (N = W rows, K = W) in the same layout, region stride W rows.
template <int W>
__device__ __forceinline__ int boff(int nrow, int m) {
    return (m >> 5) * (W * 32) + nrow * 32 + ((((m >> 2) & 7) ^ (nrow & 7)) << 2) + (m & 3);
}

// Shared-memory plan (floats, regions 1 KB aligned):
//   Ws  W×W        transform operand (Bᵀ SW128 for TC, row-major [m][n] for FP32)
//   Zs  TR×(W+1)   TC: the UMMA A tile (SW128, TR×W); FP32: epilogue/gradient
//                  tile. During aggregation it hosts the segment slots P and
//                  the staged neighbour ids.
//   Za  TR×(W+1)   row-major accumulation tile (ZLD = W+1: a row's columns and a
//                  column's rows both spread over the 32 banks); TC: epilogue /
//                  gradient tile after the conversion into Zs.
template <int W>
struct Smem {
    static constexpr int ZLD = W + 1;
    static constexpr size_t r1k(size_t f) { return (f + 255) & ~size_t(255); }
    static constexpr size_t ws = r1k(static_cast<size_t>(W) * W);
    static constexpr size_t zt = static_cast<size_t>(TR) * ZLD;
    static constexpr size_t agg = static_cast<size_t>(kThreads / 2) * W;  // hub segment slots
    static constexpr size_t zs = r1k(zt > agg ? zt : agg);
    static constexpr size_t za = r1k(zt);
    static constexpr size_t meta_ints = 2 * (TR + 1) + TR + kThreads / 2 + 8;
    static constexpr size_t bytes = (ws + zs + za + meta_ints) * sizeof(float) + 1024;  // +1 KB alignment slack
};

__device__ __forceinline__ int nseg_of(int deg) { return (deg + kSeg - 1) / kSeg; }

// ---- tcgen05 / mbarrier primitives (PTX ISA 8.6, sm_100a) ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "GSRK_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra GSRK_DONE;\n\t"
        "bra GSRK_WAIT;\n"
        "GSRK_DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)  // suspend-time hint (ns): the waiting warp sleeps instead of re-issuing the poll
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {  // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // same warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: LBO unused (1),
// SBO = 1024 B between 8-row groups, version 1, layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// D[tmem] (+)= A[smem] · B[smem], kind::tf32, cta_group::1.
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Instruction descriptor: D = F32 (bits 4-5 = 1), A = B = TF32 (2), both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24 (cute UMMA::InstrDescriptor).
template <int N>
__host__ __device__ constexpr uint32_t idesc_tf32_m128() {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(TR >> 4) << 24);
}

// tcgen05.ld 32 lanes × 32 bit × H columns (this warp's lane quadrant).
template <int H>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[H]);

#define GSRK_LD_REGS8(o) "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]), "=r"(r[o + 6]), "=r"(r[o + 7])

template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : GSRK_LD_REGS8(0) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : GSRK_LD_REGS8(0), GSRK_LD_REGS8(8)
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : GSRK_LD_REGS8(0), GSRK_LD_REGS8(8), GSRK_LD_REGS8(16), GSRK_LD_REGS8(24)
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
__device__ __forceinline__ void tmem_ld<64>(uint32_t taddr, float (&v)[64]) {
    float* h0 = v;
    float* h1 = v + 32;
    float (&a)[32] = *reinterpret_cast<float(*)[32]>(h0);
    float (&b)[32] = *reinterpret_cast<float(*)[32]>(h1);
    tmem_ld<32>(taddr, a);
    tmem_ld<32>(taddr + 32, b);
}
#undef GSRK_LD_REGS8

// ---------------------------------------------------------------------------
// Aggregation in the canonical segmented order of the oracle: a row's edge
// list is cut into kSeg-edge segments, each summed in CSR order from +0, and
// the row total folds the segment sums left to right (rows of ≤ kSeg edges =
// one plain sequential sum). Per column this is exactly the oracle's order.
//
// Work split: every "regular" row (≤ kSeg edges — all but ~0.2% of circuit
// nodes) is owned by one thread that walks its edges with 128-bit record loads
// (software-pipelined one edge ahead) and accumulates in its row of the
// row-major tile (sparse: scatter-add of the k selected values; dense: W/2
// columns in registers, two threads per row). Hub rows (> kSeg edges, up to
// 20 000 in the power-law config) are split into their kSeg-edge segments,
// each owned by one thread (pair) writing a private slot; slots are folded
// into the tile in segment order. For the sparse path the hub segments run on
// warps 4-7 concurrently with the regular rows on warps 0-3.
// The row scale (Â's row factor) is applied by the tile's consumers.
// ---------------------------------------------------------------------------
template <int W>
struct AggMeta {
    static constexpr int NP = kThreads / 2;           // hub segment slots per round
    int* rp;     // TR + 1 row pointers
    int* hoff;   // TR + 1 hub-segment offsets
    float* rfs;  // TR row scales
    int* hrow;   // NP slot rows
    __device__ AggMeta(int* meta) : rp(meta), hoff(meta + TR + 1), rfs(reinterpret_cast<float*>(meta + 2 * (TR + 1))),
                                    hrow(meta + 2 * (TR + 1) + TR) {}
};

// An fp32 value as the UMMA kind::tf32 path reads it: low 13 mantissa bits
// truncated (tests/test_gpu_config_parity.py test_fast_path_tf32_operand_truncation; oracle tf32_op).
// Used where the CUDA cores must reproduce a tensor-core operand.
__device__ __forceinline__ float tf32_op(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__device__ __forceinline__ uint4 ld4u(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

struct SparseRec {  // one CBSR record with k ≤ 16: 16 index bytes + up to 16 values
    uint4 idx;
    float4 v[4];
};

__device__ __forceinline__ void load_rec16(SparseRec& r, const uint8_t* rc, int nv4) {
    r.idx = ld4u(rc);
#pragma unroll
    for (int q = 0; q < 4; ++q) r.v[q] = q < nv4 ? ld4(reinterpret_cast<const float*>(rc + 16) + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
}

// dst[m] += sc·v for the record's k (index, value) pairs, in slot order.
__device__ __forceinline__ void scatter_rec16(float* dst, const SparseRec& r, int k, bool unit, float sc) {
    const uint32_t iw[4] = {r.idx.x, r.idx.y, r.idx.z, r.idx.w};
    const float vv[16] = {r.v[0].x, r.v[0].y, r.v[0].z, r.v[0].w, r.v[1].x, r.v[1].y, r.v[1].z, r.v[1].w,
                          r.v[2].x, r.v[2].y, r.v[2].z, r.v[2].w, r.v[3].x, r.v[3].y, r.v[3].z, r.v[3].w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (j < k) {
            const int m = static_cast<int>((iw[j >> 2] >> (8 * (j & 3))) & 0xffu);
            dst[m] = __fadd_rn(dst[m], unit ? vv[j] : __fmul_rn(sc, vv[j]));
        }
    }
}

// Sequential scatter-accumulation of edges [e_lo, e_hi) (≤ kSeg) into dst
// (sparse). All neighbour ids are loaded up front, records one edge ahead.
__device__ __forceinline__ void accumulate_sparse(const TileArgs& a, int e_lo, int e_hi, float* dst, bool unit) {
    const int k = a.k_in;
    const int ne = e_hi - e_lo;
    if (ne <= 0) return;
    if (k <= 16) {
        const int RB = rec_bytes(k), nv4 = (k + 3) >> 2;
        int cs[kSeg];
#pragma unroll
        for (int u = 0; u < kSeg; ++u) cs[u] = u < ne ? __ldg(a.dir.idx + e_lo + u) : 0;
        SparseRec buf[2];
        load_rec16(buf[0], a.rec_in + static_cast<size_t>(cs[0]) * RB, nv4);
#pragma unroll
        for (int u = 0; u < kSeg; ++u) {
            if (u < ne) {
                if (u + 1 < ne) load_rec16(buf[(u + 1) & 1], a.rec_in + static_cast<size_t>(cs[u + 1 < kSeg ? u + 1 : 0]) * RB, nv4);
                const float sc = unit ? 1.f : __ldg(a.dir.edge_f + cs[u]);
                scatter_rec16(dst, buf[u & 1], k, unit, sc);
            }
        }
    } else {
        const int KH = rec_kh(k), RB = rec_bytes(k);
        for (int e = e_lo; e < e_hi; ++e) {
            const int c = __ldg(a.dir.idx + e);
            const float sc = unit ? 1.f : __ldg(a.dir.edge_f + c);
            const uint8_t* rc = a.rec_in + static_cast<size_t>(c) * RB;
            for (int j = 0; j < k; ++j) {
                const int m = __ldg(rc + j);
                const float v = __ldg(reinterpret_cast<const float*>(rc + KH) + j);
                dst[m] = __fadd_rn(dst[m], unit ? v : __fmul_rn(sc, v));
            }
        }
    }
}

// Sequential accumulation of dense neighbour rows, columns [col0, col0 + HC).
template <int HC, bool RELU>
__device__ __forceinline__ void accumulate_dense(const TileArgs& a, int e_lo, int e_hi, int col0, float (&acc)[HC], bool unit) {
#pragma unroll
    for (int q = 0; q < HC; ++q) acc[q] = 0.f;
    const int ne = e_hi - e_lo;
    int cs[kSeg];
#pragma unroll
    for (int u = 0; u < kSeg; ++u) cs[u] = u < ne ? __ldg(a.dir.idx + e_lo + u) : 0;
#pragma unroll
    for (int u = 0; u < kSeg; ++u) {
        if (u < ne) {
            const int c = cs[u];
            const float sc = unit ? 1.f : __ldg(a.dir.edge_f + c);
            const float* src = a.x_in + static_cast<size_t>(c) * a.ld + col0;
            float v[HC];
#pragma unroll
            for (int q = 0; q < HC; q += 4) {
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                if (col0 + q < a.ld) f = ld4(src + q);
                v[q] = f.x; v[q + 1] = f.y; v[q + 2] = f.z; v[q + 3] = f.w;
            }
#pragma unroll
            for (int q = 0; q < HC; ++q) {
                float xv = v[q];
                if (RELU) xv = xv > 0.f ? xv : 0.f;
                acc[q] = __fadd_rn(acc[q], unit ? xv : __fmul_rn(sc, xv));
            }
        }
    }
}

template <int W, int AGG>
__device__ __forceinline__ void aggregate_tile(const TileArgs& a, int row0, float* Za, float* P, int* meta) {
    constexpr bool SPARSE = AGG == AGG_SPARSE;
    constexpr bool RELU = AGG == AGG_DENSE_RELU;
    constexpr int ZLD = Smem<W>::ZLD;
    constexpr int NP = AggMeta<W>::NP;
    constexpr int HC = W / 2;
    AggMeta<W> M(meta);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rows = min(TR, a.n - row0);

    for (int i = tid; i <= TR; i += kThreads) {
        if (i <= rows) M.rp[i] = __ldg(a.dir.ptr + row0 + i);
        if (i < TR) M.rfs[i] = i < rows ? __ldg(a.dir.out_f + row0 + i) : 0.f;
    }
    __syncthreads();
    if (wid == 0) {  // hub-segment prefix, 4 rows per lane
        int c[4];
        int sum = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = 4 * lane + j;
            const int deg = r < rows ? M.rp[r + 1] - M.rp[r] : 0;
            c[j] = deg > kSeg ? nseg_of(deg) : 0;
            sum += c[j];
        }
        int incl = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += v;
        }
        int run = incl - sum;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            M.hoff[4 * lane + j] = run;
            run += c[j];
        }
        if (lane == 31) M.hoff[TR] = incl;
    }
    __syncthreads();
    const int nhub = M.hoff[TR];
    const bool unit = a.dir.unit_edge != 0;

    // regular rows
    if constexpr (SPARSE) {
        if (tid < rows) {
            const int e0 = M.rp[tid], e1 = M.rp[tid + 1];
            if (e1 - e0 <= kSeg) accumulate_sparse(a, e0, e1, Za + tid * ZLD, unit);
        }
    } else {
        const int r = tid % TR, half = tid / TR;
        if (r < rows) {
            const int e0 = M.rp[r], e1 = M.rp[r + 1];
            if (e1 - e0 <= kSeg) {
                float acc[HC];
                accumulate_dense<HC, RELU>(a, e0, e1, half * HC, acc, unit);
                float* z = Za + r * ZLD + half * HC;
#pragma unroll
                for (int q = 0; q < HC; ++q) z[q] = acc[q];
            }
        }
        if (nhub) __syncthreads();
    }
    // hub segments, rounds of NP slots (sparse: warps 4-7, concurrent with the regular rows)
    for (int h0 = 0; h0 < nhub; h0 += NP) {
        const int slot = tid % NP;
        const int h = h0 + slot;
        const bool mine = SPARSE ? (tid >= NP && h < nhub) : (h < nhub);
        if (mine) {
            int lo = 0, hi = rows - 1;  // last row with hoff[row] <= h
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (M.hoff[mid] <= h) lo = mid; else hi = mid - 1;
            }
            const int r = lo;
            const int e_lo = M.rp[r] + (h - M.hoff[r]) * kSeg;
            const int e_hi = min(M.rp[r + 1], e_lo + kSeg);
            if (SPARSE || tid < NP) M.hrow[slot] = r;
            if constexpr (SPARSE) {
                float* pr = P + slot * W;
                for (int c = 0; c < W; ++c) pr[c] = 0.f;
                accumulate_sparse(a, e_lo, e_hi, pr, unit);
            } else {
                const int half = tid / NP;
                float acc[HC];
                accumulate_dense<HC, RELU>(a, e_lo, e_hi, half * HC, acc, unit);
                float* pr = P + slot * W + half * HC;
#pragma unroll
                for (int q = 0; q < HC; ++q) pr[q] = acc[q];
            }
        }
        __syncthreads();
        {   // fold this round's segment slots into their rows, in segment order
            constexpr int NG = kThreads / W;
            const int g = tid / W, c = tid % W;
            const int nr = min(NP, nhub - h0);
            for (int i = 0; i < nr; ++i) {
                const int r = M.hrow[i];
                if (r % NG != g) continue;
                const float pv = P[i * W + c];
                float* z = Za + r * ZLD + c;
                *z = (h0 + i == M.hoff[r]) ? pv : __fadd_rn(*z, pv);
            }
        }
        __syncthreads();
    }
}

template <int W>
struct KCfg {
    static constexpr int H = W / 2;                    // epilogue columns per thread
    static constexpr int DWE = W * W / kThreads;       // dW entries per thread
    static constexpr int DMB = DWE >= 4 ? DWE / 4 : 1; // dW m-rows per thread (×4 n-cols)
    static constexpr int DNB = W / 4;                  // dW n-blocks
    static constexpr bool kRegAcc = (W <= 64);
    static constexpr int kMinBlocks = W >= 128 ? 1 : 2;
};

template <int W, int AGG, int TPR, int TC>
__global__ void __launch_bounds__(kThreads, KCfg<W>::kMinBlocks) k_tile(TileArgs a) {
    using C = KCfg<W>;
    using S = Smem<W>;
    constexpr int H = C::H;
    constexpr int ZLD = S::ZLD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* Ws = base;                    // transform: Bᵀ SW128 (TC) or row-major [m][n] (FP32)
    float* Zs = Ws + S::ws;              // TC: UMMA A tile | FP32: epilogue/gradient tile | aggregation slots
    float* Za = Zs + S::zs;              // row-major accumulation tile (ZLD)
    float* U = Zs;                       // hub-segment slots (phase A only)
    float* Et = TC ? Za : Zs;            // epilogue (Es) / gradient (Gs) tile, row-major ZLD
    int* meta = reinterpret_cast<int*>(Za + S::za);
    uint64_t* bar = reinterpret_cast<uint64_t*>(meta + 2 * (TR + 1) + TR + kThreads / 2 + 2);
    const float* rfs = AggMeta<W>(meta).rfs;  // Â row scales of the tile (aggregating variants)
    constexpr bool kScale = AGG != AGG_NONE;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int n_tiles = (a.n + TR - 1) / TR;
    const bool do_dw = a.G != nullptr;
    const bool do_gemm = a.gemm != GEMM_NONE;
    const bool scatter_epi = a.epi == EPI_SCATTER_ADD || a.epi == EPI_SCATTER_SUB;
    const bool res_epi = a.epi == EPI_ADD || a.epi == EPI_SUB;
    const int kr = a.k_r, KHr = rec_kh(kr), RBr = rec_bytes(kr);

    // transform operand, once per CTA (zero padded to W×W)
    if (do_gemm) {
        for (int i = tid; i < W * W; i += kThreads) {
            const int r = i / W, c = i % W;  // W[r][c], r = contraction index
            float v = 0.f;
            if (r < a.w && c < a.w) v = (a.gemm == GEMM_W) ? a.Wm[r * a.w + c] : a.Wm[c * a.w + r];
            if constexpr (TC) Ws[boff<W>(c, r)] = v;  // Bᵀ[n = c][k = r]
            else Ws[i] = v;
        }
    }
    uint32_t tmem = 0;
    if constexpr (TC) {
        if (tid == 0) mbar_init(bar, 1);
        if (wid == 0) tmem_alloc(tslot, W < 32 ? 32 : W);
        fence_proxy_async();
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        tmem = *tslot;
    }
    uint32_t phase = 0;

    // epilogue mapping: warp → (lane quadrant, column half); thread → row
    const int q4 = wid & 3, hv = wid >> 2;
    const int er = 32 * q4 + lane;       // tile row
    const int ec0 = hv * H;              // first column

    // dW mapping
    const int dnb = tid % C::DNB, dmb = tid / C::DNB;
    const int dn0 = dnb * 4, dm0 = dmb * C::DMB;
    const bool dw_active = dm0 < W;
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

    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int row0 = tile * TR;
        const int row = row0 + er;
        const bool rvalid = row < a.n;
        // ---- phase 0: clear the accumulation tile
        for (int i = tid; i < TR * ZLD; i += kThreads) Za[i] = 0.f;
        __syncthreads();
        // ---- phase A: aggregation (or a plain row tile)
        if constexpr (AGG != AGG_NONE) {
            aggregate_tile<W, AGG>(a, row0, Za, U, meta);
        } else {
            for (int i = tid; i < TR * (W / 4); i += kThreads) {
                const int r = i / (W / 4), c = (i % (W / 4)) * 4;
                if (row0 + r < a.n && c < a.ld) {
                    const float4 v = ld4(a.x_in + static_cast<size_t>(row0 + r) * a.ld + c);
                    Za[r * ZLD + c] = v.x; Za[r * ZLD + c + 1] = v.y; Za[r * ZLD + c + 2] = v.z; Za[r * ZLD + c + 3] = v.w;
                }
            }
        }
        __syncthreads();
        // ---- phase B: transform
        if constexpr (TC) {
            if (do_gemm || do_dw) {
                // row-major tile → UMMA K-major SW128 A operand
                for (int i = tid; i < TR * (W / 4); i += kThreads) {
                    const int r = i / (W / 4), c = (i % (W / 4)) * 4;
                    const float* z = Za + r * ZLD + c;
                    float4 v = make_float4(z[0], z[1], z[2], z[3]);
                    if (kScale) {
                        const float f = rfs[r];
                        v.x = __fmul_rn(f, v.x); v.y = __fmul_rn(f, v.y); v.z = __fmul_rn(f, v.z); v.w = __fmul_rn(f, v.w);
                    }
                    *reinterpret_cast<float4*>(Zs + zoff(r, c)) = v;
                }
                fence_proxy_async();
                __syncthreads();
            }
            if (do_gemm && tid == 0) {
                tc_fence_after();
                constexpr uint32_t idesc = idesc_tf32_m128<W>();
                const uint32_t za = smem_u32(Zs), wa = smem_u32(Ws);
#pragma unroll
                for (int kk = 0; kk < W / 8; ++kk) {
                    const uint64_t ad = umma_desc_sw128(za + (kk >> 2) * (TR * 128) + (kk & 3) * 32);
                    const uint64_t bd = umma_desc_sw128(wa + (kk >> 2) * (W * 128) + (kk & 3) * 32);
                    umma_tf32(tmem, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
                umma_commit(bar);
            }
        }
        // residual rows prefetched while the transform runs
        float Rv[H];
        if (res_epi && rvalid) {
#pragma unroll
            for (int j = 0; j < H; j += 4) {
                float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
                if (ec0 + j < a.ld) t = *reinterpret_cast<const float4*>(a.R + static_cast<size_t>(row) * a.ld + ec0 + j);
                Rv[j] = t.x; Rv[j + 1] = t.y; Rv[j + 2] = t.z; Rv[j + 3] = t.w;
            }
        }
        float acc[H];
        if (do_gemm) {
            if constexpr (TC) {
                mbar_wait(bar, phase);
                phase ^= 1u;
                tc_fence_after();
                tmem_ld<H>(tmem + (static_cast<uint32_t>(32 * q4) << 16) + static_cast<uint32_t>(ec0), acc);
            } else {
#pragma unroll
                for (int j = 0; j < H; ++j) acc[j] = 0.f;
                const float* zr = Za + er * ZLD;
                const float rf = kScale ? rfs[er] : 1.f;
#pragma unroll 2
                for (int m = 0; m < W; ++m) {
                    const float z = kScale ? __fmul_rn(rf, zr[m]) : zr[m];
#pragma unroll
                    for (int j = 0; j < H; j += 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(Ws + m * W + ec0 + j);
                        acc[j] = fmaf(z, w4.x, acc[j]);
                        acc[j + 1] = fmaf(z, w4.y, acc[j + 1]);
                        acc[j + 2] = fmaf(z, w4.z, acc[j + 2]);
                        acc[j + 3] = fmaf(z, w4.w, acc[j + 3]);
                    }
                }
            }
        } else {
            const float* zr = Za + er * ZLD + ec0;
            const float rf = kScale ? rfs[er] : 1.f;
#pragma unroll
            for (int j = 0; j < H; ++j) acc[j] = kScale ? __fmul_rn(rf, zr[j]) : zr[j];
        }
        // Et may alias Za (TC) — every thread has its accumulator rows in registers
        __syncthreads();
        // scatter residual source (Alg. 1 line 10, Alg. 2 line 7)
        if (scatter_epi) {
            for (int i = tid; i < TR * ZLD; i += kThreads) Et[i] = 0.f;
            __syncthreads();
            for (int i = tid; i < TR * 16; i += kThreads) {
                const int r = i / 16, l = i % 16;
                if (row0 + r >= a.n) continue;
                const uint8_t* rc = a.rrec + static_cast<size_t>(row0 + r) * RBr;
                for (int j = l; j < kr; j += 16) Et[r * ZLD + rc[j]] = reinterpret_cast<const float*>(rc + KHr)[j];
            }
            __syncthreads();
        }
        // ---- phase C: epilogue on this thread's row segment
        {
            const size_t goff = static_cast<size_t>(row) * a.ld + ec0;
            const bool write_out = a.epi <= EPI_SCATTER_SUB;
            const bool keep_tile = a.gs_out != nullptr || a.epi == EPI_MASKED_ADD || a.epi == EPI_GATHER_REC;
            float* et = Et + er * ZLD + ec0;
#pragma unroll
            for (int j = 0; j < H; j += 4) {
                float o[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int c = ec0 + j + t;
                    float h = acc[j + t];
                    if (a.bias) h = __fadd_rn(h, c < a.w ? __ldg(a.bias + c) : 0.f);
                    float v = h;
                    if (a.epi == EPI_ADD) v = __fadd_rn(Rv[j + t], dev::quant(h, a.qs, a.qi));
                    else if (a.epi == EPI_SUB) v = __fsub_rn(Rv[j + t], dev::quant(h, a.qs, a.qi));
                    else if (a.epi == EPI_SCATTER_ADD) v = __fadd_rn(et[j + t], h);
                    else if (a.epi == EPI_SCATTER_SUB) v = __fsub_rn(et[j + t], h);
                    o[t] = v;
                }
                const bool cok = ec0 + j < a.ld;
                if (write_out && rvalid && cok) *reinterpret_cast<float4*>(a.out + goff + j) = make_float4(o[0], o[1], o[2], o[3]);
                if (a.epi == EPI_MASKED_ADD_RELU && rvalid && cok) {
                    const float4 M = *reinterpret_cast<const float4*>(a.mask_plane + goff + j);
                    for (int p = 0; p < a.ndst; ++p) {
                        float4* d = reinterpret_cast<float4*>(a.dst[p] + goff + j);
                        float4 dv = *d;
                        if (M.x > 0.f) dv.x = __fadd_rn(dv.x, o[0]);
                        if (M.y > 0.f) dv.y = __fadd_rn(dv.y, o[1]);
                        if (M.z > 0.f) dv.z = __fadd_rn(dv.z, o[2]);
                        if (M.w > 0.f) dv.w = __fadd_rn(dv.w, o[3]);
                        *d = dv;
                    }
                }
                if (keep_tile) { et[j] = o[0]; et[j + 1] = o[1]; et[j + 2] = o[2]; et[j + 3] = o[3]; }
                if (do_dw) {
                    float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (rvalid && cok) gv = ld4(a.G + goff + j);
                    et[j] = gv.x; et[j + 1] = gv.y; et[j + 2] = gv.z; et[j + 3] = gv.w;
                }
            }
        }
        if constexpr (TC) tc_fence_before();
        __syncthreads();
        // ---- phase D: row epilogues on the tile
        if (a.epi == EPI_MASKED_ADD || a.epi == EPI_GATHER_REC) {
            for (int i = tid; i < TR * 16; i += kThreads) {
                const int r = i / 16, l = i % 16;
                const int rr = row0 + r;
                if (rr >= a.n) continue;
                const uint8_t* rc = a.rrec + static_cast<size_t>(rr) * RBr;
                for (int j = l; j < kr; j += 16) {
                    const int col = rc[j];
                    const float v = Et[r * ZLD + col];
                    if (a.epi == EPI_MASKED_ADD) {
                        for (int p = 0; p < a.ndst; ++p) {
                            float* d = a.dst[p] + static_cast<size_t>(rr) * a.ld + col;
                            *d = __fadd_rn(*d, v);
                        }
                    } else {
                        uint8_t* orc = a.out_rec + static_cast<size_t>(rr) * RBr;
                        orc[j] = static_cast<uint8_t>(col);
                        reinterpret_cast<float*>(orc + KHr)[j] = v;
                    }
                }
            }
        }
        if constexpr (TPR > 0) {
            // GS top-k of the output tile: one thread per row (TPR = group size G)
            if (a.gs_out && tid < TR && row0 + tid < a.n)
                dev::gs_select_row<W, TPR>(Et + tid * ZLD, a.w, a.k_gs, a.gs_out + static_cast<size_t>(row0 + tid) * rec_bytes(a.k_gs));
        }
        if (do_dw) {
            if (dw_active) {
                float t[C::DMB][4];
#pragma unroll
                for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) t[i][j] = 0.f;
                for (int r = 0; r < TR; ++r) {
                    const float* gr = Et + r * ZLD + dn0;
                    float g0 = gr[0], g1 = gr[1], g2 = gr[2], g3 = gr[3];
                    if (TC && do_gemm) { g0 = tf32_op(g0); g1 = tf32_op(g1); g2 = tf32_op(g2); g3 = tf32_op(g3); }  // dW operands as the tensor core reads them
                    const float rf = (!TC && kScale) ? rfs[r] : 1.f;
#pragma unroll
                    for (int i = 0; i < C::DMB; ++i) {
                        const float z = TC ? (do_gemm ? tf32_op(Zs[zoff(r, dm0 + i)]) : Zs[zoff(r, dm0 + i)])
                                           : (kScale ? __fmul_rn(rf, Za[r * ZLD + dm0 + i]) : Za[r * ZLD + dm0 + i]);
                        t[i][0] = fmaf(z, g0, t[i][0]);
                        t[i][1] = fmaf(z, g1, t[i][1]);
                        t[i][2] = fmaf(z, g2, t[i][2]);
                        t[i][3] = fmaf(z, g3, t[i][3]);
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
                for (int r = 0; r < TR; ++r) s = __fadd_rn(s, Et[r * ZLD + tid]);
                dbacc += static_cast<double>(s);
            }
        }
        __syncthreads();
    }
    if (do_dw) {
        double* pp = a.part + static_cast<size_t>(blockIdx.x) * plen;
        if constexpr (C::kRegAcc) {
            if (dw_active) {
#pragma unroll
                for (int i = 0; i < C::DMB; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int m = dm0 + i, nn = dn0 + j;
                        if (m < a.w && nn < a.w) pp[m * a.w + nn] = dacc[i][j];
                    }
            }
        }
        if (tid < a.w) pp[a.w * a.w + tid] = a.want_db ? dbacc : 0.0;
    }
    if constexpr (TC) {
        tc_fence_before();
        __syncthreads();
        if (wid == 0) tmem_dealloc(tmem, W < 32 ? 32 : W);
    }
}

// ---- host-side launch helpers for one width ---------------------------------
int sm_count_host();

// Resident CTAs per SM from the kernel's registers and dynamic smem (the
// occupancy API under-reports kernels that allocate TMEM); TMEM caps the
// tensor-core variants at 512 columns per SM.
template <int W, int AGG, int TPR, int TC>
int occupancy_t() {
    static int occ = 0;
    if (!occ) {
        cudaFuncAttributes fa{};
        int dev = 0, smem_sm = 0, regs_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
        if (cudaFuncGetAttributes(&fa, k_tile<W, AGG, TPR, TC>) != cudaSuccess) {
            cudaGetLastError();
            occ = 1;
            return occ;
        }
        const int by_smem = smem_sm / static_cast<int>(Smem<W>::bytes + 1024);
        const int regs = fa.numRegs > 0 ? fa.numRegs : 255;
        const int by_regs = regs_sm / (((regs + 7) & ~7) * kThreads);
        occ = by_smem < by_regs ? by_smem : by_regs;
        if (occ > 8) occ = 8;
        if (TC && occ > 512 / (W < 32 ? 32 : W)) occ = 512 / (W < 32 ? 32 : W);
        if (occ < 1) occ = 1;
    }
    return occ;
}

template <int W, int AGG, int TPR, int TC>
cudaError_t launch_t(const TileArgs& a, cudaStream_t s, int* grid_out) {
    const int tiles = (a.n + TR - 1) / TR;
    const int cap = sm_count_host() * occupancy_t<W, AGG, TPR, TC>();
    const int grid = tiles < cap ? tiles : cap;
    if (grid_out) *grid_out = grid;
    k_tile<W, AGG, TPR, TC><<<grid, kThreads, Smem<W>::bytes, s>>>(a);
    return cudaGetLastError();
}

template <int W, int AGG, int TPR, int TC>
cudaError_t set_attr_t() {
    return cudaFuncSetAttribute(k_tile<W, AGG, TPR, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Smem<W>::bytes));
}

template <int W, int TC>
cudaError_t set_attrs() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {set_attr_t<W, AGG_SPARSE, 0, TC>(), set_attr_t<W, AGG_SPARSE, 16, TC>(), set_attr_t<W, AGG_SPARSE, W, TC>(),
                          set_attr_t<W, AGG_DENSE, 0, TC>(), set_attr_t<W, AGG_DENSE_RELU, 0, TC>(), set_attr_t<W, AGG_NONE, 0, TC>()})
        if (r != cudaSuccess) e = r;
    return e;
}

template <int W, int TC>
cudaError_t launch_w(const TileArgs& a, cudaStream_t s, int* g) {
    const int k = a.k_gs;
    const int gsg = (a.gs_out == nullptr) ? 0 : (k <= 16 ? 16 : W);  // selection group size (≥ k)
    switch (a.agg) {
        case AGG_SPARSE:
            if (gsg == 0) return launch_t<W, AGG_SPARSE, 0, TC>(a, s, g);
            if (gsg == 16) return launch_t<W, AGG_SPARSE, 16, TC>(a, s, g);
            return launch_t<W, AGG_SPARSE, W, TC>(a, s, g);
        case AGG_DENSE: return launch_t<W, AGG_DENSE, 0, TC>(a, s, g);
        case AGG_DENSE_RELU: return launch_t<W, AGG_DENSE_RELU, 0, TC>(a, s, g);
        default: return launch_t<W, AGG_NONE, 0, TC>(a, s, g);
    }
}

}  // namespace tile
}  // namespace gsrk
