// Thread-per-row tcgen05 kernels for the GSR-C training step in TF32 mode.
//
// The GSR-C step (Eq. 6-7 grouped reversible layers with GS-sparse blocks,
// SURVEY.md §8a rows a20-a22/a33) runs three block shapes, 3 × C × L launches
// per step. k_tile (tile.cuh) implements every shape generically; these are
// the lean sm_100a versions of the three the bench step actually runs:
//
//   FWD  y'_i = x_i + (Â·scatter(V,I))·W_i + b_i, then GS_k(y'_i) → records
//        (gsr_forward_block SPEC.md:253-261 + Eq. 6 add + gs_topk SPEC.md:67-76)
//   INV  x_i = y'_i − (Â·scatter(V,I))·W_i − b_i   (Eq. 7)
//   BIN  Y = Âᵀ·G_i;  dst_p[r, I[r]] += (Y·W_iᵀ)[r, I[r]]  (exact GS-masked
//        input gradient, SPEC.md:262-270 restated for Eq. 6-7) and
//        dW_i += Sᵀ·Y = (Â·S)ᵀ·G_i, S = scatter(V,I), on the tensor core — the
//        parameter gradient rides on the aggregation BIN already does, so the
//        inverse pass never reads G_i (db_i = colsum G_i: k_colsum, bias only)
//
// Design (persistent CTAs, one 128-row tile at a time):
//   * FWD / INV run as k_fws (below): the CTA's aggregation warps build tile
//     j's A operand from a shared-memory window of the neighbour records while
//     its epilogue warps finish tile j − 1 (residual, TMA store, GS top-k), with
//     two TMEM accumulators. k_fast is the single-group form of the same
//     arithmetic (the rev-baseline's dense FWD / INV, and the A/B switch
//     GSRC_NO_WS). In k_fast thread t owns tile row t end to end. It reads its
//     row's 8 neighbour slots (Dir::ell, row-addressed), walks its ≤ kSeg
//     edges (longer "hub" rows come pre-aggregated from k_hub_rows in the
//     oracle's canonical segment order), accumulates in its column of a
//     column-major view of the A buffer (bank = row: a conflict-free scatter
//     for any indices), then moves the row, scaled, into the UMMA A operand
//     (K-major SWIZZLE_128B) one 32-column region at a time,
//     reads its accumulator row back from TMEM (warp w ↔ lane quadrant w), adds
//     or subtracts the residual row (a TMA tile load into the released A
//     buffer), and runs its row's GS top-k alone (FWD: the next block's
//     records; INV: the lower layer's records in the backward sweep);
//   * the output tile leaves by TMA store; the next tile's residual and
//     neighbour slots are prefetched to L2 at tile start;
//   * BIN (256 threads): 8-lane groups gather each row of Y = Âᵀ·G_i with
//     whole-line loads, the thread pair of a row splits the epilogue columns;
//     the masked tile is TMA reduce-added into the destination planes;
//   * one elected thread issues tcgen05.mma kind::tf32 (M = 128, N = W) and,
//     for BIN, a second MN-major MMA accumulating dW = Sᵀ·Y in TMEM across all
//     tiles of the CTA (per-CTA partials, reduced in fixed order afterwards);
//   * every kernel is launched with programmatic dependent launch: the
//     on-chip prologue overlaps the predecessor (dev::pdl_wait / pdl_trigger).
// Arithmetic per row is the oracle's (oracle/gsr_oracle.hpp, TF32 mode):
// canonical segmented aggregation, row scale; fp32 operands are handed to the
// tensor core as they are, which reads them as TF32 by truncating the low 13
// mantissa bits (tests/test_gpu_config_parity.py test_fast_path_tf32_operand_truncation) — the oracle
// truncates the same operands.
#include "tile.cuh"

#include <cstdlib>

namespace gsrk {
namespace fast {

using tile::mbar_init;
using tile::mbar_wait;
using tile::smem_u32;
using tile::tmem_ld;

constexpr int TR = 128;       // rows per tile == threads per CTA
constexpr int kSegF = tile::kSeg;

enum Kind : int { FWD = 0, INV = 1, BIN = 2 };

// Swizzled [TR][W] fp32 tile (UMMA SWIZZLE_128B canonical form, K-major for
// the row-as-M operand, MN-major when rows are K): 32-column regions of
// TR × 128 B; the 16 B chunk j of row r sits at chunk j ^ (r & 7). A row's
// float4 chunks hit 8 distinct bank groups across 8 consecutive rows, so
// thread-per-row LDS/STS.128 are conflict-free.
__device__ __forceinline__ int zo(int r, int m) { return (m >> 5) * (TR * 32) + r * 32 + ((m ^ ((r & 7) << 2)) & 31); }

// MN-major tf32 operands must use the SWIZZLE_128B_BASE32B canonical layout
// (32 B granules; granule j of row r at j ^ (r & 3)); rows are the K index.
__device__ __forceinline__ int zb(int r, int m) { return (m >> 5) * (TR * 32) + r * 32 + ((((m >> 3) & 3) ^ (r & 3)) << 3) + (m & 7); }

// Shared memory (floats; every operand region 1 KB aligned):
//   FWD / INV: Ws | Zs      BIN: Ws | Zs | Y2
// Zs is the UMMA A operand; once the MMA has completed it holds the tile's
// output rows (FWD: for the GS top-k; BIN: h for the masked scatter, then S
// in BASE32B MN-major for dW). Y2 = Y in BASE32B MN-major for dW. The
// residual row is read straight from global into registers while the MMA runs.
template <int W>
struct Plan {
    static constexpr int ws = W * W;
    static constexpr int tile = TR * W;
    // the dW MMA runs with M = 128 (A = Sᵀ: four 32-column atoms at TR·128 B
    // stride from Zs); rows m ≥ W read past Zs into Y2 and land in TMEM lanes
    // that are never read, so Zs + 4 atoms must stay inside the allocation.
    static constexpr int bin_tail = 2 * tile > 4 * TR * 32 ? 2 * tile : 4 * TR * 32;
    static constexpr int floats(int kind) { return kind == BIN ? ws + tile + bin_tail : ws + tile; }
    static constexpr size_t bytes(int kind) { return static_cast<size_t>(floats(kind) + 64) * sizeof(float); }
};

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// next tile's neighbour slots and row scales toward L2 (one bulk request each)
__device__ __forceinline__ void prefetch_tile_meta(const Dir& d, int tile_next, int n_tiles, int n) {
    if (tile_next >= n_tiles) return;
    const int r0 = tile_next * TR, nr = n - r0 < TR ? n - r0 : TR;
    prefetch_l2_bulk(d.ell + static_cast<size_t>(r0) * kSegF, static_cast<uint32_t>(nr) * kSegF * 8u);
    if ((nr & 3) == 0) prefetch_l2_bulk(d.out_f + r0, static_cast<uint32_t>(nr) * 4u);
}
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// ---- TMA (cp.async.bulk.tensor) for the residual / output row tiles ----------
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int c0, int r0) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(m), "r"(c0), "r"(r0) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int r0) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(dst)), "l"(m), "r"(c0), "r"(r0), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int r0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(m), "r"(c0), "r"(r0), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int r0) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(m), "r"(c0), "r"(r0), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// K-major SWIZZLE_128B (layout type 2): LBO as given, SBO = 8-row group stride (1 KB).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
    return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo_bytes >> 4) << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

// MN-major SWIZZLE_128B_BASE32B (layout type 1): LBO = 32-column atom stride
// (TR·128 B), SBO = 4-row group stride (512 B).
__device__ __forceinline__ uint64_t desc_mn32(uint32_t saddr) {
    return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>((TR * 128) >> 4) << 16) | (static_cast<uint64_t>(512 >> 4) << 32) |
           (1ull << 46) | (1ull << 61);
}

// kind::tf32, D = F32, M = 128, N = W; a/b major: 0 = K, 1 = MN.
template <int N>
__host__ __device__ constexpr uint32_t idesc(int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(TR >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { tile::umma_tf32(d, a, b, id, acc); }

// ---- sparse row aggregation (regular rows, deg ≤ kSeg) ----------------------
// z[m] += sc · v over the row's edges in CSR order, the k (index, value)
// pairs of each record in slot order — the oracle's spmm_sparse_row order
// (sc = 1 for unit edges: the multiply is exact). KS = k at compile time
// (8 or 16), or 0 for any k ≤ 16 with predicated slots. The edge loop is not
// unrolled (one record in flight ahead): the kernel's code must stay small
// enough for the instruction cache. The accumulator is column-major,
// acc[m·TR + r]: thread r always hits bank r mod 32, so the scatter is
// conflict-free whatever the indices (a row-major tile costs ~3.5-way
// conflicts for random columns).
// Record window (k_fws): the records of rows [wlo, wlo + wcnt) staged in
// shared memory by one bulk copy; a neighbour inside it is read from there
// (generic loads), any other from global memory.
struct RecWin {
    const uint8_t* p = nullptr;
    int lo = 0, cnt = 0;
};
__device__ __forceinline__ void load_rec_any(tile::SparseRec& r, const uint8_t* rc, int nv4) {
    r.idx = *reinterpret_cast<const uint4*>(rc);
#pragma unroll
    for (int q = 0; q < 4; ++q) r.v[q] = q < nv4 ? *reinterpret_cast<const float4*>(rc + 16 + 16 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
}
template <bool WIN>
__device__ __forceinline__ const uint8_t* rec_src(const FastArgs& a, const RecWin& w, int c, int RB, bool& local) {
    if constexpr (WIN) {
        local = static_cast<unsigned>(c - w.lo) < static_cast<unsigned>(w.cnt);
        return local ? w.p + (c - w.lo) * RB : a.rec_in + static_cast<size_t>(c) * RB;
    } else {
        local = false;
        return a.rec_in + static_cast<size_t>(c) * RB;
    }
}

template <int W, int KS, bool WIN = false>
__device__ __forceinline__ void agg_sparse_row(const FastArgs& a, const int (&cv)[kSegF], const float (&sv)[kSegF], int ne, float* acc, int r,
                                               const RecWin& win = RecWin{}) {
    const int k = KS ? KS : a.k;
    const int RB = rec_bytes(k), nv4 = (k + 3) >> 2;
    const bool unit = a.dir.unit_edge != 0;
    int c1 = cv[1], c2 = cv[2], c3 = cv[3], c4 = cv[4], c5 = cv[5], c6 = cv[6], c7 = cv[7];
    float s1 = sv[1], s2 = sv[2], s3 = sv[3], s4 = sv[4], s5 = sv[5], s6 = sv[6], s7 = sv[7];
    bool loc;
    if (ne > 2) { const uint8_t* q2 = rec_src<WIN>(a, win, c2, RB, loc); if (!loc) prefetch_l2(q2); }
    if (ne > 3) { const uint8_t* q3 = rec_src<WIN>(a, win, c3, RB, loc); if (!loc) prefetch_l2(q3); }
    float* col = acc + r;
    float cur_s = sv[0];
    tile::SparseRec cur;
    if (ne > 0) {
        if constexpr (WIN) load_rec_any(cur, rec_src<WIN>(a, win, cv[0], RB, loc), nv4);
        else tile::load_rec16(cur, a.rec_in + static_cast<size_t>(cv[0]) * RB, nv4);
    }
#pragma unroll 1
    for (int u = 0; u < ne; ++u) {
        const int nc = c1;  // shift registers of the remaining neighbour ids / scales
        const float ns = s1;
        c1 = c2; c2 = c3; c3 = c4; c4 = c5; c5 = c6; c6 = c7;
        s1 = s2; s2 = s3; s3 = s4; s4 = s5; s5 = s6; s6 = s7;
        tile::SparseRec nxt = cur;
        if (u + 1 < ne) {
            if constexpr (WIN) load_rec_any(nxt, rec_src<WIN>(a, win, nc, RB, loc), nv4);
            else tile::load_rec16(nxt, a.rec_in + static_cast<size_t>(nc) * RB, nv4);
        }
        if (u + 3 < ne) { const uint8_t* q2 = rec_src<WIN>(a, win, c2, RB, loc); if (!loc) prefetch_l2(q2); }
        const float sc = unit ? 1.f : cur_s;
        const uint32_t iw[4] = {cur.idx.x, cur.idx.y, cur.idx.z, cur.idx.w};
        const float vv[16] = {cur.v[0].x, cur.v[0].y, cur.v[0].z, cur.v[0].w, cur.v[1].x, cur.v[1].y, cur.v[1].z, cur.v[1].w,
                              cur.v[2].x, cur.v[2].y, cur.v[2].z, cur.v[2].w, cur.v[3].x, cur.v[3].y, cur.v[3].z, cur.v[3].w};
        // a record's k indices are distinct: load all k accumulators, add,
        // store (no read-after-write chain inside a record)
        constexpr int NJ = KS ? KS : 16;
        int off[NJ];
        float old[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            off[j] = static_cast<int>(__byte_perm(iw[j >> 2], 0u, 0x4440u | static_cast<uint32_t>(j & 3))) * TR;
            if (KS || j < k) old[j] = col[off[j]];
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j)
            if (KS || j < k) col[off[j]] = __fadd_rn(old[j], __fmul_rn(sc, vv[j]));
        cur = nxt;
        cur_s = ns;
    }
}

// a row's neighbour slots (Dir::ell): ids (−1 padding, −2 in slot 0 for a hub
// row) and edge scales, four independent 16 B loads
__device__ __forceinline__ int load_ell_row(const int2* ell, int row, int (&cv)[kSegF], float (&sv)[kSegF]) {
    const int4* ep = reinterpret_cast<const int4*>(ell + static_cast<size_t>(row) * kSegF);
    int ne = 0;
#pragma unroll
    for (int q = 0; q < kSegF / 2; ++q) {
        const int4 v = __ldg(ep + q);
        cv[2 * q] = v.x; sv[2 * q] = __int_as_float(v.y);
        cv[2 * q + 1] = v.z; sv[2 * q + 1] = __int_as_float(v.w);
    }
#pragma unroll
    for (int q = 0; q < kSegF; ++q) ne += cv[q] >= 0 ? 1 : 0;
    return cv[0] == -2 ? -1 : ne;  // −1: hub row
}

// ---- dense row aggregation (rev-baseline FWD / INV) ----------------------
// Z = Â·relu(x_in) for the tile's rows, the BIN gather scheme: an 8-lane
// group per row, lane q owning the 16 B column chunks q (and q + 8 at W = 64),
// so every neighbour-row load is whole 128 B lines; 16 rows per pass. Edges in
// CSR order from +0 (the oracle's spmm_row order for ≤ kSeg edges); hub rows
// start from their canonical segmented sum (k_hub_seg_dense + k_hub_fold with
// relu); then Â's row scale. Rows go straight into the K-major SW128 A operand.
__device__ __forceinline__ float relu0(float v) { return v > 0.f ? v : 0.f; }  // the oracle's v > 0 ? v : 0 (−0, NaN → +0)

template <int W>
__device__ __forceinline__ void agg_dense_tile(const FastArgs& a, float* Zs, int row0, int t) {
    constexpr int NCH = W == 64 ? 2 : 1, LPR = W / 4 / NCH, RPP = TR / LPR, NP = TR / RPP;
    static_assert(LPR == kSegF, "lane q holds neighbour slot q");
    const int grp = t / LPR, q = t % LPR;
    const bool unit = a.dir.unit_edge != 0;
    int mycv[NP];
    float myscv[NP], rfv[NP];
#pragma unroll
    for (int ps = 0; ps < NP; ++ps) {  // every pass's neighbour slots first (row-addressed, no load chain)
        const int rw = row0 + ps * RPP + grp;
        int2 e = make_int2(-1, 0);
        rfv[ps] = 0.f;
        if (rw < a.n) {
            e = __ldg(a.dir.ell + static_cast<size_t>(rw) * kSegF + q);
            rfv[ps] = __ldg(a.dir.out_f + rw);
        }
        mycv[ps] = e.x;
        myscv[ps] = __int_as_float(e.y);
    }
#pragma unroll 1
    for (int pass = 0; pass < NP; ++pass) {
        const int r = pass * RPP + grp, rw = row0 + r;
        int myc = -1;
        float mysc = 1.f, rfr = 0.f;
#pragma unroll
        for (int ps = 0; ps < NP; ++ps)
            if (ps == pass) { myc = mycv[ps]; mysc = myscv[ps]; rfr = rfv[ps]; }
        const bool hub = __shfl_sync(0xffffffffu, myc, 0, LPR) == -2;
        float4 acc[NCH];
#pragma unroll
        for (int h = 0; h < NCH; ++h) acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hub) {
            const float* zh = a.Zh + static_cast<size_t>(rw) * a.ld;
#pragma unroll
            for (int h = 0; h < NCH; ++h)
                if (4 * (q + LPR * h) < a.ld) acc[h] = dev::ld4(zh + 4 * (q + LPR * h));
        }
        float4 x[kSegF][NCH];
        bool ok[kSegF];
#pragma unroll
        for (int u = 0; u < kSegF; ++u) {
            const int c = __shfl_sync(0xffffffffu, myc, u, LPR);
            ok[u] = c >= 0;
#pragma unroll
            for (int h = 0; h < NCH; ++h)
                x[u][h] = (ok[u] && 4 * (q + LPR * h) < a.ld) ? dev::ld4(a.x_in + static_cast<size_t>(c) * a.ld + 4 * (q + LPR * h))
                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < kSegF; ++u) {
            const float sc = unit ? 1.f : __shfl_sync(0xffffffffu, mysc, u, LPR);
            if (ok[u]) {
#pragma unroll
                for (int h = 0; h < NCH; ++h) {
                    acc[h].x = __fadd_rn(acc[h].x, __fmul_rn(sc, relu0(x[u][h].x)));
                    acc[h].y = __fadd_rn(acc[h].y, __fmul_rn(sc, relu0(x[u][h].y)));
                    acc[h].z = __fadd_rn(acc[h].z, __fmul_rn(sc, relu0(x[u][h].z)));
                    acc[h].w = __fadd_rn(acc[h].w, __fmul_rn(sc, relu0(x[u][h].w)));
                }
            }
        }
#pragma unroll
        for (int h = 0; h < NCH; ++h)
            *reinterpret_cast<float4*>(Zs + zo(r, 4 * (q + LPR * h))) =
                make_float4(__fmul_rn(rfr, acc[h].x), __fmul_rn(rfr, acc[h].y), __fmul_rn(rfr, acc[h].z), __fmul_rn(rfr, acc[h].w));
    }
}

// GS top-k of a row held in a swizzled smem tile → CBSR record.
// Selection: the k largest magnitudes, ties at the threshold T (the k-th
// largest key) taken lowest column first, columns ascending — the oracle's
// gs_topk. T comes from a top-G tree over the W keys: each G-key group sorted
// by Batcher's odd-even merge network (63 compare-exchanges for G = 16), groups
// merged pairwise by a half-cleaner + bitonic merge; when k == G the last level
// needs only the half-cleaner and a min (T = the smallest of the top G).
// Selection mask: keys ≥ T; only rows with extra ties at T take the slow path.
// Batcher odd-even merge sort, n = 16: 63 compare-exchanges (i, j), max → i
constexpr int kOem16N = 63;
__host__ __device__ constexpr int oem16(int i) {
    constexpr int p[126] = {0, 1, 2, 3, 0, 2, 1, 3, 1, 2, 4, 5, 6, 7, 4, 6, 5, 7, 5, 6, 0, 4, 2, 6, 2, 4, 1, 5, 3, 7, 3, 5,
                                   1, 2, 3, 4, 5, 6, 8, 9, 10, 11, 8, 10, 9, 11, 9, 10, 12, 13, 14, 15, 12, 14, 13, 15, 13, 14, 8, 12,
                                   10, 14, 10, 12, 9, 13, 11, 15, 11, 13, 9, 10, 11, 12, 13, 14, 0, 8, 4, 12, 4, 8, 2, 10, 6, 14, 6, 10,
                                   2, 4, 6, 8, 10, 12, 1, 9, 5, 13, 5, 9, 3, 11, 7, 15, 7, 11, 3, 5, 7, 9, 11, 13, 1, 2, 3, 4, 5, 6, 7,
                                   8, 9, 10, 11, 12, 13, 14};
    return p[i];
}

template <int W, bool FULLW>
__device__ __forceinline__ uint32_t gs_key(float v, int col, int w) {
    // |x| bit pattern; +1 only when padding columns (key 0) must rank below real zeros
    if (FULLW) return __float_as_uint(v) & 0x7fffffffu;
    return col < w ? (__float_as_uint(v) & 0x7fffffffu) + 1u : 0u;
}

template <int W, bool FULLW, int K = 0, bool FM = false>
__device__ __forceinline__ void gs_row_impl(const float* Ts, int r, int w, int k_rt, uint8_t* rec_out) {
    const int k = K ? K : k_rt;  // K: k at compile time (0: any k ≤ 16)
    constexpr int G = 16;
    constexpr int LW = W == 64 ? 6 : 5;
    static_assert((1 << LW) == W, "W must be 32 or 64");
    uint32_t s[W];
#pragma unroll
    for (int c = 0; c < W; c += 4) {
        const float4 v = *reinterpret_cast<const float4*>(Ts + zo(r, c));
        s[c] = gs_key<W, FULLW>(v.x, c, w);
        s[c + 1] = gs_key<W, FULLW>(v.y, c + 1, w);
        s[c + 2] = gs_key<W, FULLW>(v.z, c + 2, w);
        s[c + 3] = gs_key<W, FULLW>(v.w, c + 3, w);
    }
#pragma unroll
    for (int g = 0; g < W; g += G)
#pragma unroll
        for (int i = 0; i < kOem16N; ++i) {
            const int x = g + oem16(2 * i), y = g + oem16(2 * i + 1);
            const uint32_t hi = max(s[x], s[y]), lo = min(s[x], s[y]);
            s[x] = hi;
            s[y] = lo;
        }
    auto merge = [&](int ga, int gb, bool sort) {  // top-G of sorted groups ga ∪ gb → ga
#pragma unroll
        for (int i = 0; i < G; ++i) s[ga + i] = max(s[ga + i], s[gb + G - 1 - i]);
        if (!sort) return;
#pragma unroll
        for (int lt = 3; lt >= 0; --lt) {
            const int stride = 1 << lt;
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const uint32_t x = s[ga + i], y = s[ga + j];
                    s[ga + i] = max(x, y);
                    s[ga + j] = min(x, y);
                }
            }
        }
    };
#pragma unroll
    for (int lsp = 4; lsp < LW - 1; ++lsp) {  // all but the last level keep the groups sorted
        const int span = 1 << lsp;
#pragma unroll
        for (int g = 0; g < W; g += 2 * span) merge(g, g + span, true);
    }
    uint32_t T = 0xffffffffu;
    if (k == G) {  // last level: the top G as a set; T is its minimum
        merge(0, W / 2, false);
#pragma unroll
        for (int i = 0; i < G; i += 2) T = __vimin3_u32(T, s[i], s[i + 1]);  // VIMNMX3
    } else {
        merge(0, W / 2, true);
#pragma unroll
        for (int i = 0; i < G; ++i) T = min(T, i < k ? s[i] : 0xffffffffu);
    }
    // selection mask: every key ≥ T, unless extra ties at T must be cut
    constexpr int NWD = W / 32;
    uint32_t ge[NWD];
#pragma unroll
    for (int q = 0; q < NWD; ++q) ge[q] = 0u;
    if constexpr (FULLW && FM) {
        // "not |v| < T" (one unordered float compare, |.| an operand modifier) is
        // exactly the key compare while T is a number: a NaN's key exceeds every
        // number's, and the unordered compare counts it as ≥ T. (T itself a NaN:
        // the mask is recomputed from the keys on the tie path below.)
        const float Tf = __uint_as_float(T);
#pragma unroll
        for (int c = 0; c < W; c += 4) {
            const float4 v4 = *reinterpret_cast<const float4*>(Ts + zo(r, c));
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!(fabsf(vv[q]) < Tf)) ge[(c + q) >> 5] |= 1u << ((c + q) & 31);
        }
    } else {
#pragma unroll
        for (int c = 0; c < W; c += 4) {
            const float4 v4 = *reinterpret_cast<const float4*>(Ts + zo(r, c));
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) ge[(c + q) >> 5] |= static_cast<uint32_t>(gs_key<W, FULLW>(vv[q], c + q, w) >= T) << ((c + q) & 31);
        }
    }
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < NWD; ++q) cnt += __popc(ge[q]);
    const bool t_nan = FULLW && FM && T > 0x7f800000u;
    if (cnt != k || t_nan) {  // ties at T beyond k: keep keys > T, then the lowest-column ties
        uint32_t gt[NWD];
#pragma unroll
        for (int q = 0; q < NWD; ++q) gt[q] = 0u;
        if (t_nan)
#pragma unroll
            for (int q = 0; q < NWD; ++q) ge[q] = 0u;
        for (int c = 0; c < W; ++c) {
            const uint32_t key = gs_key<W, FULLW>(Ts[zo(r, c)], c, w);
            gt[c >> 5] |= static_cast<uint32_t>(key > T) << (c & 31);
            if (t_nan) ge[c >> 5] |= static_cast<uint32_t>(key >= T) << (c & 31);
        }
        int take = k;
#pragma unroll
        for (int q = 0; q < NWD; ++q) take -= __popc(gt[q]);
#pragma unroll
        for (int q = 0; q < NWD; ++q) {
            uint32_t eq = ge[q] & ~gt[q];
            while (take > 0 && eq) {
                gt[q] |= eq & (0u - eq);
                eq &= eq - 1u;
                --take;
            }
            ge[q] = gt[q];
        }
    }
    // emit the k selected columns in ascending order with compile-time slots
    // (k ≤ 16): index bytes and values assembled in registers, record written
    // with 128-bit stores (layout: 16 index bytes, then k values, 16 B padded)
    uint32_t iw[4] = {0u, 0u, 0u, 0u};
    float rv[16];
    uint32_t m0 = ge[0], m1 = NWD > 1 ? ge[NWD - 1] : 0u;
    const float* trow = Ts + r * 32;
    const int rx = (r & 7) << 2;
#pragma unroll
    for (int slot = 0; slot < 16; ++slot) {
        rv[slot] = 0.f;
        if (slot < k) {  // branch-free: the lowest set bit of m0, else of m1
            const bool lo = m0 != 0u;
            const uint32_t mm = lo ? m0 : m1;
            const int col = __ffs(mm) - 1 + (lo ? 0 : 32);
            const uint32_t cl = mm & (mm - 1u);
            m0 = lo ? cl : m0;
            m1 = lo ? m1 : cl;
            iw[slot >> 2] |= static_cast<uint32_t>(col) << (8 * (slot & 3));
            rv[slot] = trow[(col >> 5) * (TR * 32) + ((col ^ rx) & 31)];  // Ts[zo(r, col)]
        }
    }
    uint4* o = reinterpret_cast<uint4*>(rec_out);
    o[0] = make_uint4(iw[0], iw[1], iw[2], iw[3]);
    const int nv4 = (k + 3) >> 2;
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (q < nv4) reinterpret_cast<float4*>(rec_out + 16)[q] = make_float4(rv[4 * q], rv[4 * q + 1], rv[4 * q + 2], rv[4 * q + 3]);
}

// FM: the selection mask by unordered float compares (fewer instructions; used
// where the GS epilogue bounds the kernel, k_fws)
template <int W, int G, int K = 0, bool FM = false>
__device__ __forceinline__ void gs_row(const float* Ts, int r, int w, int k, uint8_t* rec_out) {
    static_assert(G == 16, "top-16 tree (k ≤ 16)");
    if (K && k == K && w == W) gs_row_impl<W, true, K, FM>(Ts, r, w, k, rec_out);
    else if (w == W) gs_row_impl<W, true>(Ts, r, w, k, rec_out);
    else gs_row_impl<W, false>(Ts, r, w, k, rec_out);
}

template <int W, int KIND, int KS>
__global__ void __launch_bounds__(TR, 4) k_fast(const __grid_constant__ FastArgs a) {
    using Pl = Plan<W>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* base = reinterpret_cast<float*>(smem_raw);
    if ((smem_u32(base) & 1023u) != 0) __trap();  // UMMA SW128 atoms need 1 KB alignment
    float* Ws = base;
    float* Zs = Ws + Pl::ws;
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + Pl::floats(KIND));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);

    const int t = threadIdx.x, wid = t >> 5;
    const int n_tiles = (a.n + TR - 1) / TR;
    static_assert(KIND == FWD || KIND == INV, "BIN is k_bin2");
    constexpr uint32_t TCOLS = W < 32 ? 32 : W;

    // transform operand Bᵀ[n][m] (K-major SW128, region stride W·32)
    for (int i = t; i < W * W; i += TR) {
        const int r = i / W, c = i % W;  // contraction index r, output column c
        float v = 0.f;
        if (r < a.w && c < a.w) v = a.gemm_t ? a.Wm[c * a.w + r] : a.Wm[r * a.w + c];
        Ws[tile::boff<W>(c, r)] = v;
    }
    if (t == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1); }
    if (wid == 0) tile::tmem_alloc(tslot, TCOLS);
    tile::fence_proxy_async();
    tile::tc_fence_before();
    __syncthreads();
    tile::tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t tlane = static_cast<uint32_t>(32 * wid) << 16;
    uint32_t ph0 = 0, ph2 = 0;
    dev::pdl_wait();  // the prologue above touched only W and on-chip state

    for (int tile_i = blockIdx.x; tile_i < n_tiles; tile_i += gridDim.x) {
        const int row0 = tile_i * TR;
        if (KIND == INV && tile_i + static_cast<int>(gridDim.x) >= n_tiles) dev::pdl_trigger();  // measured: FWD is better without
        const int row = row0 + t;
        const bool valid = row < a.n;
        // stage the residual (FWD / INV) and gradient (INV) rows

        // residual tile toward L2 now (TMA prefetch); it is TMA-loaded into Zs
        // once the MMA has consumed the A operand
        if (t == 0) {
#pragma unroll
            for (int c = 0; c < W; c += 32) tma_prefetch_2d(&a.tm_x, c, row0);
            prefetch_tile_meta(a.dir, tile_i + static_cast<int>(gridDim.x), n_tiles, a.n);
        }
        // ---- aggregation: this thread's row accumulates in column t of the
        // column-major view acc[m·TR + t] of the A buffer (conflict-free
        // scatter), then moves, scaled by Â's row factor, into row t of the
        // K-major SW128 A operand. KS < 0: rev-baseline dense rows.
        if constexpr (KS < 0) {
            agg_dense_tile<W>(a, Zs, row0, t);
        } else {
            float* acc = Zs;
            float rf = 0.f;
            int ne = 0;
            int cv[kSegF];
            float sv[kSegF];
            if (valid) {
                ne = load_ell_row(a.dir.ell, row, cv, sv);
                rf = __ldg(a.dir.out_f + row);
            }
            if (ne >= 0) {
#pragma unroll
                for (int m = 0; m < W; ++m) acc[m * TR + t] = 0.f;
                if (ne > 0) agg_sparse_row<W, KS>(a, cv, sv, ne, acc, t);
            }
            // columns [h, h + 32) of acc occupy exactly the storage of the A
            // operand's 32-column region h / 32: one region at a time (32 live
            // values; a barrier between its reads and its writes)
            const float* zh = a.Zh + static_cast<size_t>(row) * a.ld;
#pragma unroll
            for (int h = 0; h < W; h += 32) {
                float v[32];
                if (ne < 0) {  // hub row: canonical segmented sum precomputed by k_hub_*
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 z = h + c < a.ld ? dev::ld4(zh + h + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[c] = z.x; v[c + 1] = z.y; v[c + 2] = z.z; v[c + 3] = z.w;
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < 32; ++m) v[m] = acc[(h + m) * TR + t];
                }
                __syncthreads();
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                    *reinterpret_cast<float4*>(Zs + zo(t, h + c)) =
                        make_float4(__fmul_rn(rf, v[c]), __fmul_rn(rf, v[c + 1]), __fmul_rn(rf, v[c + 2]), __fmul_rn(rf, v[c + 3]));
            }
        }
        tile::fence_proxy_async();
        __syncthreads();
        if (t == 0) {
            tile::tc_fence_after();
            const uint32_t za = smem_u32(Zs), wa = smem_u32(Ws);
#pragma unroll
            for (int kk = 0; kk < W / 8; ++kk)
                umma(tmem, desc_sw128(za + (kk >> 2) * (TR * 128) + (kk & 3) * 32, 16), desc_sw128(wa + (kk >> 2) * (W * 128) + (kk & 3) * 32, 16),
                     idesc<W>(0, 0), kk > 0 ? 1u : 0u);
            tile::umma_commit(&bar[0]);
        }
        mbar_wait(&bar[0], ph0);
        ph0 ^= 1u;
        tile::tc_fence_after();
        // the MMA has read Zs: bring the residual tile in (rows ≥ n read as 0)
        if (t == 0) {
            mbar_expect_tx(&bar[2], static_cast<uint32_t>(TR * W * 4));
#pragma unroll
            for (int c = 0; c < W; c += 32) tma_load_2d(&a.tm_x, Zs + (c >> 5) * (TR * 32), &bar[2], c, row0);
        }
        mbar_wait(&bar[2], ph2);
        ph2 ^= 1u;

        // ---- epilogue: this thread's accumulator row (TMEM lane = tile row)
#pragma unroll
        for (int c0 = 0; c0 < W; c0 += 16) {
            float h[16];
            tmem_ld<16>(tmem + tlane + static_cast<uint32_t>(c0), h);
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
                const int c = c0 + q;
                float o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float hv = h[q + j];
                    if (a.bias) hv = __fadd_rn(hv, c + j < a.w ? __ldg(a.bias + c + j) : 0.f);
                    o[j] = dev::quant(hv, a.qs, a.qi);
                }
                float4* rp = reinterpret_cast<float4*>(Zs + zo(t, c));
                const float4 R = *rp;
                if (KIND == FWD) { o[0] = __fadd_rn(R.x, o[0]); o[1] = __fadd_rn(R.y, o[1]); o[2] = __fadd_rn(R.z, o[2]); o[3] = __fadd_rn(R.w, o[3]); }
                else { o[0] = __fsub_rn(R.x, o[0]); o[1] = __fsub_rn(R.y, o[1]); o[2] = __fsub_rn(R.z, o[2]); o[3] = __fsub_rn(R.w, o[3]); }
                *rp = make_float4(o[0], o[1], o[2], o[3]);  // output row: TMA store source and GS input
            }
        }
        // output tile back in place by TMA (rows ≥ n clipped)
        tile::fence_proxy_async();
        __syncthreads();
        if (t == 0) {
#pragma unroll
            for (int c = 0; c < W; c += 32) tma_store_2d(&a.tm_x, Zs + (c >> 5) * (TR * 32), c, row0);
            tma_store_commit();
        }
        if constexpr (KS >= 0)
            if (a.gs_out && valid) gs_row<W, 16>(Zs, t, a.w, a.k_gs, a.gs_out + static_cast<size_t>(row) * rec_bytes(a.k_gs));
        if (t == 0) tma_store_wait_read();  // Zs is rewritten by the next tile
        tile::tc_fence_before();
        __syncthreads();
    }
    tile::tc_fence_before();
    __syncthreads();
    if (wid == 0) tile::tmem_dealloc(tmem, TCOLS);
}

// ---- warp-specialised FWD / INV (sparse records) ----------------------------
// k_fast runs every phase of a tile on the same 128 threads: its record
// gathers (a chain of dependent L2/DRAM latencies per row) and its GS top-k
// selection (ALU-bound, ~1.1k instructions per row) never overlap (ncu, c3:
// 0.27 vs 0.22 ms per launch with / without the GS epilogue). Here the CTA has
// two warp groups:
//   * warps 0-3 (aggregation; thread t = tile row t): tile j's sparse
//     aggregation into the A operand Zs — the k_fast arithmetic — reading
//     neighbour records from a shared-memory window of the records of rows
//     [row0 − kWinH, row0 + TR + kWinH) (one bulk copy, issued a tile ahead,
//     double-buffered) and from global memory outside it; thread 0 then issues
//     the MMA into TMEM accumulator j & 1;
//   * warps 4-7 (epilogue; thread e = tile row e, warp ↔ TMEM lane quadrant
//     warp & 3): tile j − 1 meanwhile — accumulator row + bias, residual grid,
//     ± the residual row (TMA-loaded into Out), TMA store, then the GS top-k of
//     the output row (the next block's records).
// Handshakes: mbarriers mma_done[b] (tcgen05.commit: accumulator b full, and
// Zs free again), res_full (the residual tile is in Out), acc_free[b] (the 128
// epilogue threads have drained accumulator b), win_full[b] (record window
// b); named barriers 1 / 2 keep each group's own phases apart.
constexpr int kWinH = 16;  // record-window halo rows on each side of a tile

template <int W>
struct PlanWs {
    static constexpr int tile = TR * W;
    static constexpr int win = (TR + 2 * kWinH) * 80 / 4;  // floats per window (records ≤ 80 B)
    static constexpr int floats = W * W + 2 * tile + 2 * win;  // Ws | Zs | Out | Win[0] | Win[1]
    static constexpr size_t bytes = static_cast<size_t>(floats + 64) * sizeof(float);
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int W, int KIND, int KS>
__global__ void __launch_bounds__(2 * TR, 2) k_fws(const __grid_constant__ FastArgs a) {
    static_assert((KIND == FWD || KIND == INV) && KS >= 0, "sparse FWD / INV");
    using Pl = PlanWs<W>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* base = reinterpret_cast<float*>(smem_raw);
    if ((smem_u32(base) & 1023u) != 0) __trap();
    float* Ws = base;
    float* Zs = Ws + W * W;
    float* Ob = Zs + Pl::tile;
    uint8_t* Win = reinterpret_cast<uint8_t*>(Ob + Pl::tile);  // Win[b] = Win + b·Pl::win·4
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + Pl::floats);  // mma_done[2] | acc_free[2] | win_full[2] | res_full
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
    const int tid = threadIdx.x, wid = tid >> 5, t = tid & (TR - 1);
    const int n_tiles = (a.n + TR - 1) / TR;
    const int my_tiles = static_cast<int>(blockIdx.x) < n_tiles ? (n_tiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;
    constexpr uint32_t TCOLS = 2 * W < 32 ? 32 : 2 * W;  // two accumulators
    const int RB = rec_bytes(KS ? KS : a.k);

    // transform operand Bᵀ[n][m] (K-major SW128). On the residual grid it holds
    // tf32(W)·2^s: the tensor core reads tf32(W) unchanged, and every product and
    // partial sum scales by the power of two exactly, so the accumulator holds
    // h·2^s and the epilogue's rounding (dev::quant) needs no multiply in
    const bool grid = a.qs != 0.f;
    for (int i = tid; i < W * W; i += 2 * TR) {
        const int r = i / W, c = i % W;
        float v = 0.f;
        if (r < a.w && c < a.w) v = a.gemm_t ? a.Wm[c * a.w + r] : a.Wm[r * a.w + c];
        Ws[tile::boff<W>(c, r)] = grid ? __fmul_rn(tile::tf32_op(v), a.qs) : v;
    }
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) { mbar_init(&bar[b], 1); mbar_init(&bar[2 + b], TR); mbar_init(&bar[4 + b], 1); }
        mbar_init(&bar[6], 1);
    }
    if (wid == 0) tile::tmem_alloc(tslot, TCOLS);
    tile::fence_proxy_async();
    tile::tc_fence_before();
    __syncthreads();
    tile::tc_fence_after();
    const uint32_t tmem = *tslot;
    dev::pdl_wait();  // the prologue above touched only W and on-chip state

    auto tile_of = [&](int jj) { return static_cast<int>(blockIdx.x) + jj * static_cast<int>(gridDim.x); };
    if (tid < TR) {
        // ================= aggregation group (warps 0-3) =================
        auto win_span = [&](int jj, int& lo, int& cnt) {
            const int r0 = tile_of(jj) * TR;
            lo = r0 - kWinH > 0 ? r0 - kWinH : 0;
            const int hi = r0 + TR + kWinH < a.n ? r0 + TR + kWinH : a.n;
            cnt = hi - lo;
        };
        auto issue_win = [&](int jj) {  // records of tile jj's window → Win[jj & 1]
            int lo, cnt;
            win_span(jj, lo, cnt);
            uint64_t* wb = &bar[4 + (jj & 1)];
            mbar_expect_tx(wb, static_cast<uint32_t>(cnt * RB));
            bulk_load(Win + (jj & 1) * (Pl::win * 4), a.rec_in + static_cast<size_t>(lo) * RB, static_cast<uint32_t>(cnt * RB), wb);
        };
        if (t == 0 && my_tiles > 0) issue_win(0);
        // this row's neighbour slots and row scale, loaded one tile ahead
        int cv[kSegF];
        float sv[kSegF];
        int ne = 0;
        float rf = 0.f;
        auto load_meta = [&](int jj) {
            const int rw = tile_of(jj) * TR + t;
            ne = 0;
            rf = 0.f;
            if (jj < my_tiles && rw < a.n) {
                ne = load_ell_row(a.dir.ell, rw, cv, sv);
                rf = __ldg(a.dir.out_f + rw);
            }
        };
        load_meta(0);
        for (int j = 0; j < my_tiles; ++j) {
            const int tile_i = tile_of(j);
            const int row0 = tile_i * TR, row = row0 + t;
            const int b = j & 1;
            // no early pdl_trigger: with it, the successor's CTAs crowd this grid's tail (measured)
            if (t == 0) {
                prefetch_tile_meta(a.dir, tile_i + 2 * static_cast<int>(gridDim.x), n_tiles, a.n);
                if (j + 1 < my_tiles) {  // Win[(j + 1) & 1] was last read by tile j − 1 (before its barriers)
                    tile::fence_proxy_async();
                    issue_win(j + 1);
                }
            }
            RecWin wn;
            win_span(j, wn.lo, wn.cnt);
            wn.p = Win + b * (Pl::win * 4);
            mbar_wait(&bar[4 + b], static_cast<uint32_t>(j >> 1) & 1u);  // window j is in
            if (j > 0) mbar_wait(&bar[(j - 1) & 1], static_cast<uint32_t>((j - 1) >> 1) & 1u);  // MMA j − 1 has read Zs
            float* acc = Zs;
            if (ne >= 0) {
#pragma unroll
                for (int m = 0; m < W; ++m) acc[m * TR + t] = 0.f;
                if (ne > 0) agg_sparse_row<W, KS, true>(a, cv, sv, ne, acc, t, wn);
            }
            const float* zh = a.Zh + static_cast<size_t>(row) * a.ld;
#pragma unroll
            for (int h = 0; h < W; h += 32) {
                float v[32];
                if (ne < 0) {  // hub row: canonical segmented sum precomputed by k_hub_rows
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const float4 z = h + c < a.ld ? dev::ld4(zh + h + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                        v[c] = z.x; v[c + 1] = z.y; v[c + 2] = z.z; v[c + 3] = z.w;
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < 32; ++m) v[m] = acc[(h + m) * TR + t];
                }
                named_bar_sync(1, TR);
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                    *reinterpret_cast<float4*>(Zs + zo(t, h + c)) =
                        make_float4(__fmul_rn(rf, v[c]), __fmul_rn(rf, v[c + 1]), __fmul_rn(rf, v[c + 2]), __fmul_rn(rf, v[c + 3]));
            }
            tile::fence_proxy_async();
            named_bar_sync(1, TR);
            if (t == 0) {
                if (j >= 2) mbar_wait(&bar[2 + b], static_cast<uint32_t>((j >> 1) - 1) & 1u);  // tile j − 2 has left accumulator b
                tile::tc_fence_after();
                const uint32_t za = smem_u32(Zs), wa = smem_u32(Ws);
#pragma unroll
                for (int kk = 0; kk < W / 8; ++kk)
                    umma(tmem + static_cast<uint32_t>(b * W), desc_sw128(za + (kk >> 2) * (TR * 128) + (kk & 3) * 32, 16),
                         desc_sw128(wa + (kk >> 2) * (W * 128) + (kk & 3) * 32, 16), idesc<W>(0, 0), kk > 0 ? 1u : 0u);
                tile::umma_commit(&bar[b]);
            }
            load_meta(j + 1);
        }
    } else {
        // ================= epilogue group (warps 4-7) =================
        const uint32_t tlane = static_cast<uint32_t>(32 * (wid & 3)) << 16;
        auto issue_res = [&](int jj) {  // residual tile jj → Out (rows ≥ n read as 0)
            mbar_expect_tx(&bar[6], static_cast<uint32_t>(TR * W * 4));
#pragma unroll
            for (int c = 0; c < W; c += 32) tma_load_2d(&a.tm_x, Ob + (c >> 5) * (TR * 32), &bar[6], c, tile_of(jj) * TR);
        };
        if (t == 0 && my_tiles > 0) issue_res(0);
        for (int j = 0; j < my_tiles; ++j) {
            const int row0 = tile_of(j) * TR, row = row0 + t;
            const bool valid = row < a.n;
            const int b = j & 1;
            if (t == 0 && j + 1 < my_tiles) {
#pragma unroll
                for (int c = 0; c < W; c += 32) tma_prefetch_2d(&a.tm_x, c, tile_of(j + 1) * TR);
            }
            mbar_wait(&bar[b], static_cast<uint32_t>(j >> 1) & 1u);  // accumulator b holds tile j
            tile::tc_fence_after();
            mbar_wait(&bar[6], static_cast<uint32_t>(j) & 1u);  // residual tile j is in Out
#pragma unroll
            for (int c0 = 0; c0 < W; c0 += 16) {
                float h[16];
                tmem_ld<16>(tmem + tlane + static_cast<uint32_t>(b * W + c0), h);
                if (a.bias) {  // (scaled with the accumulator on the grid: (h + b)·2^s exactly)
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const float bv = c0 + q < a.w ? __ldg(a.bias + c0 + q) : 0.f;
                        h[q] = __fadd_rn(h[q], grid ? __fmul_rn(bv, a.qs) : bv);
                    }
                }
                if (grid) {  // dev::quant(h + b): rint((h + b)·2^s)·2^-s
#pragma unroll
                    for (int q = 0; q < 16; ++q) h[q] = __fmul_rn(rintf(h[q]), a.qi);
                }
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const int c = c0 + q;
                    float o[4] = {h[q], h[q + 1], h[q + 2], h[q + 3]};
                    float4* rp = reinterpret_cast<float4*>(Ob + zo(t, c));
                    const float4 R = *rp;
                    if (KIND == FWD) { o[0] = __fadd_rn(R.x, o[0]); o[1] = __fadd_rn(R.y, o[1]); o[2] = __fadd_rn(R.z, o[2]); o[3] = __fadd_rn(R.w, o[3]); }
                    else { o[0] = __fsub_rn(R.x, o[0]); o[1] = __fsub_rn(R.y, o[1]); o[2] = __fsub_rn(R.z, o[2]); o[3] = __fsub_rn(R.w, o[3]); }
                    *rp = make_float4(o[0], o[1], o[2], o[3]);
                }
            }
            tile::tc_fence_before();
            mbar_arrive(&bar[2 + b]);  // accumulator b drained
            tile::fence_proxy_async();
            named_bar_sync(2, TR);
            if (t == 0) {
#pragma unroll
                for (int c = 0; c < W; c += 32) tma_store_2d(&a.tm_x, Ob + (c >> 5) * (TR * 32), c, row0);
                tma_store_commit();
            }
            if (a.gs_out && valid) gs_row<W, 16, KS == 16 ? 16 : 0, true>(Ob, t, a.w, a.k_gs, a.gs_out + static_cast<size_t>(row) * rec_bytes(a.k_gs));
            named_bar_sync(2, TR);  // every read of Out is done
            if (t == 0) {
                tma_store_wait_read();
                if (j + 1 < my_tiles) {
                    tile::fence_proxy_async();
                    issue_res(j + 1);
                }
            }
        }
    }
    tile::tc_fence_before();
    __syncthreads();
    if (wid == 0) tile::tmem_dealloc(tmem, TCOLS);
}

// ---- BIN: input gradient and dW, two threads per row ------------------------
// The dense transposed aggregation gathers a full neighbour row (4w bytes) per
// edge: an 8-lane group per row makes each neighbour-row load whole 128 B
// lines; the epilogue gives threads t and t + 128 one column half each of tile
// row t & 127. The CTA has 8 warps.
// DM (rev-baseline): S = relu(u) and the mask u > 0 come from the dense row of
// u (a.mplane) instead of the block's GS record.
template <int W, int TPR, bool DM>
__global__ void __launch_bounds__(TPR * TR, 2) k_bin2(const __grid_constant__ FastArgs a) {
    using Pl = Plan<W>;
    constexpr int NT = TPR * TR, HW = W / TPR;  // HW: this thread's epilogue columns
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* base = reinterpret_cast<float*>(smem_raw);
    if ((smem_u32(base) & 1023u) != 0) __trap();
    float* Ws = base;
    float* Zs = Ws + Pl::ws;     // Y (K-major, MMA A), then du for the TMA reduce-add
    float* S2 = Zs + Pl::tile;   // S (BASE32B): the dW MMA's A = Sᵀ reads four atoms, into Y2
    float* Y2 = S2 + Pl::tile;   // Y (BASE32B), the dW MMA's B
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + Pl::floats(BIN));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 3);
    const int tid = threadIdx.x, wid = tid >> 5;
    const int t = tid & (TR - 1), hf = tid >> 7;  // tile row, column part
    const int c_lo = hf * HW;
    const int n_tiles = (a.n + TR - 1) / TR;
    constexpr uint32_t TCOLS = 2 * W < 64 ? 64 : 2 * W;

    for (int i = tid; i < W * W; i += NT) {  // Bᵀ[n][m] = W[n][m] (h = Y·Wᵀ)
        const int r = i / W, c = i % W;
        Ws[tile::boff<W>(c, r)] = (r < a.w && c < a.w) ? a.Wm[c * a.w + r] : 0.f;
    }
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    if (wid == 0) tile::tmem_alloc(tslot, TCOLS);
    tile::fence_proxy_async();
    tile::tc_fence_before();
    __syncthreads();
    tile::tc_fence_after();
    const uint32_t tmem = *tslot;
    const uint32_t tlane = static_cast<uint32_t>(32 * (wid & 3)) << 16;
    uint32_t ph0 = 0, ph1 = 0;
    bool dw_pending = false;
    dev::pdl_wait();  // the prologue above touched only W and on-chip state
    // the mask source of a tile: its GS records, or (DM) its rows of u
    auto mask_span = [&](int ti, const void*& p, uint32_t& bytes) {
        const int nr = a.n - ti * TR < TR ? a.n - ti * TR : TR;
        if (DM) { p = a.mplane + static_cast<size_t>(ti) * TR * a.ld; bytes = static_cast<uint32_t>(nr * a.ld * 4); }
        else { p = a.mrec + static_cast<size_t>(ti) * TR * rec_bytes(a.k_m); bytes = static_cast<uint32_t>(nr * rec_bytes(a.k_m)); }
    };
    if (tid == 0 && static_cast<int>(blockIdx.x) < n_tiles) {  // the first tile's mask source
        const void* p;
        uint32_t b;
        mask_span(static_cast<int>(blockIdx.x), p, b);
        prefetch_l2_bulk(p, b);
    }

    for (int tile_i = blockIdx.x; tile_i < n_tiles; tile_i += gridDim.x) {
        const int row0 = tile_i * TR, row = row0 + t;
        const bool valid = row < a.n;
        if (tile_i + static_cast<int>(gridDim.x) >= n_tiles) dev::pdl_trigger();
        if (dw_pending) {
            mbar_wait(&bar[1], ph1);
            ph1 ^= 1u;
            tile::tc_fence_after();
            dw_pending = false;
        }
        const int tnext = tile_i + static_cast<int>(gridDim.x);
        if (tid == 0) {  // the next tile's slots, mask records and its own rows of G_i (± a halo)
            prefetch_tile_meta(a.dir, tnext, n_tiles, a.n);
            if (tnext < n_tiles) {
                const void* p;
                uint32_t b;
                mask_span(tnext, p, b);
                prefetch_l2_bulk(p, b);
                // most of a circuit row's neighbours are the rows next to it: their
                // G rows toward L2 now, so the next tile's gather passes hit L2
                constexpr int kH = 8;
                const int lo = tnext * TR - kH > 0 ? tnext * TR - kH : 0;
                const int hi = tnext * TR + TR + kH < a.n ? tnext * TR + TR + kH : a.n;
                prefetch_l2_bulk(a.x_in + static_cast<size_t>(lo) * a.ld, static_cast<uint32_t>(hi - lo) * static_cast<uint32_t>(a.ld) * 4u);
            }
        }
        uint32_t hm = 0u;  // this thread's mask columns (mask of a padding / invalid row: empty)
        if constexpr (DM) {
            // ---- S = relu(u) and the mask u > 0 from the row of u, this thread's columns (BASE32B)
            const float* ur = a.mplane + static_cast<size_t>(row) * a.ld;
#pragma unroll
            for (int c = 0; c < HW; c += 4) {
                const float4 u4 = (valid && c_lo + c < a.ld) ? dev::ld4(ur + c_lo + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float uv[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) hm |= static_cast<uint32_t>(uv[j] > 0.f) << (c + j);
                *reinterpret_cast<float4*>(S2 + zb(t, c_lo + c)) = make_float4(relu0(u4.x), relu0(u4.y), relu0(u4.z), relu0(u4.w));
            }
        } else {
            // mask record of the row (the block's input records: S and the input-gradient mask)
            const uint8_t* rc = a.mrec + static_cast<size_t>(row) * rec_bytes(a.k_m);
            uint4 iw4 = make_uint4(0u, 0u, 0u, 0u);
            if (valid) iw4 = *reinterpret_cast<const uint4*>(rc);
            const uint32_t iw[4] = {iw4.x, iw4.y, iw4.z, iw4.w};
            // ---- S = scatter(V, I) of the row, this thread's columns (BASE32B): dW += Sᵀ·Y
            // (the previous tile's dW MMA has released S2 / Y2); values loaded only
            // for this thread's columns (the row's record is in L1 for its threads)
#pragma unroll
            for (int c = 0; c < HW; c += 4) *reinterpret_cast<float4*>(S2 + zb(t, c_lo + c)) = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int c = static_cast<int>((iw[j >> 2] >> (8 * (j & 3))) & 0xffu);
                if (valid && j < a.k_m && c / HW == hf) {
                    S2[zb(t, c)] = *reinterpret_cast<const float*>(rc + 16 + 4 * j);
                    hm |= 1u << (c - c_lo);
                }
            }
        }
        if (tid == 0) tma_store_wait_read();  // the previous tile's du (Zs) has been read by its reduce-add
        __syncthreads();
        // ---- Y = Âᵀ·x_in, gathered cooperatively: an 8-lane group per row, lane
        // q owning the 16 B column chunks q and q + 8 (W = 64), so every
        // neighbour-row load is four whole 128 B lines per warp instruction
        // (not 32 scattered sectors); up to 8 edges of loads in flight per lane.
        {
            constexpr int NCH = (TPR == 2 && W == 64) ? 2 : 1;  // 16 B chunks per lane: columns 4q (+4·LPR)
            constexpr int LPR = W / 4 / NCH;                    // lanes per row
            static_assert(LPR == kSegF, "lane q of a row's group holds neighbour slot q");
            constexpr int RPP = NT / LPR;                       // rows per pass
            constexpr int NP = TR / RPP;                        // passes
            const int grp = tid / LPR, q = tid % LPR;
            const bool unit = a.dir.unit_edge != 0;
            // the neighbour slots of all passes first (Dir::ell: one row-addressed
            // load per lane, no row_ptr → col_idx → edge_f chain); lane q holds slot q
            int mycv[NP];
            float myscv[NP], rfv[NP];
#pragma unroll
            for (int ps = 0; ps < NP; ++ps) {
                const int rw = row0 + ps * RPP + grp;
                int2 e = make_int2(-1, 0);
                rfv[ps] = 0.f;
                if (rw < a.n) {
                    if (q < kSegF) e = __ldg(a.dir.ell + static_cast<size_t>(rw) * kSegF + q);
                    rfv[ps] = __ldg(a.dir.out_f + rw);
                }
                mycv[ps] = e.x;
                myscv[ps] = __int_as_float(e.y);
            }
#pragma unroll 1
            for (int pass = 0; pass < NP; ++pass) {
                const int r = pass * RPP + grp, rw = row0 + r;
                int myc = -1;
                float mysc = 1.f, rfr = 0.f;
#pragma unroll
                for (int ps = 0; ps < NP; ++ps)
                    if (ps == pass) { myc = mycv[ps]; mysc = myscv[ps]; rfr = rfv[ps]; }
                const bool hub = __shfl_sync(0xffffffffu, myc, 0, LPR) == -2;
                float4 acc[NCH];
#pragma unroll
                for (int h = 0; h < NCH; ++h) acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (hub) {
                    const float* zh = a.Zh + static_cast<size_t>(rw) * a.ld;
#pragma unroll
                    for (int h = 0; h < NCH; ++h)
                        if (4 * (q + LPR * h) < a.ld) acc[h] = dev::ld4(zh + 4 * (q + LPR * h));
                }
                // every lane runs the shuffles (whole-warp masks); rows differ only in
                // predicates. Slots are filled in CSR order (−1 after the last edge), so
                // the warp walks only as many slots as its longest row has edges.
                int nmax = 0;
                {
                    const uint32_t bal = __ballot_sync(0xffffffffu, myc >= 0);
#pragma unroll
                    for (int g = 0; g < 32 / LPR; ++g) nmax = max(nmax, __popc((bal >> (g * LPR)) & 0xffu));
                }
                float4 x[kSegF][NCH];
                bool ok[kSegF];
#pragma unroll
                for (int u = 0; u < kSegF; ++u) {
                    ok[u] = false;
                    if (u < nmax) {
                        const int c = __shfl_sync(0xffffffffu, myc, u, LPR);
                        ok[u] = c >= 0;
#pragma unroll
                        for (int h = 0; h < NCH; ++h)
                            x[u][h] = (ok[u] && 4 * (q + LPR * h) < a.ld) ? dev::ld4(a.x_in + static_cast<size_t>(c) * a.ld + 4 * (q + LPR * h))
                                                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
#pragma unroll
                for (int u = 0; u < kSegF; ++u) {
                    if (u >= nmax) break;
                    const float sc = unit ? 1.f : __shfl_sync(0xffffffffu, mysc, u, LPR);
                    if (ok[u]) {
#pragma unroll
                        for (int h = 0; h < NCH; ++h) {
                            acc[h].x = __fadd_rn(acc[h].x, __fmul_rn(sc, x[u][h].x));
                            acc[h].y = __fadd_rn(acc[h].y, __fmul_rn(sc, x[u][h].y));
                            acc[h].z = __fadd_rn(acc[h].z, __fmul_rn(sc, x[u][h].z));
                            acc[h].w = __fadd_rn(acc[h].w, __fmul_rn(sc, x[u][h].w));
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < NCH; ++h) {  // Â scale; Y in K-major (MMA A) and BASE32B (dW B)
                    const float4 v = make_float4(__fmul_rn(rfr, acc[h].x), __fmul_rn(rfr, acc[h].y), __fmul_rn(rfr, acc[h].z), __fmul_rn(rfr, acc[h].w));
                    *reinterpret_cast<float4*>(Zs + zo(r, 4 * (q + LPR * h))) = v;
                    *reinterpret_cast<float4*>(Y2 + zb(r, 4 * (q + LPR * h))) = v;
                }
            }
        }
        tile::fence_proxy_async();
        tile::tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tile::tc_fence_after();
            const uint32_t za = smem_u32(Zs), wa = smem_u32(Ws);
#pragma unroll
            for (int kk = 0; kk < W / 8; ++kk)
                umma(tmem, desc_sw128(za + (kk >> 2) * (TR * 128) + (kk & 3) * 32, 16), desc_sw128(wa + (kk >> 2) * (W * 128) + (kk & 3) * 32, 16),
                     idesc<W>(0, 0), kk > 0 ? 1u : 0u);
            tile::umma_commit(&bar[0]);
            const uint32_t sa = smem_u32(S2), ya = smem_u32(Y2);
            const bool first = tile_i == static_cast<int>(blockIdx.x);
#pragma unroll
            for (int kk = 0; kk < TR / 8; ++kk)
                umma(tmem + W, desc_mn32(sa + kk * 1024), desc_mn32(ya + kk * 1024), idesc<W>(1, 1), (first && kk == 0) ? 0u : 1u);
            tile::umma_commit(&bar[1]);
        }
        dw_pending = true;
        mbar_wait(&bar[0], ph0);
        ph0 ^= 1u;
        tile::tc_fence_after();
        // ---- du = mask ⊙ (Y·Wᵀ), this thread's half → Zs: the tile TMA
        // reduce-adds into every destination plane (each element receives one
        // add, so the result is deterministic; off-mask entries add +0)
        constexpr int CW = HW < 16 ? HW : 16;  // TMEM columns per load
#pragma unroll
        for (int c0 = 0; c0 < HW; c0 += CW) {
            float h[CW];
            tmem_ld<CW>(tmem + tlane + static_cast<uint32_t>(c_lo + c0), h);
#pragma unroll
            for (int q = 0; q < CW; ++q) h[q] = (hm >> (c0 + q)) & 1u ? h[q] : 0.f;
#pragma unroll
            for (int q = 0; q < CW; q += 4)
                *reinterpret_cast<float4*>(Zs + zo(t, c_lo + c0 + q)) = make_float4(h[q], h[q + 1], h[q + 2], h[q + 3]);
        }
        tile::fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            for (int p = 0; p < a.ndst; ++p)
#pragma unroll
                for (int c = 0; c < W; c += 32) tma_reduce_add_2d(&a.tm_dst[p], Zs + (c >> 5) * (TR * 32), c, row0);
            tma_store_commit();
        }
    }
    if (dw_pending) {
        mbar_wait(&bar[1], ph1);
        tile::tc_fence_after();
    }
    // per-CTA dW partial: TMEM lane m, columns W + n; each half writes its columns
    const int plen = a.w * a.w + a.w;
    double* pp = a.part + static_cast<size_t>(blockIdx.x) * plen;
    constexpr int CW2 = HW < 16 ? HW : 16;
#pragma unroll
    for (int c0 = 0; c0 < HW; c0 += CW2) {
        float v[CW2];
        tmem_ld<CW2>(tmem + tlane + static_cast<uint32_t>(W + c_lo + c0), v);
        if (t < a.w) {
#pragma unroll
            for (int j = 0; j < CW2; ++j)
                if (c_lo + c0 + j < a.w) pp[t * a.w + c_lo + c0 + j] = static_cast<double>(v[j]);
        }
    }
    if (hf == 0 && t < a.w) pp[a.w * a.w + t] = 0.0;  // db: k_colsum (bias only)
    if (tid == 0) tma_store_wait_read();  // the last du tile leaves shared memory before exit
    tile::tc_fence_before();
    __syncthreads();
    if (wid == 0) tile::tmem_dealloc(tmem, TCOLS);
}

// ---- hub rows (deg > kSeg) ----------------------------------------------------
// Canonical order for a long row: kSeg-edge segments, each summed from +0 in
// CSR order, then folded left to right. Sparse rows (FWD / INV): one CTA per
// work item = (hub row, chunk of ≤ kHubChunk consecutive segments) computes the
// chunk's segment partials into shared rows, a thread per segment. A row of one
// chunk is folded right there; a longer row's
// chunks write their partials to Pseg and the last chunk to finish (an atomic
// count per hub row, reset by that CTA) folds the whole row from Pseg. The fold
// order is the same either way, so the result does not depend on which CTA
// folds. Work is spread over all SMs regardless of how skewed the hub degrees are.
// one segment (≤ kSeg records) of a sparse hub row into the private row pr:
// 128-bit record loads one ahead, two 8-slot halves per record
// pr = acc + thread: column m of the thread's partial row is pr[m·kHubChunk]
// (bank = thread: a conflict-free scatter for any indices)
__device__ __forceinline__ void hub_seg_sparse(const FastArgs& a, int lo, int ne, float* pr) {
    const int k = a.k, RB = rec_bytes(k), nv4 = (k + 3) >> 2;
    const bool unit = a.dir.unit_edge != 0;
    int cs[kSegF];
#pragma unroll
    for (int u = 0; u < kSegF; ++u) cs[u] = u < ne ? __ldg(a.dir.idx + lo + u) : 0;
#pragma unroll
    for (int u = 1; u < kSegF; ++u)
        if (u < ne) prefetch_l2(a.rec_in + static_cast<size_t>(cs[u]) * RB);
    tile::SparseRec buf[2];
    tile::load_rec16(buf[0], a.rec_in + static_cast<size_t>(cs[0]) * RB, nv4);
#pragma unroll
    for (int u = 0; u < kSegF; ++u) {
        if (u < ne) {
            if (u + 1 < ne) tile::load_rec16(buf[(u + 1) & 1], a.rec_in + static_cast<size_t>(cs[u + 1 < kSegF ? u + 1 : 0]) * RB, nv4);
            const float sc = unit ? 1.f : __ldg(a.dir.edge_f + cs[u]);
            const tile::SparseRec& rc = buf[u & 1];
            const uint32_t iw[4] = {rc.idx.x, rc.idx.y, rc.idx.z, rc.idx.w};
            const float vv[16] = {rc.v[0].x, rc.v[0].y, rc.v[0].z, rc.v[0].w, rc.v[1].x, rc.v[1].y, rc.v[1].z, rc.v[1].w,
                                  rc.v[2].x, rc.v[2].y, rc.v[2].z, rc.v[2].w, rc.v[3].x, rc.v[3].y, rc.v[3].z, rc.v[3].w};
#pragma unroll
            for (int h = 0; h < 16; h += 8) {
                int mm[8];
                float old[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    mm[j] = static_cast<int>(__byte_perm(iw[(h + j) >> 2], 0u, 0x4440u | static_cast<uint32_t>(j & 3))) * kHubChunk;
                    if (h + j < k) old[j] = pr[mm[j]];
                }
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (h + j < k) pr[mm[j]] = __fadd_rn(old[j], __fmul_rn(sc, vv[h + j]));
            }
        }
    }
}

template <int W>
__global__ void __launch_bounds__(kHubChunk) k_hub_rows(FastArgs a, const int4* __restrict__ items, int* __restrict__ cnt,
                                                                       float* __restrict__ Pseg) {
    constexpr int PL = W + 4, CH = kHubChunk, NT = CH;
    // the segment partials accumulate column-major, acc[m·CH + s] (conflict-free
    // scatter), then move to row-major slot[s·PL + m] for the in-order fold
    __shared__ __align__(16) float slot[CH * PL];
    __shared__ int last;
    float* acc = slot;
    const int tid = threadIdx.x;
    dev::pdl_wait();
    dev::pdl_trigger();  // the block kernel that follows may start its on-chip prologue while the hub rows finish
    // work item: {row, first edge, end edge, first segment of the chunk}, {hub index, row's first partial}
    const int4 ia = __ldg(items + 2 * blockIdx.x), ib = __ldg(items + 2 * blockIdx.x + 1);
    const int r = ia.x, e0 = ia.y, e1 = ia.z, c0 = ia.w, h = ib.x;
    const int nseg = (e1 - e0 + kSegF - 1) / kSegF;
    const int ns = min(CH, nseg - c0);
#pragma unroll 8
    for (int m = 0; m < W; ++m) acc[m * CH + tid] = 0.f;
    if (tid < ns) {
        const int lo = e0 + (c0 + tid) * kSegF;
        hub_seg_sparse(a, lo, min(kSegF, e1 - lo), acc + tid);
    }
    {  // column-major → row-major (in place: every value is in registers across the barrier)
        float v[W];
#pragma unroll
        for (int m = 0; m < W; ++m) v[m] = acc[m * CH + tid];
        __syncthreads();
#pragma unroll
        for (int m = 0; m < W; m += 4) *reinterpret_cast<float4*>(slot + tid * PL + m) = make_float4(v[m], v[m + 1], v[m + 2], v[m + 3]);
    }
    __syncthreads();
    const int ld = a.ld;
    if (nseg <= CH) {  // the whole row is here: fold left to right
        for (int col = tid; col < ld; col += NT) {
            float z = slot[col];
            for (int j = 1; j < ns; ++j) z = __fadd_rn(z, slot[j * PL + col]);
            a.Zh[static_cast<size_t>(r) * ld + col] = z;
        }
        return;
    }
    // a chunk of a longer row: partials out, then the last chunk folds the row
    const int s0 = ib.y;
    float* P = Pseg + static_cast<size_t>(s0 + c0) * ld;
    for (int i = tid; i < ns * (ld >> 2); i += NT) {
        const int rr = i / (ld >> 2), c4 = i % (ld >> 2);
        *reinterpret_cast<float4*>(P + static_cast<size_t>(rr) * ld + 4 * c4) = *reinterpret_cast<const float4*>(slot + rr * PL + 4 * c4);
    }
    __syncthreads();
    if (tid == 0) {  // the barrier orders the CTA's partial stores before this release
        __threadfence();
        const int nch = (nseg + CH - 1) / CH;
        last = atomicAdd(cnt + h, 1) == nch - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const float* Pr = Pseg + static_cast<size_t>(s0) * ld;
    for (int col = tid; col < ld; col += NT) {
        float z = __ldcg(Pr + col);
        int s = 1;
        for (; s + 16 <= nseg; s += 16) {  // sixteen partials in flight, folded in order
            float p[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) p[i] = __ldcg(Pr + static_cast<size_t>(s + i) * ld + col);
#pragma unroll
            for (int i = 0; i < 16; ++i) z = __fadd_rn(z, p[i]);
        }
        for (; s < nseg; ++s) z = __fadd_rn(z, __ldcg(Pr + static_cast<size_t>(s) * ld + col));
        a.Zh[static_cast<size_t>(r) * ld + col] = z;
    }
    if (tid == 0) cnt[h] = 0;  // ready for the next launch
}

// dense hub rows (BIN): flattened, one warp per segment over all hub segments
// of the graph (every neighbour row one coalesced load; at the gather's
// roofline), then one warp per hub row folds its partials in order.
template <int W>
__global__ void __launch_bounds__(256) k_hub_seg_dense(FastArgs a, const int2* __restrict__ segs, int nseg, float* __restrict__ Pseg) {
    // one warp per segment, lanes over columns: every neighbour row is one coalesced load
    constexpr int CPL = W / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sgi = blockIdx.x * 8 + wid;
    dev::pdl_wait();
    if (sgi >= nseg) return;
    const int2 se = __ldg(segs + sgi);
    const int lo = se.x, ne = se.y - se.x;
    const bool unit = a.dir.unit_edge != 0;
    const int myc = lane < ne ? __ldg(a.dir.idx + lo + lane) : 0;
    const float mysc = (!unit && lane < ne) ? __ldg(a.dir.edge_f + myc) : 1.f;
    float x[kSegF][CPL];
#pragma unroll
    for (int u = 0; u < kSegF; ++u) {
        const int c = __shfl_sync(0xffffffffu, myc, u);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
            const int col = lane + 32 * q;
            x[u][q] = (u < ne && col < a.ld) ? __ldg(a.x_in + static_cast<size_t>(c) * a.ld + col) : 0.f;
            if (a.relu) x[u][q] = relu0(x[u][q]);
        }
    }
    float acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] = 0.f;
#pragma unroll
    for (int u = 0; u < kSegF; ++u) {
        const float sc = __shfl_sync(0xffffffffu, mysc, u);
        if (u < ne)
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[q] = __fadd_rn(acc[q], __fmul_rn(sc, x[u][q]));
    }
    float* out = Pseg + static_cast<size_t>(sgi) * a.ld;
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        if (lane + 32 * q < a.ld) out[lane + 32 * q] = acc[q];
}

template <int W>
__global__ void __launch_bounds__(256) k_hub_fold(FastArgs a, const int* __restrict__ rows, const int* __restrict__ seg_off, int nhub,
                                                  const float* __restrict__ Pseg) {
    constexpr int CPL = W / 32;
    const int lane = threadIdx.x & 31;
    const int h = blockIdx.x * 8 + (threadIdx.x >> 5);
    dev::pdl_wait();
    if (h >= nhub) return;
    const int s0 = __ldg(seg_off + h), s1 = __ldg(seg_off + h + 1);
    float z[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) z[q] = (lane + 32 * q < a.ld) ? __ldg(Pseg + static_cast<size_t>(s0) * a.ld + lane + 32 * q) : 0.f;
    int s = s0 + 1;
    for (; s + 16 <= s1; s += 16) {  // sixteen partial rows in flight, folded in order
        float p[16][CPL];
#pragma unroll
        for (int i = 0; i < 16; ++i)
#pragma unroll
            for (int q = 0; q < CPL; ++q)
                p[i][q] = (lane + 32 * q < a.ld) ? __ldg(Pseg + static_cast<size_t>(s + i) * a.ld + lane + 32 * q) : 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i)
#pragma unroll
            for (int q = 0; q < CPL; ++q) z[q] = __fadd_rn(z[q], p[i][q]);
    }
    for (; s < s1; ++s)
#pragma unroll
        for (int q = 0; q < CPL; ++q)
            z[q] = __fadd_rn(z[q], (lane + 32 * q < a.ld) ? __ldg(Pseg + static_cast<size_t>(s) * a.ld + lane + 32 * q) : 0.f);
    const int r = __ldg(rows + h);
#pragma unroll
    for (int q = 0; q < CPL; ++q)
        if (lane + 32 * q < a.ld) a.Zh[static_cast<size_t>(r) * a.ld + lane + 32 * q] = z[q];
}

// ---- GS top-k of planes (backward recompute, Eq. 6 group sum) ---------------
// u = p0 + p1 + … (left to right) per row, then GS_k(u) → records. Plane
// tiles (128 rows × W) arrive by TMA into two alternating shared buffers (the
// next tile's load overlaps this one's selection); thread t owns row t.
template <int W>
__global__ void __launch_bounds__(TR, 3) k_gs_tma(const __grid_constant__ GsArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float* buf = reinterpret_cast<float*>(smem_raw);
    if ((smem_u32(buf) & 1023u) != 0) __trap();
    uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 2 * TR * W);
    const int t = threadIdx.x;
    const int n_tiles = (a.n + TR - 1) / TR;
    const int my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int nl = my_tiles * a.nplanes;  // this CTA's loads: (tile, plane) in order
    if (t == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    __syncthreads();
    dev::pdl_wait();
    auto issue = [&](int j) {
        const int tile_i = blockIdx.x + (j / a.nplanes) * gridDim.x, p = j % a.nplanes;
        float* dst = buf + (j & 1) * TR * W;
        mbar_expect_tx(&bar[j & 1], static_cast<uint32_t>(TR * W * 4));
#pragma unroll
        for (int c = 0; c < W; c += 32) tma_load_2d(&a.maps[p], dst + (c >> 5) * (TR * 32), &bar[j & 1], c, tile_i * TR);
    };
    if (t == 0 && nl > 0) issue(0);
    uint32_t ph[2] = {0u, 0u};
    float acc[W];
    for (int j = 0; j < nl; ++j) {
        if (j + a.nplanes >= nl) dev::pdl_trigger();  // this CTA's last tile
        if (t == 0 && j + 1 < nl) issue(j + 1);  // the other buffer was released by the barrier below
        mbar_wait(&bar[j & 1], ph[j & 1]);
        ph[j & 1] ^= 1u;
        float* Ts = buf + (j & 1) * TR * W;
        const int tile_i = blockIdx.x + (j / a.nplanes) * gridDim.x, p = j % a.nplanes;
        const int row = tile_i * TR + t;
        if (a.nplanes > 1) {
#pragma unroll
            for (int c = 0; c < W; c += 4) {
                const float4 v = *reinterpret_cast<const float4*>(Ts + zo(t, c));
                if (p == 0) { acc[c] = v.x; acc[c + 1] = v.y; acc[c + 2] = v.z; acc[c + 3] = v.w; }
                else {
                    acc[c] = __fadd_rn(acc[c], v.x); acc[c + 1] = __fadd_rn(acc[c + 1], v.y);
                    acc[c + 2] = __fadd_rn(acc[c + 2], v.z); acc[c + 3] = __fadd_rn(acc[c + 3], v.w);
                }
            }
            if (p == a.nplanes - 1) {  // the sum goes back into this thread's row for the selection
#pragma unroll
                for (int c = 0; c < W; c += 4)
                    *reinterpret_cast<float4*>(Ts + zo(t, c)) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            }
        }
        if (p == a.nplanes - 1 && row < a.n) gs_row<W, 16>(Ts, t, a.w, a.k, a.rec + static_cast<size_t>(row) * rec_bytes(a.k));
        __syncthreads();
    }
}

// db = colsum(G) (bias only): per-CTA partials over 128-row tiles in row
// order (float within a tile, double across tiles), reduced in fixed order.
__global__ void __launch_bounds__(128) k_colsum(const float* __restrict__ G, int n, int w, int ld, double* __restrict__ part) {
    const int t = threadIdx.x;
    double acc = 0.0;
    for (int r0 = blockIdx.x * TR; r0 < n; r0 += gridDim.x * TR) {
        float s = 0.f;
        const int r1 = min(n, r0 + TR);
        if (t < w)
            for (int r = r0; r < r1; ++r) s = __fadd_rn(s, __ldg(G + static_cast<size_t>(r) * ld + t));
        acc += static_cast<double>(s);
    }
    if (t < w) part[static_cast<size_t>(blockIdx.x) * w + t] = acc;
}

template <int W, int KIND, int KS>
int occupancy() {
    static int occ = 0;
    if (!occ) {
        int dev = 0, smem_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k_fast<W, KIND, KS>);
        const int by_smem = smem_sm / static_cast<int>(Plan<W>::bytes(KIND) + 1024);  // + per-CTA reserved smem
        const int regs = fa.numRegs > 0 ? ((fa.numRegs + 7) & ~7) : 255;
        const int by_regs = 65536 / (regs * TR);
        constexpr int tcols = W < 32 ? 32 : W;
        occ = by_smem < by_regs ? by_smem : by_regs;
        if (occ > 512 / tcols) occ = 512 / tcols;
        if (occ > 8) occ = 8;
        if (occ < 1) occ = 1;
    }
    return occ;
}

template <int W, int KIND, int KS>
cudaError_t launch(const FastArgs& a, cudaStream_t s, int* grid_out) {
    const int tiles = (a.n + TR - 1) / TR;
    const int cap = tile::sm_count_host() * occupancy<W, KIND, KS>();
    const int grid = tiles < cap ? tiles : cap;
    if (grid_out) *grid_out = grid;
    if (grid == 0) return cudaSuccess;
    return launch_pdl(k_fast<W, KIND, KS>, dim3(grid), dim3(TR), Plan<W>::bytes(KIND), s, a);
}

template <int W, int KIND, int KS>
int occupancy_ws() {
    static int occ = 0;
    if (!occ) {
        int dev = 0, smem_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k_fws<W, KIND, KS>);
        const int by_smem = smem_sm / static_cast<int>(PlanWs<W>::bytes + 1024);
        const int regs = fa.numRegs > 0 ? ((fa.numRegs + 7) & ~7) : 255;
        const int by_regs = 65536 / (regs * 2 * TR);
        constexpr int tcols = 2 * W < 32 ? 32 : 2 * W;
        occ = by_smem < by_regs ? by_smem : by_regs;
        if (occ > 512 / tcols) occ = 512 / tcols;
        if (occ < 1) occ = 1;
    }
    return occ;
}

bool use_ws() {
    static const int v = std::getenv("GSRC_NO_WS") ? 0 : 1;  // A/B switch: the single-group k_fast
    return v != 0;
}

template <int W, int KIND, int KS>
cudaError_t launch_ws(const FastArgs& a, cudaStream_t s, int* grid_out) {
    const int tiles = (a.n + TR - 1) / TR;
    const int cap = tile::sm_count_host() * occupancy_ws<W, KIND, KS>();
    const int grid = tiles < cap ? tiles : cap;
    if (grid_out) *grid_out = grid;
    if (grid == 0) return cudaSuccess;
    return launch_pdl(k_fws<W, KIND, KS>, dim3(grid), dim3(2 * TR), PlanWs<W>::bytes, s, a);
}

template <int W, int KIND, int KS>
cudaError_t set_attr() {
    cudaError_t e = cudaFuncSetAttribute(k_fast<W, KIND, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Plan<W>::bytes(KIND)));
    if constexpr (KS >= 0)
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fws<W, KIND, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(PlanWs<W>::bytes));
    return e;
}

constexpr int kBinTPR = 2;  // BIN threads per tile row (epilogue columns W / kBinTPR each)

template <int W>
int occupancy_bin2() {
    static int occ = 0;
    if (!occ) {
        int dev = 0, smem_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k_bin2<W, kBinTPR, false>);
        const int by_smem = smem_sm / static_cast<int>(Plan<W>::bytes(BIN) + 1024);
        const int regs = fa.numRegs > 0 ? ((fa.numRegs + 7) & ~7) : 255;
        const int by_regs = 65536 / (regs * kBinTPR * TR);
        occ = by_smem < by_regs ? by_smem : by_regs;
        const int tcols = 2 * W < 64 ? 64 : 2 * W;
        if (occ > 512 / tcols) occ = 512 / tcols;
        if (occ < 1) occ = 1;
    }
    return occ;
}

template <int W>
cudaError_t launch_bin2(const FastArgs& a, cudaStream_t s, int* grid_out) {
    const int tiles = (a.n + TR - 1) / TR;
    const int cap = tile::sm_count_host() * occupancy_bin2<W>();
    const int grid = tiles < cap ? tiles : cap;
    if (grid_out) *grid_out = grid;
    if (grid == 0) return cudaSuccess;
    if (a.mplane) return launch_pdl(k_bin2<W, kBinTPR, true>, dim3(grid), dim3(kBinTPR * TR), Plan<W>::bytes(BIN), s, a);
    return launch_pdl(k_bin2<W, kBinTPR, false>, dim3(grid), dim3(kBinTPR * TR), Plan<W>::bytes(BIN), s, a);
}

template <int W>
cudaError_t set_attrs() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {set_attr<W, FWD, 0>(), set_attr<W, FWD, 8>(), set_attr<W, FWD, 16>(), set_attr<W, INV, 0>(), set_attr<W, INV, 8>(),
                          set_attr<W, INV, 16>(), set_attr<W, FWD, -1>(), set_attr<W, INV, -1>(),
                          cudaFuncSetAttribute(k_bin2<W, kBinTPR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Plan<W>::bytes(BIN))),
                          cudaFuncSetAttribute(k_bin2<W, kBinTPR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Plan<W>::bytes(BIN)))})
        if (r != cudaSuccess) e = r;
    return e;
}

// KS: record k as a compile-time constant when it is 8 or 16 (the configs'
// values), else the predicated any-k variant.
template <int W, int KIND>
cudaError_t launch_k(const FastArgs& a, cudaStream_t s, int* g) {
    if (a.dense) return launch<W, KIND, -1>(a, s, g);
    if (use_ws()) {
        if (a.k == 16) return launch_ws<W, KIND, 16>(a, s, g);
        if (a.k == 8) return launch_ws<W, KIND, 8>(a, s, g);
        return launch_ws<W, KIND, 0>(a, s, g);
    }
    if (a.k == 16) return launch<W, KIND, 16>(a, s, g);
    if (a.k == 8) return launch<W, KIND, 8>(a, s, g);
    return launch<W, KIND, 0>(a, s, g);
}

template <int W>
cudaError_t launch_w(int kind, const FastArgs& a, cudaStream_t s, int* g) {
    switch (kind) {
        case FWD: return launch_k<W, FWD>(a, s, g);
        case INV: return launch_k<W, INV>(a, s, g);
        default: return launch_bin2<W>(a, s, g);
    }
}

}  // namespace fast

cudaError_t encode_plane_map(CUtensorMap* m, const float* base, int n, int ld) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        enc = reinterpret_cast<Encode>(fn);
    }
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(n)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(fast::TR)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// W = 128 would need 256 KB of shared memory for INV: k_tile serves it.
bool fast_supported(int w, int k) { return w >= 1 && w <= 64 && k >= 1 && k <= 16; }

cudaError_t init_fast_attributes() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {fast::set_attrs<32>(), fast::set_attrs<64>(),
                          cudaFuncSetAttribute(fast::k_gs_tma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * fast::TR * 32 * 4 + 64),
                          cudaFuncSetAttribute(fast::k_gs_tma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * fast::TR * 64 * 4 + 64)})
        if (r != cudaSuccess) e = r;
    return e;
}

int fast_bin_grid_max() {
    const int a = fast::occupancy_bin2<32>(), b = fast::occupancy_bin2<64>();
    return tile::sm_count_host() * (a > b ? a : b);
}

cudaError_t launch_fast(int kind, const FastArgs& a, cudaStream_t s, int* grid_out) {
    if (grid_out) *grid_out = 0;
    if (a.n == 0) return cudaSuccess;
    if (kind != fast::BIN && !a.dense && (a.k < 1 || a.k > 16)) return cudaErrorInvalidValue;
    if (a.gs_out && (a.k_gs < 1 || a.k_gs > 16)) return cudaErrorInvalidValue;
    if (a.w <= 32) return fast::launch_w<32>(kind, a, s, grid_out);
    if (a.w <= 64) return fast::launch_w<64>(kind, a, s, grid_out);
    return cudaErrorInvalidValue;
}

cudaError_t launch_gs_tma(const GsArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    if (a.k < 1 || a.k > 16 || a.w > 64 || a.nplanes < 1 || a.nplanes > kMaxDst) return cudaErrorInvalidValue;
    const int tiles = (a.n + fast::TR - 1) / fast::TR;
    const int cap = tile::sm_count_host() * 3;
    const int grid = tiles < cap ? tiles : cap;
    if (a.w <= 32) {
        constexpr size_t bytes = 2 * fast::TR * 32 * 4 + 64;
        return launch_pdl(fast::k_gs_tma<32>, dim3(grid), dim3(fast::TR), bytes, s, a);
    } else {
        constexpr size_t bytes = 2 * fast::TR * 64 * 4 + 64;
        return launch_pdl(fast::k_gs_tma<64>, dim3(grid), dim3(fast::TR), bytes, s, a);
    }
    return cudaGetLastError();
}

cudaError_t launch_hub_rows(const FastArgs& a, const int4* items, int nitem, int* cnt, float* Pseg, cudaStream_t s) {
    if (nitem == 0) return cudaSuccess;
    if (a.w <= 32) return launch_pdl(fast::k_hub_rows<32>, dim3(nitem), dim3(kHubChunk), 0, s, a, items, cnt, Pseg);
    if (a.w <= 64) return launch_pdl(fast::k_hub_rows<64>, dim3(nitem), dim3(kHubChunk), 0, s, a, items, cnt, Pseg);
    return cudaErrorInvalidValue;
}

cudaError_t launch_hub_dense(const FastArgs& a, const int2* segs, int nseg, const int* rows, const int* seg_off, int nhub, float* Pseg,
                             cudaStream_t s) {
    if (nhub == 0) return cudaSuccess;
    const int gs = (nseg + 7) / 8, gf = (nhub + 7) / 8;
    if (a.w <= 32) {
        cudaError_t e = launch_pdl(fast::k_hub_seg_dense<32>, dim3(gs), dim3(256), 0, s, a, segs, nseg, Pseg);
        if (e != cudaSuccess) return e;
        return launch_pdl(fast::k_hub_fold<32>, dim3(gf), dim3(256), 0, s, a, rows, seg_off, nhub, static_cast<const float*>(Pseg));
    } else if (a.w <= 64) {
        cudaError_t e = launch_pdl(fast::k_hub_seg_dense<64>, dim3(gs), dim3(256), 0, s, a, segs, nseg, Pseg);
        if (e != cudaSuccess) return e;
        return launch_pdl(fast::k_hub_fold<64>, dim3(gf), dim3(256), 0, s, a, rows, seg_off, nhub, static_cast<const float*>(Pseg));
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_colsum(const float* G, int n, int w, int ld, double* part, int* grid_out, cudaStream_t s) {
    const int tiles = (n + fast::TR - 1) / fast::TR;
    const int cap = tile::sm_count_host() * 8;
    const int grid = tiles < cap ? (tiles > 0 ? tiles : 1) : cap;
    if (grid_out) *grid_out = grid;
    fast::k_colsum<<<grid, 128, 0, s>>>(G, n, w, ld, part);
    return cudaGetLastError();
}


}  // namespace gsrk
