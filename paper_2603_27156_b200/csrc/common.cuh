// Device helpers shared by the GS and tile kernels (sm_100a).
#pragma once

#include <cstdint>
#include <utility>

#include "kernels.cuh"

namespace gsrk {
namespace dev {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Exactly invertible residual stream (gsrc_set_residual_quant): the block
// output h is rounded to the grid 2^-s (round half to even) before the Eq. 6
// add / Eq. 7 subtract, so x + q(h) and (x + q(h)) − q(h) are exact for |x| <
// 2^(24-s) and the inverse recompute reproduces the forward bit for bit.
// qs = 2^s, qi = 2^-s; qs == 0 disables it. Both multiplies are exact.
__device__ __forceinline__ float quant(float h, float qs, float qi) { return qs != 0.f ? __fmul_rn(rintf(__fmul_rn(h, qs)), qi) : h; }

// Programmatic dependent launch (launch_pdl): a kernel launched with it may
// start while its stream predecessor finishes. pdl_wait() blocks until the
// predecessor has completed and its memory is visible — every PDL kernel calls
// it before touching global memory that a predecessor writes or reads
// (only parameters, the graph structure and on-chip state come before).
// pdl_trigger() lets the successor launch once every CTA of this grid has
// called it (or exited): persistent kernels call it on their last tile.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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

// Thread-per-row GS (one thread owns all P = W columns of a row): the k-th
// largest key via a bitonic top-G selection tree — sort groups of G keys,
// then repeatedly keep the top G of two groups with the half-cleaner
// max(a_i, b_{G-1-i}) + bitonic merge — no shuffles. G ≥ k (power of two).
template <int G, int P>
__device__ __forceinline__ void sort_group(uint32_t (&s)[P], int base_) {
#pragma unroll
    for (int size = 2; size <= G; size <<= 1) {
#pragma unroll
        for (int stride = size / 2; stride > 0; stride >>= 1) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int j = i ^ stride;
                if (j > i) {
                    const uint32_t a = s[base_ + i], b = s[base_ + j];
                    const uint32_t hi = max(a, b), lo = min(a, b);
                    if ((i & size) == 0) { s[base_ + i] = hi; s[base_ + j] = lo; }
                    else { s[base_ + i] = lo; s[base_ + j] = hi; }
                }
            }
        }
    }
}

template <int G, int P>
__device__ __forceinline__ void merge_groups(uint32_t (&s)[P], int ga, int gb) {  // top-G of groups a ∪ b → a (sorted)
#pragma unroll
    for (int i = 0; i < G; ++i) s[ga + i] = max(s[ga + i], s[gb + G - 1 - i]);
#pragma unroll
    for (int stride = G / 2; stride > 0; stride >>= 1) {
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const int j = i ^ stride;
            if (j > i) {
                const uint32_t a = s[ga + i], b = s[ga + j];
                s[ga + i] = max(a, b);
                s[ga + j] = min(a, b);
            }
        }
    }
}

// xrow: the row's P values in shared memory (columns ≥ w are padding).
// Keys are rebuilt from smem in each pass so only the sort buffer lives in
// registers. Writes one CBSR record.
__device__ __forceinline__ uint32_t mag_key(float v) { return (__float_as_uint(v) & 0x7fffffffu) + 1u; }

template <int P, int G>
__device__ __forceinline__ void gs_select_row(const float* xrow, int w, int k, uint8_t* rec) {
    uint32_t s[P];
#pragma unroll
    for (int i = 0; i < P; ++i) s[i] = (i < w) ? mag_key(xrow[i]) : 0u;
#pragma unroll
    for (int g = 0; g < P; g += G) sort_group<G>(s, g);
#pragma unroll
    for (int span = G; span < P; span *= 2) {
#pragma unroll
        for (int g = 0; g < P; g += 2 * span) merge_groups<G>(s, g, g + span);
    }
    uint32_t T = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) if (i == k - 1) T = s[i];
    int gt = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) gt += s[i] > T;   // every key > T is among the top G
    int take = k - gt;                               // ties at T, lowest columns first
    int slot = 0;
    float* rv = reinterpret_cast<float*>(rec + rec_kh(k));
    for (int i = 0; i < w; ++i) {
        const float v = xrow[i];
        const uint32_t key = mag_key(v);
        const bool is_eq = key == T;
        const bool pick = key > T || (is_eq && take > 0);
        take -= (is_eq && take > 0) ? 1 : 0;
        if (pick) {
            rec[slot] = static_cast<uint8_t>(i);
            rv[slot] = v;
            ++slot;
        }
    }
}

}  // namespace dev

// host: launch `kern` with programmatic stream serialization (see pdl_wait)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace gsrk
