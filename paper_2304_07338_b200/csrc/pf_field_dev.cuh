// pf_field_dev.cuh -- device pieces of the field query shared by the split
// (encode kernel -> TMA-fed MLP kernel) and the fused warp-specialised field
// kernels: fp16 table entry gathers, multilinear accumulation, canonical
// UMMA-layout shared-memory stores, tcgen05 layer issue.
#pragma once

#include <cuda_fp16.h>

#include "pf_field.h"
#include "pf_hashgrid.cuh"
#include "pf_umma.cuh"

namespace pfk {

template <int F>
struct Raw;  // one table entry (F fp16 features)
template <>
struct Raw<8> {
    uint4 v;
};
template <>
struct Raw<4> {
    uint2 v;
};
template <>
struct Raw<2> {
    uint32_t v;
};

template <int F>
__device__ __forceinline__ Raw<F> load_raw(const __half *tab, uint32_t e) {
    Raw<F> r;
    if constexpr (F == 8) r.v = __ldg(reinterpret_cast<const uint4 *>(tab) + e);
    else if constexpr (F == 4) r.v = __ldg(reinterpret_cast<const uint2 *>(tab) + e);
    else r.v = __ldg(reinterpret_cast<const uint32_t *>(tab) + e);
    return r;
}

template <int F>
__device__ __forceinline__ void accum_raw(const Raw<F> &r, float w, float *acc) {
    const __half2 *h = reinterpret_cast<const __half2 *>(&r.v);
#pragma unroll
    for (int i = 0; i < F / 2; ++i) {
        const float2 f = __half22float2(h[i]);
        acc[2 * i] = fmaf(w, f.x, acc[2 * i]);
        acc[2 * i + 1] = fmaf(w, f.y, acc[2 * i + 1]);
    }
}

// st.shared of F fp16 features of row r at column k of an UMMA tile.
template <int F>
__device__ __forceinline__ void store_feats(uint32_t A_s, int r, int k, uint32_t sbo, const float *acc) {
    const uint32_t a = A_s + (uint32_t)(r >> 3) * sbo + (uint32_t)(k >> 3) * 128u + (uint32_t)(r & 7) * 16u +
                       (uint32_t)(k & 7) * 2u;
    uint32_t h[F / 2];
#pragma unroll
    for (int i = 0; i < F / 2; ++i) {
        __half2 v = __floats2half2_rn(acc[2 * i], acc[2 * i + 1]);
        h[i] = *reinterpret_cast<uint32_t *>(&v);
    }
    if constexpr (F == 8)
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]));
    else if constexpr (F == 4)
        asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(a), "r"(h[0]), "r"(h[1]));
    else
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(h[0]));
}

__device__ __forceinline__ void st_shared_zero16(uint32_t a) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(a), "r"(0u));
}

__device__ __forceinline__ void issue_layer(uint32_t a_s, uint32_t b_s, int K, int N, uint32_t tmem_d) {
    const uint32_t sbo = (uint32_t)K * 16u;
    const uint32_t idesc = umma_idesc_f16(128, N);
    for (int j = 0; j < K / 16; ++j) {
        const uint64_t ad = umma_sdesc(a_s + 256u * j, 128u, sbo);
        const uint64_t bd = umma_sdesc(b_s + 256u * j, 128u, sbo);
        umma_f16(tmem_d, ad, bd, idesc, j > 0 ? 1u : 0u);
    }
}

// Encode ONE level of one input (pinned in oracle
// or_hashgrid_encode): 2^D gathers issued back to back, fp32 accumulation.
// (Tried: one 256-bit load per x-edge corner pair when both entries share an
// aligned pair, else a predicated second load -- 1.5 instead of 2 sectors per
// edge, but it spills at 40 registers and at 4 CTAs/SM the field took 1.29 ms
// vs 1.22 ms; reverted.)
template <int D, int F>
__device__ __forceinline__ void encode_level(const __half *tables, const FieldLevel L, const float *pin, float *acc) {
    constexpr int NC = 1 << D;
    uint32_t c[D];
    float f[D];
    level_cell<D>(L, pin, c, f);
    const __half *tab = tables + L.offset_halves;
    Raw<F> e[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) e[k] = load_raw<F>(tab, corner_index<D>(L, c, k));
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) accum_raw<F>(e[k], corner_weight<D>(f, k), acc);
}

template <int D, int F>
__device__ __forceinline__ void encode_level(const FieldParams &P, int lv, const float *pin, float *acc) {
    encode_level<D, F>(P.tables, P.lv[lv], pin, acc);
}

}  // namespace pfk
