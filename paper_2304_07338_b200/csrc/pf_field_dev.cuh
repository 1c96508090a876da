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

// Two consecutive table entries (2F fp16) starting at an even entry: one
// 256-bit load at F = 8 (LDG.256, one 32-byte sector).
template <int F>
struct Pair {
    Raw<F> lo, hi;
};

template <int F>
__device__ __forceinline__ Pair<F> load_pair(const __half *tab, uint32_t e_even) {
    Pair<F> r;
    const __half *q = tab + (size_t)e_even * F;
    if constexpr (F == 8) {
        asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(r.lo.v.x), "=r"(r.lo.v.y), "=r"(r.lo.v.z), "=r"(r.lo.v.w), "=r"(r.hi.v.x), "=r"(r.hi.v.y),
              "=r"(r.hi.v.z), "=r"(r.hi.v.w)
            : "l"(q));
    } else if constexpr (F == 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(q));
        r.lo.v = make_uint2(v.x, v.y), r.hi.v = make_uint2(v.z, v.w);
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(q));
        r.lo.v = v.x, r.hi.v = v.y;
    }
    return r;
}

#ifndef PF_ENC_PAIR
#define PF_ENC_PAIR 0  // A/B on C2: field 1.29 ms (pair loads, 4 CTAs/SM; 6 CTAs spill) vs 1.22 ms (off)
#endif

// Encode ONE level of one input (pinned in oracle
// or_hashgrid_encode): 2^D gathers issued back to back, fp32 accumulation in
// corner order.  PF_ENC_PAIR: the two corners of an x-edge are fetched by one
// pair load when they are the two entries of one aligned pair -- always for a
// dense level with an even first index (x + 1 -> index + 1), and for a hashed
// level when the cell's x is even (x ^ 1 flips only bit 0 of the hash) -- else
// the second corner is one extra (predicated) load: 1.5 instead of 2 sectors
// per edge on average, same values, same summation order.
template <int D, int F>
__device__ __forceinline__ void encode_level(const __half *tables, const FieldLevel L, const float *pin, float *acc) {
    constexpr int NC = 1 << D;
    uint32_t c[D];
    float f[D];
    level_cell<D>(L, pin, c, f);
    const __half *tab = tables + L.offset_halves;
#if PF_ENC_PAIR
    constexpr int NP = NC / 2;
    Pair<F> p[NP];
    Raw<F> s[NP];
    bool odd[NP], same[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const uint32_t e0 = corner_index<D>(L, c, 2 * k), e1 = corner_index<D>(L, c, 2 * k + 1);
        odd[k] = (e0 & 1u) != 0u;
        same[k] = e1 == (e0 ^ 1u);
        p[k] = load_pair<F>(tab, e0 & ~1u);
        if (!same[k]) s[k] = load_raw<F>(tab, e1);
    }
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = 0.f;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const Raw<F> a = odd[k] ? p[k].hi : p[k].lo;
        const Raw<F> b = same[k] ? (odd[k] ? p[k].lo : p[k].hi) : s[k];
        accum_raw<F>(a, corner_weight<D>(f, 2 * k), acc);
        accum_raw<F>(b, corner_weight<D>(f, 2 * k + 1), acc);
    }
#else
    Raw<F> e[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) e[k] = load_raw<F>(tab, corner_index<D>(L, c, k));
#pragma unroll
    for (int k = 0; k < F; ++k) acc[k] = 0.f;
#pragma unroll
    for (int k = 0; k < NC; ++k) accum_raw<F>(e[k], corner_weight<D>(f, k), acc);
#endif
}

template <int D, int F>
__device__ __forceinline__ void encode_level(const FieldParams &P, int lv, const float *pin, float *acc) {
    encode_level<D, F>(P.tables, P.lv[lv], pin, acc);
}

}  // namespace pfk
