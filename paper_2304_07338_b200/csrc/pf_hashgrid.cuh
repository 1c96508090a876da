// pf_hashgrid.cuh -- multiresolution hash-grid addressing shared by the
// inference encoder (pf_field.cu) and the trainer (pf_train.cu).
//
// SPEC.md:385-388, pinned in oracle/pf_oracle.c or_hashgrid_encode /
// or_grid_corners: cell = floor(p * N_l) clamped to N_l - 1 (p in [0,1]),
// corner bit i <-> axis i, dense (N_l+1)^d addressing when it fits in T,
// else (v0 * 1 ^ v1 * 2654435761 ^ v2 * 805459861) mod T.
#pragma once

#include <stdint.h>

#include "pf_field.h"

namespace pfk {

constexpr uint32_t kPrime1 = 2654435761u, kPrime2 = 805459861u;

// Cell + fractional weights of one level (exact p*N split: s + e == p*N).
template <int D>
__device__ __forceinline__ void level_cell(const FieldLevel &L, const float *pin, uint32_t *c, float *f) {
    const float resf = (float)L.res;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const float s = pin[i] * resf;
        const float e = fmaf(pin[i], resf, -s);
        const float fl = floorf(s);
        float fr = (s - fl) + e;
        int ci = (int)fl;
        if (fr < 0.f) {
            ci -= 1;
            fr += 1.f;
        }
        if (ci > (int)L.res - 1) {
            ci = (int)L.res - 1;
            fr = (s - (float)ci) + e;
        }
        c[i] = (uint32_t)ci;
        f[i] = fr;
    }
}

template <int D>
__device__ __forceinline__ uint32_t corner_index(const FieldLevel &L, const uint32_t *c, int corner) {
    uint32_t v[D];
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = c[i] + (uint32_t)((corner >> i) & 1);
    if (L.dense) {
        uint32_t idx = v[0] + L.n1 * v[1];
        if (D == 3) idx += L.n1 * L.n1 * v[D - 1];
        return idx;
    }
    uint32_t h = v[0] ^ (v[1] * kPrime1);
    if (D == 3) h ^= v[D - 1] * kPrime2;
    return h & L.mask;
}

template <int D>
__device__ __forceinline__ float corner_weight(const float *f, int corner) {
    float w = 1.f;
#pragma unroll
    for (int i = 0; i < D; ++i) w *= ((corner >> i) & 1) ? f[i] : (1.f - f[i]);
    return w;
}

}  // namespace pfk
