// pf_dda.cuh -- FAST-mode macro-cell majorant walk shared by the render
// tracer (pf_trace_fast.cu) and the path tracer (pf_pathtrace.cuh).
//
// A flight samples an optical depth tau = -log(1-u) and walks the macro grid
// (PF_MACRO^3-voxel cells) with a 3-D DDA, spending tau at rate maj[cell];
// empty cells cost a few ALU ops and no texture fetch.  Delta / ratio
// tracking against any majorant >= sigma stays unbiased.
#pragma once

#include "pf_device.cuh"

namespace pfk {

// DDA state in named scalars (no dynamic indexing -> stays in registers).
struct Dda {
    int cell;                  // linear macro-cell index
    int cx, cy, cz;            // macro cell coordinates
    int sx, sy, sz;            // +1 / -1 / 0
    float tmx, tmy, tmz;       // ray parameter of the next boundary crossing per axis
    float tdx, tdy, tdz;       // parameter increment per cell per axis
};

__device__ __forceinline__ void dda_axis(float o, float d, float t, float minv_h, float mh, int mc, int &c, int &st,
                                         float &tm, float &td) {
    const float p = fmaf(d, t, o);
    c = min(max((int)floorf(p * minv_h), 0), mc - 1);
    const float inv = 1.0f / d;  // +-inf for axis-parallel rays
    if (d > 0.0f) {
        st = 1;
        tm = ((float)(c + 1) * mh - o) * inv;
        td = mh * inv;
    } else if (d < 0.0f) {
        st = -1;
        tm = ((float)c * mh - o) * inv;
        td = -mh * inv;
    } else {
        st = 0;
        tm = __int_as_float(0x7f800000);
        td = __int_as_float(0x7f800000);
    }
}

__device__ __forceinline__ void dda_init(const DevScene &S, const float o[3], const float d[3], float t, Dda &D) {
    dda_axis(o[0], d[0], t, S.minv_h[0], S.mh[0], S.mc[0], D.cx, D.sx, D.tmx, D.tdx);
    dda_axis(o[1], d[1], t, S.minv_h[1], S.mh[1], S.mc[1], D.cy, D.sy, D.tmy, D.tdy);
    dda_axis(o[2], d[2], t, S.minv_h[2], S.mh[2], S.mc[2], D.cz, D.sz, D.tmz, D.tdz);
    D.cell = D.cx + S.mc[0] * (D.cy + S.mc[1] * D.cz);
}

// Spend optical depth tau through the majorant grid from t.  Returns true at a
// tentative collision (t updated, m = that cell's majorant); false when the
// flight reaches t1 first.
// kGuard: also stop the flight if the linear cell index ever leaves the grid
// (the batch entries; see pf_trace_fast_batch.cu).
template <bool kGuard = false>
__device__ __forceinline__ bool dda_advance(const DevScene &S, Dda &D, float &t, float t1, float &tau, float &m) {
    const int stride_y = S.mc[0], stride_z = S.mc[0] * S.mc[1];
    for (;;) {
        if (kGuard && (unsigned)D.cell >= (unsigned)(stride_z * S.mc[2])) return false;
        m = __ldg(S.maj + D.cell);
        const float tn = fminf(D.tmx, fminf(D.tmy, D.tmz));
        const float t_exit = fminf(tn, t1);
        const float od = m * (t_exit - t);
        if (od >= tau && m > 0.0f) {
            t += tau / m;
            return true;
        }
        tau -= od;
        t = t_exit;
        if (t_exit >= t1) return false;
        if (D.tmx == tn) {
            D.cx += D.sx;
            if ((unsigned)D.cx >= (unsigned)S.mc[0]) return false;
            D.cell += D.sx;
            D.tmx += D.tdx;
        } else if (D.tmy == tn) {
            D.cy += D.sy;
            if ((unsigned)D.cy >= (unsigned)S.mc[1]) return false;
            D.cell += D.sy * stride_y;
            D.tmy += D.tdy;
        } else {
            D.cz += D.sz;
            if ((unsigned)D.cz >= (unsigned)S.mc[2]) return false;
            D.cell += D.sz * stride_z;
            D.tmz += D.tdz;
        }
    }
}

// Clip a flight [t0, t1] to the occupied-cell box (slightly expanded so
// rounding can never cut off an occupied cell).  False: the flight only
// crosses empty cells (sigma = 0), i.e. it passes unattenuated.
__device__ __forceinline__ bool occ_clip(const DevScene &S, const float o[3], const float d[3], float &t0, float &t1) {
    const int lo_x = __ldg(S.occ), hi_x = __ldg(S.occ + 3);
    if (hi_x < lo_x) return false;  // no occupied cell at all
    const int lo_c[3] = {lo_x, __ldg(S.occ + 1), __ldg(S.occ + 2)};
    const int hi_c[3] = {hi_x, __ldg(S.occ + 4), __ldg(S.occ + 5)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float lo = (float)lo_c[a] * S.mh[a] - 1e-4f, hi = (float)(hi_c[a] + 1) * S.mh[a] + 1e-4f;
        const float inv = 1.0f / d[a];
        float tn = (lo - o[a]) * inv, tf = (hi - o[a]) * inv;
        if (inv < 0.0f) {
            const float x = tn;
            tn = tf;
            tf = x;
        }
        t0 = fmaxf(t0, tn);
        t1 = fminf(t1, tf);
    }
    return t0 <= t1;
}

__device__ __forceinline__ float sample_tau(Pcg &r) { return -__logf(pcg_one_minus_u_f(r)); }

}  // namespace pfk
