// pf_parstep.cuh -- the binary64 tentative-collision step of the reference's
// delta tracking loop (proj/src/volume.cpp:216-224 / 245-253), shared by every
// PARITY kernel (render tracer, path tracer, photon tracer, batch entry points).
//
// Reference step:                        Here:
//   t -= log(1 - next_double()) * inv;     t -= pf_log(1 - u1) * inv       (pf_log.h)
//   if (t > t1) exit;                      same
//   sigma = sigma(ray.at(t));              certain-null test first (below)
//   if (next_double()*sigma_max < sigma)   u2sm = k53 * (sigma_max 2^-53)  (== (k53 2^-53) sigma_max,
//     accept;                                                              exact power-of-2 scale)
// Certain null: if u2sm >= B(cell(x)) >= sigma(x) the reference rejects, so
// sigma(x) is not evaluated (no voxel fetch, no classify, no binary64 x).
// B comes from DevScene::maj_tex: hardware point lookup at float coordinates
// q = qo + qd * (float)(t - tb) with qo = x(tb) * minv_h, qd = d * minv_h.
// The float position error (< 1e-3 voxel) is far inside the one-voxel
// support margin each macro-cell bound already carries (k_macro_minmax), so
// the test never rejects a collision the reference could accept.  Nothing
// here changes the RNG sequence or any decision.
#pragma once

#include "pf_device.cuh"
#include "pf_log.h"

namespace pfk {

// Flight coordinates for the majorant texture, set once per flight segment.
struct ParFlight {
    float qo[3], qd[3];
};

__device__ __forceinline__ void par_flight(const DevScene &S, const double o[3], const double d[3], double tb,
                                           ParFlight &f) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double xb = o[a] + d[a] * tb;
        f.qo[a] = (float)(xb * (double)S.minv_h[a]);
        f.qd[a] = (float)(d[a] * (double)S.minv_h[a]);
    }
}

// log(1 - next_double()) * inv   (volume.cpp:217 / 247).  1 - k 2^-53 is
// exact in binary64, so it equals (2^53 - k) 2^-53 with the integer 2^53 - k
// converted exactly; the 2^-53 is folded into pf_log's exponent (pf_log_scaled)
// -- bit-identical to pf_log(1.0 - pcg_double(r)), two binary64 ops cheaper.
__device__ __forceinline__ double par_step(Pcg &r, double inv) {
    const uint64_t m = (1ull << 53) - (pcg_u64(r) >> 11);
    return pf_log_scaled<false>((double)m, -53) * inv;
}
// the same with pf_log's table read from a shared-memory copy at byte address tab
__device__ __forceinline__ double par_step_smem(Pcg &r, double inv, uint32_t tab) {
    const uint64_t m = (1ull << 53) - (pcg_u64(r) >> 11);
    return pf_log_scaled<true>((double)m, -53, tab) * inv;
}

// next_double() * sigma_max with one multiply: sm53 = sigma_max * 2^-53.
__device__ __forceinline__ double par_u2sm(Pcg &r, double sm53) { return (double)(pcg_u64(r) >> 11) * sm53; }

// Shared-memory home of a lane's ParFlight (column per thread, 24 B):
// {qo0, qo1, qo2, qd0} as one float4 + {qd1, qd2} as one float2, so the step
// reads it with two vector LDS instead of holding six registers.
struct ParFlightSmem {
    float4 *a;
    float2 *b;
};
__device__ __forceinline__ void par_store(const ParFlightSmem &m, int tx, const ParFlight &f) {
    m.a[tx] = make_float4(f.qo[0], f.qo[1], f.qo[2], f.qd[0]);
    m.b[tx] = make_float2(f.qd[1], f.qd[2]);
}
__device__ __forceinline__ ParFlight par_load(const ParFlightSmem &m, int tx) {
    const float4 a = m.a[tx];
    const float2 b = m.b[tx];
    ParFlight f;
    f.qo[0] = a.x, f.qo[1] = a.y, f.qo[2] = a.z, f.qd[0] = a.w, f.qd[1] = b.x, f.qd[2] = b.y;
    return f;
}

// High word of the majorant bound of the cell holding x(t) (one TEX).
__device__ __forceinline__ unsigned par_bound(const DevScene &S, const ParFlight &f, double t, double tb) {
    const float s = (float)(t - tb);
    return tex3DLod<unsigned>(S.maj_tex, fmaf(f.qd[0], s, f.qo[0]), fmaf(f.qd[1], s, f.qo[1]),
                              fmaf(f.qd[2], s, f.qo[2]), 0.0f);
}
// u2sm >= 0: u2sm >= as_double(b, 0)  <=>  hi32(u2sm) >= b
__device__ __forceinline__ bool par_null_given(double u2sm, unsigned b) {
    return (uint32_t)((unsigned long long)__double_as_longlong(u2sm) >> 32) >= b;
}
// true => the reference certainly rejects this tentative collision.
__device__ __forceinline__ bool par_certain_null(const DevScene &S, const ParFlight &f, double t, double tb,
                                                 double u2sm) {
    return par_null_given(u2sm, par_bound(S, f, t, tb));
}

}  // namespace pfk
