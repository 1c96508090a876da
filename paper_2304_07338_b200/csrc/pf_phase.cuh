// pf_phase.cuh -- direction sampling shared by the photon tracer (Alg. 1) and
// the reference path tracer.
//
// binary64 routines restate the reference operation-for-operation (their
// translation units are compiled --fmad=false):
//   sample_uniform_sphere ... proj/include/pf/rng.hpp:78-83
//   orthonormal_basis + from_local_frame  proj/include/pf/math.hpp:113-126
//   hg_sample_cos / hg_sample  proj/include/pf/phase.hpp:26-40
// The binary32 variants serve FAST mode (statistical parity only); they
// consume the stream exactly like the binary64 ones (2 x u32 per uniform).
#pragma once

#include "pf_device.cuh"

namespace pfk {

constexpr double kTwoPiD = 6.283185307179586476925286766559;

// sample_uniform_sphere (rng.hpp:78-83).
__device__ __forceinline__ void uniform_sphere(Pcg &r, double out[3]) {
    const double z = 1.0 - 2.0 * pcg_double(r);
    const double phi = kTwoPiD * pcg_double(r);
    const double rr = sqrt(stdmax(0.0, 1.0 - z * z));
    out[0] = rr * cos(phi);
    out[1] = rr * sin(phi);
    out[2] = z;
}

// orthonormal_basis (Duff et al.) + from_local_frame (math.hpp:113-126).
__device__ __forceinline__ void from_local(const double n[3], const double l[3], double out[3]) {
    const double sign = copysign(1.0, n[2]);
    const double a = -1.0 / (sign + n[2]);
    const double c = n[0] * n[1] * a;
    const double t[3] = {1.0 + sign * n[0] * n[0] * a, sign * c, -sign * n[0]};
    const double b[3] = {c, sign + n[1] * n[1] * a, -n[1]};
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = t[k] * l[0] + b[k] * l[1] + n[k] * l[2];
}

// hg_sample_cos (phase.hpp:26-31).
__device__ __forceinline__ double hg_cos(double g, double u) {
    g = g < -0.999 ? -0.999 : (g > 0.999 ? 0.999 : g);
    if (fabs(g) < 1e-6) return 1.0 - 2.0 * u;
    const double sq = (1.0 - g * g) / (1.0 - g + 2.0 * g * u);
    const double c = (1.0 + g * g - sq * sq) / (2.0 * g);
    return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}

// cos/sin of the azimuth and the cone/lobe frame (phase.hpp:34-40).
__device__ __forceinline__ void frame_dir(const double axis[3], double ct, double u2, double out[3]) {
    const double st = sqrt(stdmax(0.0, 1.0 - ct * ct));
    const double phi = kTwoPiD * u2;
    const double local[3] = {st * cos(phi), st * sin(phi), ct};
    from_local(axis, local, out);
}

// hg_sample(g, w, rng) (phase.hpp:42-46): u1 then u2 from the stream.
__device__ __forceinline__ void hg_sample(double g, const double w[3], Pcg &r, double out[3]) {
    const double u1 = pcg_double(r);
    const double u2 = pcg_double(r);
    frame_dir(w, hg_cos(g, u1), u2, out);
}

// ---- binary32 (FAST mode) ----------------------------------------------
__device__ __forceinline__ void from_local(const float n[3], const float l[3], float out[3]) {
    const float sign = copysignf(1.0f, n[2]);
    const float a = -1.0f / (sign + n[2]);
    const float c = n[0] * n[1] * a;
    const float t[3] = {1.0f + sign * n[0] * n[0] * a, sign * c, -sign * n[0]};
    const float b[3] = {c, sign + n[1] * n[1] * a, -n[1]};
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] = t[k] * l[0] + b[k] * l[1] + n[k] * l[2];
}

__device__ __forceinline__ float hg_cos(float g, float u) {
    g = fminf(fmaxf(g, -0.999f), 0.999f);
    if (fabsf(g) < 1e-6f) return 1.0f - 2.0f * u;
    const float sq = (1.0f - g * g) / (1.0f - g + 2.0f * g * u);
    const float c = (1.0f + g * g - sq * sq) / (2.0f * g);
    return fminf(fmaxf(c, -1.0f), 1.0f);
}

__device__ __forceinline__ void hg_sample(float g, const float w[3], Pcg &r, float out[3]) {
    const float u1 = pcg_u_f(r);
    const float u2 = pcg_u_f(r);
    const float ct = hg_cos(g, u1);
    const float st = sqrtf(fmaxf(0.0f, 1.0f - ct * ct));
    float sp, cp;
    sincospif(2.0f * u2, &sp, &cp);
    const float local[3] = {st * cp, st * sp, ct};
    from_local(w, local, out);
    // renormalise: the binary32 frame drifts by a few ulp per bounce
    const float rl = rsqrtf(out[0] * out[0] + out[1] * out[1] + out[2] * out[2]);
#pragma unroll
    for (int k = 0; k < 3; ++k) out[k] *= rl;
}

}  // namespace pfk
