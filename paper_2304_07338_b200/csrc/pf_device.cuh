// pf_device.cuh -- device primitives shared by the sm_100a kernels.
//
// Every binary64 routine here restates the reference operation-for-operation
// (the parity translation units are compiled with --fmad=false so nvcc never
// contracts a*b+c into an FMA the x86 reference does not perform):
//   PCG32 / make_rng ........ proj/include/pf/rng.hpp:14-76
//   Aabb::intersect ......... proj/include/pf/math.hpp:95-108
//   VolumeGrid::sample ...... proj/src/volume.cpp:41-77
//   TransferFunction::classify proj/src/volume.cpp:151-161
//   hg_eval ................. proj/include/pf/phase.hpp:18-23
// The binary32 variants are the FAST mode (statistical parity only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define PF_MAX_TF 16
#define PF_MAX_LIGHTS 8

namespace pfk {

constexpr double kPi = 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);

// ---------------------------------------------------------------- scene --
// Passed by value as a kernel parameter (lives in the constant bank).
struct DevScene {
    // Volume "slice atlas": a 2-D binary32 texture holding every z-slice as an
    // (nx+1) x (ny+1) tile (last row/column duplicated), 2^atlas_log2 tiles per
    // atlas row.  One tex2Dgather returns the exact 2x2 footprint a trilinear
    // sample needs in one slice, so a tracking step issues 2 texture
    // instructions instead of 8 point fetches -- values are the stored floats,
    // so results stay bit-identical to the reference's voxel() reads.
    cudaTextureObject_t atlas;
    int atlas_log2;
    int nx, ny, nz;
    int n_tf;
    int n_lights;
    double density_scale, sigma_max, inv_sigma_max;
    double sm53;  // sigma_max * 2^-53 (exact): next_double() * sigma_max in one multiply
    float density_scale_f, sigma_max_f, inv_sigma_max_f;
    double tf_s[PF_MAX_TF];
    double tf_c[PF_MAX_TF][4];
    float tf_sf[PF_MAX_TF];
    float tf_cf[PF_MAX_TF][4];
    double light_p[PF_MAX_LIGHTS][3];
    double light_i[PF_MAX_LIGHTS][3];
    // FAST mode only: macro-cell majorants (PF_MACRO voxels per cell edge).
    // maj[c] >= density_scale * alpha(s) for every trilinear sample inside
    // cell c (built from the min/max of the cell's voxel support + the TF's
    // max_alpha, volume.cpp:163-168), so delta / ratio tracking against it is
    // unbiased; empty cells are skipped without a texture fetch.
    const float *maj;
    // FAST mode: bounding box of the macro cells with a nonzero majorant
    // (min cell x,y,z, max cell x,y,z; max < min when the medium is empty).
    // sigma(x) = 0 outside it, so flights are clipped to it exactly.
    const int *occ;
    int mc[3];
    float mh[3], minv_h[3];
    // PARITY mode: the same majorants as a point-sampled 3-D texture of the
    // high 32 bits of each bound as a binary64, rounded up (so
    // as_double(hi, 0) >= maj).  For u2*sigma_max >= 0 the certain-null test
    // u2*sigma_max >= bound is then one integer compare of high words, and
    // the hardware does the cell lookup (floor + clamp) from float
    // coordinates x * minv_h (pf_parstep.cuh).
    cudaTextureObject_t maj_tex;
};

// ------------------------------------------------------------------ rng --
struct Pcg {
    uint64_t state, inc;
};

// Pcg32::next_u32 (rng.hpp:27-33): XSH-RR output of the pre-advance state.
__device__ __forceinline__ uint32_t pcg_u32(Pcg &r) {
    uint64_t old = r.state;
    r.state = old * 6364136223846793005ULL + r.inc;
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return __funnelshift_r(xs, xs, rot);
}

// make_rng(seed, stream, index) with initstate = splitmix64(seed ^ stream*phi)
// precomputed on the host (rng.hpp:73-76); Pcg32::seed (rng.hpp:19-25).
__device__ __forceinline__ void pcg_init(Pcg &r, uint64_t initstate, uint64_t index) {
    r.state = 0ull;
    r.inc = (index << 1) | 1ull;
    pcg_u32(r);
    r.state += initstate;
    pcg_u32(r);
}

// next_u64: high word first (rng.hpp:35-38).
__device__ __forceinline__ uint64_t pcg_u64(Pcg &r) {
    uint64_t hi = pcg_u32(r);
    uint64_t lo = pcg_u32(r);
    return (hi << 32) | lo;
}

// next_double (rng.hpp:41): exact 53-bit uniform in [0,1).
__device__ __forceinline__ double pcg_double(Pcg &r) {
    return (double)(pcg_u64(r) >> 11) * 0x1.0p-53;
}

// FAST mode uniforms: still 2 x u32 per uniform so stream positions match.
// 1-u derived from the integer bits -> (0, 1].
__device__ __forceinline__ float pcg_one_minus_u_f(Pcg &r) {
    uint64_t k = pcg_u64(r) >> 11;
    return (float)((1ull << 53) - k) * 0x1.0p-53f;
}
__device__ __forceinline__ float pcg_u_f(Pcg &r) {
    return (float)(uint32_t)(pcg_u64(r) >> 40) * 0x1.0p-24f;
}

// --------------------------------------------------------------- math ----
// std::max / std::min argument order (NaN in the 2nd operand ignored).
__device__ __forceinline__ double stdmax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double stdmin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ float stdmaxf(float a, float b) { return (a < b) ? b : a; }
__device__ __forceinline__ float stdminf(float a, float b) { return (b < a) ? b : a; }

// Aabb::intersect against the unit cube (math.hpp:95-108).
template <typename R>
__device__ __forceinline__ bool aabb_unit(const R o[3], const R d[3], R tmin, R tmax, R &t0, R &t1) {
    t0 = tmin;
    t1 = tmax;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        R inv = R(1) / d[a];
        R tn = (R(0) - o[a]) * inv;
        R tf = (R(1) - o[a]) * inv;
        if (inv < R(0)) {
            R s = tn;
            tn = tf;
            tf = s;
        }
        t0 = (t0 < tn) ? tn : t0;
        t1 = (tf < t1) ? tf : t1;
        if (t0 > t1) return false;
    }
    return true;
}

// hg_eval (phase.hpp:18-23).
__device__ __forceinline__ double hg_eval_d(double g, double c) {
    g = g < -0.999 ? -0.999 : (g > 0.999 ? 0.999 : g);
    double denom = 1.0 + g * g - 2.0 * g * c;
    denom = denom < 1e-12 ? 1e-12 : denom;
    return kInv4Pi * (1.0 - g * g) / (denom * sqrt(denom));
}
__device__ __forceinline__ float hg_eval_f(float g, float c) {
    g = fminf(fmaxf(g, -0.999f), 0.999f);
    float denom = fmaxf(1.0f + g * g - 2.0f * g * c, 1e-12f);
    return (float)kInv4Pi * (1.0f - g * g) * rsqrtf(denom) / denom;
}

// ------------------------------------------------------------- volume ----
// 2x2 footprint {(ix,iy), (ix+1,iy), (ix,iy+1), (ix+1,iy+1)} of slice iz
// (gather component order: w=(0,0) z=(1,0) x=(0,1) y=(1,1)).
struct Quad {
    float c00, c10, c01, c11;
};
__device__ __forceinline__ Quad quad(const DevScene &S, int ix, int iy, int iz) {
    const int mask = (1 << S.atlas_log2) - 1;
    const float u = (float)((iz & mask) * (S.nx + 1) + ix) + 1.0f;
    const float v = (float)((iz >> S.atlas_log2) * (S.ny + 1) + iy) + 1.0f;
    const float4 g = tex2Dgather<float4>(S.atlas, u, v, 0);
    return Quad{g.w, g.z, g.x, g.y};
}

// Cell-centred axis split with boundary clamp (volume.cpp:44-57).
__device__ __forceinline__ void axis_d(double x, int n, int &i0, double &f) {
    double c = x * (double)n - 0.5;
    double lo = floor(c);
    int i = (int)lo;
    double fr = c - lo;
    if (i < 0) {
        i = 0;
        fr = 0.0;
    } else if (i >= n - 1) {
        i = n - 1;
        fr = 0.0;
    }
    i0 = i;
    f = fr;
}

// VolumeGrid::sample in binary64: lerp x, then y, then z (volume.cpp:41-77).
__device__ __forceinline__ double sample_d(const DevScene &S, const double p[3]) {
    int ix, iy, iz;
    double fx, fy, fz;
    axis_d(p[0], S.nx, ix, fx);
    axis_d(p[1], S.ny, iy, fy);
    axis_d(p[2], S.nz, iz, fz);
    const int jz = min(iz + 1, S.nz - 1);
    const Quad q0 = quad(S, ix, iy, iz), q1 = quad(S, ix, iy, jz);
    // jx/jy = min(i+1, n-1) come from the duplicated tile edge
    double c000 = q0.c00, c100 = q0.c10, c010 = q0.c01, c110 = q0.c11;
    double c001 = q1.c00, c101 = q1.c10, c011 = q1.c01, c111 = q1.c11;
    double c00 = c000 * (1.0 - fx) + c100 * fx;
    double c10 = c010 * (1.0 - fx) + c110 * fx;
    double c01 = c001 * (1.0 - fx) + c101 * fx;
    double c11 = c011 * (1.0 - fx) + c111 * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

__device__ __forceinline__ void axis_f(float x, int n, int &i0, float &f) {
    float c = x * (float)n - 0.5f;
    float lo = floorf(c);
    int i = (int)lo;
    float fr = c - lo;
    if (i < 0) {
        i = 0;
        fr = 0.0f;
    } else if (i >= n - 1) {
        i = n - 1;
        fr = 0.0f;
    }
    i0 = i;
    f = fr;
}

__device__ __forceinline__ float sample_f(const DevScene &S, const float p[3]) {
    int ix, iy, iz;
    float fx, fy, fz;
    axis_f(p[0], S.nx, ix, fx);
    axis_f(p[1], S.ny, iy, fy);
    axis_f(p[2], S.nz, iz, fz);
    const int jz = min(iz + 1, S.nz - 1);
    const Quad q0 = quad(S, ix, iy, iz), q1 = quad(S, ix, iy, jz);
    const float c000 = q0.c00, c100 = q0.c10, c010 = q0.c01, c110 = q0.c11;
    const float c001 = q1.c00, c101 = q1.c10, c011 = q1.c01, c111 = q1.c11;
    float c00 = c000 + (c100 - c000) * fx;
    float c10 = c010 + (c110 - c010) * fx;
    float c01 = c001 + (c101 - c001) * fx;
    float c11 = c011 + (c111 - c011) * fx;
    float c0 = c00 + (c10 - c00) * fy;
    float c1 = c01 + (c11 - c01) * fy;
    return c0 + (c1 - c0) * fz;
}

// TransferFunction::classify segment search + clamped lerp (volume.cpp:151-161).
__device__ __forceinline__ int tf_segment_d(const DevScene &S, double s) {
    int hi = 1;
    while (hi + 1 < S.n_tf && S.tf_s[hi] < s) ++hi;
    return hi;
}
__device__ __forceinline__ double tf_t_d(const DevScene &S, int hi, double s) {
    double t = (s - S.tf_s[hi - 1]) / (S.tf_s[hi] - S.tf_s[hi - 1]);
    return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}
__device__ __forceinline__ double clamp01_d(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

// alpha channel of classify(s) (the only channel a tracking step needs).
__device__ __forceinline__ double tf_alpha_d(const DevScene &S, double scalar) {
    double s = clamp01_d(scalar);
    int hi = tf_segment_d(S, s);
    double t = tf_t_d(S, hi, s);
    double a = S.tf_c[hi - 1][3], b = S.tf_c[hi][3];
    return a + (b - a) * t;
}
__device__ __forceinline__ void tf_rgba_d(const DevScene &S, double scalar, double rgba[4]) {
    double s = clamp01_d(scalar);
    int hi = tf_segment_d(S, s);
    double t = tf_t_d(S, hi, s);
#pragma unroll
    for (int c = 0; c < 4; ++c) rgba[c] = S.tf_c[hi - 1][c] + (S.tf_c[hi][c] - S.tf_c[hi - 1][c]) * t;
}

__device__ __forceinline__ int tf_segment_f(const DevScene &S, float s) {
    int hi = 1;
    while (hi + 1 < S.n_tf && S.tf_sf[hi] < s) ++hi;
    return hi;
}
__device__ __forceinline__ float tf_alpha_f(const DevScene &S, float scalar) {
    float s = __saturatef(scalar);
    int hi = tf_segment_f(S, s);
    float t = __saturatef((s - S.tf_sf[hi - 1]) / (S.tf_sf[hi] - S.tf_sf[hi - 1]));
    float a = S.tf_cf[hi - 1][3], b = S.tf_cf[hi][3];
    return a + (b - a) * t;
}
__device__ __forceinline__ void tf_rgba_f(const DevScene &S, float scalar, float rgba[4]) {
    float s = __saturatef(scalar);
    int hi = tf_segment_f(S, s);
    float t = __saturatef((s - S.tf_sf[hi - 1]) / (S.tf_sf[hi] - S.tf_sf[hi - 1]));
#pragma unroll
    for (int c = 0; c < 4; ++c) rgba[c] = S.tf_cf[hi - 1][c] + (S.tf_cf[hi][c] - S.tf_cf[hi - 1][c]) * t;
}

// ------------------------------------------------------- warp helpers ----
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Warp-aggregated atomicAdd on a global counter: one atomic per converged
// group of lanes, each lane receives a distinct value.
__device__ __forceinline__ unsigned long long warp_fetch_add(unsigned long long *ctr, unsigned inc) {
    unsigned m = __activemask();
    int leader = __ffs(m) - 1;
    unsigned lane = threadIdx.x & 31u;
    unsigned total = __popc(m) * inc;
    unsigned long long base = 0;
    if (lane == (unsigned)leader) base = atomicAdd(ctr, (unsigned long long)total);
    base = __shfl_sync(m, base, leader);
    return base + (unsigned long long)__popc(m & lanemask_lt()) * inc;
}

}  // namespace pfk
