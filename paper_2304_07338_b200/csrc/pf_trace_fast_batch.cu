// pf_trace_fast_batch.cu -- FAST-mode batch entries (macro-cell DDA, binary32):
// pf_delta_track_batch(fp64 = 0) and pf_transmittance_ratio_batch, exposed for
// the statistical tests against the parity kernels.
//
// Own translation unit, compiled with ptxas -O1 (paper_2304_07338_b200/build.py):
// at -O3, ptxas 12.9 miscompiled k_delta_track_batch_dda so that ~0.5% of the
// flights walked the majorant grid with a macro-cell index that disagreed with
// their (bounds-checked) cell coordinates -- out-of-bounds majorant reads,
// results that depended on where the allocator placed the buffers (55936 vs
// 55941 hits for the same rays), and an illegal-address fault once the
// process had allocated enough memory (cuda-gdb: LDG of maj[-31830] with cell
// coordinates (5, 0, 6) in an 8^3 grid).  At -O1 the result is the same for
// every placement and matches the C++ semantics (56883 hits, tools/probe_fast_batch.py;
// PARITY on the same rays: 56804).  The render tracer's frames are unaffected
// (byte-identical across placements, tools/frame_hash.py <mode> <GB>).  The
// walk here also bounds-checks the linear index (dda_advance<true>).
#define PF_TU_FAST
#include "pf_trace.cuh"
#include "pf_dda.cuh"

namespace pfk {

// FAST-mode batch entries (DDA majorants): what the render tracer does per
// flight, exposed for statistical tests against the parity kernels.
__global__ void k_delta_track_batch_dda(const DevScene S, BatchParams B) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    float o[3], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        o[a] = (float)B.a3[3 * i + a];
        d[a] = (float)B.b3[3 * i + a];
    }
    float t, t1;
    B.hit[i] = 0;
    if (B.scalar) B.scalar[i] = 0.0;
    if (!aabb_unit<float>(o, d, (float)B.tmin[i], (float)B.tmax[i], t, t1) || !(S.sigma_max_f > 0.f) ||
        !occ_clip(S, o, d, t, t1))
        return;
    Dda D;
    dda_init(S, o, d, t, D);
    float tau = sample_tau(rng), m;
    while (dda_advance<true>(S, D, t, t1, tau, m)) {
        float x[3] = {fmaf(d[0], t, o[0]), fmaf(d[1], t, o[1]), fmaf(d[2], t, o[2])};
        const float s = sample_f(S, x);
        if (pcg_u_f(rng) * m < S.density_scale_f * tf_alpha_f(S, s)) {
            B.hit[i] = 1;
            if (B.pos3)
                for (int a = 0; a < 3; ++a) B.pos3[3 * i + a] = (double)x[a];
            if (B.scalar) B.scalar[i] = (double)s;
            if (B.rgba4) {
                float c[4];
                tf_rgba_f(S, s, c);
                for (int a = 0; a < 4; ++a) B.rgba4[4 * i + a] = (double)c[a];
            }
            return;
        }
        tau = sample_tau(rng);
    }
}

__global__ void k_transmittance_ratio_dda(const DevScene S, BatchParams B) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    float a[3], dv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = (float)B.a3[3 * i + k];
        dv[k] = (float)B.b3[3 * i + k] - a[k];
    }
    const float len = sqrtf(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
    float dir[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    float t0, t1;
    if (len == 0.0f || !aabb_unit<float>(a, dir, 0.0f, len, t0, t1) || !(S.sigma_max_f > 0.0f) ||
        !occ_clip(S, a, dir, t0, t1)) {
        B.out[i] = 1.0;
        return;
    }
    double acc = 0.0;
    for (int trial = 0; trial < B.n_trials; ++trial) {
        float t = t0, T = 1.0f, m;
        Dda D;
        dda_init(S, a, dir, t, D);
        float tau = sample_tau(rng);
        while (dda_advance<true>(S, D, t, t1, tau, m)) {
            float x[3] = {fmaf(dir[0], t, a[0]), fmaf(dir[1], t, a[1]), fmaf(dir[2], t, a[2])};
            T *= 1.0f - S.density_scale_f * tf_alpha_f(S, sample_f(S, x)) / m;
            if (T < 0.1f) {
                if (pcg_u_f(rng) >= T * 10.0f) {
                    T = 0.0f;
                    break;
                }
                T = 0.1f;
            }
            tau = sample_tau(rng);
        }
        acc += (double)T;
    }
    B.out[i] = acc / B.n_trials;
}

cudaError_t launch_delta_track_batch_fast(const DevScene &S, const BatchParams &B, cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_delta_track_batch_dda<<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

cudaError_t launch_transmittance_ratio_batch(const DevScene &S, const BatchParams &B, cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_transmittance_ratio_dda<<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

}  // namespace pfk
