// pf_trace_fast.cu -- FAST-mode render tracer (binary32); the batch entries
// are in pf_trace_fast_batch.cu.
//
// Same persistent lane state machine and the same per-sample RNG streams as
// the parity tracer (pf_trace.cuh), but the majorant is piecewise constant
// over PF_MACRO^3-voxel macro cells instead of the reference's single global
// sigma_max (volume.cpp:197-202):
//   * a flight samples an optical depth tau = -log(1-u) and walks the macro
//     grid with a 3-D DDA, spending tau at rate maj[cell] -- empty cells cost
//     a few ALU ops and no texture fetch;
//   * at a tentative collision in cell c the primary ray accepts with
//     probability sigma(x) / maj[c] (delta tracking), a shadow ray multiplies
//     its transmittance by 1 - sigma(x) / maj[c] (ratio tracking, north_star)
//     with Russian roulette below 0.1.
// Both estimators stay unbiased for any majorant >= sigma, so the FAST frame
// converges to the PARITY frame (statistical parity, tests/test_gpu_render.py);
// the RNG stream of a sample is consumed differently, so single samples differ.
#define PF_TU_FAST
#include "pf_trace.cuh"
#include "pf_dda.cuh"

namespace pfk {

// nee_term with omega_out / L_d in the caller's shared-memory columns
__device__ __forceinline__ void nee_smem(const DevScene &S, int l, const float x[3], float g, float T,
                                         float (*s_wo)[PF_TRACE_THREADS], float (*s_ld)[PF_TRACE_THREADS], int tx) {
    const float wo[3] = {s_wo[0][tx], s_wo[1][tx], s_wo[2][tx]};
    float Ld[3] = {s_ld[0][tx], s_ld[1][tx], s_ld[2][tx]};
    nee_term<float>(S, l, x, wo, g, T, Ld);
#pragma unroll
    for (int c = 0; c < 3; ++c) s_ld[c][tx] = Ld[c];
}

__global__ void __launch_bounds__(PF_TRACE_THREADS, 8) k_render_trace_fast(const DevScene S, const TraceParams P) {
    float *slots = reinterpret_cast<float *>(P.slots);
    const float ds = S.density_scale_f;
    const float g = (float)P.g;

    int phase = 0;  // 0 fetch, 1 primary flight, 2 shadow flight
    uint32_t w = 0;
    uint64_t index = 0;
    Pcg rng;
    float o[3], d[3], t = 0.f, t1 = 0.f, tau = 0.f, T = 1.f;
    float sig_s = 0.f;  // sigma_s at the interaction (only the hit record needs it)
    // per-thread Ld / wo live in shared memory (column per thread, conflict-
    // free): they are touched once per NEE term, not per tracking step, and
    // the registers go to the flight state
    __shared__ float s_ld[3][PF_TRACE_THREADS], s_wo[3][PF_TRACE_THREADS];
    const int tx = threadIdx.x;
    Dda D;
    int light = 0;
    uint32_t nprim = 0, nshad = 0;

    for (;;) {
        if (phase == 0) {
            w = (uint32_t)warp_fetch_add(&P.counters[0], 1u);
            if (w >= P.n_work) break;
            int px, py;
            if (!decode_work(P, w, px, py, index)) continue;
            pcg_init(rng, P.init_cam, index);
            const float u = (float)pcg_double(rng);
            const float v = (float)pcg_double(rng);
            const float sx = (2.0f * ((float)px + u)) / (float)P.W - 1.0f;
            const float sy = 1.0f - (2.0f * ((float)py + v)) / (float)P.H;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = (float)P.cam_o[a];
                d[a] = ((float)P.cam_f[a] + (float)P.cam_r[a] * sx) + (float)P.cam_u[a] * sy;
            }
            const float rl = rsqrtf(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                d[a] *= rl;
                s_wo[a][tx] = -d[a];
            }
            float t0;
            if (!aabb_unit<float>(o, d, 0.0f, __int_as_float(0x7f800000), t0, t1) || !(S.sigma_max_f > 0.0f) ||
                !occ_clip(S, o, d, t0, t1)) {
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (float)P.bg[c];
                continue;
            }
            t = t0;
            dda_init(S, o, d, t, D);
            tau = sample_tau(rng);
            phase = 1;
        }

        // ---- advance to the next tentative collision (majorant DDA)
        float m;
        const bool coll = dda_advance(S, D, t, t1, tau, m);
        if (phase == 1) ++nprim;
        else ++nshad;

        bool flight_done = false;
        if (!coll) {
            if (phase == 1) {
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (float)P.bg[c];
                phase = 0;
                continue;
            }
            flight_done = true;
        } else {
            float x[3] = {fmaf(d[0], t, o[0]), fmaf(d[1], t, o[1]), fmaf(d[2], t, o[2])};
            const float scalar = sample_f(S, x);
            const float sigma = ds * tf_alpha_f(S, scalar);
            if (phase == 1) {
                if (pcg_u_f(rng) * m < sigma) {
                    {
                        float rgba[4];
                        tf_rgba_f(S, scalar, rgba);
                        sig_s = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) * (1.0f / 3.0f));
                    }
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        o[a] = x[a];
                        s_ld[a][tx] = 0.f;
                    }
                    pcg_init(rng, P.init_nee, index);
                    light = -1;
                    flight_done = true;
                    T = 1.f;
                    phase = 2;
                } else {
                    tau = sample_tau(rng);
                }
            } else {
                T *= 1.0f - sigma / m;
                if (T < 0.1f) {
                    if (pcg_u_f(rng) >= T * 10.0f) {
                        T = 0.f;
                        flight_done = true;
                    } else {
                        T = 0.1f;
                    }
                }
                if (!flight_done) tau = sample_tau(rng);
            }
        }
        if (!flight_done) continue;

        if (light >= 0) nee_smem(S, light, o, g, T, s_wo, s_ld, tx);
        for (;;) {
            ++light;
            if (light >= S.n_lights) break;
            float dv[3] = {(float)S.light_p[light][0] - o[0], (float)S.light_p[light][1] - o[1],
                           (float)S.light_p[light][2] - o[2]};
            const float len = sqrtf(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            if (len > 0.0f) {
#pragma unroll
                for (int a = 0; a < 3; ++a) d[a] = dv[a] / len;
                float a0, a1;
                if (aabb_unit<float>(o, d, 0.0f, len, a0, a1) && S.sigma_max_f > 0.0f && occ_clip(S, o, d, a0, a1)) {
                    t = a0;
                    t1 = a1;
                    T = 1.f;
                    dda_init(S, o, d, t, D);
                    tau = sample_tau(rng);
                    break;
                }
            }
            nee_smem(S, light, o, g, 1.0f, s_wo, s_ld, tx);
        }
        if (light < S.n_lights) continue;

        const size_t sb = 3 * (size_t)w;
#pragma unroll
        for (int c = 0; c < 3; ++c) slots[sb + c] = (float)P.w_d * s_ld[c][tx];
        const unsigned long long h = warp_fetch_add(&P.counters[1], 1u);
        if (P.use_field) {
            HitRec rec;
            rec.x[0] = o[0];
            rec.x[1] = o[1];
            rec.x[2] = o[2];
            const float wz = fminf(fmaxf(s_wo[2][tx], -1.0f), 1.0f);
            rec.wsph[0] = acosf(wz) * (float)(1.0 / kPi);
            rec.wsph[1] = (atan2f(s_wo[1][tx], s_wo[0][tx]) + (float)kPi) * (float)(0.5 / kPi);
            rec.slot = w;
            rec.sigma_s = (double)sig_s;
            P.hits[h] = rec;
            if (P.hit_dir) {
#pragma unroll
                for (int a = 0; a < 3; ++a) P.hit_dir[3 * h + a] = (double)s_wo[a][tx];
            }
        }
        phase = 0;
    }
    atomicAdd(&P.counters[2], (unsigned long long)nprim);
    atomicAdd(&P.counters[3], (unsigned long long)nshad);
    atomicAdd(&P.counters[4], (unsigned long long)(nprim + nshad));  // every tentative collision fetches
}

cudaError_t launch_render_trace_fast(const DevScene &S, const TraceParams &P, int grid, cudaStream_t st) {
    k_render_trace_fast<<<grid, PF_TRACE_THREADS, 0, st>>>(S, P);
    return cudaGetLastError();
}

int trace_grid_size_fast(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_trace_fast, PF_TRACE_THREADS, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace pfk
