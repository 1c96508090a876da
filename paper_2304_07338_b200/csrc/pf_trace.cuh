// pf_trace.cuh -- K1/K2: persistent primary delta tracking + NEE shadow rays.
//
// One template, two translation units:
//   pf_trace_parity.cu (PF_PAR = true,  binary64, --fmad=false) reproduces
//     pf::delta_track / pf::transmittance (proj/src/volume.cpp:204-256)
//     operation-for-operation with the same RNG consumption;
//   pf_trace_fast.cu   (PF_PAR = false, binary32) is the throughput mode:
//     same streams (2 x u32 per uniform), ratio-tracked shadow rays.
//
// Design (B200): a persistent grid (resident CTAs = SM count x occupancy)
// where every lane is a small state machine {fetch sample, primary flight,
// shadow flight}.  A lane whose path terminates immediately pulls the next
// sample with a warp-aggregated atomic (lane regeneration), so the warp keeps
// stepping instead of idling behind its longest path (SIMT divergence).  All
// lanes of a warp execute the same tracking-step code whichever state they
// are in.  Results go to slot[work index] and compacted hit records carry
// their slot, so the output never depends on scheduling order.
#pragma once

#include "pf_device.cuh"
#include "pf_kernels.h"

namespace pfk {

template <bool PAR>
struct Prec;
template <>
struct Prec<true> {
    using R = double;
};
template <>
struct Prec<false> {
    using R = float;
};

__device__ __forceinline__ bool decode_work(const TraceParams &P, uint32_t w, int &px, int &py,
                                            uint64_t &index) {
    const uint32_t tile_px = (uint32_t)(P.tile_w * P.tile_h);
    const uint32_t per_tile = tile_px * (uint32_t)P.spp;
    const uint32_t lt = w / per_tile;
    const uint32_t within = w - lt * per_tile;
    const uint32_t pix = within / (uint32_t)P.spp;
    const uint32_t s = within - pix * (uint32_t)P.spp;
    const uint32_t t = lt * (uint32_t)P.shard_count + (uint32_t)P.shard_index;
    const uint32_t ty = t / (uint32_t)P.tiles_x;
    const uint32_t tx = t - ty * (uint32_t)P.tiles_x;
    const uint32_t ly = pix / (uint32_t)P.tile_w;
    px = (int)(tx * (uint32_t)P.tile_w + (pix - ly * (uint32_t)P.tile_w));
    py = (int)(ty * (uint32_t)P.tile_h + ly);
    if (px >= P.W || py >= P.H) return false;
    index = ((uint64_t)py * (uint64_t)P.W + (uint64_t)px) * (uint64_t)P.spp + s;
    return true;
}

// ----- precision-dispatched primitives ------------------------------------
__device__ __forceinline__ double step_len(Pcg &r, double inv) {
    return log(1.0 - pcg_double(r)) * inv;  // volume.cpp:217 / 247
}
__device__ __forceinline__ float step_len(Pcg &r, float inv) {
    return __logf(pcg_one_minus_u_f(r)) * inv;
}
__device__ __forceinline__ double uniform(Pcg &r, double) { return pcg_double(r); }
__device__ __forceinline__ float uniform(Pcg &r, float) { return pcg_u_f(r); }
__device__ __forceinline__ double sample(const DevScene &S, const double p[3]) { return sample_d(S, p); }
__device__ __forceinline__ float sample(const DevScene &S, const float p[3]) { return sample_f(S, p); }
__device__ __forceinline__ double tf_alpha(const DevScene &S, double s) { return tf_alpha_d(S, s); }
__device__ __forceinline__ float tf_alpha(const DevScene &S, float s) { return tf_alpha_f(S, s); }
__device__ __forceinline__ void tf_rgba(const DevScene &S, double s, double c[4]) { tf_rgba_d(S, s, c); }
__device__ __forceinline__ void tf_rgba(const DevScene &S, float s, float c[4]) { tf_rgba_f(S, s, c); }
__device__ __forceinline__ double density(const DevScene &S, double) { return S.density_scale; }
__device__ __forceinline__ float density(const DevScene &S, float) { return S.density_scale_f; }
__device__ __forceinline__ double majorant(const DevScene &S, double) { return S.sigma_max; }
__device__ __forceinline__ float majorant(const DevScene &S, float) { return S.sigma_max_f; }
__device__ __forceinline__ double inv_majorant(const DevScene &S, double) { return S.inv_sigma_max; }
__device__ __forceinline__ float inv_majorant(const DevScene &S, float) { return S.inv_sigma_max_f; }
__device__ __forceinline__ double rsqrt_len(double v) { return sqrt(v); }
__device__ __forceinline__ float rsqrt_len(float v) { return sqrtf(v); }
__device__ __forceinline__ double rinf(double) { return __longlong_as_double(0x7ff0000000000000ll); }
__device__ __forceinline__ float rinf(float) { return __int_as_float(0x7f800000); }

// Conservative bound on sigma(x) from the macro-cell majorant grid: every
// trilinear sample inside the cell is covered (cell support +-1 voxel), so
// u2 * sigma_max >= bound implies the reference rejects the tentative
// collision (volume.cpp:222-223).  Used to skip the fetch + classify of
// certain null collisions WITHOUT changing the RNG sequence or any decision.
__device__ __forceinline__ double cell_bound(const DevScene &S, const double x[3]) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        // fmax/fmin also map NaN to a valid cell (the bound is then just looser)
        const double p = fmin(fmax(x[a] * (double)S.minv_h[a], 0.0), (double)(S.mc[a] - 1));
        c[a] = (int)p;
    }
    return (double)__ldg(S.maj + c[0] + S.mc[0] * (c[1] + S.mc[1] * c[2]));
}

// One light's NEE term (pinned: oracle/pf_oracle.c or_nee_term).
template <typename R>
__device__ __forceinline__ void nee_term(const DevScene &S, int l, const R x[3], const R wo[3], R g,
                                         R T, R Ld[3]) {
    R dv[3] = {x[0] - (R)S.light_p[l][0], x[1] - (R)S.light_p[l][1], x[2] - (R)S.light_p[l][2]};
    R dist2 = dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2];
    if (!(dist2 > R(0)) || T == R(0)) return;
    R len = rsqrt_len(dist2);
    R din[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    R c = din[0] * wo[0] + din[1] * wo[1] + din[2] * wo[2];
    R hg;
    if constexpr (sizeof(R) == 8) hg = hg_eval_d(g, c);
    else hg = hg_eval_f(g, c);
    R s = (hg * T) / dist2;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) Ld[ch] += s * (R)S.light_i[l][ch];
}

// ---------------------------------------------------------------------------
// The persistent render tracer.
// ---------------------------------------------------------------------------
template <bool PAR>
__global__ void __launch_bounds__(PF_TRACE_THREADS, 7)
    k_render_trace(const DevScene S, const TraceParams P) {
    using R = typename Prec<PAR>::R;
    using Slot = R;
    Slot *slots = reinterpret_cast<Slot *>(P.slots);
    const R inv_sm = inv_majorant(S, R(0));
    const R sm = majorant(S, R(0));
    const R ds = density(S, R(0));
    const R g = (R)P.g;

    int phase = 0;  // 0 fetch, 1 primary flight, 2 shadow flight
    uint32_t w = 0;
    uint64_t index = 0;
    Pcg rng;
    R o[3], d[3], t = 0, t1 = 0, ts0 = 0;
    R sig_s = 0;  // sigma_s at the interaction (only the hit record needs it)
    // omega_out / L_d in shared memory (column per thread): touched per NEE
    // term, not per tracking step
    __shared__ R s_wo[3][PF_TRACE_THREADS], s_ld[3][PF_TRACE_THREADS];
    const int tx = threadIdx.x;
    auto nee = [&](int l, R Tl) {
        const R wo[3] = {s_wo[0][tx], s_wo[1][tx], s_wo[2][tx]};
        R Ld[3] = {s_ld[0][tx], s_ld[1][tx], s_ld[2][tx]};
        nee_term<R>(S, l, o, wo, g, Tl, Ld);
#pragma unroll
        for (int c = 0; c < 3; ++c) s_ld[c][tx] = Ld[c];
    };
    int light = 0, trial = 0, passed = 0;
    R T = 1;
    uint32_t nprim = 0, nshad = 0;

    for (;;) {
        if (phase == 0) {
            w = (uint32_t)warp_fetch_add(&P.counters[0], 1u);
            if (w >= P.n_work) break;
            int px, py;
            if (!decode_work(P, w, px, py, index)) continue;
            pcg_init(rng, P.init_cam, index);
            const double u = pcg_double(rng);
            const double v = pcg_double(rng);
            // pinned camera (oracle or_camera_ray)
            const R sx = (R(2) * ((R)px + (R)u)) / (R)P.W - R(1);
            const R sy = R(1) - (R(2) * ((R)py + (R)v)) / (R)P.H;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = (R)P.cam_o[a];
                d[a] = ((R)P.cam_f[a] + (R)P.cam_r[a] * sx) + (R)P.cam_u[a] * sy;
            }
            const R len = rsqrt_len(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                d[a] = d[a] / len;
                s_wo[a][tx] = -d[a];
            }
            R t0;
            if (!aabb_unit<R>(o, d, R(0), rinf(R(0)), t0, t1) || !(sm > R(0))) {
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (Slot)P.bg[c];
                continue;
            }
            t = t0;
            phase = 1;
        }

        // ---- one tentative-collision step (shared by both flight kinds) ----
        t -= step_len(rng, inv_sm);
        if (phase == 1) ++nprim;
        else ++nshad;

        bool flight_done = false;  // shadow flight finished this step
        bool collided = false;
        if (t > t1) {
            if (phase == 1) {  // primary ray left the volume: background
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (Slot)P.bg[c];
                phase = 0;
                continue;
            }
            flight_done = true;
        } else {
            R x[3] = {o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t};
            // u2 is drawn before sigma(x) is evaluated: nothing else touches the
            // stream in between, so the sequence is the reference's
            const R u2 = uniform(rng, R(0));
            if (u2 * sm >= (R)cell_bound(S, x)) continue;  // certain null collision
            const R scalar = sample(S, x);
            const R sigma = ds * tf_alpha(S, scalar);
            if (phase == 1) {
                if (u2 * sm < sigma) {
                    // real interaction: Interaction{x, scalar, albedo}
                    {
                        R rgba[4];
                        tf_rgba(S, scalar, rgba);
                        sig_s = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) / R(3));
                    }
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        o[a] = x[a];
                        s_ld[a][tx] = R(0);
                    }
                    pcg_init(rng, P.init_nee, index);
                    light = -1;
                    flight_done = true;  // fall through into "start next light"
                    T = R(1);
                    phase = 2;
                }
            } else if (PAR) {
                if (u2 * sm < sigma) {
                    flight_done = true;
                    collided = true;
                }
            } else {
                // ratio tracking + Russian roulette below T < 0.1
                T *= R(1) - sigma * inv_sm;
                if (T < R(0.1)) {
                    const R q = T * R(10);
                    if (uniform(rng, R(0)) >= q) {
                        T = R(0);
                        flight_done = true;
                    } else {
                        T = R(0.1);
                    }
                }
            }
        }
        if (!flight_done) continue;

        // ---- a shadow flight ended (or the primary hit just happened) ----
        if (light >= 0) {
            if (PAR) {
                if (!collided) ++passed;
                if (++trial < P.nee_trials) {
                    t = ts0;
                    continue;
                }
                T = (R)passed / (R)P.nee_trials;
            }
            nee(light, T);
        }
        // start the next light's segment x -> P (volume.cpp:230-238)
        for (;;) {
            ++light;
            if (light >= S.n_lights) break;
            R dv[3] = {(R)S.light_p[light][0] - o[0], (R)S.light_p[light][1] - o[1],
                       (R)S.light_p[light][2] - o[2]};
            const R len = rsqrt_len(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            bool trivially_lit = (len == R(0));
            if (!trivially_lit) {
#pragma unroll
                for (int a = 0; a < 3; ++a) d[a] = dv[a] / len;
                R a0, a1;
                trivially_lit = !aabb_unit<R>(o, d, R(0), len, a0, a1) || !(sm > R(0));
                if (!trivially_lit) {
                    t = a0;
                    ts0 = a0;
                    t1 = a1;
                    trial = 0;
                    passed = 0;
                    T = R(1);
                    break;
                }
            }
            nee(light, R(1));
        }
        if (light < S.n_lights) continue;  // shadow flight started

        // ---- all lights done: w_d * L_d into the slot, hit record for the field
        const size_t sb = 3 * (size_t)w;
#pragma unroll
        for (int c = 0; c < 3; ++c) slots[sb + c] = (Slot)P.w_d * s_ld[c][tx];
        if (P.use_field) {
            const unsigned long long h = warp_fetch_add(&P.counters[1], 1u);
            HitRec rec;
            rec.x[0] = (float)o[0];
            rec.x[1] = (float)o[1];
            rec.x[2] = (float)o[2];
            const float wz = fminf(fmaxf((float)s_wo[2][tx], -1.0f), 1.0f);
            rec.wsph[0] = acosf(wz) * (float)(1.0 / kPi);
            rec.wsph[1] = (atan2f((float)s_wo[1][tx], (float)s_wo[0][tx]) + (float)kPi) * (float)(0.5 / kPi);
            rec.slot = w;
            rec.sigma_s = (double)sig_s;
            P.hits[h] = rec;
            if (P.hit_dir) {
#pragma unroll
                for (int a = 0; a < 3; ++a) P.hit_dir[3 * h + a] = (double)s_wo[a][tx];
            }
        } else {
            warp_fetch_add(&P.counters[1], 1u);
        }
        phase = 0;
    }
    atomicAdd(&P.counters[2], (unsigned long long)nprim);
    atomicAdd(&P.counters[3], (unsigned long long)nshad);
}

// ---------------------------------------------------------------------------
// Batched parity entry points (one thread per ray).
// ---------------------------------------------------------------------------
template <bool PAR>
__global__ void k_delta_track_batch(const DevScene S, BatchParams B) {
    using R = typename Prec<PAR>::R;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    R o[3], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        o[a] = (R)B.a3[3 * i + a];
        d[a] = (R)B.b3[3 * i + a];
    }
    R t0, t1;
    B.hit[i] = 0;
    if (!aabb_unit<R>(o, d, (R)B.tmin[i], (R)B.tmax[i], t0, t1)) return;
    const R sm = majorant(S, R(0));
    if (sm <= R(0)) return;
    const R inv = inv_majorant(S, R(0));
    R t = t0;
    for (;;) {
        t -= step_len(rng, inv);
        if (t > t1) return;
        R x[3] = {o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t};
        const R u2 = uniform(rng, R(0));
        if (u2 * sm >= (R)cell_bound(S, x)) continue;  // certain null collision
        const R s = sample(S, x);
        const R sigma = density(S, R(0)) * tf_alpha(S, s);
        if (u2 * sm < sigma) {
            B.hit[i] = 1;
            if (B.pos3)
                for (int a = 0; a < 3; ++a) B.pos3[3 * i + a] = (double)x[a];
            if (B.rgba4) {
                R c[4];
                tf_rgba(S, s, c);
                for (int a = 0; a < 4; ++a) B.rgba4[4 * i + a] = (double)c[a];
            }
            return;
        }
    }
}

#ifdef PF_TU_PARITY
// transmittance(medium, a, b, rng, n_trials), volume.cpp:227-256 (binary64).
__global__ void k_transmittance_batch(const DevScene S, BatchParams B) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    double a[3], dv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        a[k] = B.a3[3 * i + k];
        dv[k] = B.b3[3 * i + k] - a[k];
    }
    const double len = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
    if (len == 0.0) {
        B.out[i] = 1.0;
        return;
    }
    double dir[3] = {dv[0] / len, dv[1] / len, dv[2] / len};
    double t0, t1;
    if (!aabb_unit<double>(a, dir, 0.0, len, t0, t1) || S.sigma_max <= 0.0) {
        B.out[i] = 1.0;
        return;
    }
    int passed = 0;
    for (int trial = 0; trial < B.n_trials; ++trial) {
        double t = t0;
        bool collided = false;
        const double inv = 1.0 / S.sigma_max;
        for (;;) {
            t -= log(1.0 - pcg_double(rng)) * inv;
            if (t > t1) break;
            double x[3] = {a[0] + dir[0] * t, a[1] + dir[1] * t, a[2] + dir[2] * t};
            const double u2 = pcg_double(rng);
            if (u2 * S.sigma_max >= cell_bound(S, x)) continue;  // certain null collision
            const double sigma = S.density_scale * tf_alpha_d(S, sample_d(S, x));
            if (u2 * S.sigma_max < sigma) {
                collided = true;
                break;
            }
        }
        if (!collided) ++passed;
    }
    B.out[i] = (double)passed / B.n_trials;
}

__global__ void k_rng_doubles(BatchParams B) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    for (int k = 0; k < B.n_trials; ++k) B.out[i * (size_t)B.n_trials + k] = pcg_double(rng);
}

#endif  // PF_TU_PARITY


}  // namespace pfk
