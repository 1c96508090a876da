// pf_pathtrace.cuh -- render_path_traced: the reference
// volumetric path tracer with NEE at every vertex, HG-sampled continuation
// and Russian roulette.  Pinned in oracle/pf_oracle.c or_render_path_traced /
// or_pt_indirect (composition checked against the reference's own
// delta_track / transmittance / hg_sample in oracle/ref_shim.cpp).
//
// One template, two translation units (like pf_trace.cuh):
//   pf_pathtrace_parity.cu (binary64, --fmad=false): the reference's global
//     majorant, delta-tracked shadow trials, same RNG consumption -> the
//     oracle's image up to last-ulp libm differences;
//   pf_pathtrace_fast.cu (binary32): macro-cell majorant DDA + ratio-tracked
//     shadow rays, unbiased (statistical parity).
// Up to and including the first interaction's NEE the program is exactly
// k_render_trace{,_fast}'s (same streams and operations), so max_bounces = 1
// reproduces render_neural without a field bit-for-bit.
//
// Design: the persistent lane state machine of the render tracer extended
// with a path vertex counter -- a lane walks {path flight -> shadow flights
// per light -> scatter} until the path ends, then pulls the next sample with
// a warp-aggregated atomic, so long paths never hold a warp's other lanes.
#pragma once

#include "pf_dda.cuh"
#include "pf_phase.cuh"
#include "pf_trace.cuh"

namespace pfk {

template <bool PAR>
__global__ void __launch_bounds__(PF_TRACE_THREADS, PAR ? 6 : 8) k_render_pt(const DevScene S, const TraceParams P) {
    using R = typename Prec<PAR>::R;
    R *slots = reinterpret_cast<R *>(P.slots);
    const R inv_sm = inv_majorant(S, R(0));
    const R sm = majorant(S, R(0));
    const R ds = density(S, R(0));
    const R g = (R)P.g;

    int phase = 0;  // 0 fetch, 1 path flight, 2 shadow flight
    int vert = 0;   // path vertex being searched for / lit (0 = first interaction)
    uint32_t w = 0;
    uint64_t index = 0;
    Pcg rng;
    R o[3], d[3], pd[3];  // flight origin + direction; pd = direction of the path segment
    R t = 0, t1 = 0, ts0 = 0, T = 1;
    // radiance accumulators in shared memory (column per thread): touched once
    // per NEE term / vertex, not per tracking step; [0..2] L_d of the current
    // vertex, [3..5] L_d of vertex 0, [6..8] L_i
    __shared__ R s_acc[9][PF_TRACE_THREADS];
    const int tx = threadIdx.x;
    R ss_v = 0;  // sigma_s of the current vertex (alpha * mean rgb)
#pragma unroll
    for (int k = 0; k < 9; ++k) s_acc[k][tx] = R(0);
    R thr = 1, ss0 = 0;
    int light = 0, trial = 0, passed = 0;
    ParFlight F;      // PARITY only: majorant-texture coordinates of the flight (origin at tb)
    R tb = 0;         // PARITY only: flight segment start
    Dda D;            // FAST only
    float tau = 0.f;  // FAST only
    uint32_t nprim = 0, nshad = 0;

    // begin a straight flight o + t d over [tmin, tmax] (false: no overlap with the box)
    auto start_flight = [&](R tmin, R tmax) -> bool {
        R a0, a1;
        if (!aabb_unit<R>(o, d, tmin, tmax, a0, a1) || !(sm > R(0))) return false;
        if constexpr (!PAR) {
            if (!occ_clip(S, o, d, a0, a1)) return false;  // only empty cells: no collision
        }
        t = a0;
        t1 = a1;
        if constexpr (PAR) {
            tb = a0;
            par_flight(S, o, d, a0, F);  // majorant-texture coordinates (pf_parstep.cuh)
        } else {
            dda_init(S, o, d, t, D);
            tau = sample_tau(rng);
        }
        return true;
    };
    auto nee = [&](int l, const R wo[3], R Tl) {
        R Ld[3] = {s_acc[0][tx], s_acc[1][tx], s_acc[2][tx]};
        nee_term<R>(S, l, o, wo, g, Tl, Ld);
#pragma unroll
        for (int c = 0; c < 3; ++c) s_acc[c][tx] = Ld[c];
    };
    auto finish = [&]() {
        const size_t sb = 3 * (size_t)w;
#pragma unroll
        for (int c = 0; c < 3; ++c) slots[sb + c] = (R)P.w_d * s_acc[3 + c][tx] + (R)P.w_i * (ss0 * s_acc[6 + c][tx]);
        warp_fetch_add(&P.counters[1], 1u);
        phase = 0;
    };

    for (;;) {
        if (phase == 0) {
            w = (uint32_t)warp_fetch_add(&P.counters[0], 1u);
            if (w >= P.n_work) break;
            int px, py;
            if (!decode_work(P, w, px, py, index)) continue;
            pcg_init(rng, P.init_cam, index);
            if constexpr (PAR) {
                const double u = pcg_double(rng);
                const double v = pcg_double(rng);
                const R sx = (R(2) * ((R)px + (R)u)) / (R)P.W - R(1);
                const R sy = R(1) - (R(2) * ((R)py + (R)v)) / (R)P.H;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    o[a] = (R)P.cam_o[a];
                    d[a] = ((R)P.cam_f[a] + (R)P.cam_r[a] * sx) + (R)P.cam_u[a] * sy;
                }
                const R len = rsqrt_len(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
                for (int a = 0; a < 3; ++a) d[a] = d[a] / len;
            } else {
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
                for (int a = 0; a < 3; ++a) d[a] *= rl;
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) pd[a] = d[a];
            vert = 0;
            thr = R(1);
#pragma unroll
            for (int c = 0; c < 3; ++c) s_acc[6 + c][tx] = R(0);
            if (!start_flight(R(0), rinf(R(0)))) {
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (R)P.bg[c];
                continue;
            }
            phase = 1;
        }

        // ---- one tentative collision of the current flight ----------------
        bool left = false;  // the flight left its segment
        R x[3] = {0, 0, 0}, scalar = 0;
        if constexpr (PAR) {
            t -= step_len(rng, inv_sm);
            if (phase == 1) ++nprim;
            else ++nshad;
            if (t > t1) {
                left = true;
            } else {
                const double u2sm = par_u2sm(rng, (double)sm * 0x1.0p-53);
                if (par_certain_null(S, F, t, tb, u2sm)) continue;  // certain null collision
#pragma unroll
                for (int a = 0; a < 3; ++a) x[a] = o[a] + d[a] * t;
                scalar = sample(S, x);
                if (!(u2sm < ds * tf_alpha(S, scalar))) continue;  // null collision
            }
        } else {
            float m;
            const bool coll = dda_advance(S, D, t, t1, tau, m);
            if (phase == 1) ++nprim;
            else ++nshad;
            if (!coll) {
                left = true;
            } else {
#pragma unroll
                for (int a = 0; a < 3; ++a) x[a] = fmaf(d[a], t, o[a]);
                scalar = sample_f(S, x);
                const float sigma = ds * tf_alpha_f(S, scalar);
                if (phase == 1) {
                    if (!(pcg_u_f(rng) * m < sigma)) {
                        tau = sample_tau(rng);
                        continue;
                    }
                } else {
                    // ratio tracking + Russian roulette below T < 0.1
                    T *= 1.0f - sigma / m;
                    bool stop = false;
                    if (T < 0.1f) {
                        if (pcg_u_f(rng) >= T * 10.0f) {
                            T = 0.f;
                            stop = true;
                        } else {
                            T = 0.1f;
                        }
                    }
                    if (!stop) {
                        tau = sample_tau(rng);
                        continue;
                    }
                }
            }
        }

        R wo[3] = {-pd[0], -pd[1], -pd[2]};
        if (phase == 1) {
            if (left) {  // the path segment escaped
                if (vert == 0) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = (R)P.bg[c];
                    phase = 0;
                } else {
                    finish();
                }
                continue;
            }
            // real interaction: path vertex `vert`
            {
                R rgba[4];
                tf_rgba(S, scalar, rgba);
                if constexpr (PAR) ss_v = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) / R(3));
                else ss_v = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) * (1.0f / 3.0f));
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = x[a];
                s_acc[a][tx] = R(0);
            }
            if (vert == 0) pcg_init(rng, P.init_nee, index);  // vertex 0 lights on the Nee stream
            light = -1;
            T = R(1);
            phase = 2;
        } else {
            // a shadow flight ended
            if constexpr (PAR) {
                if (left) ++passed;
                if (++trial < P.nee_trials) {
                    t = ts0;
                    continue;
                }
                T = (R)passed / (R)P.nee_trials;
            }
            nee(light, wo, T);
        }

        // start the next light's shadow segment x -> P (volume.cpp:230-238)
        for (;;) {
            ++light;
            if (light >= S.n_lights) break;
            R dv[3] = {(R)S.light_p[light][0] - o[0], (R)S.light_p[light][1] - o[1],
                       (R)S.light_p[light][2] - o[2]};
            const R len = rsqrt_len(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            // parity: transmittance's `len == 0 -> 1` test (volume.cpp:232); fast: the tracer's
            if (PAR ? !(len == R(0)) : len > R(0)) {
#pragma unroll
                for (int a = 0; a < 3; ++a) d[a] = dv[a] / len;
                if (start_flight(R(0), len)) {
                    ts0 = t;
                    trial = 0;
                    passed = 0;
                    T = R(1);
                    break;
                }
            }
            nee(light, wo, R(1));
        }
        if (light < S.n_lights) continue;  // shadow flight started

        // ---- vertex lit: accumulate, roulette, scatter --------------------
        const R ss = ss_v;
        bool go = vert + 1 < P.max_bounces;
        if (vert == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) s_acc[3 + c][tx] = s_acc[c][tx];
            ss0 = ss;
            if (go) pcg_init(rng, P.init_pt, index);  // the continuation's own stream
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c) s_acc[6 + c][tx] += thr * s_acc[c][tx];
            thr *= ss;
            if (go) {
                if (!(thr > R(0))) {
                    go = false;
                } else if (vert >= P.rr_start) {
                    const R q = thr < (R)P.rr_min ? (R)P.rr_min : (thr > (R)P.rr_max ? (R)P.rr_max : thr);
                    if (uniform(rng, R(0)) >= q) go = false;
                    else thr /= q;
                }
            }
        }
        if (!go) {
            finish();
            continue;
        }
        R nd[3];
        hg_sample(g, pd, rng, nd);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            pd[a] = nd[a];
            d[a] = nd[a];
        }
        ++vert;
        if (!start_flight(R(0), rinf(R(0)))) {
            finish();
            continue;
        }
        phase = 1;
    }
    atomicAdd(&P.counters[2], (unsigned long long)nprim);
    atomicAdd(&P.counters[3], (unsigned long long)nshad);
}

}  // namespace pfk
