// pf_trace.cuh -- K1/K2: persistent primary delta tracking + NEE shadow rays.
//
// Included by two translation units:
//   pf_trace_parity.cu (binary64, --fmad=false): k_render_trace_parity and the
//     batch entry points reproduce pf::delta_track / pf::transmittance
//     (proj/src/volume.cpp:204-256) operation-for-operation with the same RNG
//     consumption (tracking step: pf_parstep.cuh);
//   pf_trace_fast.cu (binary32): the throughput mode (own kernel), same
//     streams (2 x u32 per uniform), macro-cell DDA + ratio-tracked shadow rays;
//     it uses the precision-dispatched primitives below.
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
#include "pf_parstep.cuh"

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
    return par_step(r, inv);  // volume.cpp:217 / 247 (pf_parstep.cuh)
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

#ifdef PF_TU_PARITY  // kernels defined in pf_trace_parity.cu only
// ---------------------------------------------------------------------------
// The persistent PARITY render tracer (binary64, the reference's global
// majorant and RNG consumption; the FAST tracer is pf_trace_fast.cu).
// Per lane: {fetch sample -> primary flight -> shadow flight(s) per light}.
// The tracking step (pf_parstep.cuh) only touches the RNG state, t, and six
// float majorant-texture coordinates; the binary64 ray (origin, direction),
// omega_out, L_d and the sample index live in per-thread shared-memory
// columns and are read only at events (a voxel fetch, a flight end), which
// keeps the step loop spill-free and short (~100 instructions vs ~280).
// ---------------------------------------------------------------------------
#ifndef PF_PAR_REFILL
#define PF_PAR_REFILL 2  // waiting lanes that trigger a refill from the warp queue
#endif
#ifndef PF_PAR_FETCH
#define PF_PAR_FETCH 2  // lanes parked at a voxel fetch that trigger a fetch round
#endif
#ifndef PF_PAR_BURST
#define PF_PAR_BURST 16  // tentative collisions per lane between warp-level checks
#endif
#ifndef PF_PAR_CTAS
#define PF_PAR_CTAS 5  // resident CTAs per SM (register budget 65536 / (128 x 5) = 102 for the pipelined burst)
#endif
#ifndef PF_PAR_PIPE
#define PF_PAR_PIPE 1  // 1: software-pipelined burst (next step's log overlaps this step's TEX)
#endif
#ifndef PF_PAR_LOG_SMEM
#define PF_PAR_LOG_SMEM 1  // 1: the step's log table from a per-CTA shared-memory copy (LDS) instead of LDG
#endif
__global__ void __launch_bounds__(PF_TRACE_THREADS, PF_PAR_CTAS)
    k_render_trace_parity(const DevScene S, const TraceParams P) {
    double *slots = reinterpret_cast<double *>(P.slots);
    const double inv_sm = S.inv_sigma_max;
    const double sm = S.sigma_max;
    const double sm53 = S.sm53;
    const double ds = S.density_scale;
    const double g = P.g;

    // event-only state: per-thread shared-memory columns
    __shared__ double s_o[3][PF_TRACE_THREADS], s_d[3][PF_TRACE_THREADS];
    __shared__ double s_wo[3][PF_TRACE_THREADS], s_ld[3][PF_TRACE_THREADS];
    __shared__ double s_sig[PF_TRACE_THREADS], s_tb[PF_TRACE_THREADS];
    __shared__ unsigned long long s_idx[PF_TRACE_THREADS];
    __shared__ uint32_t s_w[PF_TRACE_THREADS];
    __shared__ int s_light[PF_TRACE_THREADS], s_trial[PF_TRACE_THREADS], s_passed[PF_TRACE_THREADS];
    // shadow-step accounting without a second per-step counter: nstep at the
    // start of the current shadow flight, and the shadow steps so far
    __shared__ uint32_t s_mark[PF_TRACE_THREADS], s_nshad[PF_TRACE_THREADS];
    __shared__ double s_u2[PF_TRACE_THREADS];      // u2 * sigma_max of a parked lane
    __shared__ uint32_t s_nfetch[PF_TRACE_THREADS];  // voxel fetches (sigma(x) evaluations)
    __shared__ float4 s_qa[PF_TRACE_THREADS];
    __shared__ float2 s_qb[PF_TRACE_THREADS];
    const ParFlightSmem Fm{s_qa, s_qb};
    const int tx = threadIdx.x;
#if PF_PAR_LOG_SMEM
    __shared__ pf_log_wide s_logtab[1 << PF_LOG_BITS];
    pf_log_fill_wide(s_logtab, tx, PF_TRACE_THREADS);
    __syncthreads();
    const uint32_t logtab = (uint32_t)__cvta_generic_to_shared(s_logtab);
#define PAR_STEP(r) par_step_smem(r, inv_sm, logtab)
#else
#define PAR_STEP(r) par_step(r, inv_sm)
#endif

    // step-loop state: registers
    // 0 waiting for a sample, 1 primary flight, 2 shadow flight, 3 queue drained;
    // | 4: parked at a voxel fetch (sigma(x) pending) of a primary / shadow flight
    int phase = 0;
    Pcg rng;
    double t = 0, t1 = 0;
    uint32_t nstep = 0;
    s_nshad[tx] = 0;
    s_nfetch[tx] = 0;

    auto nee = [&](int l, double Tl) {
        const double x[3] = {s_o[0][tx], s_o[1][tx], s_o[2][tx]};
        const double wo[3] = {s_wo[0][tx], s_wo[1][tx], s_wo[2][tx]};
        double Ld[3] = {s_ld[0][tx], s_ld[1][tx], s_ld[2][tx]};
        nee_term<double>(S, l, x, wo, g, Tl, Ld);
#pragma unroll
        for (int c = 0; c < 3; ++c) s_ld[c][tx] = Ld[c];
    };

    // Sample setup through a per-warp ready queue in shared memory: when a
    // refill finds the queue empty, the WHOLE warp (converged, 32 lanes) sets up
    // the next 32 work items at once -- work decode, camera ray, binary64
    // divisions, box clip; rays that miss the box write their background slot
    // here and are never queued -- so a waiting lane only copies one queue
    // entry (~40 instructions) instead of running the ~300-instruction setup
    // with a handful of lanes active.  Lanes wait (phase 0) until
    // PF_PAR_REFILL of them are waiting or none is tracking.
    __shared__ double q_d[3][PF_TRACE_THREADS], q_t0[PF_TRACE_THREADS], q_t1[PF_TRACE_THREADS];
    __shared__ unsigned long long q_st[PF_TRACE_THREADS], q_idx[PF_TRACE_THREADS];
    __shared__ uint32_t q_w[PF_TRACE_THREADS];
    const int lane = tx & 31, wb = tx & ~31;  // this warp's 32 queue slots: [wb, wb + 32)
    int qh = 0, qn = 0;                       // warp-uniform ring head / count
    bool drained = false;                     // warp-uniform: the work counter ran out

    auto take = [&](unsigned wmask) {
        const int r = __popc(wmask & lanemask_lt());
        if (phase == 0 && r < qn) {
            const int q = wb + ((qh + r) & 31);
            double o[3], d[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = P.cam_o[a];
                d[a] = q_d[a][q];
                s_o[a][tx] = o[a];
                s_d[a][tx] = d[a];
                s_wo[a][tx] = -d[a];
            }
            const unsigned long long index = q_idx[q];
            s_idx[tx] = index;
            s_w[tx] = q_w[q];
            rng.state = q_st[q];
            rng.inc = (index << 1) | 1ull;
            t = q_t0[q];
            t1 = q_t1[q];
            s_tb[tx] = t;
            ParFlight F;
            par_flight(S, o, d, t, F);
            par_store(Fm, tx, F);
            phase = 1;
        }
        const int got = min(__popc(wmask), qn);
        qh = (qh + got) & 31;
        qn -= got;
    };
    auto fill = [&]() {  // precondition: qn == 0, all 32 lanes converged
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&P.counters[0], 32ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base + 32ull >= (unsigned long long)P.n_work) drained = true;
        bool ok = false;
        const uint32_t w = (uint32_t)(base + (unsigned long long)lane);
        int px = 0, py = 0;
        uint64_t index = 0;
        double d[3], t0 = 0, ta = 0;
        Pcg r;
        if (base + (unsigned long long)lane < (unsigned long long)P.n_work && decode_work(P, w, px, py, index)) {
            pcg_init(r, P.init_cam, index);
            const double u = pcg_double(r);
            const double v = pcg_double(r);
            // pinned camera (oracle or_camera_ray)
            const double sx = (2.0 * ((double)px + u)) / (double)P.W - 1.0;
            const double sy = 1.0 - (2.0 * ((double)py + v)) / (double)P.H;
            double o[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                o[a] = P.cam_o[a];
                d[a] = (P.cam_f[a] + P.cam_r[a] * sx) + P.cam_u[a] * sy;
            }
            const double len = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
#pragma unroll
            for (int a = 0; a < 3; ++a) d[a] = d[a] / len;
            if (aabb_unit<double>(o, d, 0.0, rinf(0.0), t0, ta) && sm > 0.0) {
                ok = true;
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[3 * (size_t)w + c] = P.bg[c];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const int q = wb + ((qh + qn + __popc(m & lanemask_lt())) & 31);
#pragma unroll
            for (int a = 0; a < 3; ++a) q_d[a][q] = d[a];
            q_t0[q] = t0;
            q_t1[q] = ta;
            q_st[q] = r.state;
            q_idx[q] = index;
            q_w[q] = w;
        }
        qn += __popc(m);
    };

    for (;;) {
        const unsigned waiting = __ballot_sync(0xffffffffu, phase == 0);
        const unsigned tracking = __ballot_sync(0xffffffffu, phase == 1 || phase == 2);
        const unsigned parked = __ballot_sync(0xffffffffu, (phase & 4) != 0);
        if (waiting && (tracking == 0 || __popc(waiting) >= PF_PAR_REFILL)) {
            take(waiting);
            const unsigned still = __ballot_sync(0xffffffffu, phase == 0);
            if (still && qn == 0 && !drained) {
                fill();
                take(still);
            }
            if (drained && qn == 0 && phase == 0) phase = 3;  // no work left for this lane
            continue;  // re-evaluate the warp's state
        }
        if (tracking == 0 && parked == 0) break;  // every lane drained

        bool flight_done = false;  // shadow flight finished this step
        bool collided = false;
        if (parked && (tracking == 0 || __popc(parked) >= PF_PAR_FETCH)) {
            // ---- fetch round: the parked lanes evaluate sigma(x) together ----
            if ((phase & 4) == 0) continue;
            phase &= 3;
            ++s_nfetch[tx];
            const double u2sm = s_u2[tx];
            double x[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) x[a] = s_o[a][tx] + s_d[a][tx] * t;  // ray.at(t)
            const double scalar = sample_d(S, x);
            const double sigma = ds * tf_alpha_d(S, scalar);
            if (!(u2sm < sigma)) continue;  // null collision: back to stepping
            {
                if (phase == 1) {
                    // real interaction: Interaction{x, scalar, albedo}
                    double rgba[4];
                    tf_rgba_d(S, scalar, rgba);
                    s_sig[tx] = rgba[3] * ((rgba[0] + rgba[1] + rgba[2]) / 3.0);
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        s_o[a][tx] = x[a];
                        s_ld[a][tx] = 0.0;
                    }
                    pcg_init(rng, P.init_nee, s_idx[tx]);
                    s_light[tx] = -1;
                    flight_done = true;  // fall through into "start next light"
                    phase = 2;
                } else {
                    flight_done = true;
                    collided = true;
                }
            }
        } else {
            if (phase != 1 && phase != 2) continue;
            // ---- a burst of up to PF_PAR_BURST tentative-collision steps ----
            // (shared by both flight kinds; the warp-level bookkeeping above runs
            // once per burst, a lane leaves the burst at its first event)
            const ParFlight F = par_load(Fm, tx);
            const double tb = s_tb[tx];
            int ev = 0;  // 0 none, 1 left the segment, 2 parked at a voxel fetch
#if PF_PAR_PIPE
            // Software-pipelined: step k+1's u1 draw and binary64 log are computed
            // while step k's majorant TEX is in flight (they do not depend on it);
            // if step k parks (or the burst ends) the speculative u1 draw is undone
            // by restoring the stream state, so the RNG sequence and every
            // decision are exactly the unpipelined ones.
            t -= PAR_STEP(rng);
            ++nstep;
            if (t > t1) {
                ev = 1;
            } else {
                double u2sm = par_u2sm(rng, sm53);
                unsigned bnd = par_bound(S, F, t, tb);
#pragma unroll 1
                for (int k = 1;; ++k) {
                    const unsigned long long saved = rng.state;
                    const double tn = t - PAR_STEP(rng);  // speculative step k+1
                    if (!par_null_given(u2sm, bnd)) {
                        rng.state = saved;
                        s_u2[tx] = u2sm;  // park until the warp's next fetch round
                        ev = 2;
                        break;
                    }
                    if (k == PF_PAR_BURST) {
                        rng.state = saved;
                        break;
                    }
                    t = tn;
                    ++nstep;
                    if (t > t1) {
                        ev = 1;
                        break;
                    }
                    u2sm = par_u2sm(rng, sm53);
                    bnd = par_bound(S, F, t, tb);
                }
            }
#else
#pragma unroll 1
            for (int k = 0; k < PF_PAR_BURST; ++k) {
                t -= PAR_STEP(rng);
                ++nstep;
                if (t > t1) {
                    ev = 1;
                    break;
                }
                // u2 is drawn before sigma(x) is evaluated: nothing else touches
                // the stream in between, so the sequence is the reference's
                const double u2sm = par_u2sm(rng, sm53);
                if (!par_certain_null(S, F, t, tb, u2sm)) {
                    s_u2[tx] = u2sm;  // park until the warp's next fetch round
                    ev = 2;
                    break;
                }
            }
#endif
            if (ev == 0) continue;
            if (ev == 2) {
                phase |= 4;
                continue;
            }
            if (phase == 1) {  // primary ray left the volume: background
                const size_t sb = 3 * (size_t)s_w[tx];
#pragma unroll
                for (int c = 0; c < 3; ++c) slots[sb + c] = P.bg[c];
                phase = 0;
                continue;
            }
            flight_done = true;
        }
        if (!flight_done) continue;

        // ---- a shadow flight ended (or the primary hit just happened) ----
        int light = s_light[tx];
        if (light >= 0) {
            s_nshad[tx] += nstep - s_mark[tx];
            const int passed = s_passed[tx] + (collided ? 0 : 1);
            const int trial = s_trial[tx] + 1;
            if (trial < P.nee_trials) {
                s_passed[tx] = passed;
                s_trial[tx] = trial;
                s_mark[tx] = nstep;
                t = s_tb[tx];
                continue;
            }
            nee(light, (double)passed / (double)P.nee_trials);
        }
        // start the next light's segment x -> P (volume.cpp:230-238)
        for (;;) {
            ++light;
            if (light >= S.n_lights) break;
            double o[3] = {s_o[0][tx], s_o[1][tx], s_o[2][tx]};
            double dv[3] = {S.light_p[light][0] - o[0], S.light_p[light][1] - o[1], S.light_p[light][2] - o[2]};
            const double len = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
            bool trivially_lit = (len == 0.0);
            if (!trivially_lit) {
                double d[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    d[a] = dv[a] / len;
                    s_d[a][tx] = d[a];
                }
                double a0, a1;
                trivially_lit = !aabb_unit<double>(o, d, 0.0, len, a0, a1) || !(sm > 0.0);
                if (!trivially_lit) {
                    t = a0;
                    t1 = a1;
                    s_tb[tx] = a0;
                    {
                        ParFlight F;
                        par_flight(S, o, d, a0, F);
                        par_store(Fm, tx, F);
                    }
                    s_trial[tx] = 0;
                    s_passed[tx] = 0;
                    s_mark[tx] = nstep;
                    break;
                }
            }
            nee(light, 1.0);
        }
        s_light[tx] = light;
        if (light < S.n_lights) continue;  // shadow flight started

        // ---- all lights done: w_d * L_d into the slot, hit record for the field
        const uint32_t w = s_w[tx];
        const size_t sb = 3 * (size_t)w;
#pragma unroll
        for (int c = 0; c < 3; ++c) slots[sb + c] = P.w_d * s_ld[c][tx];
        if (P.use_field) {
            const unsigned long long h = warp_fetch_add(&P.counters[1], 1u);
            HitRec rec;
            rec.x[0] = (float)s_o[0][tx];
            rec.x[1] = (float)s_o[1][tx];
            rec.x[2] = (float)s_o[2][tx];
            const float wz = fminf(fmaxf((float)s_wo[2][tx], -1.0f), 1.0f);
            rec.wsph[0] = acosf(wz) * (float)(1.0 / kPi);
            rec.wsph[1] = (atan2f((float)s_wo[1][tx], (float)s_wo[0][tx]) + (float)kPi) * (float)(0.5 / kPi);
            rec.slot = w;
            rec.sigma_s = s_sig[tx];
            P.hits[h] = rec;
            if (P.hit_dir) {
#pragma unroll
                for (int a = 0; a < 3; ++a) P.hit_dir[3 * h + a] = s_wo[a][tx];
            }
        } else {
            warp_fetch_add(&P.counters[1], 1u);
        }
        phase = 0;
    }
    atomicAdd(&P.counters[2], (unsigned long long)(nstep - s_nshad[tx]));
    atomicAdd(&P.counters[3], (unsigned long long)s_nshad[tx]);
    atomicAdd(&P.counters[4], (unsigned long long)s_nfetch[tx]);
}

// ---------------------------------------------------------------------------
// Batched parity entry points (one thread per ray).
// ---------------------------------------------------------------------------
// pf::delta_track (volume.cpp:204-225), binary64: hit, Interaction{position,
// scalar, albedo}.
__global__ void k_delta_track_batch(const DevScene S, BatchParams B) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B.n) return;
    Pcg rng;
    pcg_init(rng, B.initstate, B.idx[i]);
    double o[3], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        o[a] = B.a3[3 * i + a];
        d[a] = B.b3[3 * i + a];
    }
    double t0, t1;
    B.hit[i] = 0;
    if (B.scalar) B.scalar[i] = 0.0;
    if (!aabb_unit<double>(o, d, B.tmin[i], B.tmax[i], t0, t1)) return;
    const double sm = S.sigma_max;
    if (sm <= 0.0) return;
    const double inv = S.inv_sigma_max, sm53 = S.sm53;
    ParFlight F;
    par_flight(S, o, d, t0, F);
    double t = t0;
    for (;;) {
        t -= par_step(rng, inv);
        if (t > t1) return;
        const double u2sm = par_u2sm(rng, sm53);
        if (par_certain_null(S, F, t, t0, u2sm)) continue;
        double x[3] = {o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t};
        const double s = sample_d(S, x);
        const double sigma = S.density_scale * tf_alpha_d(S, s);
        if (u2sm < sigma) {
            B.hit[i] = 1;
            if (B.pos3)
                for (int a = 0; a < 3; ++a) B.pos3[3 * i + a] = x[a];
            if (B.scalar) B.scalar[i] = s;
            if (B.rgba4) {
                double c[4];
                tf_rgba_d(S, s, c);
                for (int a = 0; a < 4; ++a) B.rgba4[4 * i + a] = c[a];
            }
            return;
        }
    }
}

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
    const double inv = S.inv_sigma_max, sm53 = S.sm53;
    ParFlight F;
    par_flight(S, a, dir, t0, F);
    for (int trial = 0; trial < B.n_trials; ++trial) {
        double t = t0;
        bool collided = false;
        for (;;) {
            t -= par_step(rng, inv);
            if (t > t1) break;
            const double u2sm = par_u2sm(rng, sm53);
            if (par_certain_null(S, F, t, t0, u2sm)) continue;
            double x[3] = {a[0] + dir[0] * t, a[1] + dir[1] * t, a[2] + dir[2] * t};
            const double sigma = S.density_scale * tf_alpha_d(S, sample_d(S, x));  // Medium::extinction
            if (u2sm < sigma) {
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
