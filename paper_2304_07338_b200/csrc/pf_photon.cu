// pf_photon.cu -- multi-phase photon tracing (Alg. 1, photon.hpp:48-57) on the
// device, binary64, compiled with --fmad=false like the parity tracer.
//
// Pinned algorithm: oracle/pf_oracle.c or_trace_photons / or_emit_direction /
// or_hg_sample.  One thread per photon i:
//   pair = i % (nL*nG), light = pair / nG, phase = pair % nG,
//   rng = make_rng(seed, Trace, i), emit toward the box's bounding sphere,
//   up to max_bounces delta-tracked interactions; bounce >= 1 deposits.
// Deposits are appended to a scratch list (warp-aggregated atomics) tagged
// with (photon, ordinal); a scan over per-photon counts then scatters them to
// the reference's concatenation order (photon index, then bounce) -- the
// result is independent of scheduling, like the reference's per-worker
// gather.
#include <cooperative_groups.h>

#include <cub/device/device_scan.cuh>

#include "pf_photon.h"
#include "pf_phase.cuh"
#include "pf_trace.cuh"

namespace cg = cooperative_groups;

namespace pfk {

namespace {

// emit_direction (photon.hpp:48-50; oracle or_emit_direction).
__device__ __forceinline__ void emit_dir(const double P[3], Pcg &r, double out[3]) {
    const double R = 0.5 * sqrt(3.0);
    const double v[3] = {0.5 - P[0], 0.5 - P[1], 0.5 - P[2]};
    const double d = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (d <= R) {
        uniform_sphere(r, out);
        return;
    }
    const double axis[3] = {v[0] / d, v[1] / d, v[2] / d};
    const double s = R / d;
    const double cos_max = sqrt(stdmax(0.0, 1.0 - s * s));
    const double u1 = pcg_double(r), u2 = pcg_double(r);
    frame_dir(axis, 1.0 - u1 * (1.0 - cos_max), u2, out);
}

// delta_track (volume.cpp:200-225) from o along d over [0, inf): binary64,
// global majorant, exact certain-null shortcut (same RNG draws as the
// reference: step, then u2, per tentative collision).
__device__ __forceinline__ bool track(const DevScene &S, const double o[3], const double d[3], Pcg &rng,
                                      double x[3], double c[4], uint32_t &steps) {
    double t0, t1;
    if (!aabb_unit<double>(o, d, 0.0, rinf(0.0), t0, t1)) return false;
    if (S.sigma_max <= 0.0) return false;
    const double inv = S.inv_sigma_max, sm53 = S.sm53;
    ParFlight F;
    par_flight(S, o, d, t0, F);
    // software-pipelined like the render tracer: the next step's u1 draw and
    // log run while this step's majorant TEX is in flight; a real collision
    // undoes the speculative draw, a rejected fetch keeps it (it is exactly
    // the reference's next draw)
    double t = t0 - par_step(rng, inv);
    if (t > t1) return false;
    ++steps;
    double u2sm = par_u2sm(rng, sm53);
    unsigned bnd = par_bound(S, F, t, t0);
    for (;;) {
        const unsigned long long saved = rng.state;
        const double tn = t - par_step(rng, inv);
        if (!par_null_given(u2sm, bnd)) {
#pragma unroll
            for (int a = 0; a < 3; ++a) x[a] = o[a] + d[a] * t;
            const double s = sample_d(S, x);
            tf_rgba_d(S, s, c);
            if (u2sm < S.density_scale * c[3]) {
                rng.state = saved;
                return true;
            }
        }
        t = tn;
        if (t > t1) return false;
        ++steps;
        u2sm = par_u2sm(rng, sm53);
        bnd = par_bound(S, F, t, t0);
    }
}

__global__ void __launch_bounds__(128, 7) k_trace_photons(const DevScene S, const PhotonTraceParams P) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t steps = 0;
    // per-photon power scale and throughput in shared memory (column per
    // thread): used once per bounce, so the tracking loop keeps the registers
    __shared__ double s_scale[3][128], s_thr[3][128];
    const int tx = threadIdx.x;
    if (i < P.n_total) {
        const uint64_t pairs = (uint64_t)S.n_lights * (uint64_t)P.n_phases;
        const uint64_t pr = i % pairs;
        const int li = (int)(pr / (uint64_t)P.n_phases), gi = (int)(pr % (uint64_t)P.n_phases);
        const double g = P.g[gi];
        const double n_pair = (double)(P.n_total / pairs + (pr < P.n_total % pairs ? 1u : 0u));
#pragma unroll
        for (int k = 0; k < 3; ++k) s_scale[k][tx] = S.light_i[li][k] / n_pair;
        Pcg rng;
        pcg_init(rng, P.initstate, i);
        double o[3] = {S.light_p[li][0], S.light_p[li][1], S.light_p[li][2]}, w[3];
        emit_dir(o, rng, w);
#pragma unroll
        for (int k = 0; k < 3; ++k) s_thr[k][tx] = 1.0;
        uint32_t dep = 0;
        for (int bounce = 0; bounce < P.max_bounces; ++bounce) {
            double x[3], c[4];
            if (!track(S, o, w, rng, x, c, steps)) break;
#pragma unroll
            for (int k = 0; k < 3; ++k) s_thr[k][tx] *= c[3] * c[k];
            double nw[3];
            {
                const double u1 = pcg_double(rng), u2 = pcg_double(rng);
                frame_dir(w, hg_cos(g, u1), u2, nw);
            }
            if (bounce >= 1) {
                cg::coalesced_group grp = cg::coalesced_threads();
                unsigned long long base = 0;
                if (grp.thread_rank() == 0) base = atomicAdd(P.counter, (unsigned long long)grp.size());
                const unsigned long long slot = grp.shfl(base, 0) + grp.thread_rank();
                if (slot < P.cap) {
                    PhotonOut r;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        r.pos[k] = (float)x[k];
                        r.dir[k] = (float)nw[k];
                        r.pow[k] = (float)(s_scale[k][tx] * s_thr[k][tx]);
                    }
                    r.g_index = (uint8_t)gi;
                    // deposit ordinal (16 bits in pad[0..1]; max_bounces <= 65536
                    // is enforced by pf_trace_photons)
                    r.pad[0] = (uint8_t)(dep & 0xff);
                    r.pad[1] = (uint8_t)(dep >> 8);
                    r.pad[2] = 0;
                    P.rec[slot] = r;
                    P.rec_photon[slot] = (uint32_t)i;
                }
                ++dep;
            }
            if (bounce >= P.rr_start) {
                double q = stdmax(stdmax(s_thr[0][tx], s_thr[1][tx]), s_thr[2][tx]);
                q = q < P.rr_min ? P.rr_min : (q > P.rr_max ? P.rr_max : q);
                if (pcg_double(rng) >= q) break;
#pragma unroll
                for (int k = 0; k < 3; ++k) s_thr[k][tx] /= q;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                o[k] = x[k];
                w[k] = nw[k];
            }
        }
        P.counts[i] = dep;
    }
    // step statistics (one atomic per warp)
    const unsigned m = __activemask();
    for (int off = 16; off > 0; off >>= 1) steps += __shfl_down_sync(m, steps, off);
    if ((threadIdx.x & 31) == 0 && steps) atomicAdd(P.steps, (unsigned long long)steps);
}

// Scatter scratch deposits to (photon, ordinal) order.
__global__ void k_photon_scatter(const PhotonOut *rec, const uint32_t *rec_photon, const uint32_t *offs,
                                 uint64_t n, PhotonOut *out) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    PhotonOut p = rec[r];
    const uint64_t dst = (uint64_t)offs[rec_photon[r]] + ((uint32_t)p.pad[0] | ((uint32_t)p.pad[1] << 8));
    p.pad[0] = p.pad[1] = 0;
    out[dst] = p;
}

}  // namespace

cudaError_t launch_trace_photons(const DevScene &S, const PhotonTraceParams &P, cudaStream_t st) {
    if (P.n_total == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((P.n_total + 127) / 128);
    k_trace_photons<<<blocks, 128, 0, st>>>(S, P);
    return cudaGetLastError();
}

cudaError_t photon_scan_bytes(uint64_t n, size_t *bytes) {
    *bytes = 0;
    return cub::DeviceScan::ExclusiveSum(nullptr, *bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                         (int64_t)n);
}

cudaError_t launch_photon_compact(const uint32_t *counts, uint32_t *offs, uint64_t n_photons, void *tmp,
                                  size_t tmp_bytes, const PhotonOut *rec, const uint32_t *rec_photon,
                                  uint64_t n_rec, PhotonOut *out, cudaStream_t st) {
    if (n_photons == 0 || n_rec == 0) return cudaSuccess;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, offs, (int64_t)n_photons, st);
    if (e != cudaSuccess) return e;
    k_photon_scatter<<<(unsigned)((n_rec + 255) / 256), 256, 0, st>>>(rec, rec_photon, offs, n_rec, out);
    return cudaGetLastError();
}

}  // namespace pfk
