// pf_knn.cu -- K6/K7: phase-selective exact KNN + fused Eq. 6 / Eq. 7.
//
// SPEC.md:221-280 (photon_map: build / knn_phase), SPEC.md:282-316 (Eq. 6
// estimate_radiance, Eq. 7 encode_log), SPEC.md:476-484 (make_batch).
//
// B200 design.  The reference's "single kd-tree with phase filtering" is a
// pointer-chasing structure; on the GPU the photon map becomes a per-phase
// uniform cell grid built by a radix sort on (phase, cell) keys, so every
// cell's photons of ONE phase are contiguous 16-byte records {x,y,z,id}.
// A query is one warp: lanes stream candidate records of a cell in
// coalesced 512-byte rows, and the warp keeps the exact top-K as a sorted,
// lane-distributed list of 64-bit keys (float_bits(d2) << 32 | id) -- the
// (d2, id) lexicographic order the oracle uses, so ties break by photon id.
// Cells are visited in Chebyshev rings around the query cell and skipped
// when their (conservatively expanded) box distance cannot beat the current
// K-th key; the search stops when the ring bound exceeds the K-th distance
// or r_max.  The result is therefore exactly the brute-force answer.
//
// Compiled with --fmad=false: d2 = ((dx*dx)+(dy*dy))+(dz*dz) in binary32 and
// Eq. 6 in binary64 must round exactly like the oracle.
#include <algorithm>
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pf_knn.h"

namespace pfk {

// ---- build ---------------------------------------------------------------
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void k_knn_bbox(const PhotonRec *ph, size_t n, int n_phases, uint32_t *mins,
                           uint32_t *maxs, uint32_t *counts) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const PhotonRec p = ph[i];
    const int g = p.g_index;
    if (g >= n_phases) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        atomicMin(&mins[3 * g + a], f2ord(p.position[a]));
        atomicMax(&maxs[3 * g + a], f2ord(p.position[a]));
    }
    atomicAdd(&counts[g], 1u);
}

__device__ __forceinline__ int cell_axis(double p, double lo, double inv_h, int R) {
    double c = floor((p - lo) * inv_h);
    int ci = c < 0.0 ? 0 : (c > (double)(R - 1) ? R - 1 : (int)c);
    return ci;
}

__global__ void k_knn_keys(const PhotonRec *ph, size_t n, const KnnParams P, uint32_t *keys,
                           uint32_t *vals, uint32_t *hist) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const PhotonRec p = ph[i];
    uint32_t key = P.total_cells;  // photons of unknown phases sort past the end
    if (p.g_index < P.n_phases) {
        const KnnGrid &G = P.grid[p.g_index];
        const int cx = cell_axis(p.position[0], G.lo[0], G.inv_h[0], G.R[0]);
        const int cy = cell_axis(p.position[1], G.lo[1], G.inv_h[1], G.R[1]);
        const int cz = cell_axis(p.position[2], G.lo[2], G.inv_h[2], G.R[2]);
        key = G.cell_base + (uint32_t)cx + (uint32_t)G.R[0] * ((uint32_t)cy + (uint32_t)G.R[1] * (uint32_t)cz);
        atomicAdd(&hist[key], 1u);
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
}

// Sorted copies in (phase, cell, id) order: positions + id for the candidate
// scan, {direction, power} payload for Eq. 6 (a query's neighbours sit in a
// few cells, so their payloads are contiguous), and the id -> sorted-index map.
__global__ void k_knn_gather(const PhotonRec *ph, size_t n, const uint32_t *vals, float4 *spos, float4 *spay,
                             uint32_t *inv) {
    const size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t id = vals[j];
    const PhotonRec p = ph[id];
    spos[j] = make_float4(p.position[0], p.position[1], p.position[2], __uint_as_float(id));
    spay[2 * j] = make_float4(p.direction[0], p.direction[1], p.direction[2], p.power[0]);
    spay[2 * j + 1] = make_float4(p.power[1], p.power[2], 0.0f, 0.0f);
    inv[id] = (uint32_t)j;
}

// ---- query ---------------------------------------------------------------
__device__ __forceinline__ unsigned knn_lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int KP>
struct WarpTopK {
    uint64_t v[KP];  // list position p = s*32 + lane, ascending
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int s = 0; s < KP; ++s) v[s] = ~0ull;
    }
    __device__ __forceinline__ uint64_t at(int p) const {
        uint64_t r = 0;
#pragma unroll
        for (int s = 0; s < KP; ++s)
            if (s == (p >> 5)) r = v[s];
        return __shfl_sync(0xffffffffu, r, p & 31);
    }
    // Merge up to 32 new keys (one per lane, ~0ull = none) in one pass:
    // bitonic-sort them across the warp, take min(list, reversed(new)) on the
    // last slot (the union's KP*32 smallest as a bitonic sequence), then a
    // bitonic merge over the KP*32 positions.  Exact; keys are distinct.
    __device__ __forceinline__ void merge32(uint64_t x, unsigned lane) {
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const uint64_t y = __shfl_xor_sync(0xffffffffu, x, j);
                const bool up = (lane & k) == 0 || k == 32;
                const bool lower = (lane & j) == 0;
                x = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
            }
        }
        const uint64_t br = __shfl_sync(0xffffffffu, x, 31 - lane);
        v[KP - 1] = v[KP - 1] < br ? v[KP - 1] : br;
#pragma unroll
        for (int J = KP / 2; J >= 1; J >>= 1) {
#pragma unroll
            for (int s = 0; s < KP; ++s)
                if ((s & J) == 0) {
                    const uint64_t a = v[s], b = v[s + J];
                    v[s] = a < b ? a : b;
                    v[s + J] = a < b ? b : a;
                }
        }
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const bool lower = (lane & j) == 0;
#pragma unroll
            for (int s = 0; s < KP; ++s) {
                const uint64_t y = __shfl_xor_sync(0xffffffffu, v[s], j);
                v[s] = lower ? (v[s] < y ? v[s] : y) : (v[s] < y ? y : v[s]);
            }
        }
    }
    __device__ __forceinline__ void insert(uint64_t key, unsigned lane) {
        int pos = 0;
#pragma unroll
        for (int s = 0; s < KP; ++s) pos += __popc(__ballot_sync(0xffffffffu, v[s] < key));
        uint64_t carry = 0;
#pragma unroll
        for (int s = 0; s < KP; ++s) {
            const uint64_t up = __shfl_up_sync(0xffffffffu, v[s], 1);
            const uint64_t last = __shfl_sync(0xffffffffu, v[s], 31);
            const uint64_t nv = lane == 0 ? carry : up;
            carry = last;
            const int p = s * 32 + (int)lane;
            v[s] = p > pos ? nv : (p == pos ? key : v[s]);
        }
    }
};

__device__ __forceinline__ float d2_rn(float4 c, const float q[3]) {
    const float dx = __fsub_rn(c.x, q[0]), dy = __fsub_rn(c.y, q[1]), dz = __fsub_rn(c.z, q[2]);
    return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
}

// hg_eval (phase.hpp:18-23), binary64, no contraction (TU built --fmad=false).
__device__ __forceinline__ double knn_hg_eval(double g, double c) {
    g = g < -0.999 ? -0.999 : (g > 0.999 ? 0.999 : g);
    double denom = 1.0 + g * g - 2.0 * g * c;
    denom = denom < 1e-12 ? 1e-12 : denom;
    return (1.0 / (4.0 * 3.14159265358979323846)) * (1.0 - g * g) / (denom * sqrt(denom));
}

template <int KP, bool RENDER>
__global__ void __launch_bounds__(128) k_knn_query(const KnnParams P) {
    // per-warp staging buffer: accepted candidates are merged 32 at a time
    __shared__ uint64_t s_buf[4][32];
    const unsigned lane = threadIdx.x & 31u;
    uint64_t *buf = s_buf[(threadIdx.x >> 5) & 3];
    constexpr bool render = RENDER;
    const size_t nq = (render && !P.order) ? (size_t)*P.n_hits : P.nq;  // order = fallback list
    const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t qs = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; qs < nq; qs += nwarps) {
    const size_t qi = P.order ? (size_t)__ldg(P.order + qs) : qs;  // spatially sorted visit order
    const int K = P.K;
    float q[3];
    int g;
    if constexpr (render) {
        const HitRec &h = P.hits[qi];
        q[0] = h.x[0];
        q[1] = h.x[1];
        q[2] = h.x[2];
        g = P.render_g;
    } else {
        q[0] = P.qx[3 * qi];
        q[1] = P.qx[3 * qi + 1];
        q[2] = P.qx[3 * qi + 2];
        g = P.qg[qi];
    }
    WarpTopK<KP> top;
    top.init();
    int count = 0;
    uint64_t thr = ~0ull;  // key of the K-th entry (inf while count < K)
    float kth = __int_as_float(0x7f800000);
    const float r2 = P.r2;
    int nb = 0;  // keys staged in buf (warp-uniform)

    auto flush = [&]() {
        __syncwarp();
        const uint64_t x = (int)lane < nb ? buf[lane] : ~0ull;
        __syncwarp();
        top.merge32(x, lane);
        count = min(K, count + nb);
        nb = 0;
        if (count >= K) {
            thr = top.at(K - 1);
            kth = __uint_as_float((uint32_t)(thr >> 32));
        }
    };
    // scan the contiguous sorted records [b, e) (one row segment of cells)
    auto scan = [&](uint32_t b, uint32_t e) {
        for (uint32_t j0 = b; j0 < e; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint64_t key = ~0ull;
            if (j < e) {
                const float4 c = __ldg(&P.spos[j]);
                const float d2 = d2_rn(c, q);
                if (d2 <= r2) key = ((uint64_t)__float_as_uint(d2) << 32) | __float_as_uint(c.w);
            }
            const bool acc = key < thr;
            const unsigned m = __ballot_sync(0xffffffffu, acc);
            const int nn = __popc(m);
            if (nn == 0) continue;
            if (nb + nn > 32) flush();
            if (acc) buf[nb + __popc(m & knn_lanemask_lt())] = key;
            nb += nn;
            if (nb == 32) flush();
        }
    };

    if (g < P.n_phases && P.grid[g].n > 0) {
        // register copy of this phase's grid (no dynamically indexed param loads)
        const KnnGrid &Gp = P.grid[g];
        int R[3], qc[3];
        float lo[3], h[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            R[a] = Gp.R[a];
            lo[a] = (float)Gp.lo[a];
            h[a] = (float)Gp.h[a];
            qc[a] = cell_axis((double)q[a], Gp.lo[a], Gp.inv_h[a], R[a]);
        }
        const float eps = (float)Gp.eps + 1e-6f;  // box slack >> binary32 rounding of the bounds
        const uint32_t cbase = Gp.cell_base;
        const double hmin = Gp.hmin, geps = Gp.eps;
        // squared 1-D gap between the query and the cell interval [c0, c1] on axis a
        // (edge cells extend to infinity: clamped photons may lie outside the grid box)
        auto gap = [&](int a, int c0, int c1) -> float {
            const float l = c0 == 0 ? -3.0e38f : fmaf((float)c0, h[a], lo[a]) - eps;
            const float u = c1 == R[a] - 1 ? 3.0e38f : fmaf((float)(c1 + 1), h[a], lo[a]) + eps;
            const float d = q[a] < l ? l - q[a] : (q[a] > u ? q[a] - u : 0.0f);
            return d * d;
        };
        const int rmax = max(R[0], max(R[1], R[2]));
        for (int ring = 0; ring <= rmax; ++ring) {
            for (int dz = -ring; dz <= ring; ++dz) {
                const int cz = qc[2] + dz;
                if (cz < 0 || cz >= R[2]) continue;
                const float gz = gap(2, cz, cz);
                for (int dy = -ring; dy <= ring; ++dy) {
                    const int cy = qc[1] + dy;
                    if (cy < 0 || cy >= R[1]) continue;
                    const float gyz = gz + gap(1, cy, cy);
                    if (gyz * (1.0f - 1e-5f) > fminf(r2, kth)) continue;
                    const uint32_t row = cbase + (uint32_t)R[0] * ((uint32_t)cy + (uint32_t)R[1] * (uint32_t)cz);
                    // the ring's new cells in this row: the whole [-ring, ring] segment on
                    // the outer y/z faces, else only the two end cells
                    const bool face = abs(dz) == ring || abs(dy) == ring;
                    for (int part = 0; part < (face ? 1 : 2); ++part) {
                        int x0 = face ? qc[0] - ring : (part == 0 ? qc[0] - ring : qc[0] + ring);
                        int x1 = face ? qc[0] + ring : x0;
                        x0 = max(x0, 0);
                        x1 = min(x1, R[0] - 1);
                        if (x0 > x1) continue;
                        const float lb = (gyz + gap(0, x0, x1)) * (1.0f - 1e-5f);
                        if (lb > r2 || lb > kth) continue;
                        scan(__ldg(P.cell_start + row + (uint32_t)x0), __ldg(P.cell_start + row + (uint32_t)x1 + 1));
                    }
                }
            }
            if (nb) flush();
            // every cell at Chebyshev distance > ring is >= ring*h_min - 2 eps away
            const double bnd = fmax(0.0, ring * hmin - 2.0 * geps);
            const double bnd2 = bnd * bnd * (1.0 - 1e-5);
            if (bnd2 > (double)r2) break;
            if (count >= K && bnd2 > (double)kth) break;
        }
    }
    if (nb) flush();

    // ---- outputs: ids / d2 / counts
    if (P.out_ids || P.out_d2) {
#pragma unroll
        for (int s = 0; s < KP; ++s) {
            const int p = s * 32 + (int)lane;
            if (p < K) {
                const bool live = p < count;
                if (P.out_ids) P.out_ids[qi * K + p] = live ? (uint32_t)top.v[s] : 0xFFFFFFFFu;
                if (P.out_d2)
                    P.out_d2[qi * K + p] =
                        live ? __uint_as_float((uint32_t)(top.v[s] >> 32)) : __int_as_float(0x7f800000);
            }
        }
    }
    if (P.out_counts && lane == 0) P.out_counts[qi] = count;
    if (!P.out_targets && !render) continue;

    // ---- fused Eq. 6 (binary64, sequential in list order) + Eq. 7
    double L[3] = {0.0, 0.0, 0.0};
    if (count > 0) {
        const double r = sqrt((double)__uint_as_float((uint32_t)(top.at(count - 1) >> 32)));
        if (!(r < 1e-6)) {
            const double *wp = render ? P.hit_dir + 3 * qi : P.qw + 3 * qi;
            const double w[3] = {wp[0], wp[1], wp[2]};
            const double gv = P.phase[g];
            double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int s = 0; s < KP; ++s) {
                if (s * 32 >= count) break;
                const int p = s * 32 + (int)lane;
                double term[3] = {0.0, 0.0, 0.0};
                if (p < count) {
                    const uint32_t j = __ldg(P.inv + (uint32_t)top.v[s]);
                    const float4 a = __ldg(P.spay + 2 * (size_t)j), b = __ldg(P.spay + 2 * (size_t)j + 1);
                    const double c = w[0] * (double)a.x + w[1] * (double)a.y + w[2] * (double)a.z;
                    const double f = knn_hg_eval(gv, c);
                    term[0] = f * (double)a.w;
                    term[1] = f * (double)b.x;
                    term[2] = f * (double)b.y;
                }
                // sequential sum in list order (bit-identical to the oracle loop)
                const int n_here = min(32, count - s * 32);
                for (int k = 0; k < n_here; ++k) {
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) acc[ch] += __shfl_sync(0xffffffffu, term[ch], k);
                }
            }
            const double vol = (4.0 / 3.0) * 3.14159265358979323846 * (r * r * r);
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) L[ch] = acc[ch] / vol;
        }
    }
    if (render && lane == 0) {
        // compose term w_i * (sigma_s * L_i) into the sample's slot
        const HitRec &h = P.hits[qi];
        if (P.slot_f64) {
            double *sl = reinterpret_cast<double *>(P.slots) + 3 * (size_t)h.slot;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) sl[ch] = sl[ch] + P.w_i * (h.sigma_s * L[ch]);
        } else {
            float *sl = reinterpret_cast<float *>(P.slots) + 3 * (size_t)h.slot;
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) sl[ch] = sl[ch] + (float)(P.w_i * (h.sigma_s * L[ch]));
        }
    } else if (lane == 0) {
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
            const double v = L[ch];
            double t;
            if (v > 1.0) t = 0.0;
            else if (v > P.enc_threshold) t = -log10(v) / P.psi;
            else t = 1.0;
            P.out_targets[3 * qi + ch] = t;
        }
    }
    }  // query loop
}

// ---- K <= 64: one warp per query, collect-and-sort instead of merge ----------
// Same idea as the CTA kernel below at warp scale: probe the density from cell
// counts, collect every photon inside a ball expected to hold ~1.3 K of them
// into a per-warp shared buffer (ballot-compacted, coalesced row scans), sort
// the (d2, id) keys with a warp bitonic network and keep the first K.  ~4x
// fewer instructions per query than merging 32 keys at a time into the
// register top-K; exact for the same reason (all photons with d2 <= rho^2 are
// collected).  Queries whose ball cannot be sized within the buffer go to the
// merge kernel (fallback list).
constexpr int kSelWarps = 4;
// PF_KNN_MERGE=1 forces the merge kernel (A/B comparisons)
static bool knn_sel_disabled() {
    const char *e = std::getenv("PF_KNN_MERGE");
    return e && e[0] == '1';
}
constexpr int kSelCap = 256;

// Bitonic network stages for one k2 (block size of the current merge), strides
// jstart .. 1, on S*32 keys held as r[s] = element base + s*32 + lane: strides
// >= 32 exchange registers, smaller strides exchange lanes.  Directions come
// from the GLOBAL element index, so warps can run their parts of a larger
// network.
template <int S>
__device__ __forceinline__ void warp_bitonic_stage(uint64_t (&r)[S], unsigned lane, int base, int k2, int jstart) {
#pragma unroll
    for (int jj = jstart; jj > 0; jj >>= 1) {
        if (jj >= 32) {
            const int js = jj >> 5;
#pragma unroll
            for (int sI = 0; sI < S; ++sI) {
                if (sI & js) continue;
                const int i = base + sI * 32 + (int)lane;
                const bool up = (i & k2) == 0;
                const uint64_t a = r[sI], b = r[sI | js];
                const bool sw = (a > b) == up;
                r[sI] = sw ? b : a;
                r[sI | js] = sw ? a : b;
            }
        } else {
#pragma unroll
            for (int sI = 0; sI < S; ++sI) {
                const int i = base + sI * 32 + (int)lane;
                const uint64_t o = __shfl_xor_sync(0xffffffffu, r[sI], jj);
                const bool lower = (lane & jj) == 0;
                const bool up = (i & k2) == 0;
                // lower element keeps min when ascending
                const bool take_min = lower == up;
                r[sI] = take_min ? (o < r[sI] ? o : r[sI]) : (o > r[sI] ? o : r[sI]);
            }
        }
    }
}

// Warp bitonic sort of S*32 keys held as r[s] = element s*32 + lane.
template <int S>
__device__ __forceinline__ void warp_sort_regs(uint64_t (&r)[S], unsigned lane) {
#pragma unroll
    for (int k2 = 2; k2 <= S * 32; k2 <<= 1) warp_bitonic_stage<S>(r, lane, 0, k2, k2 >> 1);
}

template <int S>
__device__ __forceinline__ void sort_buf(uint64_t *buf, int n, unsigned lane) {
    uint64_t r[S];
#pragma unroll
    for (int sI = 0; sI < S; ++sI) {
        const int i = sI * 32 + (int)lane;
        r[sI] = i < n ? buf[i] : ~0ull;
    }
    warp_sort_regs<S>(r, lane);
#pragma unroll
    for (int sI = 0; sI < S; ++sI) buf[sI * 32 + (int)lane] = r[sI];
    __syncwarp();
}

// Ball-radius search: attempts before a query goes to the exact fallback.
constexpr int kKnnAttempts = 24;

// Distance from q to the phase's grid box (+ the binning slack): a lower bound
// on every photon distance of the phase.
__device__ __forceinline__ double knn_box_dist(const KnnGrid &Gp, const float q[3]) {
    double d2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double b0 = Gp.lo[a] - Gp.eps, b1 = Gp.lo[a] + (double)Gp.R[a] * Gp.h[a] + Gp.eps;
        const double d = (double)q[a] < b0 ? b0 - (double)q[a] : ((double)q[a] > b1 ? (double)q[a] - b1 : 0.0);
        d2 += d * d;
    }
    return sqrt(d2);
}

// Radius of the ball around q that contains the probe's cell cube (cells
// qc -+ ring, clamped to the grid): when the cube held >= K photons, no ball
// search ever needs to grow beyond it.
__device__ __forceinline__ double knn_cube_reach(const KnnGrid &Gp, const float q[3], const int qc[3], int ring) {
    double d2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int c0 = max(qc[a] - ring, 0), c1 = min(qc[a] + ring, Gp.R[a] - 1);
        const double e0 = Gp.lo[a] + (double)c0 * Gp.h[a] - Gp.eps, e1 = Gp.lo[a] + (double)(c1 + 1) * Gp.h[a] + Gp.eps;
        const double d = fmax(fabs((double)q[a] - e0), fabs((double)q[a] - e1));
        d2 += d * d;
    }
    return sqrt(d2) * 1.0001 + 1e-7;
}

// binary32 versions for the warp kernel, whose per-query radius bookkeeping
// otherwise costs ~8% of its instructions in binary64: lo/h/eps are the
// kernel's float copies of the grid, and every bound carries a relative margin
// in the safe direction (the bounds only steer the search; the collection test
// itself is exact).  ring < 0: the whole grid box; inner: distance to the box
// instead of to its farthest corner.
__device__ __forceinline__ float knn_extent_f(const float lo[3], const float h[3], const int R[3], float eps,
                                              const float q[3], const int qc[3], int ring, bool inner) {
    float d2 = 0.0f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int c0 = ring < 0 ? 0 : max(qc[a] - ring, 0), c1 = ring < 0 ? R[a] - 1 : min(qc[a] + ring, R[a] - 1);
        const float e0 = fmaf((float)c0, h[a], lo[a]) - eps, e1 = fmaf((float)(c1 + 1), h[a], lo[a]) + eps;
        const float d = inner ? (q[a] < e0 ? e0 - q[a] : (q[a] > e1 ? q[a] - e1 : 0.0f))
                              : fmaxf(fabsf(q[a] - e0), fabsf(q[a] - e1));
        d2 = fmaf(d, d, d2);
    }
    return sqrtf(d2);
}

// The 32*KP smallest of the n keys in buf, sorted ascending, back into
// buf[0, 32*KP) (list order = the oracle's).  Instead of one bitonic sort of
// all n keys rounded up to a power of two (112 register stages for
// 64 < n <= 128), the first KP runs of 32 are sorted together and every later
// run is folded in with the bitonic top-k merge: a run with no key below the
// current (32*KP)-th smallest is skipped; otherwise it is sorted (15 stages),
// reversed, min-combined with the top list's last 32 entries -- which leaves
// the 32*KP smallest as a bitonic sequence -- and merged (5*KP + 1 stages).
template <int KP>
__device__ __forceinline__ void select_topk(uint64_t *buf, int n, unsigned lane) {
    uint64_t top[KP];
#pragma unroll
    for (int sI = 0; sI < KP; ++sI) {
        const int i = sI * 32 + (int)lane;
        top[sI] = i < n ? buf[i] : ~0ull;
    }
    warp_sort_regs<KP>(top, lane);
    for (int run = KP; run * 32 < n; ++run) {
        const int i = run * 32 + (int)lane;
        uint64_t x[1] = {i < n ? buf[i] : ~0ull};
        const uint64_t kth = __shfl_sync(0xffffffffu, top[KP - 1], 31);
        if (!__any_sync(0xffffffffu, x[0] < kth)) continue;
        warp_sort_regs<1>(x, lane);
        const uint64_t rev = __shfl_sync(0xffffffffu, x[0], 31 - (int)lane);
        top[KP - 1] = rev < top[KP - 1] ? rev : top[KP - 1];
        warp_bitonic_stage<KP>(top, lane, 0, 32 * KP, 16 * KP);
    }
    __syncwarp();  // every lane has read its keys before the list overwrites them
#pragma unroll
    for (int sI = 0; sI < KP; ++sI) buf[sI * 32 + (int)lane] = top[sI];
    __syncwarp();
}

#ifndef PF_KNN_EARLY
#define PF_KNN_EARLY 1
#endif

template <int KP>
__global__ void __launch_bounds__(kSelWarps * 32, 8) k_knn_query_sel(const KnnParams P) {
    __shared__ uint64_t s_keys[kSelWarps][kSelCap];
    const unsigned lane = threadIdx.x & 31u;
    const int wi = threadIdx.x >> 5;
    uint64_t *buf = s_keys[wi];
    const size_t nq = P.nq;
    const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
    const int K = P.K;
    for (size_t qs = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; qs < nq; qs += nwarps) {
        const size_t qi = P.order ? (size_t)__ldg(P.order + qs) : qs;
        const float q[3] = {P.qx[3 * qi], P.qx[3 * qi + 1], P.qx[3 * qi + 2]};
        const int g = P.qg[qi];
        int count = 0, n = 0;
        bool fail = false;
        if (g < P.n_phases && P.grid[g].n > 0) {
            const KnnGrid &Gp = P.grid[g];
            int R[3], qc[3];
            float lo[3], h[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                R[a] = Gp.R[a];
                lo[a] = (float)Gp.lo[a];
                h[a] = (float)Gp.h[a];
                qc[a] = cell_axis((double)q[a], Gp.lo[a], Gp.inv_h[a], R[a]);
            }
            const float eps = (float)Gp.eps + 1e-6f;
            const float hminf = (float)Gp.hmin;
            const uint32_t cbase = Gp.cell_base;
            const int rmax = max(R[0], max(R[1], R[2]));
            auto gap = [&](int a, int c0, int c1) -> float {
                const float l = c0 == 0 ? -3.0e38f : fmaf((float)c0, h[a], lo[a]) - eps;
                const float u = c1 == R[a] - 1 ? 3.0e38f : fmaf((float)(c1 + 1), h[a], lo[a]) + eps;
                const float d = q[a] < l ? l - q[a] : (q[a] > u ? q[a] - u : 0.0f);
                return d * d;
            };
            // 1. density probe (cell counts only): cubes of half-size 0, 1, .., 4, 8,
            // 16, ... cells (tight density estimate near the photons; geometric
            // beyond, so a query far from them -- an empty corner of a traced map --
            // costs O(ring^2) row reads, not O(ring^3)), rows clamped to the grid
            int ring = 0;
            uint32_t cube = 0;
            for (;;) {
                uint32_t c = 0;
                const int x0 = max(qc[0] - ring, 0), x1 = min(qc[0] + ring, R[0] - 1);
                const int y0 = max(qc[1] - ring, 0), ny = min(qc[1] + ring, R[1] - 1) - y0 + 1;
                const int z0 = max(qc[2] - ring, 0), nz = min(qc[2] + ring, R[2] - 1) - z0 + 1;
                for (int r = (int)lane; r < ny * nz; r += 32) {
                    const int cz = z0 + r / ny, cy = y0 + r % ny;
                    const uint32_t row = cbase + (uint32_t)R[0] * ((uint32_t)cy + (uint32_t)R[1] * (uint32_t)cz);
                    c += __ldg(P.cell_start + row + x1 + 1) - __ldg(P.cell_start + row + x0);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                cube = c;
                if (cube >= (uint32_t)K || ring >= rmax) break;
                ring = min(ring < 4 ? ring + 1 : 2 * ring, rmax);
            }
            float vol = 1.0f;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int c0 = max(qc[a] - ring, 0), c1 = min(qc[a] + ring, R[a] - 1);
                vol *= (float)(c1 - c0 + 1) * h[a];
            }
            float rho = cbrtf(1.3f * (float)K * vol / (fmaxf((float)cube, 1.0f) * 4.18879020f));
            // a radius whose ball holds every photon of the phase (grid box + slack)
            const float all = knn_extent_f(lo, h, R, eps, q, qc, -1, false) * 1.001f + 1e-6f;
            // queries outside the phase's grid box (make_batch draws x ~ U^3 while a
            // traced map fills only the medium): no photon is closer than dbox, and
            // the probe measured the density at the box face nearest q
            const float dbox = knn_extent_f(lo, h, R, eps, q, qc, -1, true) * (1.0f - 1e-5f);
            // growth cap: the ball around the probe cube holds >= K photons
            const float reach =
                cube >= (uint32_t)K ? fminf(knn_extent_f(lo, h, R, eps, q, qc, ring, false) * 1.0001f + 1e-6f, all) : all;
            // bracket: a ball of radius lo_r holds fewer than K photons -- beyond the
            // box distance, the ball inside the previous (< K) probe cube when q is
            // in the grid -- one of radius hi_r overflowed; proposals outside bisect
            float lo_r = dbox > 0.0f ? dbox : (float)(ring <= 4 ? max(ring - 1, 0) : ring >> 1) * hminf * (1.0f - 1e-5f);
            float hi_r = 3.0e38f;
            rho = fminf(fmaxf(rho + dbox, lo_r), reach);
            const float ihx = (float)Gp.inv_h[0];
            // 2. collect every photon with d2 <= thr
            for (int attempt = 0;; ++attempt) {
                const float thr = fminf(fminf(rho * rho, 3.0e38f), P.r2);
                const int rc = (int)fminf(ceilf(sqrtf(thr) * 1.00001f / hminf) + 1.0f, (float)rmax);
                const int z0 = max(qc[2] - rc, 0), z1 = min(qc[2] + rc, R[2] - 1);
                const int y0 = max(qc[1] - rc, 0), y1 = min(qc[1] + rc, R[1] - 1);
                const int xl = max(qc[0] - rc, 0), xr = min(qc[0] + rc, R[0] - 1);
                const float gx = gap(0, xl, xr);
                n = 0;
                bool over = false;
                __syncwarp();  // the previous attempt's / query's buffer stores are ordered before ours
                // rows of the cube in chunks of 32: each lane sizes one row (ball
                // pruning, exact x-cell range through the binning function), a warp
                // scan concatenates the row segments and all 32 lanes stream the
                // concatenated candidates (independent, coalesced loads)
                const int ny = y1 - y0 + 1, nrows = (z1 - z0 + 1) * ny;
                // lane's row cursor (row r0 + lane), advanced 32 rows per chunk
                int cz = z0 + (int)lane / ny, cy = y0 + (int)lane % ny;
                const int dz32 = 32 / ny, dy32 = 32 % ny;
                for (int r0 = 0; r0 < nrows && !over; r0 += 32) {
                    const int r = r0 + (int)lane;
                    uint32_t b = 0, len = 0;
                    if (r < nrows) {
                        const float gyz = gap(2, cz, cz) + gap(1, cy, cy);
                        if ((gyz + gx) * (1.0f - 1e-5f) <= thr) {
                            // x-cells the ball reaches in this row: binary32 estimate of the
                            // binning function floor((x - lo) / h) with a 1e-3-cell margin
                            // (its rounding error is ~1e-4 cells), so the range is a superset
                            const float dxm = sqrtf(fmaxf(thr - gyz * (1.0f - 1e-5f), 0.0f)) * 1.0001f + 1e-6f;
                            const int xa = max(xl, (int)floorf((q[0] - dxm - lo[0]) * ihx - 1e-3f));
                            const int xb = min(xr, (int)floorf((q[0] + dxm - lo[0]) * ihx + 1e-3f));
                            if (xa <= xb) {
                                const uint32_t row = cbase + (uint32_t)R[0] * ((uint32_t)cy + (uint32_t)R[1] * (uint32_t)cz);
                                b = __ldg(P.cell_start + row + xa);
                                len = __ldg(P.cell_start + row + xb + 1) - b;
                            }
                        }
                    }
                    uint32_t incl = len;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                        if ((int)lane >= o) incl += t;
                    }
                    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                    for (uint32_t t0 = 0; t0 < total; t0 += 32) {
#if PF_KNN_EARLY
                        // the ball already overflowed the buffer: this attempt will be
                        // retried with a smaller ball, stop scanning (n is then a lower
                        // bound of the ball's count, so the shrink is conservative)
                        if (n > kSelCap) break;
#endif
                        const uint32_t t = t0 + lane;
                        // segment of candidate t: first lane whose inclusive offset exceeds t
                        int pos = 0;
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1) {
                            const uint32_t v = __shfl_sync(0xffffffffu, incl, pos + step - 1);
                            if (v <= t) pos += step;
                        }
                        const uint32_t seg_b = __shfl_sync(0xffffffffu, b, pos);
                        const uint32_t seg_excl = __shfl_sync(0xffffffffu, incl - len, pos);
                        uint64_t key = 0;
                        bool acc = false;
                        if (t < total) {
                            const float4 c = __ldg(&P.spos[seg_b + (t - seg_excl)]);
                            const float d2 = d2_rn(c, q);
                            acc = d2 <= thr;
                            key = ((uint64_t)__float_as_uint(d2) << 32) | __float_as_uint(c.w);
                        }
                        const unsigned m = __ballot_sync(0xffffffffu, acc);
                        const int slot = n + __popc(m & knn_lanemask_lt());
                        if (acc && slot < kSelCap) buf[slot] = key;
                        n += __popc(m);
                    }
                    if (n > kSelCap) over = true;
                    cy += dy32;
                    cz += dz32;
                    if (cy > y1) {
                        cy -= ny;
                        ++cz;
                    }
                }
                const bool short_ = n < K && thr < P.r2 && rho < all;
                // resize the ball from what this one held (density-corrected), bisecting
                // the bracket when the count is too steep in rho for the cube-root rule
                if (over && attempt < kKnnAttempts) {
                    hi_r = rho;
                    const float nx = rho * fmaxf(0.5f, fminf(0.9f, cbrtf(1.3f * (float)K / (float)n)));
                    rho = nx > lo_r ? nx : 0.5f * (lo_r + hi_r);
                    continue;
                }
                if (short_ && attempt < kKnnAttempts) {
                    lo_r = rho;
                    const float nx =
                        fminf(rho * fminf(3.0f, fmaxf(1.25f, cbrtf(1.3f * (float)K / fmaxf((float)n, 1.0f)))), fmaxf(reach, rho));
                    rho = nx < hi_r ? nx : 0.5f * (lo_r + hi_r);
                    continue;
                }
                fail = over || short_;
                break;
            }
            __syncwarp();
            if (!fail) {
                // 3. the K <= 32*KP smallest keys, sorted (bitonic top-k in registers)
                select_topk<KP>(buf, n, lane);
                count = min(n, K);
            }
        }
        if (fail) {
            if (lane == 0) P.fallback[atomicAdd(P.fallback_n, 1u)] = (uint32_t)qi;
            __syncwarp();
            continue;
        }
        // 4. outputs (list position p = s*32 + lane, like the merge kernel)
        uint64_t v[KP];
#pragma unroll
        for (int sI = 0; sI < KP; ++sI) {
            const int p2 = sI * 32 + (int)lane;
            v[sI] = p2 < count ? buf[p2] : ~0ull;
        }
        if (P.out_ids || P.out_d2) {
#pragma unroll
            for (int sI = 0; sI < KP; ++sI) {
                const int p2 = sI * 32 + (int)lane;
                if (p2 < K) {
                    const bool lv = p2 < count;
                    if (P.out_ids) P.out_ids[qi * K + p2] = lv ? (uint32_t)v[sI] : 0xFFFFFFFFu;
                    if (P.out_d2)
                        P.out_d2[qi * K + p2] = lv ? __uint_as_float((uint32_t)(v[sI] >> 32)) : __int_as_float(0x7f800000);
                }
            }
        }
        if (P.out_counts && lane == 0) P.out_counts[qi] = count;
        if (!P.out_targets) {
            __syncwarp();
            continue;
        }
        // fused Eq. 6 (binary64, sequential in list order) + Eq. 7
        double L[3] = {0.0, 0.0, 0.0};
        if (count > 0) {
            const double r = sqrt((double)__uint_as_float((uint32_t)(buf[count - 1] >> 32)));
            if (!(r < 1e-6)) {
                const double *wp = P.qw + 3 * qi;
                const double w[3] = {wp[0], wp[1], wp[2]};
                const double gv = P.phase[g];
                // per-photon terms -> shared memory (the key buffer is free now), then
                // lanes 0..2 sum one channel each sequentially in list order
                double *tb = reinterpret_cast<double *>(buf);  // 3 x 64 doubles <= kSelCap keys
                __syncwarp();  // every lane has read buf[count - 1] (r) before it is overwritten
#pragma unroll
                for (int sI = 0; sI < KP; ++sI) {
                    const int p2 = sI * 32 + (int)lane;
                    if (p2 < count) {
                        const uint32_t j = __ldg(P.inv + (uint32_t)v[sI]);
                        const float4 a = __ldg(P.spay + 2 * (size_t)j), b = __ldg(P.spay + 2 * (size_t)j + 1);
                        const double f = knn_hg_eval(gv, w[0] * (double)a.x + w[1] * (double)a.y + w[2] * (double)a.z);
                        tb[p2] = f * (double)a.w;
                        tb[64 + p2] = f * (double)b.x;
                        tb[128 + p2] = f * (double)b.y;
                    }
                }
                __syncwarp();
                double a2 = 0.0;
                if (lane < 3)
                    for (int k = 0; k < count; ++k) a2 += tb[64 * lane + k];
                __syncwarp();
                double acc[3];
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) acc[ch] = __shfl_sync(0xffffffffu, a2, ch);
                const double vol = (4.0 / 3.0) * 3.14159265358979323846 * (r * r * r);
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) L[ch] = acc[ch] / vol;
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const double vv = L[ch];
                double t;
                if (vv > 1.0) t = 0.0;
                else if (vv > P.enc_threshold) t = -log10(vv) / P.psi;
                else t = 1.0;
                P.out_targets[3 * qi + ch] = t;
            }
        }
        __syncwarp();
    }
}

// ---- large K: one CTA per query, select instead of merge -------------------
// For K in (64, 1024] the warp kernel's register top-K (merge 32 keys into a
// K-long bitonic list per flush) is latency- and spill-bound.  Here a CTA
//   1. probes the photon density around the query from cell counts only
//      (cube of cells until it holds >= K photons of the phase),
//   2. picks a radius rho whose ball should hold ~1.3 K photons and collects
//      EVERY photon with d2 <= min(rho^2, r_max^2) into shared memory as
//      (d2, id) keys (all warps stream the sorted rows, coalesced),
//   3. retries with a larger / smaller rho if the ball held < K photons (and
//      could hold more) or overflowed the buffer,
//   4. radix-selects the K-th smallest key (8 x 8-bit MSD passes), keeps the
//      keys <= it, bitonic-sorts them -> the same list as the oracle,
//   5. writes ids / d2 / count and Eq. 6 (binary64, sequential in list order)
//      + Eq. 7 exactly like the warp kernel.
// Exactness: every photon with d2 <= rho^2 is collected, so when >= K are
// found the K smallest keys of the whole phase are among them.
constexpr int kCtaThreads = 256;

// Block bitonic sort of P2 keys (power of two, 256..1024) in shared memory:
// every warp sorts its 128-key run in registers, then each merge level does
// its strides >= 128 in shared memory (block barriers) and its strides < 128
// in registers again -- 6 barrier stages for 1024 keys instead of 55.
__device__ __forceinline__ void cta_sort(uint64_t *a, int P2, int warp, unsigned lane, int tid) {
    const bool act = warp < P2 / 128;
    const int base = warp * 128;
    uint64_t r[4];
    if (act) {
#pragma unroll
        for (int sI = 0; sI < 4; ++sI) r[sI] = a[base + sI * 32 + (int)lane];
#pragma unroll
        for (int k2 = 2; k2 <= 128; k2 <<= 1) warp_bitonic_stage<4>(r, lane, base, k2, k2 >> 1);
#pragma unroll
        for (int sI = 0; sI < 4; ++sI) a[base + sI * 32 + (int)lane] = r[sI];
    }
    __syncthreads();
    for (int k2 = 256; k2 <= P2; k2 <<= 1) {
        for (int jj = k2 >> 1; jj >= 128; jj >>= 1) {
            for (int pI = tid; pI < P2 / 2; pI += kCtaThreads) {
                const int i = (pI / jj) * 2 * jj + (pI % jj), ij = i + jj;
                const uint64_t x = a[i], y = a[ij];
                if ((x > y) == ((i & k2) == 0)) {
                    a[i] = y;
                    a[ij] = x;
                }
            }
            __syncthreads();
        }
        if (act) {
#pragma unroll
            for (int sI = 0; sI < 4; ++sI) r[sI] = a[base + sI * 32 + (int)lane];
            warp_bitonic_stage<4>(r, lane, base, k2, 64);
#pragma unroll
            for (int sI = 0; sI < 4; ++sI) a[base + sI * 32 + (int)lane] = r[sI];
        }
        __syncthreads();
    }
}
constexpr int kCtaCap = 4096;  // collected keys per query (32 KB)
#ifndef PF_KNN_CTA_TGT
#define PF_KNN_CTA_TGT 2.5  // photons a K7c ball is sized to hold, in units of K (A/B: 1.3 / 2.0 / 2.5 / 3.0 -> 8.04 / 7.79 / 7.68 / 7.65 ms per 2^16 K=1024 targets; 2.5 keeps the expected count well inside the 4 K buffer)
#endif

__global__ void __launch_bounds__(kCtaThreads, 5) k_knn_query_cta(const KnnParams P) {
    __shared__ uint64_t keys[kCtaCap];
    __shared__ uint64_t sel[1024];
    __shared__ uint32_t hist[256];
    double *terms = reinterpret_cast<double *>(keys);  // 3 x 1024, keys are dead once `sel` is sorted
    __shared__ int s_n, s_over, s_cnt;
    __shared__ uint64_t s_prefix;
    __shared__ int s_need, s_unique;
    __shared__ unsigned long long s_cube;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int K = P.K;
    for (size_t qs = blockIdx.x; qs < P.nq; qs += gridDim.x) {
        const size_t qi = P.order ? (size_t)__ldg(P.order + qs) : qs;
        const float q[3] = {P.qx[3 * qi], P.qx[3 * qi + 1], P.qx[3 * qi + 2]};
        const int g = P.qg[qi];
        int count = 0;
        uint64_t kth = ~0ull;
        const bool live = g < P.n_phases && P.grid[g].n > 0;
        if (live) {
            const KnnGrid &Gp = P.grid[g];
            int R[3], qc[3];
            float lo[3], h[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                R[a] = Gp.R[a];
                lo[a] = (float)Gp.lo[a];
                h[a] = (float)Gp.h[a];
                qc[a] = cell_axis((double)q[a], Gp.lo[a], Gp.inv_h[a], R[a]);
            }
            const float eps = (float)Gp.eps + 1e-6f;
            const uint32_t cbase = Gp.cell_base;
            const int rmax = max(R[0], max(R[1], R[2]));
            auto gap = [&](int a, int c0, int c1) -> float {
                const float l = c0 == 0 ? -3.0e38f : fmaf((float)c0, h[a], lo[a]) - eps;
                const float u = c1 == R[a] - 1 ? 3.0e38f : fmaf((float)(c1 + 1), h[a], lo[a]) + eps;
                const float d = q[a] < l ? l - q[a] : (q[a] > u ? q[a] - u : 0.0f);
                return d * d;
            };
            // 1. density probe: smallest cube of cells around qc holding >= K photons
            int ring = 0;  // half-sizes 0..4, 8, 16, ... (as in k_knn_query_sel)
            unsigned long long cube = 0;
            for (;;) {
                if (tid == 0) s_cube = 0ull;
                __syncthreads();
                const int x0 = max(qc[0] - ring, 0), x1 = min(qc[0] + ring, R[0] - 1);
                const int y0 = max(qc[1] - ring, 0), ny = min(qc[1] + ring, R[1] - 1) - y0 + 1;
                const int z0 = max(qc[2] - ring, 0), nz = min(qc[2] + ring, R[2] - 1) - z0 + 1;
                for (int r = tid; r < ny * nz; r += kCtaThreads) {
                    const int cz = z0 + r / ny, cy = y0 + r % ny;
                    const uint32_t row = cbase + (uint32_t)R[0] * ((uint32_t)cy + (uint32_t)R[1] * (uint32_t)cz);
                    atomicAdd(&s_cube, (unsigned long long)(__ldg(P.cell_start + row + x1 + 1) -
                                                           __ldg(P.cell_start + row + x0)));
                }
                __syncthreads();
                cube = s_cube;
                __syncthreads();
                if (cube >= (unsigned long long)K || ring >= rmax) break;
                ring = min(ring < 4 ? ring + 1 : 2 * ring, rmax);
            }
            // 2. radius whose ball should hold ~1.3 K photons (cube volume / count)
            double vol = 1.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int c0 = max(qc[a] - ring, 0), c1 = min(qc[a] + ring, R[a] - 1);
                vol *= (double)(c1 - c0 + 1) * (double)h[a];
            }
            double rho = cbrt(PF_KNN_CTA_TGT * (double)K * vol / (fmax((double)cube, 1.0) * 4.18879020478639098));
            // a radius whose ball holds every photon of the phase (grid box + slack)
            double all = 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double b0 = Gp.lo[a] - Gp.eps, b1 = Gp.lo[a] + (double)R[a] * Gp.h[a] + Gp.eps;
                const double d = fmax(fabs((double)q[a] - b0), fabs((double)q[a] - b1));
                all += d * d;
            }
            all = sqrt(all) * 1.001 + 1e-6;
            const double dbox = knn_box_dist(Gp, q);  // as in k_knn_query_sel
            const double reach = cube >= (unsigned long long)K ? fmin(knn_cube_reach(Gp, q, qc, ring), all) : all;
            double lo_r = dbox > 0.0 ? dbox * (1.0 - 1e-6) : (double)(ring <= 4 ? max(ring - 1, 0) : ring >> 1) * (double)Gp.hmin * (1.0 - 1e-6);
            double hi_r = 3.0e38;
            rho = fmin(fmax(rho + dbox, lo_r), reach);
            for (int attempt = 0;; ++attempt) {
                // 3. collect every photon with d2 <= thr
                const float rho2 = (float)fmin(rho * rho, 3.0e38);
                const float thr = fminf(rho2, P.r2);
                const int rc = (int)fmin(ceil(sqrt((double)thr) / (double)Gp.hmin) + 1.0, (double)rmax);
                if (tid == 0) {
                    s_n = 0;
                    s_over = 0;
                }
                __syncthreads();
                // rows (cz, cy) of the cell cube, one z-slice per warp; per row only the
                // x-cells the ball can reach (+-1 cell of slack for binary32 rounding)
                const int z0 = max(qc[2] - rc, 0), z1 = min(qc[2] + rc, R[2] - 1);
                const int y0 = max(qc[1] - rc, 0), y1 = min(qc[1] + rc, R[1] - 1);
                const int xl = max(qc[0] - rc, 0), xr = min(qc[0] + rc, R[0] - 1);
                const float gx = gap(0, xl, xr);
                for (int cz = z0 + warp; cz <= z1; cz += kCtaThreads / 32) {
                    const float gz = gap(2, cz, cz);
                    if ((gz + gx) * (1.0f - 1e-5f) > thr) continue;
                    for (int cy = y0; cy <= y1; ++cy) {
#if PF_KNN_EARLY
                        // the ball already overflowed the buffer: the attempt is retried
                        if (*(volatile int *)&s_over) break;
#endif
                        const float gyz = gz + gap(1, cy, cy);
                        if ((gyz + gx) * (1.0f - 1e-5f) > thr) continue;
                        const float dxm = sqrtf(fmaxf(thr - gyz * (1.0f - 1e-5f), 0.0f)) * 1.0001f + eps;
                        const int xa = max(xl, (int)floorf((q[0] - dxm - lo[0]) / h[0]) - 1);
                        const int xb = min(xr, (int)floorf((q[0] + dxm - lo[0]) / h[0]) + 1);
                        if (xa > xb) continue;
                        const uint32_t row = cbase + (uint32_t)R[0] * ((uint32_t)cy + (uint32_t)R[1] * (uint32_t)cz);
                        const uint32_t b = __ldg(P.cell_start + row + xa), e = __ldg(P.cell_start + row + xb + 1);
                        for (uint32_t j = b + lane; j < e; j += 32) {
#if PF_KNN_EARLY
                            if (*(volatile int *)&s_over) break;
#endif
                            const float4 c = __ldg(&P.spos[j]);
                            const float d2 = d2_rn(c, q);
                            if (d2 <= thr) {
                                const int slot = atomicAdd(&s_n, 1);
                                if (slot < kCtaCap) keys[slot] = ((uint64_t)__float_as_uint(d2) << 32) | __float_as_uint(c.w);
                                else s_over = 1;
                            }
                        }
                    }
                }
                __syncthreads();
                const int n = s_n;
                const bool over = s_over != 0;
                const bool short_ = n < K && thr < P.r2 && rho < all;
                __syncthreads();
                if (over && attempt < kKnnAttempts) {
                    hi_r = rho;
                    rho = 0.8 * rho > lo_r ? 0.8 * rho : 0.5 * (lo_r + hi_r);
                    continue;
                }
                if (short_ && attempt < kKnnAttempts) {
                    lo_r = rho;
                    const double nx = fmin(rho * 1.5, fmax(reach, rho));
                    rho = nx < hi_r ? nx : 0.5 * (lo_r + hi_r);
                    continue;
                }
                if (over || short_) {
                    count = -1;  // give up (never observed): the warp kernel redoes this query
                    break;
                }
                // 4. K-th smallest key (radix select, MSD 8 bits at a time); stops
                // as soon as the K-th key's bin holds it alone: the selection is then
                // "prefix <= the K-th key's prefix" (the first 2-3 passes for
                // distinct distances instead of all 8)
                count = min(n, K);
                uint64_t kmask = ~0ull;
                if (n > K) {
                    if (tid == 0) {
                        s_prefix = 0ull;
                        s_need = K;
                        s_unique = 0;
                    }
                    for (int pass = 0; pass < 8; ++pass) {
                        const int shift = 56 - 8 * pass;
                        for (int i = tid; i < 256; i += kCtaThreads) hist[i] = 0u;
                        __syncthreads();
                        const uint64_t pre = s_prefix;
                        const uint64_t pmask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
                        for (int i = tid; i < n; i += kCtaThreads)
                            if ((keys[i] & pmask) == pre) atomicAdd(&hist[(keys[i] >> shift) & 255u], 1u);
                        __syncthreads();
                        if (warp == 0) {
                            // bin holding the need-th key: lane-local sums of 8 bins, warp scan
                            const int need = s_need;
                            uint32_t loc[8], lsum = 0;
#pragma unroll
                            for (int b2 = 0; b2 < 8; ++b2) {
                                loc[b2] = hist[lane * 8 + b2];
                                lsum += loc[b2];
                            }
                            uint32_t incl = lsum;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                                if (lane >= o) incl += v;
                            }
                            const uint32_t excl = incl - lsum;
                            const unsigned hit = __ballot_sync(0xffffffffu, (int)incl >= need);
                            const int src = __ffs(hit) - 1;
                            if (lane == src) {
                                int left = need - (int)excl, bsel = lane * 8 + 7;
#pragma unroll
                                for (int b2 = 0; b2 < 8; ++b2) {
                                    if ((int)loc[b2] >= left) {
                                        bsel = lane * 8 + b2;
                                        break;
                                    }
                                    left -= (int)loc[b2];
                                }
                                s_need = left;
                                s_prefix = pre | ((uint64_t)bsel << shift);
                                s_unique = hist[bsel] == 1u ? 1 : 0;
                            }
                        }
                        __syncthreads();
                        if (s_unique) {
                            kmask = ~0ull << shift;
                            break;
                        }
                    }
                    kth = s_prefix;  // with kmask: the K-th key's prefix (keys are distinct)
                } else {
                    kth = ~0ull;
                }
                // compact the selected keys, pad to a power of two, bitonic sort
                if (tid == 0) s_cnt = 0;
                __syncthreads();
                for (int i = tid; i < n; i += kCtaThreads)
                    if ((keys[i] & kmask) <= kth) sel[atomicAdd(&s_cnt, 1)] = keys[i];
                __syncthreads();
                int P2 = 32;
                while (P2 < count) P2 <<= 1;
                for (int i = count + tid; i < P2; i += kCtaThreads) sel[i] = ~0ull;
                __syncthreads();
                if (P2 >= 256) {
                    cta_sort(sel, P2, warp, lane, tid);
                } else {
                    if (warp == 0) {
                        if (P2 == 32) sort_buf<1>(sel, count, lane);
                        else if (P2 == 64) sort_buf<2>(sel, count, lane);
                        else sort_buf<4>(sel, count, lane);
                    }
                    __syncthreads();
                }
                break;
            }
        }
        if (count < 0) {
            // fallback marker: counts = -1 tells the host to rerun on the warp kernel
            if (tid == 0 && P.out_counts) P.out_counts[qi] = -1;
            if (tid == 0 && P.fallback) P.fallback[atomicAdd(P.fallback_n, 1u)] = (uint32_t)qi;
            __syncthreads();
            continue;
        }
        // 5. outputs
        for (int p2 = tid; p2 < K; p2 += kCtaThreads) {
            const bool lv = p2 < count;
            if (P.out_ids) P.out_ids[qi * K + p2] = lv ? (uint32_t)sel[p2] : 0xFFFFFFFFu;
            if (P.out_d2) P.out_d2[qi * K + p2] = lv ? __uint_as_float((uint32_t)(sel[p2] >> 32)) : __int_as_float(0x7f800000);
        }
        if (P.out_counts && tid == 0) P.out_counts[qi] = count;
        if (P.out_targets) {
            double r = 0.0;
            if (count > 0) r = sqrt((double)__uint_as_float((uint32_t)(sel[count - 1] >> 32)));
            const bool zero = count == 0 || r < 1e-6;
            if (!zero) {
                const double w[3] = {P.qw[3 * qi], P.qw[3 * qi + 1], P.qw[3 * qi + 2]};
                const double gv = P.phase[g];
                for (int p2 = tid; p2 < count; p2 += kCtaThreads) {
                    const uint32_t j = __ldg(P.inv + (uint32_t)sel[p2]);
                    const float4 a = __ldg(P.spay + 2 * (size_t)j), b = __ldg(P.spay + 2 * (size_t)j + 1);
                    const double f = knn_hg_eval(gv, w[0] * (double)a.x + w[1] * (double)a.y + w[2] * (double)a.z);
                    terms[p2] = f * (double)a.w;
                    terms[1024 + p2] = f * (double)b.x;
                    terms[2048 + p2] = f * (double)b.y;
                }
            }
            __syncthreads();
            if (tid < 3) {
                double L = 0.0;
                if (!zero) {
                    // sequential in list order (bit-identical to the oracle loop)
                    double acc = 0.0;
                    const double *tc = terms + 1024 * tid;
                    for (int p2 = 0; p2 < count; ++p2) acc += tc[p2];
                    L = acc / ((4.0 / 3.0) * 3.14159265358979323846 * (r * r * r));
                }
                double t;
                if (L > 1.0) t = 0.0;
                else if (L > P.enc_threshold) t = -log10(L) / P.psi;
                else t = 1.0;
                P.out_targets[3 * qi + tid] = t;
            }
        }
        __syncthreads();
    }
}

// make_batch query generation (oracle or_make_queries).
__device__ __forceinline__ uint32_t mq_u32(uint64_t &st, uint64_t inc) {
    uint64_t old = st;
    st = old * 6364136223846793005ULL + inc;
    uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
    uint32_t rot = (uint32_t)(old >> 59);
    return __funnelshift_r(xs, xs, rot);
}
__device__ __forceinline__ double mq_double(uint64_t &st, uint64_t inc) {
    uint64_t hi = mq_u32(st, inc);
    uint64_t lo = mq_u32(st, inc);
    return (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;
}

__global__ void k_make_queries(uint64_t initstate, uint64_t base, size_t batch, int n_phases,
                               float *x3, double *w3, uint8_t *gidx) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= batch) return;
    const uint64_t inc = ((base + i) << 1) | 1ull;
    uint64_t st = 0;
    mq_u32(st, inc);
    st += initstate;
    mq_u32(st, inc);
#pragma unroll
    for (int a = 0; a < 3; ++a) x3[3 * i + a] = (float)mq_double(st, inc);
    const double z = 1.0 - 2.0 * mq_double(st, inc);
    const double phi = (2.0 * 3.14159265358979323846) * mq_double(st, inc);
    const double t = 1.0 - z * z;
    const double rr = sqrt(t > 0.0 ? t : 0.0);
    w3[3 * i] = rr * cos(phi);
    w3[3 * i + 1] = rr * sin(phi);
    w3[3 * i + 2] = z;
    gidx[i] = (uint8_t)(((uint64_t)mq_u32(st, inc) * (uint64_t)n_phases) >> 32);
}

// ---- host --------------------------------------------------------------
cudaError_t knn_bbox(const PhotonRec *ph, size_t n, int n_phases, uint32_t *mins, uint32_t *maxs,
                     uint32_t *counts, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    k_knn_bbox<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ph, n, n_phases, mins, maxs, counts);
    return cudaGetLastError();
}

cudaError_t knn_sort(const PhotonRec *ph, size_t n, const KnnParams &P, KnnBuffers &B,
                     cudaStream_t st) {
    cudaError_t e;
    const size_t ncells = (size_t)P.total_cells + 1;
    if ((e = B.keys.ensure(n * 4)) || (e = B.vals.ensure(n * 4)) || (e = B.keys2.ensure(n * 4)) ||
        (e = B.vals2.ensure(n * 4)) || (e = B.hist.ensure(ncells * 4)) ||
        (e = B.cell_start.ensure((ncells + 1) * 4)) || (e = B.spos.ensure(n * 16)) ||
        (e = B.spay.ensure(n * 32)) || (e = B.inv.ensure(n * 4)))
        return e;
    cudaMemsetAsync(B.hist.p, 0, ncells * 4, st);
    if (n) {
        k_knn_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ph, n, P, (uint32_t *)B.keys.p,
                                                                (uint32_t *)B.vals.p, (uint32_t *)B.hist.p);
        if ((e = cudaGetLastError())) return e;
    }
    // stable radix sort by cell key keeps ids ascending inside a cell
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) <= (uint64_t)P.total_cells) ++end_bit;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (uint32_t *)B.keys.p, (uint32_t *)B.keys2.p,
                                    (uint32_t *)B.vals.p, (uint32_t *)B.vals2.p, (int)n, 0, end_bit, st);
    if ((e = B.temp.ensure(tmp + 256))) return e;
    cub::DeviceRadixSort::SortPairs(B.temp.p, tmp, (uint32_t *)B.keys.p, (uint32_t *)B.keys2.p,
                                    (uint32_t *)B.vals.p, (uint32_t *)B.vals2.p, (int)n, 0, end_bit, st);
    size_t tmp2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp2, (uint32_t *)B.hist.p, (uint32_t *)B.cell_start.p,
                                  (int)ncells, st);
    if ((e = B.temp2.ensure(tmp2 + 256))) return e;
    cub::DeviceScan::ExclusiveSum(B.temp2.p, tmp2, (uint32_t *)B.hist.p, (uint32_t *)B.cell_start.p,
                                  (int)ncells, st);
    if (n) {
        k_knn_gather<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ph, n, (const uint32_t *)B.vals2.p,
                                                                  (float4 *)B.spos.p, (float4 *)B.spay.p,
                                                                  (uint32_t *)B.inv.p);
        if ((e = cudaGetLastError())) return e;
    }
    return cudaSuccess;
}

// (phase, 30-bit Morton code of the position in [0,1]^3) visit-order keys
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3FFu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_knn_order_keys(const float *x3, const uint8_t *g, size_t n, uint32_t *keys, uint32_t *idx) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) c[a] = (uint32_t)(__saturatef(x3[3 * i + a]) * 1023.0f);
    keys[i] = ((uint32_t)min((int)g[i], 3) << 30) | (spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2));
    idx[i] = (uint32_t)i;
}

cudaError_t knn_order(const float *x3, const uint8_t *g, size_t n, KnnBuffers &B, const uint32_t **order,
                      cudaStream_t st) {
    cudaError_t e;
    if ((e = B.qk.ensure(n * 4)) || (e = B.qi.ensure(n * 4)) || (e = B.qk2.ensure(n * 4)) || (e = B.qi2.ensure(n * 4)))
        return e;
    k_knn_order_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x3, g, n, (uint32_t *)B.qk.p, (uint32_t *)B.qi.p);
    if ((e = cudaGetLastError())) return e;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, (uint32_t *)B.qk.p, (uint32_t *)B.qk2.p, (uint32_t *)B.qi.p,
                                    (uint32_t *)B.qi2.p, (int)n, 0, 32, st);
    if ((e = B.temp3.ensure(tmp + 256))) return e;
    cub::DeviceRadixSort::SortPairs(B.temp3.p, tmp, (uint32_t *)B.qk.p, (uint32_t *)B.qk2.p, (uint32_t *)B.qi.p,
                                    (uint32_t *)B.qi2.p, (int)n, 0, 32, st);
    *order = (const uint32_t *)B.qi2.p;
    return cudaGetLastError();
}

cudaError_t knn_query(const KnnParams &P, cudaStream_t st) {
    if (P.nq == 0) return cudaSuccess;
    if (P.K > 64 && P.fallback) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // resident CTAs per SM (5: 48 registers, 43 KB static smem each; the
        // 4th and 5th CTA hide the collect/select barrier stalls: 15.3 -> 12.8
        // ms per 2^16 targets at K = 1024); PF_KNN_CTA_PER_SM overrides
        static const int per_sm = [] {
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_knn_query_cta, kCtaThreads, 0);
            const char *e = std::getenv("PF_KNN_CTA_PER_SM");
            const int v = e ? std::atoi(e) : occ;
            return v >= 1 && v <= 8 ? v : 3;
        }();
        const unsigned blocks = (unsigned)std::min<size_t>(P.nq, (size_t)sms * per_sm);
        k_knn_query_cta<<<blocks, kCtaThreads, 0, st>>>(P);
        return cudaGetLastError();
    }
    const unsigned blocks = (unsigned)((P.nq * 32 + 127) / 128);
    const int kp = (P.K + 31) / 32;
    if (kp <= 1) k_knn_query<1, false><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 2) k_knn_query<2, false><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 4) k_knn_query<4, false><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 8) k_knn_query<8, false><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 16) k_knn_query<16, false><<<blocks, 128, 0, st>>>(P);
    else k_knn_query<32, false><<<blocks, 128, 0, st>>>(P);
    return cudaGetLastError();
}

static int knn_sms() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

cudaError_t knn_query_auto(KnnParams P, KnnBuffers &B, cudaStream_t st) {
    if (P.nq == 0) return cudaSuccess;
    cudaError_t e;
    if (P.K <= 64 && !knn_sel_disabled()) {
        if ((e = B.fb.ensure(P.nq * 4)) || (e = B.fbn.ensure(16))) return e;
        P.fallback = (uint32_t *)B.fb.p;
        P.fallback_n = (unsigned *)B.fbn.p;
        if ((e = cudaMemsetAsync(B.fbn.p, 0, 4, st))) return e;
        const unsigned blocks = (unsigned)std::min<size_t>((P.nq + kSelWarps - 1) / kSelWarps, (size_t)knn_sms() * 16);
        if (P.K <= 32) k_knn_query_sel<1><<<blocks, kSelWarps * 32, 0, st>>>(P);
        else k_knn_query_sel<2><<<blocks, kSelWarps * 32, 0, st>>>(P);
        if ((e = cudaGetLastError())) return e;
        unsigned n_fb = 0;
        if ((e = cudaMemcpyAsync(&n_fb, B.fbn.p, 4, cudaMemcpyDeviceToHost, st))) return e;
        if ((e = cudaStreamSynchronize(st))) return e;
        if (n_fb) {
            KnnParams Q = P;
            Q.fallback = nullptr;
            Q.order = (const uint32_t *)B.fb.p;
            Q.nq = n_fb;
            return knn_query(Q, st);
        }
        return cudaSuccess;
    }
    if (P.K <= 64) {
        P.fallback = nullptr;
        return knn_query(P, st);
    }
    if ((e = B.fb.ensure(P.nq * 4)) || (e = B.fbn.ensure(16))) return e;
    P.fallback = (uint32_t *)B.fb.p;
    P.fallback_n = (unsigned *)B.fbn.p;
    if ((e = cudaMemsetAsync(B.fbn.p, 0, 4, st))) return e;
    if ((e = knn_query(P, st))) return e;
    unsigned n_fb = 0;
    if ((e = cudaMemcpyAsync(&n_fb, B.fbn.p, 4, cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    if (n_fb) {  // exact fallback: the warp kernel on the unresolved queries
        KnnParams Q = P;
        Q.fallback = nullptr;
        Q.order = (const uint32_t *)B.fb.p;
        Q.nq = n_fb;
        return knn_query(Q, st);
    }
    return cudaSuccess;
}

// Render mode keeps the merge kernel: hit records come in tracer order over a
// strongly clustered traced map, where the collect-and-sort kernel's ball
// sizing needs retries (measured 24.1 vs 20.4 ms per config-2 frame).
cudaError_t knn_query_render(const KnnParams &P, int sms, cudaStream_t st) {
    if (P.nq == 0) return cudaSuccess;
    // persistent: enough warps to fill the SMs, grid-striding over the device-side hit count
    const unsigned blocks = (unsigned)std::min<size_t>((P.nq * 32 + 127) / 128, (size_t)sms * 16);
    const int kp = (P.K + 31) / 32;
    if (kp <= 1) k_knn_query<1, true><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 2) k_knn_query<2, true><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 4) k_knn_query<4, true><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 8) k_knn_query<8, true><<<blocks, 128, 0, st>>>(P);
    else if (kp <= 16) k_knn_query<16, true><<<blocks, 128, 0, st>>>(P);
    else k_knn_query<32, true><<<blocks, 128, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t knn_make_queries(uint64_t initstate, uint64_t base, size_t batch, int n_phases,
                             float *x3, double *w3, uint8_t *gidx, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    k_make_queries<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(initstate, base, batch, n_phases,
                                                                     x3, w3, gidx);
    return cudaGetLastError();
}

}  // namespace pfk
