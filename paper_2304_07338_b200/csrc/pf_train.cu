// pf_train.cu -- photon-field training on the device: train_step (SPEC.md:
// 403-411) = forward, relative-MSE loss, full backward through the MLP and
// the hash-grid interpolation into the embedding tables, Adam with the
// SPEC's learning-rate schedule; pinned in oracle/pf_oracle.c
// or_train_grad / or_adam_update (binary64, finite-difference checked).
//
// B200 design (binary32 master parameters, like tiny-cuda-nn's fp32 master
// copy; the fp16 tables / tcgen05 MLP of the renderer are refreshed from
// them by pf_train_commit):
//   k_train_pack   W_L -> W_L^T image (one per step, ~134 KB for the paper
//                  field) that every CTA pulls into shared memory;
//   k_train_fwd    one thread per query: hash-grid encode (the renderer's
//                  addressing, pf_hashgrid.cuh) fused with layer 0, then the
//                  hidden layers from smem-broadcast W^T rows; activations are
//                  kept feature-major [k][query] (coalesced across the warp)
//                  for the backward pass; loss term + dloss/dz_H;
//   k_train_bwd    one thread per query: dz_{L-1} = (W_L^T dz_L) . [a_L > 0],
//                  then dfeat = W_0^T dz_0 (feature-major rows);
//   k_train_scatter one thread per (query, level), level-major grid (the
//                  level's gradient slab stays L2-resident): dfeat scattered
//                  into the tables with fixed-point integer atomics
//                  (deterministic: integer adds are associative) + touched
//                  flags (sparse Adam);
//   k_train_wgrad  dW_L = dZ_L . In_L^T (+ db_L via a virtual ones row) as
//                  a tiled SIMT GEMM over query chunks -> per-chunk partials;
//   k_train_wsum   partials summed in chunk order (deterministic);
//   k_train_adam   Adam with bias correction on the global step: every MLP
//                  parameter, table parameters of touched entries only.
// Every reduction has a fixed order, so a step is bit-reproducible.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "pf_hashgrid.cuh"
#include "pf_train.h"

namespace pfk {

namespace {

// 512 threads share one smem W^T image (134 KB for the paper field, one CTA
// per SM) so an SM still runs 16 warps; 128 registers per thread fit.
constexpr int kThreads = 512;
constexpr int kChunk = 256;  // queries per weight-gradient partial
#ifndef PF_TRAIN_SMEM_SCATTER
#define PF_TRAIN_SMEM_SCATTER 1
#endif

__device__ __forceinline__ float relu(float x) { return x < 0.f ? 0.f : x; }

__device__ __forceinline__ void fix_add(unsigned long long *p, float v) {
    const long long fx = __double2ll_rn((double)v * kGradFix);
    if (fx != 0) atomicAdd(p, (unsigned long long)fx);
}

// W_L (row-major [o][k] in the flat vector) -> W_L^T [k][o] image + biases.
__global__ void k_train_pack(const TrainParams T, const uint32_t *off_w, float *img, int total_layers) {
    const int L = blockIdx.y;
    if (L >= total_layers) return;
    const int nin = L == 0 ? T.din : 64, nout = L < T.H ? 64 : 3, os = L < T.H ? 64 : T.out_stride;
    const float *W = T.params + off_w[L];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nin * os; i += gridDim.x * blockDim.x) {
        const int k = i / os, o = i - k * os;
        img[T.wt_off[L] + i] = o < nout ? W[(size_t)o * nin + k] : 0.f;
    }
    if (blockIdx.x == 0)
        for (int o = threadIdx.x; o < os; o += blockDim.x)
            img[T.b_off[L] + o] = o < nout ? W[(size_t)nout * nin + o] : 0.f;
}

__device__ __forceinline__ void load_image(const float4 *img, int n4, float4 *sm) {
    for (int i = threadIdx.x; i < n4; i += blockDim.x) sm[i] = __ldg(img + i);
    __syncthreads();
}

// acc[0..63] += W^T[k][0..63] * x  (smem broadcast rows)
__device__ __forceinline__ void axpy64(const float *row, float x, float *acc) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float4 w = r4[j];
        acc[4 * j] = fmaf(w.x, x, acc[4 * j]);
        acc[4 * j + 1] = fmaf(w.y, x, acc[4 * j + 1]);
        acc[4 * j + 2] = fmaf(w.z, x, acc[4 * j + 2]);
        acc[4 * j + 3] = fmaf(w.w, x, acc[4 * j + 3]);
    }
}

__device__ __forceinline__ float dot64(const float *row, const float *v) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float4 w = r4[j];
        s0 = fmaf(w.x, v[4 * j], s0);
        s1 = fmaf(w.y, v[4 * j + 1], s1);
        s2 = fmaf(w.z, v[4 * j + 2], s2);
        s3 = fmaf(w.w, v[4 * j + 3], s3);
    }
    return (s0 + s1) + (s2 + s3);
}

// Features of one level (binary32 master tables, same addressing as the renderer).
template <int D, int F>
__device__ __forceinline__ void level_feats(const TrainParams &T, int lv, const float *pin, float *feat) {
    const FieldLevel L = T.lv[lv];
    uint32_t c[D];
    float f[D];
    level_cell<D>(L, pin, c, f);
#pragma unroll
    for (int k = 0; k < F; ++k) feat[k] = 0.f;
#pragma unroll
    for (int corner = 0; corner < (1 << D); ++corner) {
        const float w = corner_weight<D>(f, corner);
        const float *e = T.params + L.offset_halves + (size_t)corner_index<D>(L, c, corner) * F;
#pragma unroll
        for (int k = 0; k < F; k += 2) {
            const float2 v = __ldg(reinterpret_cast<const float2 *>(e + k));
            feat[k] = fmaf(w, v.x, feat[k]);
            feat[k + 1] = fmaf(w, v.y, feat[k + 1]);
        }
    }
}

template <int FP, int FD>
__global__ void __launch_bounds__(kThreads, 1) k_train_fwd(const TrainParams T, const float4 *img, int n4) {
    extern __shared__ float4 sm4[];
    load_image(img, n4, sm4);
    const float *sm = reinterpret_cast<const float *>(sm4);
    const size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (q >= T.n) return;
    const size_t ld = T.ld;
    float acc[64];
#pragma unroll
    for (int o = 0; o < 64; ++o) acc[o] = sm[T.b_off[0] + o];
    // ---- encode fused with layer 0 (features also kept for dW_0)
    const float *W0 = sm + T.wt_off[0];
    {
        const float pin[3] = {__saturatef(T.qx[3 * q]), __saturatef(T.qx[3 * q + 1]), __saturatef(T.qx[3 * q + 2])};
        for (int l = 0; l < T.n_pos_levels; ++l) {
            float feat[FP];
            level_feats<3, FP>(T, l, pin, feat);
#pragma unroll
            for (int k = 0; k < FP; ++k) {
                T.A0[(size_t)(l * FP + k) * ld + q] = feat[k];
                axpy64(W0 + (l * FP + k) * 64, feat[k], acc);
            }
        }
    }
    {
        const float pin[2] = {__saturatef(T.qw[2 * q]), __saturatef(T.qw[2 * q + 1])};
        const int k0 = T.n_pos_levels * FP;
        for (int l = 0; l < T.n_dir_levels; ++l) {
            float feat[FD];
            level_feats<2, FD>(T, T.n_pos_levels + l, pin, feat);
#pragma unroll
            for (int k = 0; k < FD; ++k) {
                T.A0[(size_t)(k0 + l * FD + k) * ld + q] = feat[k];
                axpy64(W0 + (k0 + l * FD + k) * 64, feat[k], acc);
            }
        }
    }
    {
        const float gin = (T.qg[q] + 1.0f) * 0.5f;
        T.A0[(size_t)(T.din - 1) * ld + q] = gin;
        axpy64(W0 + (T.din - 1) * 64, gin, acc);
    }
#pragma unroll
    for (int o = 0; o < 64; ++o) T.A[(size_t)o * ld + q] = relu(acc[o]);
    // ---- hidden layers 1 .. H-1 (inputs streamed back from the thread's own rows)
    for (int L = 1; L < T.H; ++L) {
        const float *in = T.A + (size_t)(L - 1) * 64 * ld;
        const float *Wt = sm + T.wt_off[L];
#pragma unroll
        for (int o = 0; o < 64; ++o) acc[o] = sm[T.b_off[L] + o];
#pragma unroll 4
        for (int k = 0; k < 64; ++k) axpy64(Wt + k * 64, in[(size_t)k * ld + q], acc);
        float *out = T.A + (size_t)L * 64 * ld;
#pragma unroll
        for (int o = 0; o < 64; ++o) out[(size_t)o * ld + q] = relu(acc[o]);
    }
    // ---- output layer (identity) + loss + dloss/dz_H
    const float *in = T.A + (size_t)(T.H - 1) * 64 * ld;
    const float *Wt = sm + T.wt_off[T.H];
    float p[3] = {sm[T.b_off[T.H]], sm[T.b_off[T.H] + 1], sm[T.b_off[T.H] + 2]};
#pragma unroll 4
    for (int k = 0; k < 64; ++k) {
        const float a = in[(size_t)k * ld + q];
        const float4 w = *reinterpret_cast<const float4 *>(Wt + k * T.out_stride);
        p[0] = fmaf(w.x, a, p[0]);
        p[1] = fmaf(w.y, a, p[1]);
        p[2] = fmaf(w.z, a, p[2]);
    }
    float lq = 0.f;
    float *dzH = T.dZ + (size_t)T.H * 64 * ld;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float e = p[ch] - T.qt[3 * q + ch];
        const float den = fmaf(p[ch], p[ch], T.eps_rel);  // prediction detached
        lq += e * e / den;
        dzH[(size_t)ch * ld + q] = 2.0f * e / den * T.inv_3n;
    }
    T.loss_q[q] = lq;
}

template <int D, int F>
__device__ __forceinline__ void level_scatter(const TrainParams &T, int lv, const float *pin, int k0, size_t q,
                                              uint32_t entry_base, uint32_t tab_base, int Fdiv) {
    const FieldLevel L = T.lv[lv];
    float dfeat[F];
#pragma unroll
    for (int k = 0; k < F; ++k) dfeat[k] = T.dF[(size_t)(k0 + k) * T.ld + q];
    uint32_t c[D];
    float f[D];
    level_cell<D>(L, pin, c, f);
#pragma unroll
    for (int corner = 0; corner < (1 << D); ++corner) {
        const float w = corner_weight<D>(f, corner);
        const uint32_t idx = corner_index<D>(L, c, corner);
        unsigned long long *gp = T.gtab + L.offset_halves + (size_t)idx * F;
#pragma unroll
        for (int k = 0; k < F; ++k) fix_add(gp + k, w * dfeat[k]);
        T.touched[entry_base + (L.offset_halves - tab_base) / (uint32_t)Fdiv + idx] = 1;
    }
}

// Coarse dense levels (<= kSmemSlots gradient words: e.g. the paper field's
// pos levels 0-1 and dir levels 0-2) are the hottest atomic targets -- every
// query of the batch hits the same few hundred entries.  A CTA first sums its
// queries' contributions in shared memory, then adds each nonzero word to
// the table once: the same integer total (fixed-point adds are associative,
// so the step stays bit-reproducible) with ~256x fewer global atomics.
constexpr int kSmemSlots = 6144;  // 48 KB of int64
struct SmallLevels {
    int n;
    int lv[16];
};
// at most 16 small levels take the shared-memory path; any further ones stay on the global path

template <int D, int F>
__device__ __forceinline__ void level_scatter_smem(const TrainParams &T, int lv, const float *pin, int k0, size_t q,
                                                   bool live, uint32_t entry_base, uint32_t tab_base, int Fdiv,
                                                   unsigned long long *acc, uint32_t words) {
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) acc[i] = 0ull;
    __syncthreads();
    const FieldLevel L = T.lv[lv];
    if (live) {
        float dfeat[F];
#pragma unroll
        for (int k = 0; k < F; ++k) dfeat[k] = T.dF[(size_t)(k0 + k) * T.ld + q];
        uint32_t c[D];
        float f[D];
        level_cell<D>(L, pin, c, f);
#pragma unroll
        for (int corner = 0; corner < (1 << D); ++corner) {
            const float w = corner_weight<D>(f, corner);
            const uint32_t idx = corner_index<D>(L, c, corner);
#pragma unroll
            for (int k = 0; k < F; ++k) {
                const long long fx = __double2ll_rn((double)(w * dfeat[k]) * kGradFix);
                if (fx != 0) atomicAdd(acc + (size_t)idx * F + k, (unsigned long long)fx);
            }
            T.touched[entry_base + (L.offset_halves - tab_base) / (uint32_t)Fdiv + idx] = 1;
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
        if (acc[i] != 0ull) atomicAdd(T.gtab + L.offset_halves + i, acc[i]);
}

// Level lv of the table is "small": dense with <= kSmemSlots gradient words.
__host__ __device__ __forceinline__ bool scatter_small(const TrainParams &T, int lv, int FP, int FD) {
    const FieldLevel L = T.lv[lv];
    const int D = lv < T.n_pos_levels ? 3 : 2, F = lv < T.n_pos_levels ? FP : FD;
    uint64_t ent = 1;
    for (int a = 0; a < D; ++a) ent *= L.n1;
    return L.dense && ent * (uint64_t)F <= (uint64_t)kSmemSlots;
}

// the small levels: one CTA per (256 queries, small level), smem pre-sum
template <int FP, int FD>
__global__ void __launch_bounds__(256) k_train_scatter_small(const TrainParams T, const SmallLevels SL) {
    __shared__ unsigned long long acc[kSmemSlots];
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = SL.lv[blockIdx.y];
    const FieldLevel L = T.lv[lv];
    const bool live = q < T.n;
    const size_t qq = live ? q : 0;
    if (lv < T.n_pos_levels) {
        const uint32_t words = L.n1 * L.n1 * L.n1 * (uint32_t)FP;
        const float pin[3] = {__saturatef(T.qx[3 * qq]), __saturatef(T.qx[3 * qq + 1]), __saturatef(T.qx[3 * qq + 2])};
        level_scatter_smem<3, FP>(T, lv, pin, lv * FP, qq, live, 0u, 0u, FP, acc, words);
    } else {
        const int l = lv - T.n_pos_levels;
        const uint32_t words = L.n1 * L.n1 * (uint32_t)FD;
        const float pin[2] = {__saturatef(T.qw[2 * qq]), __saturatef(T.qw[2 * qq + 1])};
        level_scatter_smem<2, FD>(T, lv, pin, T.n_pos_levels * FP + l * FD, qq, live, T.n_pos_tab / (uint32_t)FP,
                                  T.n_pos_tab, FD, acc, words);
    }
}

// grid (query blocks, levels): blockIdx.y is the level, so the CTAs of one
// level run together and its fixed-point gradient slab stays in L2 (small
// levels are k_train_scatter_small's)
template <int FP, int FD>
__global__ void __launch_bounds__(256) k_train_scatter(const TrainParams T, uint32_t small_mask) {
    const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lv = blockIdx.y;
    if ((small_mask >> lv) & 1u) return;  // CTA-uniform: done by k_train_scatter_small
    if (q >= T.n) return;
    if (lv < T.n_pos_levels) {
        const float pin[3] = {__saturatef(T.qx[3 * q]), __saturatef(T.qx[3 * q + 1]), __saturatef(T.qx[3 * q + 2])};
        level_scatter<3, FP>(T, lv, pin, lv * FP, q, 0u, 0u, FP);
    } else {
        const int l = lv - T.n_pos_levels;
        const float pin[2] = {__saturatef(T.qw[2 * q]), __saturatef(T.qw[2 * q + 1])};
        level_scatter<2, FD>(T, lv, pin, T.n_pos_levels * FP + l * FD, q, T.n_pos_tab / (uint32_t)FP, T.n_pos_tab,
                             FD);
    }
}

template <int FP, int FD>
__global__ void __launch_bounds__(kThreads, 1) k_train_bwd(const TrainParams T, const float4 *img, int n4) {
    extern __shared__ float4 sm4[];
    load_image(img, n4, sm4);
    const float *sm = reinterpret_cast<const float *>(sm4);
    const size_t q = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (q >= T.n) return;
    const size_t ld = T.ld;
    float dz[64];
    // ---- output layer: dz_{H-1} = (W_H^T dz_H) . [a_H > 0]
    {
        const float *dzH = T.dZ + (size_t)T.H * 64 * ld;
        const float d0 = dzH[q], d1 = dzH[ld + q], d2 = dzH[2 * ld + q];
        const float *Wt = sm + T.wt_off[T.H];
        const float *aH = T.A + (size_t)(T.H - 1) * 64 * ld;
        float *out = T.dZ + (size_t)(T.H - 1) * 64 * ld;
#pragma unroll
        for (int k = 0; k < 64; ++k) {
            const float4 w = *reinterpret_cast<const float4 *>(Wt + k * T.out_stride);
            const float da = fmaf(w.x, d0, fmaf(w.y, d1, w.z * d2));
            dz[k] = aH[(size_t)k * ld + q] > 0.f ? da : 0.f;
            out[(size_t)k * ld + q] = dz[k];
        }
    }
    // ---- hidden layers: dz_{L-1} = (W_L^T dz_L) . [a_L > 0], L = H-1 .. 1
    for (int L = T.H - 1; L >= 1; --L) {
        const float *Wt = sm + T.wt_off[L];
        const float *aL = T.A + (size_t)(L - 1) * 64 * ld;
        float *out = T.dZ + (size_t)(L - 1) * 64 * ld;
#pragma unroll 2
        for (int k = 0; k < 64; ++k) {
            // (W_L^T dz)_k = sum_o W_L[o][k] dz_o = row k of W_L^T . dz
            const float da = dot64(Wt + k * 64, dz);
            out[(size_t)k * ld + q] = aL[(size_t)k * ld + q] > 0.f ? da : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 64; ++k) dz[k] = out[(size_t)k * ld + q];
    }
    // ---- dfeat = W_0^T dz_0 (row j of W_0^T is W_0[:, j]) -> feature-major
    // rows for k_train_scatter.  W_0^T is stored [k][o], so
    // (W_0^T dz)_k = sum_o W0T[k][o] dz_o
    const float *W0 = sm + T.wt_off[0];
    const int n_tab_feats = T.n_pos_levels * FP + T.n_dir_levels * FD;
#pragma unroll 2
    for (int k = 0; k < n_tab_feats; ++k) T.dF[(size_t)k * ld + q] = dot64(W0 + k * 64, dz);
}

// dW_L partials: part[chunk][o][k] = sum_{q in chunk} dZ_L[o][q] In_L[k][q],
// k == nin is the virtual ones row (db_L).  64 x 64 tile per CTA, 4 x 4 per thread.
__global__ void __launch_bounds__(256) k_train_wgrad(const float *Z, const float *X, int nout, int nin, size_t n,
                                                     size_t ld, int kpad, float *part) {
    __shared__ float Zs[32][68];
    __shared__ float Xs[32][68];
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int k0 = blockIdx.x * 64;
    const size_t q0 = (size_t)blockIdx.y * kChunk;
    float acc[4][4] = {};
    for (size_t qb = q0; qb < q0 + kChunk && qb < n; qb += 32) {
        // load 64 rows x 32 queries of Z and X (coalesced along the query axis)
        for (int i = tid; i < 64 * 32; i += 256) {
            const int r = i >> 5, j = i & 31;
            const size_t qq = qb + j;
            const bool ok = qq < n;
            Zs[j][r] = (ok && r < nout) ? Z[(size_t)r * ld + qq] : 0.f;
            const int k = k0 + r;
            Xs[j][r] = !ok ? 0.f : (k < nin ? X[(size_t)k * ld + qq] : (k == nin ? 1.f : 0.f));
        }
        __syncthreads();
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
            const float4 a = *reinterpret_cast<const float4 *>(&Zs[j][ty * 4]);
            const float4 b = *reinterpret_cast<const float4 *>(&Xs[j][tx * 4]);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
        }
        __syncthreads();
    }
    float *out = part + (size_t)blockIdx.y * 64 * kpad;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) out[(size_t)(ty * 4 + u) * kpad + k0 + tx * 4 + v] = acc[u][v];
}

// Sum the chunk partials in chunk order into the dense MLP gradient.
__global__ void k_train_wsum(const float *part, int n_chunks, int nout, int nin, int kpad, float *gW) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nout * (nin + 1)) return;
    const int o = i / (nin + 1), k = i - o * (nin + 1);
    float s = 0.f;
    for (int c = 0; c < n_chunks; ++c) s += part[((size_t)c * 64 + o) * kpad + k];
    if (k < nin) gW[(size_t)o * nin + k] = s;
    else gW[(size_t)nout * nin + o] = s;
}

// Deterministic loss sum (fixed strided order + fixed tree), binary64.
__global__ void __launch_bounds__(1024) k_train_loss(const float *lq, size_t n, double scale, double *out) {
    __shared__ double s[1024];
    double a = 0.0;
    for (size_t i = threadIdx.x; i < n; i += 1024) a += (double)lq[i];
    s[threadIdx.x] = a;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0] * scale;
}

struct AdamArgs {
    size_t n_params, n_tab, n_pos_tab;
    int Fp, Fd;
    float lr, b1, b2, eps, bc1, bc2;
    float *params, *m, *v;
    const float *gmlp;
    unsigned long long *gtab;
    const uint8_t *touched;
};

template <int F>
__device__ __forceinline__ void ld_vec(const float *a, float (&r)[F]) {
    if constexpr (F % 4 == 0) {
#pragma unroll
        for (int k = 0; k < F; k += 4) {
            const float4 x = *reinterpret_cast<const float4 *>(a + k);
            r[k] = x.x, r[k + 1] = x.y, r[k + 2] = x.z, r[k + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < F; k += 2) {
            const float2 x = *reinterpret_cast<const float2 *>(a + k);
            r[k] = x.x, r[k + 1] = x.y;
        }
    }
}
template <int F>
__device__ __forceinline__ void st_vec(float *a, const float (&r)[F]) {
    if constexpr (F % 4 == 0) {
#pragma unroll
        for (int k = 0; k < F; k += 4) *reinterpret_cast<float4 *>(a + k) = make_float4(r[k], r[k + 1], r[k + 2], r[k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < F; k += 2) *reinterpret_cast<float2 *>(a + k) = make_float2(r[k], r[k + 1]);
    }
}

// One thread per table ENTRY (touched test once; the F contiguous parameters,
// moments and fixed-point gradients are all loaded before any store, so the
// loads of a thread overlap) or per MLP parameter.
template <int F>
__device__ __forceinline__ void adam_entry(const AdamArgs &A, size_t i0) {
    float *__restrict__ P = A.params + i0;
    float *__restrict__ M = A.m + i0;
    float *__restrict__ V = A.v + i0;
    unsigned long long *__restrict__ G = A.gtab + i0;
    // 16-byte vector loads / stores (an entry's F values are F*4-byte
    // aligned: tables start at 0 and n_pos_tab, entries are F wide)
    unsigned long long gq[F];
    float p[F], m[F], v[F];
    ld_vec<F>(P, p);
    ld_vec<F>(M, m);
    ld_vec<F>(V, v);
#pragma unroll
    for (int k = 0; k < F; k += 2) {
        const ulonglong2 x = *reinterpret_cast<const ulonglong2 *>(G + k);
        gq[k] = x.x;
        gq[k + 1] = x.y;
    }
#pragma unroll
    for (int k = 0; k < F; ++k) {
        const float g = (float)((double)(long long)gq[k] * (1.0 / kGradFix));
        m[k] = A.b1 * m[k] + (1.f - A.b1) * g;
        v[k] = A.b2 * v[k] + (1.f - A.b2) * g * g;
        p[k] -= A.lr * (m[k] / A.bc1) / (sqrtf(v[k] / A.bc2) + A.eps);
    }
#pragma unroll
    for (int k = 0; k < F; k += 2) *reinterpret_cast<ulonglong2 *>(G + k) = make_ulonglong2(0ull, 0ull);
    st_vec<F>(P, p);
    st_vec<F>(M, m);
    st_vec<F>(V, v);
}

__global__ void k_train_adam(const AdamArgs A, size_t n_pos_entries, size_t n_entries) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_entries) {
        if (!A.touched[t]) return;  // sparse: untouched entries keep params and moments
        const bool pos = t < n_pos_entries;
        const int F = pos ? A.Fp : A.Fd;
        const size_t i0 = pos ? t * (size_t)A.Fp : A.n_pos_tab + (t - n_pos_entries) * (size_t)A.Fd;
        if (F == 8) adam_entry<8>(A, i0);
        else if (F == 4) adam_entry<4>(A, i0);
        else adam_entry<2>(A, i0);
        return;
    }
    const size_t i = A.n_tab + (t - n_entries);
    if (i >= A.n_params) return;
    const float g = A.gmlp[i - A.n_tab];
    const float m = A.b1 * A.m[i] + (1.f - A.b1) * g;
    const float v = A.b2 * A.v[i] + (1.f - A.b2) * g * g;
    A.m[i] = m;
    A.v[i] = v;
    A.params[i] -= A.lr * (m / A.bc1) / (sqrtf(v / A.bc2) + A.eps);
}

// Dense gradient export (pf_train_grad) + accumulator reset.
__global__ void k_train_export(const AdamArgs A, float *grad, uint8_t *touched_out, size_t n_entries) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < A.n_params) {
        float g;
        if (i < A.n_tab) {
            g = (float)((double)(long long)A.gtab[i] * (1.0 / kGradFix));
            A.gtab[i] = 0ull;
        } else {
            g = A.gmlp[i - A.n_tab];
        }
        if (grad) grad[i] = g;
    }
    if (touched_out && i < n_entries) touched_out[i] = A.touched[i];
}

__global__ void k_train_prep(const double *w3, const uint8_t *gidx, const double *t3d, TrainPhases ph, size_t n,
                             float *w2, float *g, float *t3) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // (theta/pi, (phi+pi)/2pi), phi = atan2(w_y, w_x)  (oracle or_dir_to_sph)
    const double z = fmin(fmax(w3[3 * i + 2], -1.0), 1.0);
    w2[2 * i] = (float)(acos(z) / 3.14159265358979323846);
    w2[2 * i + 1] = (float)((atan2(w3[3 * i + 1], w3[3 * i]) + 3.14159265358979323846) / 6.283185307179586476925);
    const int gi = gidx[i];
    g[i] = (float)(gi < ph.n ? ph.v[gi] : 0.0);
#pragma unroll
    for (int c = 0; c < 3; ++c) t3[3 * i + c] = (float)t3d[3 * i + c];
}

template <int FP, int FD>
cudaError_t launch_fb(const TrainParams &T, const float4 *img, int n4, size_t smem, bool fwd, cudaStream_t st) {
    const unsigned blocks = (unsigned)((T.n + kThreads - 1) / kThreads);
    if (fwd) {
        cudaFuncSetAttribute(k_train_fwd<FP, FD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_train_fwd<FP, FD><<<blocks, kThreads, smem, st>>>(T, img, n4);
    } else {
        cudaFuncSetAttribute(k_train_bwd<FP, FD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_train_bwd<FP, FD><<<blocks, kThreads, smem, st>>>(T, img, n4);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        SmallLevels SL{};
        SL.n = 0;
#if PF_TRAIN_SMEM_SCATTER
        for (int lv = 0; lv < T.n_pos_levels + T.n_dir_levels && SL.n < 16; ++lv)
            if (scatter_small(T, lv, FP, FD)) SL.lv[SL.n++] = lv;
#endif
        const unsigned qb = (unsigned)((T.n + 255) / 256);
        if (SL.n > 0) {
            k_train_scatter_small<FP, FD><<<dim3(qb, (unsigned)SL.n), 256, 0, st>>>(T, SL);
            const cudaError_t e2 = cudaGetLastError();
            if (e2 != cudaSuccess) return e2;
        }
        uint32_t small_mask = 0u;
        for (int i = 0; i < SL.n; ++i) small_mask |= 1u << SL.lv[i];
        k_train_scatter<FP, FD><<<dim3(qb, (unsigned)(T.n_pos_levels + T.n_dir_levels)), 256, 0, st>>>(T, small_mask);
    }
    return cudaGetLastError();
}

cudaError_t launch_fb_dispatch(int fp, int fd, const TrainParams &T, const float4 *img, int n4, size_t smem, bool fwd,
                               cudaStream_t st) {
#define PF_FB(A, B) \
    if (fp == A && fd == B) return launch_fb<A, B>(T, img, n4, smem, fwd, st);
    PF_FB(2, 2) PF_FB(2, 4) PF_FB(2, 8) PF_FB(4, 2) PF_FB(4, 4) PF_FB(4, 8) PF_FB(8, 2) PF_FB(8, 4) PF_FB(8, 8)
#undef PF_FB
    return cudaErrorInvalidValue;
}

}  // namespace

double train_lr(const TrainState &S, uint64_t step, uint64_t total) {
    double s = (double)step - S.decay_start * (double)total;
    if (s < 0.0) s = 0.0;
    return S.lr * std::pow(S.decay, std::floor(s / (double)S.decay_interval));
}

cudaError_t train_init(TrainState &S, const FieldDesc &fd, const std::vector<FieldLevel> &levels,
                       const float *params_dev, cudaStream_t st) {
    S.fd = fd;
    S.levels = levels;
    S.Fp = fd.pos.features;
    S.Fd = fd.dir.features;
    S.H = fd.hidden_layers;
    S.din = fd.pos.levels * fd.pos.features + fd.dir.levels * fd.dir.features + 1;
    S.n_pos_tab = field_grid_param_count(fd.pos);
    S.n_tab = S.n_pos_tab + field_grid_param_count(fd.dir);
    S.n_params = field_param_count(fd);
    S.n_entries = S.n_pos_tab / S.Fp + (S.n_tab - S.n_pos_tab) / S.Fd;
    size_t off = S.n_tab, img = 0;
    for (int L = 0; L <= S.H; ++L) {
        const int nin = L == 0 ? S.din : 64, nout = L < S.H ? 64 : 3, os = L < S.H ? 64 : 4;
        S.off_w[L] = (uint32_t)off;
        off += (size_t)nout * nin + nout;
        S.wt_off[L] = (uint32_t)img;
        img += (size_t)nin * os;
        S.b_off[L] = (uint32_t)img;
        img += 64;
    }
    S.img_floats = (img + 3) & ~(size_t)3;
    cudaError_t e;
    if ((e = S.params.ensure(S.n_params * 4)) || (e = S.m.ensure(S.n_params * 4)) || (e = S.v.ensure(S.n_params * 4)) ||
        (e = S.gmlp.ensure((S.n_params - S.n_tab) * 4)) || (e = S.gtab.ensure(S.n_tab * 8)) ||
        (e = S.touched.ensure(S.n_entries)) || (e = S.img.ensure(S.img_floats * 4 + 16)))
        return e;
    if ((e = cudaMemcpyAsync(S.params.p, params_dev, S.n_params * 4, cudaMemcpyDefault, st))) return e;
    cudaMemsetAsync(S.m.p, 0, S.n_params * 4, st);
    cudaMemsetAsync(S.v.p, 0, S.n_params * 4, st);
    cudaMemsetAsync(S.gtab.p, 0, S.n_tab * 8, st);
    cudaMemsetAsync(S.touched.p, 0, S.n_entries, st);
    S.ready = true;
    return cudaGetLastError();
}

cudaError_t train_prep(const double *w3, const uint8_t *gidx, const double *t3d, const double *phase, int n_phases,
                       size_t n, float *w2, float *g, float *t3, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    TrainPhases ph;
    ph.n = n_phases;
    for (int i = 0; i < n_phases && i < 8; ++i) ph.v[i] = phase[i];
    k_train_prep<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w3, gidx, t3d, ph, n, w2, g, t3);
    return cudaGetLastError();
}

cudaError_t train_backward(TrainState &S, size_t n, const float *x3, const float *w2, const float *g, const float *t3,
                           size_t n_global, size_t loss_slot, cudaStream_t st) {
    cudaError_t e;
    if (n_global < n || n_global == 0) n_global = n ? n : 1;
    const size_t ld = (n + 3) & ~(size_t)3;
    const size_t rows = 2 * (size_t)S.din + (size_t)S.H * 64 + (size_t)(S.H + 1) * 64;
    if ((e = S.act.ensure(rows * ld * 4))) return e;
    if ((e = S.lossq.ensure(n * 4 + 16))) return e;
    if ((e = S.loss_dev.ensure((loss_slot + 1) * 8))) return e;
    const int n_chunks = (int)((n + kChunk - 1) / kChunk);
    const int kpad_max = ((S.din + 1 + 63) / 64) * 64;
    if ((e = S.part.ensure((size_t)n_chunks * 64 * kpad_max * 4))) return e;
    // kernel view
    TrainParams T;
    std::memset(&T, 0, sizeof(T));
    T.n_pos_levels = S.fd.pos.levels;
    T.n_dir_levels = S.fd.dir.levels;
    T.Fp = S.Fp;
    T.Fd = S.Fd;
    T.din = S.din;
    T.H = S.H;
    for (size_t i = 0; i < S.levels.size() && i < PF_FIELD_MAX_LEVELS; ++i) T.lv[i] = S.levels[i];
    T.params = (const float *)S.params.p;
    T.n_pos_tab = (uint32_t)S.n_pos_tab;
    for (int L = 0; L <= S.H; ++L) {
        T.wt_off[L] = S.wt_off[L];
        T.b_off[L] = S.b_off[L];
    }
    T.out_stride = 4;
    T.n = n;
    T.ld = ld;
    T.qx = x3;
    T.qw = w2;
    T.qg = g;
    T.qt = t3;
    T.eps_rel = (float)S.eps_rel;
    T.inv_3n = (float)(1.0 / (3.0 * (double)n_global));  // this shard's part of the global mean
    float *act = (float *)S.act.p;
    T.A0 = act;
    T.A = act + (size_t)S.din * ld;
    T.dZ = T.A + (size_t)S.H * 64 * ld;
    T.dF = T.dZ + (size_t)(S.H + 1) * 64 * ld;
    T.loss_q = (float *)S.lossq.p;
    T.gtab = (unsigned long long *)S.gtab.p;
    T.touched = (uint8_t *)S.touched.p;

    // W^T image (offsets of W_L passed through a tiny device table)
    if ((e = S.offw.ensure(32))) return e;
    if ((e = cudaMemcpyAsync(S.offw.p, S.off_w, 32, cudaMemcpyHostToDevice, st))) return e;
    k_train_pack<<<dim3(64, S.H + 1), 256, 0, st>>>(T, (const uint32_t *)S.offw.p, (float *)S.img.p, S.H + 1);
    if ((e = cudaGetLastError())) return e;
    const int n4 = (int)(S.img_floats / 4);
    const size_t smem = S.img_floats * 4;
    if (n) {
        if ((e = launch_fb_dispatch(S.Fp, S.Fd, T, (const float4 *)S.img.p, n4, smem, true, st))) return e;
    }
    k_train_loss<<<1, 1024, 0, st>>>(T.loss_q, n, 1.0 / (3.0 * (double)n_global), (double *)S.loss_dev.p + loss_slot);
    if (n) {
        if ((e = launch_fb_dispatch(S.Fp, S.Fd, T, (const float4 *)S.img.p, n4, smem, false, st))) return e;
    }
    // dW_L, db_L (deterministic two-pass reduction)
    float *gmlp = (float *)S.gmlp.p;
    for (int L = 0; L <= S.H; ++L) {
        const int nin = L == 0 ? S.din : 64, nout = L < S.H ? 64 : 3;
        const int kpad = ((nin + 1 + 63) / 64) * 64;
        const float *Z = T.dZ + (size_t)L * 64 * ld;
        const float *X = L == 0 ? T.A0 : T.A + (size_t)(L - 1) * 64 * ld;
        if (n) {
            k_train_wgrad<<<dim3(kpad / 64, n_chunks), 256, 0, st>>>(Z, X, nout, nin, n, ld, kpad, (float *)S.part.p);
            if ((e = cudaGetLastError())) return e;
        }
        const int cnt = nout * (nin + 1);
        k_train_wsum<<<(cnt + 255) / 256, 256, 0, st>>>((const float *)S.part.p, n ? n_chunks : 0, nout, nin, kpad,
                                                        gmlp + (S.off_w[L] - S.n_tab));
        if ((e = cudaGetLastError())) return e;
    }
    return cudaSuccess;
}

cudaError_t train_finish(TrainState &S, uint64_t step, uint64_t total, bool do_update, float *grad_out,
                         uint8_t *touched_out, cudaStream_t st) {
    cudaError_t e;
    float *gmlp = (float *)S.gmlp.p;
    AdamArgs A;
    A.n_params = S.n_params;
    A.n_tab = S.n_tab;
    A.n_pos_tab = S.n_pos_tab;
    A.Fp = S.Fp;
    A.Fd = S.Fd;
    A.params = (float *)S.params.p;
    A.m = (float *)S.m.p;
    A.v = (float *)S.v.p;
    A.gmlp = gmlp;
    A.gtab = (unsigned long long *)S.gtab.p;
    A.touched = (const uint8_t *)S.touched.p;
    const double t = (double)(step + 1);
    A.lr = (float)train_lr(S, step, total);
    A.b1 = (float)S.beta1;
    A.b2 = (float)S.beta2;
    A.eps = (float)S.eps;
    A.bc1 = (float)(1.0 - std::pow(S.beta1, t));
    A.bc2 = (float)(1.0 - std::pow(S.beta2, t));
    const size_t nb = std::max(S.n_params, S.n_entries);
    if (do_update) {
        const size_t nt = S.n_entries + (S.n_params - S.n_tab);
        k_train_adam<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(A, S.n_pos_tab / (size_t)S.Fp, S.n_entries);
    } else {
        k_train_export<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(A, grad_out, touched_out, S.n_entries);
    }
    if ((e = cudaGetLastError())) return e;
    return cudaMemsetAsync(S.touched.p, 0, S.n_entries, st);
}

cudaError_t train_step(TrainState &S, size_t n, const float *x3, const float *w2, const float *g, const float *t3,
                       uint64_t step, uint64_t total, bool do_update, float *grad_out, uint8_t *touched_out,
                       size_t loss_slot, int sms, cudaStream_t st) {
    (void)sms;
    cudaError_t e = train_backward(S, n, x3, w2, g, t3, n, loss_slot, st);
    if (e != cudaSuccess) return e;
    return train_finish(S, step, total, do_update, grad_out, touched_out, st);
}

}  // namespace pfk
