// pf_field.cu -- K3+K4: batched photon-field query on the 5th-gen tensor cores.
//
// SPEC.md:352-447 (encode_input + forward + infer_radiance); Alg. 2's
// "L_i^pred <- Decode(P_phi(samples))".
//
// One persistent CTA per SM holds the whole MLP (fp16, UMMA canonical
// layout, pulled in once by a 1-D bulk TMA copy) in shared memory.  Each
// 128-thread warpgroup owns an independent tile pipeline:
//   1. every thread encodes ONE query (hash-grid gather, fp32 accumulate)
//      and writes its fp16 feature row straight into the A-operand tile;
//   2. one elected thread issues tcgen05.mma (M=128, N=64, K=16 steps) with
//      the fp32 accumulator in TMEM (64 columns per warpgroup);
//   3. the warpgroup pulls its rows back with tcgen05.ld (thread i <-> TMEM
//      lane i), adds bias + ReLU, packs fp16 into the same A tile, and the
//      next layer's MMA is issued -- 6 dependent MMA chains per tile;
//   4. the last layer (N=16, 3 live columns) is decoded with Eq. 8 and, in
//      render mode, w_i * sigma_s * L_i is added into the sample's slot.
// 2-4 warpgroups per CTA interleave their encode / epilogue / MMA phases so
// the tensor pipe and the gather units overlap.
#include <cuda_fp16.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "pf_field.h"
#include "pf_umma.cuh"

namespace pfk {

constexpr uint32_t kPrime1 = 2654435761u, kPrime2 = 805459861u;

__device__ __forceinline__ void load_feats(const __half *tab, uint32_t e, float *v, int F) {
    if (F == 8) {
        uint4 u = __ldg(reinterpret_cast<const uint4 *>(tab) + e);
        const __half2 *h = reinterpret_cast<const __half2 *>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float2 f = __half22float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    } else if (F == 4) {
        uint2 u = __ldg(reinterpret_cast<const uint2 *>(tab) + e);
        const __half2 *h = reinterpret_cast<const __half2 *>(&u);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            float2 f = __half22float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    } else {
        uint32_t u = __ldg(reinterpret_cast<const uint32_t *>(tab) + e);
        float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&u));
        v[0] = f.x;
        v[1] = f.y;
    }
}

__device__ __forceinline__ void store_feats(uint8_t *A, int r, int k, uint32_t sbo, const float *acc,
                                            int F) {
    uint8_t *p = A + (r >> 3) * sbo + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
    if (F == 8) {
        uint4 u;
        __half2 *h = reinterpret_cast<__half2 *>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(acc[2 * i], acc[2 * i + 1]);
        *reinterpret_cast<uint4 *>(p) = u;
    } else if (F == 4) {
        uint2 u;
        __half2 *h = reinterpret_cast<__half2 *>(&u);
        h[0] = __floats2half2_rn(acc[0], acc[1]);
        h[1] = __floats2half2_rn(acc[2], acc[3]);
        *reinterpret_cast<uint2 *>(p) = u;
    } else {
        __half2 h = __floats2half2_rn(acc[0], acc[1]);
        *reinterpret_cast<__half2 *>(p) = h;
    }
}

// Multilinear hash-grid encoding of one D-dim input into A row r, columns
// [kbase, kbase + levels*F) (pinned in oracle or_hashgrid_encode).
template <int D, int F>
__device__ __forceinline__ void encode_grid(const FieldParams &P, int lv0, int nlv, const float *in,
                                            uint8_t *A, int r, int kbase, uint32_t sbo) {
    float pin[D];
#pragma unroll
    for (int i = 0; i < D; ++i) pin[i] = __saturatef(in[i]);
    for (int l = 0; l < nlv; ++l) {
        const FieldLevel L = P.lv[lv0 + l];
        const float resf = (float)L.res;
        uint32_t c[D];
        float f[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            // exact p*N split: s + e == p*N, so the cell fraction keeps full precision
            const float s = pin[i] * resf;
            const float e = fmaf(pin[i], resf, -s);
            float fl = floorf(s);
            float fr = (s - fl) + e;
            int ci = (int)fl;
            if (fr < 0.f) {
                ci -= 1;
                fr += 1.f;
            }
            if (ci > (int)L.res - 1) {
                ci = (int)L.res - 1;
                fr = (s - (float)ci) + e;
            }
            c[i] = (uint32_t)ci;
            f[i] = fr;
        }
        float acc[F];
#pragma unroll
        for (int k = 0; k < F; ++k) acc[k] = 0.f;
#pragma unroll
        for (int corner = 0; corner < (1 << D); ++corner) {
            float w = 1.f;
            uint32_t v[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const int bit = (corner >> i) & 1;
                w *= bit ? f[i] : (1.f - f[i]);
                v[i] = c[i] + (uint32_t)bit;
            }
            uint32_t idx;
            if (L.dense) {
                idx = v[0] + L.n1 * v[1];
                if (D == 3) idx += L.n1 * L.n1 * v[D - 1];
            } else {
                uint32_t h = v[0] ^ (v[1] * kPrime1);
                if (D == 3) h ^= v[D - 1] * kPrime2;
                idx = h & L.mask;
            }
            float e[F];
            load_feats(P.tables + L.offset_halves, idx, e, F);
#pragma unroll
            for (int k = 0; k < F; ++k) acc[k] = fmaf(w, e[k], acc[k]);
        }
        store_feats(A, r, kbase + l * F, sbo, acc, F);
    }
}

__device__ __forceinline__ void issue_layer(uint32_t a_s, uint32_t b_s, int K, int N, uint32_t tmem_d) {
    const uint32_t sbo = (uint32_t)K * 16u;
    const uint32_t idesc = umma_idesc_f16(128, N);
    for (int j = 0; j < K / 16; ++j) {
        const uint64_t ad = umma_sdesc(a_s + 256u * j, 128u, sbo);
        const uint64_t bd = umma_sdesc(b_s + 256u * j, 128u, sbo);
        umma_f16(tmem_d, ad, bd, idesc, j > 0 ? 1u : 0u);
    }
}

// Zero-pad columns [k0, k1) of row r in a chunk tile of width W (multiples of 8).
__device__ __forceinline__ void zero_cols(uint8_t *A, int r, int k0, int k1, uint32_t sbo) {
    for (int k = k0; k < k1; k += 8)
        *reinterpret_cast<uint4 *>(A + (r >> 3) * sbo + (k >> 3) * 128 + (r & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
}

template <int FP, int FD>
__global__ void __launch_bounds__(512, 1) k_field(const FieldParams P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *img = smem;
    uint8_t *abase = smem + P.img_bytes;
    // per warpgroup: two 128 x 64 fp16 chunk tiles (16 KB each) + 2 mbarriers
    uint64_t *bars = reinterpret_cast<uint64_t *>(abase + (size_t)P.n_wg * 32768);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 1 + 2 * P.n_wg);

    const int tid = threadIdx.x, wg = tid >> 7, r = tid & 127, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i <= 2 * P.n_wg; ++i) mbar_init(smem_u32(&bars[i]), 1);
        mbar_fence_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(tmem_slot), P.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
        mbar_expect_tx(smem_u32(&bars[0]), P.img_bytes);
        bulk_g2s(smem_u32(img), P.img, P.img_bytes, smem_u32(&bars[0]));
    }
    const uint32_t tmem_base = *tmem_slot;
    mbar_wait(smem_u32(&bars[0]), 0);

    const size_t n_items = P.mode == 0 ? (size_t)(*P.n_hits) : P.n_query;
    const size_t n_tiles = (n_items + 127) / 128;
    uint8_t *buf[2] = {abase + (size_t)wg * 32768, abase + (size_t)wg * 32768 + 16384};
    const uint32_t buf_s[2] = {smem_u32(buf[0]), smem_u32(buf[1])};
    const uint32_t img_s = smem_u32(img);
    const uint32_t tmem_wg = tmem_base + (uint32_t)(wg * 64);
    const uint32_t tmem_rows = tmem_wg + ((uint32_t)(32 * (warp & 3)) << 16);
    const uint32_t mbar[2] = {smem_u32(&bars[1 + 2 * wg]), smem_u32(&bars[2 + 2 * wg])};
    uint32_t ph[2] = {0u, 0u};
    bool pending[2] = {false, false};
    const float *bias = reinterpret_cast<const float *>(img + P.off_bias);
    const int kdir = P.n_pos_levels * FP;
    const int kg = kdir + P.n_dir_levels * FD;     // column of the g input
    const int nch = (P.K0 + 63) / 64;
    const uint32_t sbo_w0 = (uint32_t)P.K0 * 16u;

    auto wait_buf = [&](int b) {
        if (pending[b]) {
            mbar_wait(mbar[b], ph[b]);
            ph[b] ^= 1u;
            pending[b] = false;
        }
    };

    for (size_t tile = (size_t)blockIdx.x * P.n_wg + wg; tile < n_tiles; tile += (size_t)gridDim.x * P.n_wg) {
        const size_t row = tile * 128 + r;
        const bool valid = row < n_items;
        float x[3] = {0.f, 0.f, 0.f}, ws[2] = {0.f, 0.f}, gin = 0.f;
        uint32_t slot = 0;
        double sigma_s = 0.0;
        if (valid) {
            if (P.mode == 0) {
                const HitRec h = P.hits[row];
                x[0] = h.x[0];
                x[1] = h.x[1];
                x[2] = h.x[2];
                ws[0] = h.wsph[0];
                ws[1] = h.wsph[1];
                slot = h.slot;
                sigma_s = h.sigma_s;
                gin = P.g_render;
            } else {
                x[0] = P.qx[3 * row];
                x[1] = P.qx[3 * row + 1];
                x[2] = P.qx[3 * row + 2];
                ws[0] = P.qw[2 * row];
                ws[1] = P.qw[2 * row + 1];
                gin = P.qg[row];
            }
        }
        // ---- K3 + layer-0 MMA, chunk by chunk (encode j+1 overlaps MMA j)
        for (int j = 0; j < nch; ++j) {
            const int b = j & 1;
            const int k0 = 64 * j, kw = min(64, P.K0 - k0);
            const uint32_t sbo = (uint32_t)kw * 16u;
            wait_buf(b);  // the MMA that last read this buffer is done
            uint8_t *A = buf[b];
            // position levels whose features start in [k0, k0+kw)
            const int lp0 = min(P.n_pos_levels, k0 / FP), lp1 = min(P.n_pos_levels, (k0 + kw) / FP);
            if (lp1 > lp0) encode_grid<3, FP>(P, lp0, lp1 - lp0, x, A, r, lp0 * FP - k0, sbo);
            const int ld0 = min(P.n_dir_levels, max(0, (k0 - kdir + FD - 1) / FD));
            const int ld1 = min(P.n_dir_levels, max(0, (k0 + kw - kdir + FD - 1) / FD));
            if (ld1 > ld0) encode_grid<2, FD>(P, P.n_pos_levels + ld0, ld1 - ld0, ws, A, r, kdir + ld0 * FD - k0, sbo);
            if (kg >= k0 && kg < k0 + kw) {
                const int kk = kg - k0;
                uint8_t *p = A + (r >> 3) * sbo + (kk >> 3) * 128 + (r & 7) * 16;
                uint4 u = make_uint4(0u, 0u, 0u, 0u);
                u.x = (uint32_t)__half_as_ushort(__float2half_rn((gin + 1.0f) * 0.5f));
                *reinterpret_cast<uint4 *>(p) = u;
                zero_cols(A, r, kk + 8, kw, sbo);
            } else if (kg < k0) {
                zero_cols(A, r, 0, kw, sbo);
            }
            fence_proxy_async_smem();
            named_bar_sync(1 + wg, 128);
            if (r == 0) {
                tc_fence_after();
                const uint32_t idesc = umma_idesc_f16(128, 64);
                for (int s = 0; s < kw / 16; ++s) {
                    const uint64_t ad = umma_sdesc(buf_s[b] + 256u * s, 128u, sbo);
                    const uint64_t bd = umma_sdesc(img_s + P.off_w[0] + (uint32_t)(k0 / 8) * 128u + 256u * s, 128u,
                                                   sbo_w0);
                    umma_f16(tmem_wg, ad, bd, idesc, (j > 0 || s > 0) ? 1u : 0u);
                }
                umma_commit(mbar[b]);
            }
            pending[b] = true;
        }
        wait_buf(0);
        wait_buf(1);
        tc_fence_after();

        // ---- K4: hidden layers (epilogue of layer L-1 feeds the MMA of layer L)
        for (int L = 1; L <= P.hidden_layers; ++L) {
            const int b = L & 1;
            uint8_t *A = buf[b];
            const float *bl = bias + (L - 1) * 64;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                float v[16];
                tmem_ld16(tmem_rows + 16 * c, v);
                tmem_ld_wait();
                uint4 u[2];
                __half2 *h = reinterpret_cast<__half2 *>(u);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float a0 = fmaxf(v[2 * i] + bl[16 * c + 2 * i], 0.f);
                    const float a1 = fmaxf(v[2 * i + 1] + bl[16 * c + 2 * i + 1], 0.f);
                    h[i] = __floats2half2_rn(a0, a1);
                }
                uint8_t *p = A + (r >> 3) * 1024 + (2 * c) * 128 + (r & 7) * 16;  // K = 64: SBO = 1024
                *reinterpret_cast<uint4 *>(p) = u[0];
                *reinterpret_cast<uint4 *>(p + 128) = u[1];
            }
            tc_fence_before();
            fence_proxy_async_smem();
            named_bar_sync(1 + wg, 128);
            if (r == 0) {
                tc_fence_after();
                issue_layer(buf_s[b], img_s + P.off_w[L], 64, L < P.hidden_layers ? 64 : 16, tmem_wg);
                umma_commit(mbar[b]);
            }
            pending[b] = true;
            wait_buf(b);
            tc_fence_after();
        }

        // ---- output layer epilogue: bias, Eq. 8 decode, compose term
        float v[16];
        tmem_ld16(tmem_rows, v);
        tmem_ld_wait();
        tc_fence_before();
        const float *bo = bias + P.hidden_layers * 64;
        float o3[3] = {v[0] + bo[0], v[1] + bo[1], v[2] + bo[2]};
        if (valid) {
            if (P.mode == 0) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float Li = exp2f(-__saturatef(o3[c]) * P.psi_log2_10);  // Eq. 8
                    if (P.slot_f64) {
                        double *sp = reinterpret_cast<double *>(P.slots) + 3 * (size_t)slot + c;
                        *sp = *sp + P.w_i * (sigma_s * (double)Li);
                    } else {
                        float *sp = reinterpret_cast<float *>(P.slots) + 3 * (size_t)slot + c;
                        *sp = *sp + (float)P.w_i * ((float)sigma_s * Li);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    P.qout[3 * row + c] = P.decoded ? exp2f(-__saturatef(o3[c]) * P.psi_log2_10) : o3[c];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, P.tmem_cols);
    }
}

// ------------------------------------------------------------------------
// host side: layout + packing + launch
// ------------------------------------------------------------------------
static int level_res(const FieldGridDesc &g, int l) {
    return (int)std::floor((double)g.base_res * std::pow(g.growth, (double)l));
}

static bool level_dense(const FieldGridDesc &g, int l, uint64_t &verts) {
    const uint64_t n1 = (uint64_t)level_res(g, l) + 1u, T = 1ull << g.log2_table;
    uint64_t v = 1;
    for (int i = 0; i < g.dims; ++i) {
        v *= n1;
        if (v > T) {
            verts = T;
            return false;
        }
    }
    verts = v;
    return true;
}

size_t field_grid_param_count(const FieldGridDesc &g) {
    size_t n = 0;
    for (int l = 0; l < g.levels; ++l) {
        uint64_t v;
        level_dense(g, l, v);
        n += (size_t)v * g.features;
    }
    return n;
}

size_t field_param_count(const FieldDesc &d) {
    const size_t din = (size_t)(d.pos.levels * d.pos.features + d.dir.levels * d.dir.features + 1);
    const size_t w = (size_t)d.width;
    return field_grid_param_count(d.pos) + field_grid_param_count(d.dir) + din * w + w +
           (size_t)(d.hidden_layers - 1) * (w * w + w) + 3 * w + 3;
}

const char *field_validate(const FieldDesc &d) {
    if (d.width != 64) return "field: the tcgen05 kernel supports width 64 only";
    if (d.hidden_layers < 1 || d.hidden_layers > 7) return "field: hidden_layers must be in [1,7]";
    if (d.pos.dims != 3 || d.dir.dims != 2) return "field: pos grid must be 3-D and dir grid 2-D";
    for (const FieldGridDesc *g : {&d.pos, &d.dir}) {
        if (g->features != 2 && g->features != 4 && g->features != 8)
            return "field: features per level must be 2, 4 or 8";
        if (g->levels < 1 || g->levels > 16) return "field: levels must be in [1,16]";
        if (g->base_res < 1 || !(g->growth >= 1.0)) return "field: base_res >= 1, growth >= 1";
        if (g->log2_table < 4 || g->log2_table > 24) return "field: log2_table in [4,24]";
        if (level_res(*g, g->levels - 1) > (1 << 24)) return "field: level resolution too large";
    }
    if ((d.pos.levels * d.pos.features) % 8 != 0 || (d.dir.levels * d.dir.features) % 8 != 0)
        return "field: levels*features must be a multiple of 8 for each grid";
    if (!(d.psi > 0.0)) return "field: psi must be positive";
    return nullptr;
}

// element (r, k) of a [rows x K] fp16 UMMA tile (K-major, SWIZZLE_NONE)
static inline size_t canon_off(int r, int k, int K) {
    return (size_t)(r >> 3) * (K * 16) + (size_t)(k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

void field_pack(const FieldDesc &d, const float *params, FieldHost &out) {
    const int din = d.pos.levels * d.pos.features + d.dir.levels * d.dir.features + 1;
    const int K0 = ((din + 15) / 16) * 16 < 64 ? 64 : ((din + 15) / 16) * 16;
    out.K0 = K0;
    out.n_pos_levels = d.pos.levels;
    out.n_dir_levels = d.dir.levels;
    out.fp = d.pos.features;
    out.fd = d.dir.features;
    out.hidden_layers = d.hidden_layers;
    out.psi = d.psi;
    // --- tables -> fp16, same order as the flat vector
    const size_t ntab = field_grid_param_count(d.pos) + field_grid_param_count(d.dir);
    out.tables.resize(ntab);
    for (size_t i = 0; i < ntab; ++i) out.tables[i] = __half_as_ushort(__float2half_rn(params[i]));
    out.levels.clear();
    size_t off = 0;
    for (const FieldGridDesc *g : {&d.pos, &d.dir}) {
        for (int l = 0; l < g->levels; ++l) {
            FieldLevel L{};
            uint64_t v;
            L.dense = level_dense(*g, l, v) ? 1u : 0u;
            L.res = (uint32_t)level_res(*g, l);
            L.n1 = L.res + 1u;
            L.mask = (1u << g->log2_table) - 1u;
            L.offset_halves = (uint32_t)off;
            out.levels.push_back(L);
            off += (size_t)v * g->features;
        }
    }
    // --- MLP image: W_0..W_H (canonical fp16), then fp32 biases
    const float *mlp = params + ntab;
    const int H = d.hidden_layers;
    std::vector<int> Kl(H + 1), Nl(H + 1), Nreal(H + 1), Kreal(H + 1);
    for (int L = 0; L <= H; ++L) {
        Kl[L] = L == 0 ? K0 : 64;
        Kreal[L] = L == 0 ? din : 64;
        Nl[L] = L < H ? 64 : 16;
        Nreal[L] = L < H ? 64 : 3;
    }
    size_t bytes = 0;
    for (int L = 0; L <= H; ++L) {
        out.off_w[L] = (uint32_t)bytes;
        bytes += (size_t)Nl[L] * Kl[L] * 2;
    }
    out.off_bias = (uint32_t)bytes;
    bytes += (size_t)(H * 64 + 16) * 4;
    bytes = (bytes + 1023) & ~(size_t)1023;
    out.image.assign(bytes, 0);
    size_t p = 0;
    float *bias = reinterpret_cast<float *>(out.image.data() + out.off_bias);
    for (int L = 0; L <= H; ++L) {
        uint8_t *W = out.image.data() + out.off_w[L];
        for (int n = 0; n < Nreal[L]; ++n)
            for (int k = 0; k < Kreal[L]; ++k) {
                uint16_t h = __half_as_ushort(__float2half_rn(mlp[p + (size_t)n * Kreal[L] + k]));
                std::memcpy(W + canon_off(n, k, Kl[L]), &h, 2);
            }
        p += (size_t)Nreal[L] * Kreal[L];
        for (int n = 0; n < Nreal[L]; ++n) bias[L * 64 + n] = mlp[p + n];
        p += (size_t)Nreal[L];
    }
}

int field_launch_config(const FieldHost &h, int &n_wg, size_t &smem, int device) {
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const size_t per_wg = 32768;  // two 128 x 64 fp16 chunk tiles
    const size_t fixed = h.image.size() + 256;
    n_wg = 0;
    for (int k = 4; k >= 1; --k)
        if (fixed + k * per_wg <= (size_t)max_smem) {
            n_wg = k;
            break;
        }
    smem = fixed + (size_t)n_wg * per_wg;
    return n_wg > 0 ? 0 : 1;
}

template <int FP, int FD>
static cudaError_t launch_t(const FieldParams &P, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_field<FP, FD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    k_field<FP, FD><<<grid, P.n_wg * 128, smem, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_field(const FieldParams &P, int fp, int fd, int grid, size_t smem,
                         cudaStream_t st) {
#define PF_FIELD_CASE(a, b) \
    if (fp == a && fd == b) return launch_t<a, b>(P, grid, smem, st);
    PF_FIELD_CASE(2, 2)
    PF_FIELD_CASE(2, 4)
    PF_FIELD_CASE(2, 8)
    PF_FIELD_CASE(4, 2)
    PF_FIELD_CASE(4, 4)
    PF_FIELD_CASE(4, 8)
    PF_FIELD_CASE(8, 2)
    PF_FIELD_CASE(8, 4)
    PF_FIELD_CASE(8, 8)
#undef PF_FIELD_CASE
    return cudaErrorInvalidValue;
}

}  // namespace pfk
