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

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pf_field.h"
#include "pf_field_dev.cuh"
#include "pf_hashgrid.cuh"
#include "pf_umma.cuh"

namespace pfk {


// Feature tiles are staged in chunks of PF_FIELD_CW columns (128 rows x CW
// fp16 = CW * 256 bytes, one bulk-TMA copy each): the MLP keeps
// a_bytes / chunk_bytes of them in flight per warpgroup while layer 0's MMAs
// consume the previous ones.
#ifndef PF_FIELD_CW
#define PF_FIELD_CW 32
#endif
static_assert(PF_FIELD_CW == 16 || PF_FIELD_CW == 32 || PF_FIELD_CW == 64, "chunk width 16, 32 or 64 columns");
constexpr uint32_t kFieldChunkBytes = PF_FIELD_CW * 256u;

// Byte offset of element (row, k) in the feature-tile buffer: tile-major,
// then CW-column chunks, each a canonical K-major UMMA tile.
__device__ __forceinline__ size_t feat_off(const FieldParams &P, size_t row, int k) {
    const size_t tile = row >> 7;
    const int r = (int)(row & 127), chunk = k / PF_FIELD_CW, kk = k % PF_FIELD_CW;
    const int kw = min(PF_FIELD_CW, P.K0 - PF_FIELD_CW * chunk);
    return (tile * (size_t)P.nch + (size_t)chunk) * kFieldChunkBytes +
           (size_t)((r >> 3) * kw * 16 + (kk >> 3) * 128 + (r & 7) * 16 + (kk & 7) * 2);
}

template <int F>
__device__ __forceinline__ void st_feats_global(uint8_t *p, const float *acc) {
    uint32_t h[F / 2];
#pragma unroll
    for (int i = 0; i < F / 2; ++i) {
        __half2 v = __floats2half2_rn(acc[2 * i], acc[2 * i + 1]);
        h[i] = *reinterpret_cast<uint32_t *>(&v);
    }
    // streaming stores (evict-first): the 0.9 GB of feature tiles must not
    // push the level-major encoder's hash tables out of L2
    if constexpr (F == 8) __stcs(reinterpret_cast<uint4 *>(p), make_uint4(h[0], h[1], h[2], h[3]));
    else if constexpr (F == 4) __stcs(reinterpret_cast<uint2 *>(p), make_uint2(h[0], h[1]));
    else __stcs(reinterpret_cast<unsigned int *>(p), h[0]);
}

#ifndef PF_ENC_G
#define PF_ENC_G 2
#endif
static_assert(PF_ENC_G == 2 || PF_ENC_G == 4 || PF_ENC_G == 8, "levels per encoder sweep: 2, 4 or 8");

// K3: hash-grid encoding, one thread per (query, unit); a warp covers 16
// queries x 2 units (PF_ENC_G units per level-major sweep: A/B 2 < 4 < 8 by
// 3% / 9%, the hash tables in use stay L2-resident) so each level's rows land
// as contiguous 128-byte stores.  Units: pos levels, dir levels, then one
// "g + zero padding" unit.  6 CTAs of 256 per SM (40 registers).
#ifndef PF_ENC_MINB
#define PF_ENC_MINB 6
#endif
template <int FP, int FD>
__global__ void __launch_bounds__(256, PF_ENC_MINB) k_field_encode(const FieldParams P) {
    const size_t n_all = P.mode == 0 ? (size_t)(*P.n_hits) : P.n_query;
    const size_t n = n_all > P.row0 ? min(n_all - P.row0, P.row_cap) : 0;  // rows of this launch
    const size_t n_rows = (n + 127) & ~(size_t)127;  // whole tiles (pad rows encode zeros)
    // PF_ENC_G levels per sweep (a warp covers 32 / G rows x G levels)
    constexpr int G = PF_ENC_G, RW = 32 / G;
    const int U = P.n_pos_levels + P.n_dir_levels + 1, UG = (U + G - 1) / G;
    const int lane = threadIdx.x & 31;
    const uint32_t warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_rg = (uint32_t)(n_rows / RW);  // RW-row groups (render rows < 2^32)
    // per-level addressing in shared memory: each warp reads 4 different
    // levels, which a dynamically indexed kernel-parameter load serialises
    __shared__ FieldLevel s_lv[PF_FIELD_MAX_LEVELS];
    for (int i = threadIdx.x; i < U - 1 && i < PF_FIELD_MAX_LEVELS; i += blockDim.x) s_lv[i] = P.lv[i];
    __syncthreads();
    // level-major: the whole grid sweeps all rows for one group of 4 levels
    // before the next, so the tables in use (4 x <= 8 MB at the paper config)
    // stay L2-resident instead of being gathered from DRAM
    for (int ug = 0; ug < UG; ++ug)
    for (uint32_t rg = warp0; rg < n_rg; rg += n_warps) {
        const size_t row = (size_t)rg * RW + (lane % RW);
        const int u = ug * G + lane / RW;
        if (u >= U) continue;
        const bool valid = row < n;
        const size_t gr = P.row0 + row;  // global item index
        float x[3] = {0.f, 0.f, 0.f}, ws[2] = {0.f, 0.f}, gin = 0.f;
        if (valid) {
            if (P.mode == 0) {
                // x[3] + wsph[2]: the first 20 bytes of the 32-byte record
                const float4 a = __ldg(reinterpret_cast<const float4 *>(P.hits + gr));
                x[0] = a.x, x[1] = a.y, x[2] = a.z;
                ws[0] = a.w, ws[1] = __ldg(&P.hits[gr].wsph[1]);
                gin = P.g_render;
            } else {
                x[0] = P.qx[3 * gr], x[1] = P.qx[3 * gr + 1], x[2] = P.qx[3 * gr + 2];
                ws[0] = P.qw[2 * gr], ws[1] = P.qw[2 * gr + 1];
                gin = P.qg[gr];
            }
        }
        if (u < P.n_pos_levels) {
            float pin[3] = {__saturatef(x[0]), __saturatef(x[1]), __saturatef(x[2])};
            float acc[FP];
            encode_level<3, FP>(P.tables, s_lv[u], pin, acc);
            st_feats_global<FP>(P.feat + feat_off(P, row, u * FP), acc);
        } else if (u < P.n_pos_levels + P.n_dir_levels) {
            const int l = u - P.n_pos_levels;
            float pin[2] = {__saturatef(ws[0]), __saturatef(ws[1])};
            float acc[FD];
            encode_level<2, FD>(P.tables, s_lv[P.n_pos_levels + l], pin, acc);
            st_feats_global<FD>(P.feat + feat_off(P, row, P.n_pos_levels * FP + l * FD), acc);
        } else {
            const int kg = P.n_pos_levels * FP + P.n_dir_levels * FD;  // multiple of 8
            const uint32_t gh = valid ? (uint32_t)__half_as_ushort(__float2half_rn((gin + 1.0f) * 0.5f)) : 0u;
            *reinterpret_cast<uint4 *>(P.feat + feat_off(P, row, kg)) = make_uint4(gh, 0u, 0u, 0u);
            for (int k = kg + 8; k < P.K0; k += 8)
                *reinterpret_cast<uint4 *>(P.feat + feat_off(P, row, k)) = make_uint4(0u, 0u, 0u, 0u);
        }
    }
}

// K4: the MLP on tcgen05.  Persistent CTA per SM with the whole MLP image in
// shared memory; each warpgroup owns a 128-row tile pipeline:
//   layer 0: the tile's feature chunks (PF_FIELD_CW columns each) stream in
//            by 1-D bulk TMA through NS = a_bytes / chunk-bytes slots
//            (mbarrier complete_tx), so NS chunk loads are in flight while the
//            kw/16 tcgen05.mma (M=128, N=64, K=16) of the oldest accumulate
//            into the warpgroup's 64-column TMEM accumulator;
//   layers 1..H: tcgen05.ld -> bias + ReLU -> fp16 -> st.shared into the A
//            tile -> next layer's MMA (N=16 for the 3-wide output layer);
//   epilogue: Eq. 8 decode, compose term into the sample's slot.
__global__ void __launch_bounds__(1024, 1) k_field_mlp(const FieldParams P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *img = smem;
    uint8_t *abase = smem + P.img_bytes;
    // barriers: [0] weights; per warpgroup w at 1 + (2 NS + 1) w: full[NS], empty[NS], done.
    // The warpgroup's a_bytes of shared memory hold NS layer-0 chunk slots
    // (filled by bulk TMA while the MMAs of earlier chunks run) and, from
    // layer 1 on, the 16 KB activation tile.
    const int NS = min(8, (int)(P.a_bytes / kFieldChunkBytes));
    const int NB = 2 * NS + 1;
    uint64_t *bars = reinterpret_cast<uint64_t *>(abase + (size_t)P.n_wg * P.a_bytes);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 1 + NB * P.n_wg);

    const int tid = threadIdx.x, wg = tid >> 7, r = tid & 127, warp = tid >> 5;
    if (tid == 0) {
        for (int i = 0; i <= NB * P.n_wg; ++i) mbar_init(smem_u32(&bars[i]), 1);
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

    const size_t n_all = P.mode == 0 ? (size_t)(*P.n_hits) : P.n_query;
    const size_t n_items = n_all > P.row0 ? min(n_all - P.row0, P.row_cap) : 0;
    const size_t n_tiles = (n_items + 127) / 128;
    const uint32_t abuf = smem_u32(abase + (size_t)wg * P.a_bytes);  // slot b at abuf + b * chunk bytes
    const uint32_t img_s = smem_u32(img);
    const uint32_t tmem_wg = tmem_base + (uint32_t)(wg * 64);
    const uint32_t tmem_rows = tmem_wg + ((uint32_t)(32 * (warp & 3)) << 16);
    uint64_t *wb = bars + 1 + NB * wg;
    const uint32_t full0 = smem_u32(&wb[0]), empty0 = smem_u32(&wb[NS]), done = smem_u32(&wb[2 * NS]);
    uint32_t full_par = 0u, empty_par = 0u, pending = 0u, ph_done = 0u;  // per-slot phase bits
    const float *bias = reinterpret_cast<const float *>(img + P.off_bias);
    const uint32_t sbo_w0 = (uint32_t)P.K0 * 16u;

    for (size_t tile = (size_t)blockIdx.x * P.n_wg + wg; tile < n_tiles; tile += (size_t)gridDim.x * P.n_wg) {
        const uint8_t *tsrc = P.feat + tile * (size_t)P.nch * kFieldChunkBytes;
        // ---- layer 0: TMA-fed chunks (only thread r == 0 drives the pipeline)
        if (r == 0) {
            auto load = [&](int j) {
                const int b = j % NS;
                if (pending & (1u << b)) {  // the slot's previous chunk is still being read by its MMAs
                    mbar_wait(empty0 + 8u * b, (empty_par >> b) & 1u);
                    empty_par ^= 1u << b;
                    pending &= ~(1u << b);
                }
                const uint32_t bytes = (uint32_t)min(PF_FIELD_CW, P.K0 - PF_FIELD_CW * j) * 256u;  // 128 rows x kw x 2 B
                mbar_expect_tx(full0 + 8u * b, bytes);
                bulk_g2s(abuf + (uint32_t)b * kFieldChunkBytes, tsrc + (size_t)j * kFieldChunkBytes, bytes,
                         full0 + 8u * b);
            };
            for (int j = 0; j < NS && j < P.nch; ++j) load(j);
            for (int j = 0; j < P.nch; ++j) {
                const int b = j % NS;
                mbar_wait(full0 + 8u * b, (full_par >> b) & 1u);
                full_par ^= 1u << b;
                tc_fence_after();
                const int kw = min(PF_FIELD_CW, P.K0 - PF_FIELD_CW * j);
                const uint32_t sbo = (uint32_t)kw * 16u, idesc = umma_idesc_f16(128, 64);
                const uint32_t a0 = abuf + (uint32_t)b * kFieldChunkBytes;
                const uint32_t b0 = img_s + P.off_w[0] + (uint32_t)(j * (PF_FIELD_CW / 8)) * 128u;
                for (int s = 0; s < kw / 16; ++s) {
                    const uint64_t ad = umma_sdesc(a0 + 256u * s, 128u, sbo);
                    const uint64_t bd = umma_sdesc(b0 + 256u * s, 128u, sbo_w0);
                    umma_f16(tmem_wg, ad, bd, idesc, (j > 0 || s > 0) ? 1u : 0u);
                }
                umma_commit(empty0 + 8u * b);
                pending |= 1u << b;
                if (j + NS < P.nch) load(j + NS);  // waits for this slot's MMAs, the other slots stay in flight
            }
            umma_commit(done);
        }
        // one warp polls the mbarrier, the other three sleep in the named barrier
        if ((r >> 5) == 0) mbar_wait(done, ph_done);
        named_bar_sync(1 + wg, 128);
        ph_done ^= 1u;
        tc_fence_after();
        if (r == 0) {  // keep the per-slot parities in step (every MMA is complete by now)
            for (int b = 0; b < NS; ++b)
                if (pending & (1u << b)) {
                    mbar_wait(empty0 + 8u * b, (empty_par >> b) & 1u);
                    empty_par ^= 1u << b;
                }
            pending = 0u;
        }

        // ---- hidden layers (epilogue of layer L-1 feeds the MMA of layer L)
        for (int L = 1; L <= P.hidden_layers; ++L) {
            const float *bl = bias + (L - 1) * 64;
            const uint32_t pa = abuf + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 16u;  // K=64: SBO 1024
            // two halves of 32 columns: both 16-column loads of a half in flight, one wait
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t acc[32];
                tmem_ld16(tmem_rows + 32 * hf, acc);
                tmem_ld16(tmem_rows + 32 * hf + 16, acc + 16);
                tmem_ld_wait();
                tmem_regs_ready<32>(acc);
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int col = 32 * hf + 16 * c;
                    float a[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) a[i] = fmaxf(__uint_as_float(acc[16 * c + i]) + bl[col + i], 0.f);
                    store_feats<8>(pa, 0, col, 1024u, a);
                    store_feats<8>(pa, 0, col + 8, 1024u, a + 8);
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();
            named_bar_sync(1 + wg, 128);
            if (r == 0) {
                tc_fence_after();
                issue_layer(abuf, img_s + P.off_w[L], 64, L < P.hidden_layers ? 64 : 16, tmem_wg);
                umma_commit(done);
            }
            if ((r >> 5) == 0) mbar_wait(done, ph_done);
            named_bar_sync(1 + wg, 128);
            ph_done ^= 1u;
            tc_fence_after();
        }

        // ---- output layer epilogue: bias, Eq. 8 decode, compose term
        uint32_t vr[16];
        tmem_ld16(tmem_rows, vr);
        tmem_ld_wait();
        tmem_regs_ready<16>(vr);
        tc_fence_before();
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(vr[i]);
        named_bar_sync(1 + wg, 128);  // all rows read TMEM / A before the next tile reuses them
        const size_t row = tile * 128 + r, gr = P.row0 + row;
        if (row < n_items) {
            const float *bo = bias + P.hidden_layers * 64;
            const float o3[3] = {v[0] + bo[0], v[1] + bo[1], v[2] + bo[2]};
            if (P.mode == 0) {
                const HitRec h = P.hits[gr];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const float Li = exp2f(-__saturatef(o3[c]) * P.psi_log2_10);  // Eq. 8
                    if (P.slot_f64) {
                        double *sp = reinterpret_cast<double *>(P.slots) + 3 * (size_t)h.slot + c;
                        *sp = *sp + P.w_i * (h.sigma_s * (double)Li);
                    } else {
                        float *sp = reinterpret_cast<float *>(P.slots) + 3 * (size_t)h.slot + c;
                        *sp = *sp + (float)P.w_i * ((float)h.sigma_s * Li);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    P.qout[3 * gr + c] = P.decoded ? exp2f(-__saturatef(o3[c]) * P.psi_log2_10) : o3[c];
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
    // the direction tables start right after the position tables and are read
    // with F_dir-wide vector loads (fp16 encode, fp32 Adam): keep them aligned
    if (field_grid_param_count(d.pos) % (size_t)d.dir.features != 0)
        return "field: position table parameters must be a multiple of the direction feature count "
               "(16-byte aligned direction tables)";
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
    // --- tables -> fp16, same order as the flat vector; every level starts on
    // a 32-byte boundary, so the two entries of an x-edge whose first index is
    // even (dense: x even in the flattened index; hashed: cell x even, since
    // x ^ 1 flips only bit 0 of the hash) share one 32-byte sector at F = 8,
    // and F-wide vector loads of either grid stay aligned for any (Fp, Fd)
    out.levels.clear();
    out.enc_levels.clear();
    size_t off = 0, eoff = 0;
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
            L.offset_halves = (uint32_t)eoff;
            out.enc_levels.push_back(L);
            off += (size_t)v * g->features;
            eoff = (eoff + (size_t)v * g->features + 15) & ~(size_t)15;
        }
    }
    out.tables.assign(eoff, 0);
    for (size_t l = 0; l < out.levels.size(); ++l) {
        const size_t src = out.levels[l].offset_halves, dst = out.enc_levels[l].offset_halves;
        const size_t end = l + 1 < out.levels.size() ? out.levels[l + 1].offset_halves : off;
        for (size_t k = 0; k < end - src; ++k) out.tables[dst + k] = __half_as_ushort(__float2half_rn(params[src + k]));
    }
    const size_t ntab = off;
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

int field_launch_config(const FieldHost &h, int &n_wg, size_t &smem, size_t &a_bytes, int device) {
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const size_t fixed = h.image.size() + 2048;  // + mbarriers (<= 1 + 17 x 8) and the TMEM slot
    // preferred: 8 warpgroups x one 16 KB tile (8 tiles in flight per SM, TMEM
    // 8 x 64 columns); else up to 4 warpgroups x two 16 KB chunk buffers.
    // PF_MLP_WG=1..4 forces that many double-buffered warpgroups (A/B).
    const char *e = std::getenv("PF_MLP_WG");
    const int want = e ? std::atoi(e) : 8;
    n_wg = 0;
    if (want >= 8 && fixed + 8 * 16384 <= (size_t)max_smem) {
        n_wg = 8;
        a_bytes = 16384;
    } else {
        for (int k = std::min(4, std::max(1, want)); k >= 1; --k)
            if (fixed + k * 32768 <= (size_t)max_smem) {
                n_wg = k;
                break;
            }
        a_bytes = 32768;
    }
    smem = fixed + (size_t)n_wg * a_bytes;
    return n_wg > 0 ? 0 : 1;
}

int field_chunk_cols() { return PF_FIELD_CW; }

size_t field_feat_bytes(const FieldHost &h, size_t n_items) {
    const size_t nch = (size_t)((h.K0 + PF_FIELD_CW - 1) / PF_FIELD_CW);
    return ((n_items + 127) / 128) * nch * kFieldChunkBytes;
}

template <int FP, int FD>
static cudaError_t launch_encode(const FieldParams &P0, int grid, cudaStream_t st) {
    const FieldParams &P = P0;
    k_field_encode<FP, FD><<<grid, 256, 0, st>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_field(const FieldParams &P, int fp, int fd, int grid, size_t smem, cudaStream_t st) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int egrid = sms * 8;  // 2048 resident threads per SM
    cudaError_t e = cudaErrorInvalidValue;
#define PF_FIELD_CASE(a, b) \
    if (fp == a && fd == b) e = launch_encode<a, b>(P, egrid, st);
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
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_field_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_field_mlp<<<grid, P.n_wg * 128, smem, st>>>(P);
    return cudaGetLastError();
}

}  // namespace pfk
