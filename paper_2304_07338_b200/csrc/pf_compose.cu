// pf_compose.cu -- K5 compose + multi-GPU tile pack/unpack.
//
// compose (Alg. 2):
//   L(pixel) = (1/spp) * sum_{k=0..spp-1} slot_k
// where slot_k already holds w_d*L_d,k + w_i*sigma_s,k*L_i,k (or the
// background for samples that never interact).  The sum runs in sample order
// k = 0..spp-1 (binary64 in parity mode), exactly like the oracle, so the
// frame is deterministic and independent of the tile/GPU partition.
#include "pf_kernels.h"

namespace pfk {

__device__ __forceinline__ bool tile_pixel(const ComposeParams &C, uint32_t lt, uint32_t pix,
                                           int &px, int &py) {
    const uint32_t t = lt * (uint32_t)C.shard_count + (uint32_t)C.shard_index;
    const uint32_t ty = t / (uint32_t)C.tiles_x, tx = t - ty * (uint32_t)C.tiles_x;
    const uint32_t ly = pix / (uint32_t)C.tile_w;
    px = (int)(tx * (uint32_t)C.tile_w + (pix - ly * (uint32_t)C.tile_w));
    py = (int)(ty * (uint32_t)C.tile_h + ly);
    return px < C.W && py < C.H;
}

template <typename S>
__global__ void k_compose(const ComposeParams C) {
    const uint32_t tile_px = (uint32_t)(C.tile_w * C.tile_h);
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)C.n_local_tiles * tile_px) return;
    const uint32_t lt = (uint32_t)(i / tile_px), pix = (uint32_t)(i - (size_t)lt * tile_px);
    int px, py;
    if (!tile_pixel(C, lt, pix, px, py)) return;
    const S *s = reinterpret_cast<const S *>(C.slots) + 3 * i * (size_t)C.spp;
    S acc0 = 0, acc1 = 0, acc2 = 0;
    for (int k = 0; k < C.spp; ++k) {
        acc0 += s[3 * k];
        acc1 += s[3 * k + 1];
        acc2 += s[3 * k + 2];
    }
    float *o = C.out + 3 * ((size_t)py * C.W + px);
    o[0] = (float)(acc0 / (S)C.spp);
    o[1] = (float)(acc1 / (S)C.spp);
    o[2] = (float)(acc2 / (S)C.spp);
}

__global__ void k_tiles_pack(const ComposeParams C, const float *frame, float *packed) {
    const uint32_t tile_px = (uint32_t)(C.tile_w * C.tile_h);
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)C.n_local_tiles * tile_px) return;
    const uint32_t lt = (uint32_t)(i / tile_px), pix = (uint32_t)(i - (size_t)lt * tile_px);
    int px, py;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f;
    if (tile_pixel(C, lt, pix, px, py)) {
        const float *f = frame + 3 * ((size_t)py * C.W + px);
        v0 = f[0];
        v1 = f[1];
        v2 = f[2];
    }
    packed[3 * i] = v0;
    packed[3 * i + 1] = v1;
    packed[3 * i + 2] = v2;
}

// packed_all = shard_count consecutive buffers of per_shard floats; shard r's
// local tile j is global tile j*shard_count + r.
__global__ void k_tiles_unpack(ComposeParams C, const float *packed_all, size_t per_shard,
                               float *frame) {
    const uint32_t tile_px = (uint32_t)(C.tile_w * C.tile_h);
    const uint32_t tiles_y = (uint32_t)((C.H + C.tile_h - 1) / C.tile_h);
    const size_t n_tiles = (size_t)C.tiles_x * tiles_y;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tiles * tile_px) return;
    const uint32_t t = (uint32_t)(i / tile_px), pix = (uint32_t)(i - (size_t)t * tile_px);
    const uint32_t r = t % (uint32_t)C.shard_count, lt = t / (uint32_t)C.shard_count;
    C.shard_index = (int)r;
    int px, py;
    if (!tile_pixel(C, lt, pix, px, py)) return;
    const float *src = packed_all + r * per_shard + 3 * ((size_t)lt * tile_px + pix);
    float *dst = frame + 3 * ((size_t)py * C.W + px);
    dst[0] = src[0];
    dst[1] = src[1];
    dst[2] = src[2];
}

// Slice atlas for the volume texture: tile (z % cols, z / cols) holds slice z
// with its last row / column duplicated (the reference's min(i+1, n-1) clamp).
__global__ void k_build_atlas(const float *vol, int nx, int ny, int nz, int lg, float *atlas, size_t aw,
                              size_t ah) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= aw * ah) return;
    const size_t ay = i / aw, ax = i - ay * aw;
    const int tx = (int)(ax / (size_t)(nx + 1)), ty = (int)(ay / (size_t)(ny + 1));
    const int x = min((int)(ax - (size_t)tx * (nx + 1)), nx - 1);
    const int y = min((int)(ay - (size_t)ty * (ny + 1)), ny - 1);
    const int z = (ty << lg) + tx;
    atlas[i] = z < nz ? vol[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * (size_t)z)] : 0.0f;
}

cudaError_t launch_build_atlas(const float *vol, int nx, int ny, int nz, int lg, float *atlas, size_t aw,
                               size_t ah, cudaStream_t st) {
    const size_t n = aw * ah;
    k_build_atlas<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vol, nx, ny, nz, lg, atlas, aw, ah);
    return cudaGetLastError();
}

// Per macro cell: min/max scalar over the voxels a trilinear sample inside
// the cell can touch (indices [c*B-1, c*B+B], clamped).
__global__ void k_macro_minmax(const float *vol, int nx, int ny, int nz, float2 *mm, int mcx, int mcy, int mcz,
                               int B) {
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (size_t)mcx * mcy * mcz) return;
    const int cx = (int)(c % mcx), cy = (int)((c / mcx) % mcy), cz = (int)(c / ((size_t)mcx * mcy));
    const int x0 = max(cx * B - 1, 0), x1 = min(cx * B + B, nx - 1);
    const int y0 = max(cy * B - 1, 0), y1 = min(cy * B + B, ny - 1);
    const int z0 = max(cz * B - 1, 0), z1 = min(cz * B + B, nz - 1);
    float lo = 1e30f, hi = -1e30f;
    for (int z = z0; z <= z1; ++z)
        for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
                const float v = vol[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * (size_t)z)];
                lo = fminf(lo, v);
                hi = fmaxf(hi, v);
            }
    mm[c] = make_float2(lo, hi);
}

// majorant = density_scale * TransferFunction::max_alpha(lo, hi) (volume.cpp:163-168), padded 1e-5.
__device__ double tf_alpha_host_like(const TfPoints &T, int n, double s) {
    const double *p = T.p;
    s = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
    int hi = 1;
    while (hi + 1 < n && p[hi * 5] < s) ++hi;
    double t = (s - p[(hi - 1) * 5]) / (p[hi * 5] - p[(hi - 1) * 5]);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return p[(hi - 1) * 5 + 4] + (p[hi * 5 + 4] - p[(hi - 1) * 5 + 4]) * t;
}

__global__ void k_macro_majorant(const float2 *mm, size_t ncells, const TfPoints T, int n, double ds, float *maj,
                                 uint32_t *maj_hi, int mcx, int mcy, int *occ) {
    const double *tf = T.p;
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    const double lo = mm[c].x, hi = mm[c].y;
    double m = fmax(tf_alpha_host_like(T, n, lo), tf_alpha_host_like(T, n, hi));
    for (int i = 0; i < n; ++i)
        if (tf[5 * i] > lo && tf[5 * i] < hi) m = fmax(m, tf[5 * i + 4]);
    const float b = m > 0.0 ? (float)(ds * m * (1.0 + 1e-5)) : 0.0f;
    maj[c] = b;
    // high word of (double)b, rounded up: as_double(hi, 0) >= b
    const unsigned long long bits = (unsigned long long)__double_as_longlong((double)b);
    maj_hi[c] = (uint32_t)(bits >> 32) + ((uint32_t)bits != 0u ? 1u : 0u);
    if (m > 0.0) {  // occupied-cell bounding box
        const int cx = (int)(c % (size_t)mcx), cy = (int)((c / (size_t)mcx) % (size_t)mcy),
                  cz = (int)(c / ((size_t)mcx * (size_t)mcy));
        atomicMin(&occ[0], cx);
        atomicMin(&occ[1], cy);
        atomicMin(&occ[2], cz);
        atomicMax(&occ[3], cx);
        atomicMax(&occ[4], cy);
        atomicMax(&occ[5], cz);
    }
}

cudaError_t launch_macro_minmax(const float *vol, int nx, int ny, int nz, float2 *mm, int mcx, int mcy, int mcz,
                                int B, cudaStream_t st) {
    const size_t n = (size_t)mcx * mcy * mcz;
    k_macro_minmax<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(vol, nx, ny, nz, mm, mcx, mcy, mcz, B);
    return cudaGetLastError();
}

cudaError_t launch_macro_majorant(const float2 *mm, size_t ncells, const TfPoints &tf_pts, int n_tf, double ds,
                                  float *maj, uint32_t *maj_hi, int mcx, int mcy, int *occ, cudaStream_t st) {
    // occ = {INT_MAX-ish x3, -1 x3} before the min / max reduction
    cudaError_t e = cudaMemsetAsync(occ, 0x7f, 3 * sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(occ + 3, 0xff, 3 * sizeof(int), st);
    if (e != cudaSuccess) return e;
    k_macro_majorant<<<(unsigned)((ncells + 255) / 256), 256, 0, st>>>(mm, ncells, tf_pts, n_tf, ds, maj, maj_hi, mcx, mcy,
                                                                      occ);
    return cudaGetLastError();
}

cudaError_t launch_compose(bool parity, const ComposeParams &C, cudaStream_t st) {
    const size_t n = (size_t)C.n_local_tiles * C.tile_w * C.tile_h;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (parity) k_compose<double><<<blocks, 256, 0, st>>>(C);
    else k_compose<float><<<blocks, 256, 0, st>>>(C);
    return cudaGetLastError();
}

cudaError_t launch_tiles_pack(const ComposeParams &C, const float *frame, float *packed,
                              cudaStream_t st) {
    const size_t n = (size_t)C.n_local_tiles * C.tile_w * C.tile_h;
    if (n == 0) return cudaSuccess;
    k_tiles_pack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(C, frame, packed);
    return cudaGetLastError();
}

cudaError_t launch_tiles_unpack(const ComposeParams &C, const float *packed_all,
                                size_t per_shard_floats, float *frame, cudaStream_t st) {
    const size_t tiles_y = (size_t)((C.H + C.tile_h - 1) / C.tile_h);
    const size_t n = (size_t)C.tiles_x * tiles_y * C.tile_w * C.tile_h;
    if (n == 0) return cudaSuccess;
    k_tiles_unpack<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(C, packed_all, per_shard_floats,
                                                                 frame);
    return cudaGetLastError();
}

}  // namespace pfk
