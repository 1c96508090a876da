// pf_kernels.h -- host/device shared structs and kernel launchers (internal).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define PF_TRACE_THREADS 128
#define PF_MACRO 8  // default voxels per macro-cell edge (FAST-mode majorant grid)

namespace pfk {

struct DevScene;

// Grow-only device buffer.
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    ~DevBuf() { release(); }
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
};

// Compacted hit record: one per camera sample with a real interaction.
struct HitRec {
    float x[3];     // interaction position (field input)
    float wsph[2];  // omega_out in normalized spherical coords
    uint32_t slot;  // work index of the sample (where L_i lands)
    double sigma_s; // alpha * mean(rgb) at the interaction
};
static_assert(sizeof(HitRec) == 32, "HitRec must stay 32 B");

struct TraceParams {
    uint64_t init_cam, init_nee;  // splitmix64(seed ^ stream*phi) per stream
    double cam_o[3], cam_f[3], cam_r[3], cam_u[3];
    int W, H, spp;
    int tile_w, tile_h, tiles_x, shard_index, shard_count;
    uint32_t n_work;
    double g, w_d;
    double bg[3];
    int nee_trials, use_field;
    void *slots;                    // 3 x (double | float) per work item
    HitRec *hits;
    double *hit_dir;                // optional: omega_out per hit record (photon-map L_i source)
    unsigned long long *counters;   // [0] work, [1] hits, [2] primary steps, [3] shadow steps
    // render_path_traced only: continuation stream + roulette
    uint64_t init_pt;
    int max_bounces, rr_start;
    double rr_min, rr_max, w_i;
};

struct BatchParams {
    size_t n;
    uint64_t initstate;
    const uint64_t *idx;
    const double *a3, *b3, *tmin, *tmax;
    int n_trials;
    int *hit;
    double *pos3, *rgba4, *out;
    double *scalar;  // Interaction::scalar (volume.hpp:82-86), optional
};

// Per-pixel compose over the spp slots (K5) + tile helpers.
struct ComposeParams {
    int W, H, spp, tile_w, tile_h, tiles_x, shard_index, shard_count;
    uint32_t n_local_tiles;
    const void *slots;
    float *out;   // full frame, row-major RGB
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_render_trace(bool parity, const DevScene &S, const TraceParams &P, int grid,
                                cudaStream_t st);
cudaError_t launch_delta_track_batch(bool parity, const DevScene &S, const BatchParams &B,
                                     cudaStream_t st);
cudaError_t launch_transmittance_batch(const DevScene &S, const BatchParams &B, cudaStream_t st);
cudaError_t launch_transmittance_ratio_batch(const DevScene &S, const BatchParams &B,
                                             cudaStream_t st);
cudaError_t launch_rng_doubles(const BatchParams &B, cudaStream_t st);
cudaError_t launch_compose(bool parity, const ComposeParams &C, cudaStream_t st);
cudaError_t launch_tiles_pack(const ComposeParams &C, const float *frame, float *packed,
                              cudaStream_t st);
cudaError_t launch_tiles_unpack(const ComposeParams &C, const float *packed_all,
                                size_t per_shard_floats, float *frame, cudaStream_t st);
int trace_grid_size(bool parity, int device);
cudaError_t launch_macro_minmax(const float *vol, int nx, int ny, int nz, float2 *mm, int mcx, int mcy,
                                int mcz, int macro, cudaStream_t st);
// transfer-function control points passed by value (no host->device copy per TF change)
struct TfPoints {
    double p[16 * 5];
};
cudaError_t launch_macro_majorant(const float2 *mm, size_t ncells, const TfPoints &tf_pts, int n_tf,
                                  double density_scale, float *maj, uint32_t *maj_hi, int mcx, int mcy, int *occ,
                                  cudaStream_t st);
cudaError_t launch_build_atlas(const float *vol, int nx, int ny, int nz, int log2_cols, float *atlas,
                               size_t aw, size_t ah, cudaStream_t st);

}  // namespace pfk
