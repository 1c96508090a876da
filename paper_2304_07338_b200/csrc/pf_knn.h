// pf_knn.h -- photon map (per-phase cell grid) + KNN internals.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_kernels.h"

#define PF_MAX_PHASES 8

namespace pfk {

struct PhotonRec {  // == pf_photon (photon.hpp:17-22), 40 bytes
    float position[3];
    float direction[3];
    float power[3];
    uint8_t g_index;
    uint8_t pad_[3];
};
static_assert(sizeof(PhotonRec) == 40, "PhotonRec must be 40 B");

struct KnnGrid {
    double lo[3], h[3], inv_h[3];
    double hmin, eps;  // smallest cell edge; absolute bound slack
    int R[3];
    uint32_t cell_base;
    uint32_t n;        // photons of this phase
};

struct KnnParams {
    int n_phases;
    uint32_t total_cells;
    KnnGrid grid[PF_MAX_PHASES];
    double phase[PF_MAX_PHASES];
    const float4 *spos;           // sorted {x, y, z, id}
    const float4 *spay;           // sorted {dir xyz, power r} {power g, b, -, -}
    const uint32_t *inv;          // id -> sorted index
    const uint32_t *cell_start;   // total_cells + 1
    const PhotonRec *photons;     // load order (ids)
    size_t nq;
    const uint32_t *order;        // optional visit order (spatially sorted queries)
    const float *qx;
    const uint8_t *qg;
    const double *qw;
    int K;
    float r2;
    double psi, enc_threshold;    // Eq. 7: 10^-psi
    uint32_t *out_ids;
    float *out_d2;
    int32_t *out_counts;
    double *out_targets;
    // render_photon_map: queries are the render tracer's hit
    // records (count on the device), phase = render_g, omega = hit_dir; the
    // estimate lands in the sample slots as w_i * sigma_s * L (Eq. 6, no Eq. 7).
    // large-K CTA kernel: queries it could not resolve (never observed) are
    // appended here and re-run on the warp kernel
    uint32_t *fallback;
    unsigned *fallback_n;
    const HitRec *hits;
    const double *hit_dir;
    const unsigned long long *n_hits;
    void *slots;
    int slot_f64, render_g;
    double w_i;
};

struct KnnBuffers {
    DevBuf keys, vals, keys2, vals2, hist, cell_start, spos, spay, inv, temp, temp2;
    DevBuf qk, qi, qk2, qi2, temp3;  // query visit-order sort
    DevBuf fb, fbn;                  // large-K fallback list
};

cudaError_t knn_bbox(const PhotonRec *ph, size_t n, int n_phases, uint32_t *mins, uint32_t *maxs,
                     uint32_t *counts, cudaStream_t st);
cudaError_t knn_sort(const PhotonRec *ph, size_t n, const KnnParams &P, KnnBuffers &B,
                     cudaStream_t st);
cudaError_t knn_query(const KnnParams &P, cudaStream_t st);
// K > 64: CTA-per-query select kernel + exact warp-kernel fallback (syncs the stream)
cudaError_t knn_query_auto(KnnParams P, KnnBuffers &B, cudaStream_t st);
// render mode: P.nq = upper bound on the hit count, grid-stride over *P.n_hits
cudaError_t knn_query_render(const KnnParams &P, int sms, cudaStream_t st);
cudaError_t knn_order(const float *x3, const uint8_t *g, size_t n, KnnBuffers &B, const uint32_t **order,
                      cudaStream_t st);
cudaError_t knn_make_queries(uint64_t initstate, uint64_t base, size_t batch, int n_phases,
                             float *x3, double *w3, uint8_t *gidx, cudaStream_t st);

}  // namespace pfk
