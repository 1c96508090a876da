// pf_photon.h -- device photon tracer (Alg. 1) parameters and launchers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_device.cuh"

#define PF_MAX_TRACE_PHASES 8

namespace pfk {

// Byte layout of pf_photon (include/pf_gpu.h); pad[0] carries the deposit
// ordinal inside the scratch list and is zeroed on compaction.
struct PhotonOut {
    float pos[3];
    float dir[3];
    float pow[3];
    uint8_t g_index;
    uint8_t pad[3];
};
static_assert(sizeof(PhotonOut) == 40, "PhotonOut must match pf_photon");

struct PhotonTraceParams {
    uint64_t n_total;
    uint64_t initstate;  // splitmix64(seed ^ Trace * phi), rng.hpp:73-76
    int n_phases, max_bounces, rr_start;
    double rr_min, rr_max;
    double g[PF_MAX_TRACE_PHASES];
    PhotonOut *rec;           // scratch deposits [cap]
    uint32_t *rec_photon;     // owning photon of each scratch deposit
    unsigned long long cap;
    unsigned long long *counter;  // [0] deposits appended
    unsigned long long *steps;    // tentative collisions (statistics)
    uint32_t *counts;         // deposits per photon [n_total]
};

cudaError_t launch_trace_photons(const DevScene &S, const PhotonTraceParams &P, cudaStream_t st);
cudaError_t photon_scan_bytes(uint64_t n, size_t *bytes);
cudaError_t launch_photon_compact(const uint32_t *counts, uint32_t *offs, uint64_t n_photons, void *tmp,
                                  size_t tmp_bytes, const PhotonOut *rec, const uint32_t *rec_photon,
                                  uint64_t n_rec, PhotonOut *out, cudaStream_t st);

}  // namespace pfk
