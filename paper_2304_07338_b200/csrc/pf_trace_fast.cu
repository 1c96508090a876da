// pf_trace_fast.cu -- binary32 FAST instantiation of pf_trace.cuh (ratio-
// tracked shadow rays).  Same RNG streams as the parity path.
#define PF_TU_FAST
#include "pf_trace.cuh"

namespace pfk {

cudaError_t launch_render_trace_fast(const DevScene &S, const TraceParams &P, int grid,
                                     cudaStream_t st) {
    k_render_trace<false><<<grid, PF_TRACE_THREADS, 0, st>>>(S, P);
    return cudaGetLastError();
}

cudaError_t launch_delta_track_batch_fast(const DevScene &S, const BatchParams &B,
                                          cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_delta_track_batch<false><<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

cudaError_t launch_transmittance_ratio_batch(const DevScene &S, const BatchParams &B,
                                             cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_transmittance_ratio_batch<<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

int trace_grid_size_fast(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_trace<false>, PF_TRACE_THREADS, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace pfk
