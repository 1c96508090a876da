// pf_trace_parity.cu -- binary64 parity instantiation of pf_trace.cuh.
// Compiled with --fmad=false: the reference (x86-64, -ffp-contract=off) never
// fuses a*b+c, so neither may we.
#define PF_TU_PARITY
#include "pf_trace.cuh"

namespace pfk {

cudaError_t launch_render_trace_parity(const DevScene &S, const TraceParams &P, int grid,
                                       cudaStream_t st) {
    k_render_trace_parity<<<grid, PF_TRACE_THREADS, 0, st>>>(S, P);
    return cudaGetLastError();
}

cudaError_t launch_delta_track_batch_parity(const DevScene &S, const BatchParams &B,
                                            cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_delta_track_batch<<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

cudaError_t launch_transmittance_batch(const DevScene &S, const BatchParams &B, cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_transmittance_batch<<<blocks, 128, 0, st>>>(S, B);
    return cudaGetLastError();
}

cudaError_t launch_rng_doubles(const BatchParams &B, cudaStream_t st) {
    const unsigned blocks = (unsigned)((B.n + 127) / 128);
    k_rng_doubles<<<blocks, 128, 0, st>>>(B);
    return cudaGetLastError();
}

int trace_grid_size_parity(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_trace_parity, PF_TRACE_THREADS, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace pfk
