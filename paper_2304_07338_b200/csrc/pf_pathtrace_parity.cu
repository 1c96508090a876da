// pf_pathtrace_parity.cu -- binary64 render_path_traced (pf_pathtrace.cuh).
// Compiled with --fmad=false like the parity render tracer.
#define PF_TU_PARITY_PT
#include "pf_pathtrace.cuh"

namespace pfk {

cudaError_t launch_render_pt_parity(const DevScene &S, const TraceParams &P, int grid, cudaStream_t st) {
    k_render_pt<true><<<grid, PF_TRACE_THREADS, 0, st>>>(S, P);
    return cudaGetLastError();
}

int pt_grid_size_parity(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_pt<true>, PF_TRACE_THREADS, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace pfk
