// pf_pathtrace_fast.cu -- binary32 render_path_traced (pf_pathtrace.cuh):
// macro-cell majorant DDA + ratio-tracked shadow rays (statistical parity).
#include "pf_pathtrace.cuh"

namespace pfk {

cudaError_t launch_render_pt_fast(const DevScene &S, const TraceParams &P, int grid, cudaStream_t st) {
    k_render_pt<false><<<grid, PF_TRACE_THREADS, 0, st>>>(S, P);
    return cudaGetLastError();
}

int pt_grid_size_fast(int device) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_render_pt<false>, PF_TRACE_THREADS, 0);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace pfk
