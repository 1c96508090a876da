// pf_capi.cu -- the extern "C" boundary (include/pf_gpu.h) and the context.
//
// Host side of the drop-in: validation mirrors the reference's exceptions
// (std::invalid_argument -> PF_ERR_INVALID, runtime/CUDA -> PF_ERR_RUNTIME),
// scene state is kept device-resident per context, and every kernel runs on
// the context stream.  Calls with only device pointers are fully asynchronous;
// calls that return data into host memory synchronise the stream.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pf_gpu.h"
#include "pf_device.cuh"
#include "pf_field.h"
#include "pf_kernels.h"
#include "pf_knn.h"
#include "pf_photon.h"
#include "pf_train.h"

namespace pfk {
cudaError_t launch_render_trace_parity(const DevScene &, const TraceParams &, int, cudaStream_t);
cudaError_t launch_render_trace_fast(const DevScene &, const TraceParams &, int, cudaStream_t);
cudaError_t launch_delta_track_batch_parity(const DevScene &, const BatchParams &, cudaStream_t);
cudaError_t launch_delta_track_batch_fast(const DevScene &, const BatchParams &, cudaStream_t);
int trace_grid_size_parity(int device);
int trace_grid_size_fast(int device);
cudaError_t launch_render_pt_parity(const DevScene &, const TraceParams &, int, cudaStream_t);
cudaError_t launch_render_pt_fast(const DevScene &, const TraceParams &, int, cudaStream_t);
int pt_grid_size_parity(int device);
int pt_grid_size_fast(int device);
}  // namespace pfk

using namespace pfk;

namespace {

thread_local std::string g_err;

int set_err(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// A failed call is reported once: the runtime's (non-sticky) last-error state
// is cleared so a later, unrelated cudaGetLastError() check does not re-report it.
#define PF_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            (void)cudaGetLastError();                                                      \
            return set_err(PF_ERR_RUNTIME, "%s failed: %s", #call, cudaGetErrorString(e_)); \
        }                                                                                  \
    } while (0)

uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// make_rng's initstate (rng.hpp:73-76)
uint64_t stream_initstate(uint64_t seed, uint64_t stream) {
    return splitmix64(seed ^ (stream * 0x9e3779b97f4a7c15ULL));
}

// Host PCG32 (rng.hpp) for pf_field_init.
struct HostPcg {
    uint64_t state = 0, inc = 0;
    uint32_t next() {
        uint64_t old = state;
        state = old * 6364136223846793005ULL + inc;
        uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = (uint32_t)(old >> 59u);
        return (xs >> rot) | (xs << ((0u - rot) & 31u));
    }
    void seed(uint64_t initstate, uint64_t initseq) {
        state = 0;
        inc = (initseq << 1u) | 1u;
        next();
        state += initstate;
        next();
    }
    double next_double() {
        uint64_t hi = next();
        uint64_t lo = next();
        return (double)(((hi << 32) | lo) >> 11) * 0x1.0p-53;
    }
};

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// TransferFunction::classify on the host (volume.cpp:151-161) for max_alpha.
double tf_classify_alpha(const std::vector<double> &pts, double scalar) {
    const int n = (int)pts.size() / 5;
    double s = scalar < 0.0 ? 0.0 : (scalar > 1.0 ? 1.0 : scalar);
    int hi = 1;
    while (hi + 1 < n && pts[hi * 5] < s) ++hi;
    const double *a = &pts[(hi - 1) * 5], *b = &pts[hi * 5];
    double t = (s - a[0]) / (b[0] - a[0]);
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    return a[4] + (b[4] - a[4]) * t;
}

// Macro-cell edge in voxels (PF_MACRO; PF_MACRO_CELL overrides it for tuning sweeps).
int macro_default() {
    const char *e = std::getenv("PF_MACRO_CELL");
    const int v = e ? std::atoi(e) : 0;
    return v >= 2 && v <= 64 ? v : PF_MACRO;
}

// Target photons of one phase per KNN grid cell (PF_KNN_PPC overrides it for tuning sweeps).
double knn_photons_per_cell() {
    const char *e = std::getenv("PF_KNN_PPC");
    const double v = e ? std::atof(e) : 0.0;
    return v > 0.05 && v < 1024.0 ? v : 8.0;
}

}  // namespace

struct pf_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool timing = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // volume
    cudaArray_t vol_array = nullptr;
    cudaTextureObject_t vol_tex = 0;
    int atlas_log2 = 0;
    int mc[3] = {0, 0, 0};
    int macro = macro_default();  // voxels per macro-cell edge
    DevBuf macro_mm, maj, maj_hi, occ;
    cudaArray_t maj_array = nullptr;  // PARITY majorant texture (high words, see DevScene::maj_tex)
    cudaTextureObject_t maj_tex = 0;
    int nx = 0, ny = 0, nz = 0;
    float vmin = 0.f, vmax = 0.f;
    // medium / lights
    bool has_medium = false;
    std::vector<double> tf;
    double density_scale = 0.0, sigma_max = 0.0;
    std::vector<double> lights;
    // field
    bool has_field = false;
    FieldDesc fdesc{};
    FieldHost fhost;
    DevBuf f_tables, f_img, f_feat;
    int f_nwg = 0;
    size_t f_smem = 0, f_abytes = 32768;
    int sms = 0;
    // render scratch
    DevBuf slots, hits, hit_dir, counters, frame_stage, stage[10];
    // knn
    bool has_knn = false;
    KnnParams knn{};
    KnnBuffers kb;
    DevBuf k_photons, k_bbox;
    size_t k_n = 0;
    // photon trace (Alg. 1): resident result + scratch
    DevBuf t_rec, t_rec_photon, t_counts, t_offs, t_tmp, t_out, t_ctr;
    // asynchronous host-output frames: double-buffered device staging, D2H on a
    // copy stream overlapped with the next frame's kernels
    cudaStream_t cstream = nullptr;
    DevBuf aframe[2];
    cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    const void *a_host[2] = {nullptr, nullptr};
    int a_next = 0;
    // field training
    TrainState train;
    DevBuf tr_x, tr_w2, tr_g, tr_t, tr_w3, tr_gi, tr_t3d;
    size_t t_n = 0;
    unsigned long long trace_steps = 0;
    uint64_t t_total = 0;
    bool has_trace = false;

    cudaError_t stage_in(int slot, const void *host, size_t bytes, const void **dev) {
        if (!host || is_device_ptr(host)) {
            *dev = host;
            return cudaSuccess;
        }
        cudaError_t e = stage[slot].ensure(bytes);
        if (e) return e;
        e = cudaMemcpyAsync(stage[slot].p, host, bytes, cudaMemcpyHostToDevice, stream);
        *dev = stage[slot].p;
        return e;
    }
    cudaError_t out_ptr(int slot, void *user, size_t bytes, void **dev, bool *host) {
        *host = user && !is_device_ptr(user);
        if (!*host) {
            *dev = user;
            return cudaSuccess;
        }
        cudaError_t e = stage[slot].ensure(bytes);
        *dev = stage[slot].p;
        return e;
    }
    DevScene scene() const {
        DevScene S;
        std::memset(&S, 0, sizeof(S));
        S.atlas = vol_tex;
        S.atlas_log2 = atlas_log2;
        S.maj = (const float *)maj.p;
        S.maj_tex = maj_tex;
        S.occ = (const int *)occ.p;
        for (int a = 0; a < 3; ++a) {
            const int n = a == 0 ? nx : a == 1 ? ny : nz;
            S.mc[a] = mc[a];
            S.mh[a] = (float)macro / (float)n;
            S.minv_h[a] = (float)n / (float)macro;
        }
        S.nx = nx;
        S.ny = ny;
        S.nz = nz;
        S.n_tf = (int)tf.size() / 5;
        S.n_lights = (int)lights.size() / 6;
        S.density_scale = density_scale;
        S.sigma_max = sigma_max;
        S.inv_sigma_max = sigma_max > 0.0 ? 1.0 / sigma_max : 0.0;
        S.sm53 = sigma_max * 0x1.0p-53;
        S.density_scale_f = (float)density_scale;
        S.sigma_max_f = (float)sigma_max;
        S.inv_sigma_max_f = sigma_max > 0.0 ? (float)(1.0 / sigma_max) : 0.f;
        for (int i = 0; i < S.n_tf; ++i) {
            S.tf_s[i] = tf[5 * i];
            S.tf_sf[i] = (float)tf[5 * i];
            for (int c = 0; c < 4; ++c) {
                S.tf_c[i][c] = tf[5 * i + 1 + c];
                S.tf_cf[i][c] = (float)tf[5 * i + 1 + c];
            }
        }
        for (int l = 0; l < S.n_lights; ++l)
            for (int a = 0; a < 3; ++a) {
                S.light_p[l][a] = lights[6 * l + a];
                S.light_i[l][a] = lights[6 * l + 3 + a];
            }
        return S;
    }
    void free_volume() {
        if (vol_tex) cudaDestroyTextureObject(vol_tex);
        if (vol_array) cudaFreeArray(vol_array);
        if (maj_tex) cudaDestroyTextureObject(maj_tex);
        if (maj_array) cudaFreeArray(maj_array);
        vol_tex = 0;
        vol_array = nullptr;
        maj_tex = 0;
        maj_array = nullptr;
        nx = ny = nz = 0;
    }
};

extern "C" {

const char *pf_last_error(void) { return g_err.c_str(); }
const char *pf_version(void) { return "photonfield-b200 0.1 (sm_100a)"; }

int pf_ctx_create(int device, pf_ctx **out) {
    if (!out) return set_err(PF_ERR_INVALID, "pf_ctx_create: out is NULL");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return set_err(PF_ERR_RUNTIME, "pf_ctx_create: no CUDA device visible");
    }
    if (device < 0 || device >= n) return set_err(PF_ERR_INVALID, "pf_ctx_create: bad device %d", device);
    PF_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    PF_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(PF_ERR_RUNTIME, "pf_ctx_create: device %d is sm_%d%d; this build targets sm_100a",
                       device, prop.major, prop.minor);
    auto *c = new pf_ctx();
    c->device = device;
    c->sms = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e) {
        delete c;
        return set_err(PF_ERR_RUNTIME, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    c->own_stream = true;
    for (auto &ev : c->ev) cudaEventCreate(&ev);
    if (c->counters.ensure(64)) {
        delete c;
        return set_err(PF_ERR_RUNTIME, "cudaMalloc counters failed");
    }
    *out = c;
    return PF_OK;
}

void pf_ctx_destroy(pf_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->free_volume();
    for (auto &ev : c->ev)
        if (ev) cudaEventDestroy(ev);
    if (c->cstream) {
        cudaStreamSynchronize(c->cstream);
        cudaStreamDestroy(c->cstream);
    }
    for (int k = 0; k < 2; ++k) {
        if (c->ev_ready[k]) cudaEventDestroy(c->ev_ready[k]);
        if (c->ev_copied[k]) cudaEventDestroy(c->ev_copied[k]);
    }
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
}

int pf_ctx_set_stream(pf_ctx *c, void *s) {
    if (!c) return set_err(PF_ERR_INVALID, "null context");
    if (c->own_stream) {
        cudaStreamSynchronize(c->stream);
        cudaStreamDestroy(c->stream);
        c->own_stream = false;
        c->stream = nullptr;
    }
    if (s) {
        c->stream = (cudaStream_t)s;
    } else {
        PF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return PF_OK;
}

int pf_ctx_synchronize(pf_ctx *c) {
    if (!c) return set_err(PF_ERR_INVALID, "null argument");
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    if (c->cstream) PF_CUDA(cudaStreamSynchronize(c->cstream));
    return PF_OK;
}

int pf_ctx_set_timing(pf_ctx *c, int enabled) {
    if (!c) return set_err(PF_ERR_INVALID, "null context");
    c->timing = enabled != 0;
    return PF_OK;
}

// ---------------------------------------------------------------- scene --
int pf_volume_upload(pf_ctx *c, int nx, int ny, int nz, const float *data) {
    if (!c || !data) return set_err(PF_ERR_INVALID, "pf_volume_upload: null argument");
    if (nx <= 0 || ny <= 0 || nz <= 0)
        return set_err(PF_ERR_INVALID, "VolumeGrid: dims must be positive");
    PF_CUDA(cudaSetDevice(c->device));
    const size_t n = (size_t)nx * ny * nz;
    std::vector<float> host;
    const float *src = data;
    const bool dev = is_device_ptr(data);
    if (dev) {
        // ordered on the context stream (not the legacy default stream, which
        // does not wait for non-blocking streams such as a torch side stream)
        host.resize(n);
        PF_CUDA(cudaMemcpyAsync(host.data(), data, n * 4, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
        src = host.data();
    }
    // VolumeGrid ctor validation + attained range (volume.cpp:24-39)
    float lo = 1.f, hi = 0.f;
    for (size_t i = 0; i < n; ++i) {
        const float v = src[i];
        if (!std::isfinite(v) || v < 0.f || v > 1.f)
            return set_err(PF_ERR_INVALID, "VolumeGrid: scalars must be finite and in [0,1]");
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    c->free_volume();
    // slice atlas (see DevScene): smallest power-of-two tile columns that fit
    int max_w = 0, max_h = 0;
    cudaDeviceGetAttribute(&max_w, cudaDevAttrMaxTexture2DWidth, c->device);
    cudaDeviceGetAttribute(&max_h, cudaDevAttrMaxTexture2DHeight, c->device);
    int lg = 0;
    while ((size_t)((nz + (1 << lg) - 1) >> lg) * (size_t)(ny + 1) > (size_t)max_h) ++lg;
    const size_t aw = (size_t)(1 << lg) * (size_t)(nx + 1);
    const size_t ah = (size_t)((nz + (1 << lg) - 1) >> lg) * (size_t)(ny + 1);
    if (aw > (size_t)max_w) return set_err(PF_ERR_INVALID, "VolumeGrid: %dx%dx%d exceeds the texture atlas", nx, ny, nz);
    DevBuf lin, atl;
    PF_CUDA(lin.ensure(n * 4));
    PF_CUDA(atl.ensure(aw * ah * 4));
    PF_CUDA(cudaMemcpyAsync(lin.p, src, n * 4, cudaMemcpyHostToDevice, c->stream));
    PF_CUDA(launch_build_atlas((const float *)lin.p, nx, ny, nz, lg, (float *)atl.p, aw, ah, c->stream));
    // FAST-mode macro-cell scalar ranges (majorants are derived per TF in pf_medium_set)
    for (int a = 0; a < 3; ++a) c->mc[a] = ((a == 0 ? nx : a == 1 ? ny : nz) + c->macro - 1) / c->macro;
    const size_t ncell = (size_t)c->mc[0] * c->mc[1] * c->mc[2];
    PF_CUDA(c->macro_mm.ensure(ncell * sizeof(float2)));
    PF_CUDA(c->maj.ensure(ncell * sizeof(float)));
    PF_CUDA(c->maj_hi.ensure(ncell * sizeof(uint32_t)));
    PF_CUDA(launch_macro_minmax((const float *)lin.p, nx, ny, nz, (float2 *)c->macro_mm.p, c->mc[0], c->mc[1],
                                c->mc[2], c->macro, c->stream));
    cudaChannelFormatDesc fd = cudaCreateChannelDesc<float>();
    PF_CUDA(cudaMallocArray(&c->vol_array, &fd, aw, ah));
    PF_CUDA(cudaMemcpy2DToArrayAsync(c->vol_array, 0, 0, atl.p, aw * 4, aw * 4, ah, cudaMemcpyDeviceToDevice,
                                     c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    cudaResourceDesc rd;
    std::memset(&rd, 0, sizeof(rd));
    rd.resType = cudaResourceTypeArray;
    rd.res.array.array = c->vol_array;
    cudaTextureDesc td;
    std::memset(&td, 0, sizeof(td));
    td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint;  // gathers return the stored floats; no fixed-point lerp
    td.readMode = cudaReadModeElementType;
    td.normalizedCoords = 0;
    PF_CUDA(cudaCreateTextureObject(&c->vol_tex, &rd, &td, nullptr));
    {  // PARITY majorant texture: mc[0] x mc[1] x mc[2] uint32, point-sampled, clamped
        cudaChannelFormatDesc md = cudaCreateChannelDesc<unsigned int>();
        PF_CUDA(cudaMalloc3DArray(&c->maj_array, &md, make_cudaExtent(c->mc[0], c->mc[1], c->mc[2])));
        cudaResourceDesc mr;
        std::memset(&mr, 0, sizeof(mr));
        mr.resType = cudaResourceTypeArray;
        mr.res.array.array = c->maj_array;
        cudaTextureDesc mt;
        std::memset(&mt, 0, sizeof(mt));
        mt.addressMode[0] = mt.addressMode[1] = mt.addressMode[2] = cudaAddressModeClamp;
        mt.filterMode = cudaFilterModePoint;
        mt.readMode = cudaReadModeElementType;
        mt.normalizedCoords = 0;
        PF_CUDA(cudaCreateTextureObject(&c->maj_tex, &mr, &mt, nullptr));
    }
    c->atlas_log2 = lg;
    c->nx = nx;
    c->ny = ny;
    c->nz = nz;
    c->vmin = lo;
    c->vmax = hi;
    c->has_medium = false;  // sigma_max depends on the attained range
    return PF_OK;
}

int pf_medium_set(pf_ctx *c, const double *tf_pts, int n_pts, double density_scale, double sigma_max) {
    if (!c || !tf_pts) return set_err(PF_ERR_INVALID, "pf_medium_set: null argument");
    if (!c->vol_tex) return set_err(PF_ERR_INVALID, "pf_medium_set: upload a volume first");
    if (n_pts < 2) return set_err(PF_ERR_INVALID, "TransferFunction: need at least two control points");
    if (n_pts > PF_MAX_TF) return set_err(PF_ERR_INVALID, "TransferFunction: at most %d points", PF_MAX_TF);
    if (tf_pts[0] != 0.0 || tf_pts[5 * (n_pts - 1)] != 1.0)
        return set_err(PF_ERR_INVALID, "TransferFunction: control points must span [0,1]");
    for (int i = 0; i < n_pts; ++i) {
        for (int ch = 1; ch < 5; ++ch) {
            const double v = tf_pts[5 * i + ch];
            if (!(v >= 0.0 && v <= 1.0))
                return set_err(PF_ERR_INVALID, "TransferFunction: channels must be in [0,1]");
        }
        if (i > 0 && tf_pts[5 * i] <= tf_pts[5 * (i - 1)])
            return set_err(PF_ERR_INVALID, "TransferFunction: positions must be strictly increasing");
    }
    if (!(density_scale > 0.0) || !std::isfinite(density_scale))
        return set_err(PF_ERR_INVALID, "Medium: density_scale must be positive and finite");
    c->tf.assign(tf_pts, tf_pts + 5 * n_pts);
    c->density_scale = density_scale;
    if (sigma_max < 0.0) {
        // Medium ctor: density_scale * tf.max_alpha(value_min, value_max) (volume.cpp:163-168, 197-202)
        const double lo = (double)c->vmin, hi = (double)c->vmax;
        double ra = tf_classify_alpha(c->tf, lo), rb = tf_classify_alpha(c->tf, hi);
        double m = (ra < rb) ? rb : ra;
        for (int i = 0; i < n_pts; ++i) {
            const double s = tf_pts[5 * i];
            if (s > lo && s < hi) m = (m < tf_pts[5 * i + 4]) ? tf_pts[5 * i + 4] : m;
        }
        sigma_max = density_scale * m;
    }
    c->sigma_max = sigma_max;
    // per-macro-cell majorants for the FAST tracer
    PF_CUDA(cudaSetDevice(c->device));
    TfPoints tp;
    std::memset(&tp, 0, sizeof(tp));
    std::memcpy(tp.p, c->tf.data(), c->tf.size() * sizeof(double));
    PF_CUDA(c->occ.ensure(6 * sizeof(int)));
    PF_CUDA(launch_macro_majorant((const float2 *)c->macro_mm.p, (size_t)c->mc[0] * c->mc[1] * c->mc[2], tp, n_pts,
                                  density_scale, (float *)c->maj.p, (uint32_t *)c->maj_hi.p, c->mc[0], c->mc[1],
                                  (int *)c->occ.p, c->stream));
    {
        cudaMemcpy3DParms cp;
        std::memset(&cp, 0, sizeof(cp));
        cp.srcPtr = make_cudaPitchedPtr(c->maj_hi.p, (size_t)c->mc[0] * 4, c->mc[0], c->mc[1]);
        cp.dstArray = c->maj_array;
        cp.extent = make_cudaExtent(c->mc[0], c->mc[1], c->mc[2]);
        cp.kind = cudaMemcpyDeviceToDevice;
        PF_CUDA(cudaMemcpy3DAsync(&cp, c->stream));
    }
    c->has_medium = true;
    return PF_OK;
}

int pf_medium_sigma_max(pf_ctx *c, double *out) {
    if (!c || !out) return set_err(PF_ERR_INVALID, "null argument");
    if (!c->has_medium) return set_err(PF_ERR_INVALID, "pf_medium_sigma_max: no medium set");
    *out = c->sigma_max;
    return PF_OK;
}

int pf_lights_set(pf_ctx *c, const double *lights, int n) {
    if (!c || (n > 0 && !lights)) return set_err(PF_ERR_INVALID, "pf_lights_set: null argument");
    if (n < 0 || n > PF_MAX_LIGHTS) return set_err(PF_ERR_INVALID, "pf_lights_set: 0..%d lights", PF_MAX_LIGHTS);
    for (int i = 0; i < 6 * n; ++i)
        if (!std::isfinite(lights[i])) return set_err(PF_ERR_INVALID, "LightSource: non-finite value");
    for (int l = 0; l < n; ++l)
        for (int ch = 3; ch < 6; ++ch)
            if (lights[6 * l + ch] < 0.0) return set_err(PF_ERR_INVALID, "LightSource: intensity must be >= 0");
    c->lights.assign(lights, lights + 6 * n);
    return PF_OK;
}

// ---------------------------------------------------------------- field --
static FieldDesc to_fdesc(const pf_field_desc *d) {
    FieldDesc f;
    f.pos = {d->pos.dims, d->pos.levels, d->pos.features, d->pos.base_res, d->pos.growth, d->pos.log2_table};
    f.dir = {d->dir.dims, d->dir.levels, d->dir.features, d->dir.base_res, d->dir.growth, d->dir.log2_table};
    f.hidden_layers = d->hidden_layers;
    f.width = d->width;
    f.psi = d->psi;
    return f;
}

int pf_field_param_count(const pf_field_desc *d, size_t *out) {
    if (!d || !out) return set_err(PF_ERR_INVALID, "null argument");
    FieldDesc f = to_fdesc(d);
    if (const char *m = field_validate(f)) return set_err(PF_ERR_INVALID, "%s", m);
    *out = field_param_count(f);
    return PF_OK;
}

int pf_field_init(const pf_field_desc *d, uint64_t seed, double embed_scale, double bias_scale,
                  float *out) {
    if (!d || !out) return set_err(PF_ERR_INVALID, "null argument");
    FieldDesc f = to_fdesc(d);
    if (const char *m = field_validate(f)) return set_err(PF_ERR_INVALID, "%s", m);
    HostPcg r;
    r.seed(stream_initstate(seed, PF_STREAM_FIELDINIT), 0);
    const size_t ntab = field_grid_param_count(f.pos) + field_grid_param_count(f.dir);
    size_t p = 0;
    for (; p < ntab; ++p) out[p] = (float)((2.0 * r.next_double() - 1.0) * embed_scale);
    const int din = f.pos.levels * f.pos.features + f.dir.levels * f.dir.features + 1;
    for (int L = 0; L <= f.hidden_layers; ++L) {
        const int K = L == 0 ? din : f.width, N = L < f.hidden_layers ? f.width : 3;
        const double a = std::sqrt(6.0 / K);  // He-uniform by fan-in
        for (int i = 0; i < N * K; ++i) out[p++] = (float)((2.0 * r.next_double() - 1.0) * a);
        for (int i = 0; i < N; ++i) out[p++] = (float)((2.0 * r.next_double() - 1.0) * bias_scale);
    }
    return PF_OK;
}

static int field_load(pf_ctx *c, const FieldDesc &f, const float *params, size_t n);

int pf_field_load(pf_ctx *c, const pf_field_desc *d, const float *params, size_t n) {
    if (!c || !d || !params) return set_err(PF_ERR_INVALID, "pf_field_load: null argument");
    FieldDesc f = to_fdesc(d);
    if (const char *m = field_validate(f)) return set_err(PF_ERR_INVALID, "%s", m);
    return field_load(c, f, params, n);
}

static int field_load(pf_ctx *c, const FieldDesc &f, const float *params, size_t n) {
    const size_t need = field_param_count(f);
    if (n != need) return set_err(PF_ERR_INVALID, "pf_field_load: expected %zu params, got %zu", need, n);
    PF_CUDA(cudaSetDevice(c->device));
    std::vector<float> host;
    const float *src = params;
    if (is_device_ptr(params)) {
        host.resize(n);
        PF_CUDA(cudaMemcpyAsync(host.data(), params, n * 4, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
        src = host.data();
    }
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(src[i])) return set_err(PF_ERR_INVALID, "pf_field_load: non-finite parameter");
    FieldHost h;
    field_pack(f, src, h);
    if ((int)h.levels.size() > PF_FIELD_MAX_LEVELS) return set_err(PF_ERR_INVALID, "too many levels");
    int nwg;
    size_t smem, a_bytes;
    if (field_launch_config(h, nwg, smem, a_bytes, c->device))
        return set_err(PF_ERR_INVALID, "pf_field_load: MLP does not fit in shared memory");
    PF_CUDA(c->f_tables.ensure(h.tables.size() * 2));
    PF_CUDA(c->f_img.ensure(h.image.size()));
    PF_CUDA(cudaMemcpyAsync(c->f_tables.p, h.tables.data(), h.tables.size() * 2, cudaMemcpyHostToDevice,
                            c->stream));
    PF_CUDA(cudaMemcpyAsync(c->f_img.p, h.image.data(), h.image.size(), cudaMemcpyHostToDevice, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    c->fdesc = f;
    c->fhost = std::move(h);
    c->f_nwg = nwg;
    c->f_smem = smem;
    c->f_abytes = a_bytes;
    c->has_field = true;
    return PF_OK;
}

// Feature-tile staging budget (HBM): the hit count is only known on the
// device, so renders launch ceil(n_work / cap) encode+MLP pairs and the
// surplus pairs exit immediately (~11 us each).  12 GiB of the 180 GB keeps
// C2 (16.6M samples, paper field: 640 B/row = 10.6 GB) to one pair.
static constexpr size_t kFieldStageBytes = (size_t)12 << 30;
static constexpr size_t kFieldRowCap = (size_t)1 << 22;

// encode + MLP over n_max items (count on device for renders), in row batches
static int run_field(pf_ctx *c, FieldParams P, size_t n_max, uint32_t *launches = nullptr) {
    const size_t row_bytes = (size_t)P.nch * (size_t)field_chunk_cols() * 2u;  // fp16 columns per row
    const size_t cap = std::min(n_max, std::max(kFieldRowCap, kFieldStageBytes / row_bytes));
    PF_CUDA(c->f_feat.ensure(field_feat_bytes(c->fhost, cap)));
    P.feat = (uint8_t *)c->f_feat.p;
    P.row_cap = cap;
    for (size_t r0 = 0; r0 < n_max; r0 += cap) {
        P.row0 = r0;
        const size_t tiles = (std::min(cap, n_max - r0) + 127) / 128;
        const int grid = (int)std::max<size_t>(1, std::min<size_t>((size_t)c->sms, (tiles + P.n_wg - 1) / P.n_wg));
        PF_CUDA(launch_field(P, c->fhost.fp, c->fhost.fd, grid, c->f_smem, c->stream));
        if (launches) *launches += 2;
    }
    return PF_OK;
}

static FieldParams field_params(pf_ctx *c) {
    FieldParams P;
    std::memset(&P, 0, sizeof(P));
    const FieldHost &h = c->fhost;
    P.n_pos_levels = h.n_pos_levels;
    P.n_dir_levels = h.n_dir_levels;
    P.K0 = h.K0;
    P.hidden_layers = h.hidden_layers;
    P.n_wg = c->f_nwg;
    P.tmem_cols = c->f_nwg <= 2 ? 128u : (c->f_nwg <= 4 ? 256u : 512u);
    P.img_bytes = (uint32_t)h.image.size();
    P.a_bytes = (uint32_t)c->f_abytes;
    for (int i = 0; i < 8; ++i) P.off_w[i] = h.off_w[i];
    P.off_bias = h.off_bias;
    P.psi_log2_10 = (float)(h.psi * 3.3219280948873623478703194294894);
    for (size_t i = 0; i < h.enc_levels.size(); ++i) P.lv[i] = h.enc_levels[i];
    P.tables = (const __half *)c->f_tables.p;
    P.img = c->f_img.p;
    P.nch = (h.K0 + field_chunk_cols() - 1) / field_chunk_cols();
    P.row_cap = kFieldRowCap;
    return P;
}

int pf_field_query(pf_ctx *c, size_t n, const float *x3, const float *w2, const float *g, float *out,
                   int decoded) {
    if (!c || (n && (!x3 || !w2 || !g || !out))) return set_err(PF_ERR_INVALID, "pf_field_query: null argument");
    if (!c->has_field) return set_err(PF_ERR_INVALID, "pf_field_query: no field loaded");
    if (n == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    const void *dx, *dw, *dg;
    void *dout;
    bool host_out;
    PF_CUDA(c->stage_in(0, x3, n * 12, &dx));
    PF_CUDA(c->stage_in(1, w2, n * 8, &dw));
    PF_CUDA(c->stage_in(2, g, n * 4, &dg));
    PF_CUDA(c->out_ptr(3, out, n * 12, &dout, &host_out));
    FieldParams P = field_params(c);
    P.mode = 1;
    P.n_query = n;
    P.qx = (const float *)dx;
    P.qw = (const float *)dw;
    P.qg = (const float *)dg;
    P.qout = (float *)dout;
    P.decoded = decoded;
    if (int e = run_field(c, P, n)) return e;
    if (host_out) {
        PF_CUDA(cudaMemcpyAsync(out, dout, n * 12, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
    }
    return PF_OK;
}

// --------------------------------------------------------------- render --
int pf_camera_make(const double pos[3], const double look_at[3], const double up[3], double vfov_deg,
                   int width, int height, pf_camera *out) {
    if (!pos || !look_at || !up || !out) return set_err(PF_ERR_INVALID, "pf_camera_make: null argument");
    if (width <= 0 || height <= 0) return set_err(PF_ERR_INVALID, "Camera: dims must be positive");
    if (!(vfov_deg > 0.0 && vfov_deg < 180.0)) return set_err(PF_ERR_INVALID, "Camera: fov must be in (0, pi)");
    auto norm = [](double v[3]) {
        double len = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        v[0] = v[0] / len;
        v[1] = v[1] / len;
        v[2] = v[2] / len;
    };
    double f[3] = {look_at[0] - pos[0], look_at[1] - pos[1], look_at[2] - pos[2]};
    norm(f);
    double r[3] = {f[1] * up[2] - f[2] * up[1], f[2] * up[0] - f[0] * up[2], f[0] * up[1] - f[1] * up[0]};
    norm(r);
    double u[3] = {r[1] * f[2] - r[2] * f[1], r[2] * f[0] - r[0] * f[2], r[0] * f[1] - r[1] * f[0]};
    const double th = std::tan(vfov_deg * (3.14159265358979323846 / 180.0) * 0.5);
    const double aspect = (double)width / (double)height;
    for (int a = 0; a < 3; ++a) {
        out->origin[a] = pos[a];
        out->forward[a] = f[a];
        out->right[a] = r[a] * (aspect * th);
        out->up[a] = u[a] * th;
    }
    out->width = width;
    out->height = height;
    for (int a = 0; a < 3; ++a)
        if (!std::isfinite(out->right[a]) || !std::isfinite(out->up[a]) || !std::isfinite(out->forward[a]))
            return set_err(PF_ERR_INVALID, "Camera: degenerate basis (up parallel to view direction)");
    return PF_OK;
}

static int validate_tiles(const pf_camera *cam, const pf_render_desc *d) {
    if (d->tile_w <= 0 || d->tile_h <= 0) return set_err(PF_ERR_INVALID, "render: tile dims must be positive");
    if (d->shard_count < 1 || d->shard_index < 0 || d->shard_index >= d->shard_count)
        return set_err(PF_ERR_INVALID, "render: shard_index must be in [0, shard_count)");
    if (cam->width <= 0 || cam->height <= 0) return set_err(PF_ERR_INVALID, "Camera: dims must be positive");
    return PF_OK;
}

static uint32_t local_tiles(const pf_camera *cam, const pf_render_desc *d, int shard, uint32_t *tiles_x) {
    const uint32_t tx = (uint32_t)((cam->width + d->tile_w - 1) / d->tile_w);
    const uint32_t ty = (uint32_t)((cam->height + d->tile_h - 1) / d->tile_h);
    const uint32_t n = tx * ty;
    if (tiles_x) *tiles_x = tx;
    return n > (uint32_t)shard ? (n - (uint32_t)shard + (uint32_t)d->shard_count - 1) / (uint32_t)d->shard_count
                               : 0u;
}

int pf_tiles_count(const pf_camera *cam, const pf_render_desc *d, int shard, int *n_tiles) {
    if (!cam || !d || !n_tiles) return set_err(PF_ERR_INVALID, "null argument");
    if (int e = validate_tiles(cam, d)) return e;
    if (shard < 0 || shard >= d->shard_count) return set_err(PF_ERR_INVALID, "bad shard");
    *n_tiles = (int)local_tiles(cam, d, shard, nullptr);
    return PF_OK;
}

static ComposeParams compose_params(const pf_camera *cam, const pf_render_desc *d) {
    ComposeParams C;
    C.W = cam->width;
    C.H = cam->height;
    C.spp = d->spp;
    C.tile_w = d->tile_w;
    C.tile_h = d->tile_h;
    uint32_t tx;
    C.n_local_tiles = local_tiles(cam, d, d->shard_index, &tx);
    C.tiles_x = (int)tx;
    C.shard_index = d->shard_index;
    C.shard_count = d->shard_count;
    C.slots = nullptr;
    C.out = nullptr;
    return C;
}

// L_i source of the three first-interaction renderers
enum LiSource { kLiNeural = 0, kLiPathTraced = 1, kLiPhotonMap = 2 };

static int render_common(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, LiSource src,
                         const pf_path_desc *pt, int K, float r_max, float *out_rgb, pf_render_stats *stats) {
    const char *name = src == kLiNeural ? "render_neural" : (src == kLiPathTraced ? "render_path_traced"
                                                                                  : "render_photon_map");
    if (!c || !cam || !d || !out_rgb) return set_err(PF_ERR_INVALID, "%s: null argument", name);
    if (int e = validate_tiles(cam, d)) return e;
    if (d->spp <= 0) return set_err(PF_ERR_INVALID, "%s: spp must be >= 1", name);
    if (!c->vol_tex || !c->has_medium) return set_err(PF_ERR_INVALID, "%s: volume/medium not set", name);
    if (c->lights.empty()) return set_err(PF_ERR_INVALID, "%s: at least one light required", name);
    if (d->mode != PF_MODE_PARITY && d->mode != PF_MODE_FAST) return set_err(PF_ERR_INVALID, "render: bad mode");
    if (d->mode == PF_MODE_PARITY && d->nee_trials <= 0)
        return set_err(PF_ERR_INVALID, "transmittance: n_trials must be positive");
    if (src == kLiNeural && d->use_field && !c->has_field)
        return set_err(PF_ERR_INVALID, "render_neural: no field loaded");
    if (!std::isfinite(d->g)) return set_err(PF_ERR_INVALID, "%s: non-finite g", name);
    int render_g = -1;
    if (src == kLiPathTraced) {
        if (!pt) return set_err(PF_ERR_INVALID, "render_path_traced: null path description");
        if (pt->max_bounces < 1) return set_err(PF_ERR_INVALID, "render_path_traced: max_bounces must be >= 1");
        if (!(pt->rr_min_survival > 0.0 && pt->rr_min_survival <= pt->rr_max_survival && pt->rr_max_survival <= 1.0))
            return set_err(PF_ERR_INVALID, "render_path_traced: need 0 < rr_min_survival <= rr_max_survival <= 1");
    }
    if (src == kLiPhotonMap) {
        if (!c->has_knn) return set_err(PF_ERR_INVALID, "render_photon_map: call pf_knn_build first");
        if (K < 1 || K > 1024) return set_err(PF_ERR_INVALID, "KnnQuery: K must be in [1, 1024]");
        if (!(r_max > 0.0f)) return set_err(PF_ERR_INVALID, "KnnQuery: r_max must be > 0");
        for (int i = 0; i < c->knn.n_phases; ++i)
            if (c->knn.phase[i] == d->g) render_g = i;
        if (render_g < 0) return set_err(PF_ERR_INVALID, "render_photon_map: g is not in the map's phase set");
    }
    PF_CUDA(cudaSetDevice(c->device));
    const bool parity = d->mode == PF_MODE_PARITY;
    ComposeParams C = compose_params(cam, d);
    const size_t tile_px = (size_t)d->tile_w * d->tile_h;
    const size_t n_work = (size_t)C.n_local_tiles * tile_px * (size_t)d->spp;
    if (n_work >= (1ull << 32)) return set_err(PF_ERR_INVALID, "render: > 2^32 samples per shard");
    const size_t slot_bytes = n_work * 3 * (parity ? 8 : 4);
    PF_CUDA(c->slots.ensure(slot_bytes));
    const bool want_hits = (src == kLiNeural && d->use_field) || src == kLiPhotonMap;
    if (want_hits) PF_CUDA(c->hits.ensure(n_work * sizeof(HitRec)));
    if (src == kLiPhotonMap) PF_CUDA(c->hit_dir.ensure(n_work * 24));
    void *frame;
    bool host_out;
    PF_CUDA(c->out_ptr(7, out_rgb, (size_t)cam->width * cam->height * 12, &frame, &host_out));
    if (host_out) PF_CUDA(cudaMemsetAsync(frame, 0, (size_t)cam->width * cam->height * 12, c->stream));
    PF_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));

    TraceParams P;
    std::memset(&P, 0, sizeof(P));
    P.init_cam = stream_initstate(d->seed, PF_STREAM_CAMERA);
    P.init_nee = stream_initstate(d->seed, PF_STREAM_NEE);
    for (int a = 0; a < 3; ++a) {
        P.cam_o[a] = cam->origin[a];
        P.cam_f[a] = cam->forward[a];
        P.cam_r[a] = cam->right[a];
        P.cam_u[a] = cam->up[a];
        P.bg[a] = d->background[a];
    }
    P.W = cam->width;
    P.H = cam->height;
    P.spp = d->spp;
    P.tile_w = d->tile_w;
    P.tile_h = d->tile_h;
    P.tiles_x = C.tiles_x;
    P.shard_index = d->shard_index;
    P.shard_count = d->shard_count;
    P.n_work = (uint32_t)n_work;
    P.g = d->g;
    P.w_d = d->w_d;
    P.nee_trials = d->nee_trials > 0 ? d->nee_trials : 1;
    P.use_field = want_hits ? 1 : 0;
    P.slots = c->slots.p;
    P.hits = (HitRec *)c->hits.p;
    P.hit_dir = src == kLiPhotonMap ? (double *)c->hit_dir.p : nullptr;
    P.counters = (unsigned long long *)c->counters.p;
    P.w_i = d->w_i;
    if (src == kLiPathTraced) {
        P.init_pt = stream_initstate(d->seed, PF_STREAM_PATHTRACE);
        P.max_bounces = pt->max_bounces;
        P.rr_start = pt->rr_start_bounce;
        P.rr_min = pt->rr_min_survival;
        P.rr_max = pt->rr_max_survival;
    }
    const DevScene S = c->scene();

    uint32_t n_launch = 0;
    if (c->timing) cudaEventRecord(c->ev[0], c->stream);
    if (n_work && src == kLiPathTraced) {
        ++n_launch;
        const int grid = parity ? pt_grid_size_parity(c->device) : pt_grid_size_fast(c->device);
        PF_CUDA(parity ? launch_render_pt_parity(S, P, grid, c->stream) : launch_render_pt_fast(S, P, grid, c->stream));
    } else if (n_work) {
        ++n_launch;
        const int grid = parity ? trace_grid_size_parity(c->device) : trace_grid_size_fast(c->device);
        PF_CUDA(parity ? launch_render_trace_parity(S, P, grid, c->stream)
                       : launch_render_trace_fast(S, P, grid, c->stream));
    }
    if (c->timing) cudaEventRecord(c->ev[1], c->stream);
    if (src == kLiPhotonMap && n_work) {
        KnnParams Q = c->knn;
        Q.nq = n_work;  // upper bound; the kernel reads the device-side hit count
        Q.K = K;
        Q.r2 = r_max * r_max;
        Q.order = nullptr;
        Q.hits = P.hits;
        Q.hit_dir = P.hit_dir;
        Q.n_hits = P.counters + 1;
        Q.slots = c->slots.p;
        Q.slot_f64 = parity ? 1 : 0;
        Q.render_g = render_g;
        Q.w_i = d->w_i;
        PF_CUDA(knn_query_render(Q, c->sms, c->stream));
        ++n_launch;
    }
    if (src == kLiNeural && d->use_field && n_work) {
        FieldParams F = field_params(c);
        F.mode = 0;
        F.hits = P.hits;
        F.n_hits = P.counters + 1;
        F.slots = c->slots.p;
        F.slot_f64 = parity ? 1 : 0;
        F.w_i = d->w_i;
        F.g_render = (float)d->g;
        if (int e = run_field(c, F, n_work, &n_launch)) return e;
    }
    if (c->timing) cudaEventRecord(c->ev[2], c->stream);
    C.slots = c->slots.p;
    C.out = (float *)frame;
    PF_CUDA(launch_compose(parity, C, c->stream));
    if (C.n_local_tiles) ++n_launch;
    if (c->timing) cudaEventRecord(c->ev[3], c->stream);
    if (host_out)
        PF_CUDA(cudaMemcpyAsync(out_rgb, frame, (size_t)cam->width * cam->height * 12, cudaMemcpyDeviceToHost,
                                c->stream));
    if (stats) {
        unsigned long long cnt[5];
        PF_CUDA(cudaMemcpyAsync(cnt, c->counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
        std::memset(stats, 0, sizeof(*stats));
        stats->samples = 0;
        stats->hits = cnt[1];
        stats->primary_steps = cnt[2];
        stats->shadow_steps = cnt[3];
        stats->voxel_fetches = cnt[4];
        // samples = work items that map into the frame
        uint64_t samples = 0;
        {
            const uint32_t tiles_y = (uint32_t)((cam->height + d->tile_h - 1) / d->tile_h);
            for (uint32_t lt = 0; lt < C.n_local_tiles; ++lt) {
                const uint32_t t = lt * (uint32_t)d->shard_count + (uint32_t)d->shard_index;
                const uint32_t ty = t / (uint32_t)C.tiles_x, tx = t % (uint32_t)C.tiles_x;
                (void)tiles_y;
                const uint64_t w = (uint64_t)std::min(d->tile_w, cam->width - (int)tx * d->tile_w);
                const uint64_t h = (uint64_t)std::min(d->tile_h, cam->height - (int)ty * d->tile_h);
                samples += w * h * (uint64_t)d->spp;
            }
        }
        stats->samples = samples;
        stats->kernel_launches = n_launch;
        if (c->timing) {
            cudaEventElapsedTime(&stats->ms_trace, c->ev[0], c->ev[1]);
            cudaEventElapsedTime(&stats->ms_field, c->ev[1], c->ev[2]);
            cudaEventElapsedTime(&stats->ms_compose, c->ev[2], c->ev[3]);
        }
    } else if (host_out) {
        PF_CUDA(cudaStreamSynchronize(c->stream));
    }
    PF_CUDA(cudaGetLastError());
    return PF_OK;
}

int pf_render_neural(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, float *out_rgb,
                     pf_render_stats *stats) {
    return render_common(c, cam, d, kLiNeural, nullptr, 0, 0.0f, out_rgb, stats);
}

int pf_render_path_traced(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, const pf_path_desc *pt,
                          float *out_rgb, pf_render_stats *stats) {
    return render_common(c, cam, d, kLiPathTraced, pt, 0, 0.0f, out_rgb, stats);
}

int pf_render_photon_map(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, int K, float r_max,
                         float *out_rgb, pf_render_stats *stats) {
    return render_common(c, cam, d, kLiPhotonMap, nullptr, K, r_max, out_rgb, stats);
}

int pf_render_neural_async(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, float *host_out) {
    if (!c || !cam || !d || !host_out) return set_err(PF_ERR_INVALID, "pf_render_neural_async: null argument");
    if (is_device_ptr(host_out)) return set_err(PF_ERR_INVALID, "pf_render_neural_async: host output expected");
    PF_CUDA(cudaSetDevice(c->device));
    if (!c->cstream) {
        PF_CUDA(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            PF_CUDA(cudaEventCreateWithFlags(&c->ev_ready[k], cudaEventDisableTiming));
            PF_CUDA(cudaEventCreateWithFlags(&c->ev_copied[k], cudaEventDisableTiming));
            PF_CUDA(cudaEventRecord(c->ev_copied[k], c->cstream));
        }
    }
    const int k = c->a_next;
    const size_t bytes = (size_t)cam->width * cam->height * 12;
    // staging buffer k is free once its previous frame has been copied out
    PF_CUDA(cudaStreamWaitEvent(c->stream, c->ev_copied[k], 0));
    if (c->aframe[k].cap < bytes) {
        PF_CUDA(cudaStreamSynchronize(c->stream));
        PF_CUDA(c->aframe[k].ensure(bytes));
    }
    if (d->shard_count > 1) PF_CUDA(cudaMemsetAsync(c->aframe[k].p, 0, bytes, c->stream));
    if (int e = pf_render_neural(c, cam, d, (float *)c->aframe[k].p, nullptr)) return e;
    PF_CUDA(cudaEventRecord(c->ev_ready[k], c->stream));
    PF_CUDA(cudaStreamWaitEvent(c->cstream, c->ev_ready[k], 0));
    PF_CUDA(cudaMemcpyAsync(host_out, c->aframe[k].p, bytes, cudaMemcpyDeviceToHost, c->cstream));
    PF_CUDA(cudaEventRecord(c->ev_copied[k], c->cstream));
    c->a_host[k] = host_out;
    c->a_next = k ^ 1;
    return PF_OK;
}

int pf_frame_wait(pf_ctx *c, const float *host_out) {
    if (!c || !host_out) return set_err(PF_ERR_INVALID, "pf_frame_wait: null argument");
    PF_CUDA(cudaSetDevice(c->device));
    for (int k = 0; k < 2; ++k)
        if (c->a_host[k] == host_out) {
            PF_CUDA(cudaEventSynchronize(c->ev_copied[k]));
            return PF_OK;
        }
    return set_err(PF_ERR_INVALID, "pf_frame_wait: no frame in flight for this buffer");
}

int pf_tiles_pack(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, const float *frame, float *packed) {
    if (!c || !cam || !d || !frame || !packed) return set_err(PF_ERR_INVALID, "null argument");
    if (int e = validate_tiles(cam, d)) return e;
    if (!is_device_ptr(frame) || !is_device_ptr(packed))
        return set_err(PF_ERR_INVALID, "pf_tiles_pack: device pointers required");
    PF_CUDA(cudaSetDevice(c->device));
    ComposeParams C = compose_params(cam, d);
    PF_CUDA(launch_tiles_pack(C, frame, packed, c->stream));
    return PF_OK;
}

int pf_tiles_unpack(pf_ctx *c, const pf_camera *cam, const pf_render_desc *d, const float *packed_all,
                    size_t per_shard, float *frame) {
    if (!c || !cam || !d || !packed_all || !frame) return set_err(PF_ERR_INVALID, "null argument");
    if (int e = validate_tiles(cam, d)) return e;
    if (!is_device_ptr(frame) || !is_device_ptr(packed_all))
        return set_err(PF_ERR_INVALID, "pf_tiles_unpack: device pointers required");
    PF_CUDA(cudaSetDevice(c->device));
    ComposeParams C = compose_params(cam, d);
    PF_CUDA(launch_tiles_unpack(C, packed_all, per_shard, frame, c->stream));
    return PF_OK;
}

// ------------------------------------------------------- parity batches --
static int batch_common(pf_ctx *c, size_t n, const double *a3, const double *b3, const uint64_t *idx,
                        BatchParams &B) {
    std::memset(&B, 0, sizeof(B));
    B.n = n;
    const void *da, *db, *di;
    PF_CUDA(c->stage_in(0, a3, n * 24, &da));
    PF_CUDA(c->stage_in(1, b3, n * 24, &db));
    PF_CUDA(c->stage_in(2, idx, n * 8, &di));
    B.a3 = (const double *)da;
    B.b3 = (const double *)db;
    B.idx = (const uint64_t *)di;
    return PF_OK;
}

int pf_delta_track_batch(pf_ctx *c, size_t n, const double *o3, const double *d3, const double *tmin,
                         const double *tmax, uint64_t seed, uint64_t stream, const uint64_t *idx, int fp64,
                         int *hit, double *pos3, double *scalar1, double *rgba4) {
    if (!c || (n && (!o3 || !d3 || !tmin || !tmax || !idx || !hit)))
        return set_err(PF_ERR_INVALID, "pf_delta_track_batch: null argument");
    if (!c->vol_tex || !c->has_medium) return set_err(PF_ERR_INVALID, "delta_track: volume/medium not set");
    if (n == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    // ray validation (volume.cpp:205-207) needs host-visible rays
    {
        std::vector<double> ho, hd, hmin, hmax;
        const double *po = o3, *pd = d3, *pmin = tmin, *pmax = tmax;
        auto fetch = [&](const double *p, size_t cnt, std::vector<double> &v) -> const double * {
            if (!is_device_ptr(p)) return p;
            v.resize(cnt);
            cudaMemcpyAsync(v.data(), p, cnt * 8, cudaMemcpyDeviceToHost, c->stream);
            cudaStreamSynchronize(c->stream);
            return v.data();
        };
        po = fetch(o3, 3 * n, ho);
        pd = fetch(d3, 3 * n, hd);
        pmin = fetch(tmin, n, hmin);
        pmax = fetch(tmax, n, hmax);
        for (size_t i = 0; i < n; ++i) {
            bool ok = std::isfinite(pmin[i]) && pmin[i] >= 0.0 && pmin[i] <= pmax[i];
            for (int a = 0; a < 3 && ok; ++a) ok = std::isfinite(po[3 * i + a]) && std::isfinite(pd[3 * i + a]);
            if (!ok) return set_err(PF_ERR_INVALID, "delta_track: invalid ray (index %zu)", i);
        }
    }
    BatchParams B;
    if (int e = batch_common(c, n, o3, d3, idx, B)) return e;
    const void *dmin, *dmax;
    PF_CUDA(c->stage_in(3, tmin, n * 8, &dmin));
    PF_CUDA(c->stage_in(4, tmax, n * 8, &dmax));
    B.tmin = (const double *)dmin;
    B.tmax = (const double *)dmax;
    B.initstate = stream_initstate(seed, stream);
    void *dhit, *dpos = nullptr, *drgba = nullptr, *dsc = nullptr;
    bool hh, hp = false, hr = false, hs = false;
    PF_CUDA(c->out_ptr(5, hit, n * 4, &dhit, &hh));
    if (pos3) PF_CUDA(c->out_ptr(6, pos3, n * 24, &dpos, &hp));
    if (rgba4) PF_CUDA(c->out_ptr(7, rgba4, n * 32, &drgba, &hr));
    if (scalar1) PF_CUDA(c->out_ptr(8, scalar1, n * 8, &dsc, &hs));
    B.hit = (int *)dhit;
    B.pos3 = (double *)dpos;
    B.rgba4 = (double *)drgba;
    B.scalar = (double *)dsc;
    const DevScene S = c->scene();
    PF_CUDA(fp64 ? launch_delta_track_batch_parity(S, B, c->stream) : launch_delta_track_batch_fast(S, B, c->stream));
    if (hh) PF_CUDA(cudaMemcpyAsync(hit, dhit, n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (hp) PF_CUDA(cudaMemcpyAsync(pos3, dpos, n * 24, cudaMemcpyDeviceToHost, c->stream));
    if (hr) PF_CUDA(cudaMemcpyAsync(rgba4, drgba, n * 32, cudaMemcpyDeviceToHost, c->stream));
    if (hs) PF_CUDA(cudaMemcpyAsync(scalar1, dsc, n * 8, cudaMemcpyDeviceToHost, c->stream));
    if (hh || hp || hr || hs) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

static int transmittance_common(pf_ctx *c, size_t n, const double *a3, const double *b3, uint64_t seed,
                                uint64_t stream, const uint64_t *idx, int n_trials, double *out, bool ratio) {
    if (!c || (n && (!a3 || !b3 || !idx || !out))) return set_err(PF_ERR_INVALID, "transmittance: null argument");
    if (n_trials <= 0) return set_err(PF_ERR_INVALID, "transmittance: n_trials must be positive");
    if (!c->vol_tex || !c->has_medium) return set_err(PF_ERR_INVALID, "transmittance: volume/medium not set");
    if (n == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    BatchParams B;
    if (int e = batch_common(c, n, a3, b3, idx, B)) return e;
    B.initstate = stream_initstate(seed, stream);
    B.n_trials = n_trials;
    void *dout;
    bool ho;
    PF_CUDA(c->out_ptr(5, out, n * 8, &dout, &ho));
    B.out = (double *)dout;
    const DevScene S = c->scene();
    PF_CUDA(ratio ? launch_transmittance_ratio_batch(S, B, c->stream) : launch_transmittance_batch(S, B, c->stream));
    if (ho) {
        PF_CUDA(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
    }
    return PF_OK;
}

int pf_transmittance_batch(pf_ctx *c, size_t n, const double *a3, const double *b3, uint64_t seed,
                           uint64_t stream, const uint64_t *idx, int n_trials, double *out) {
    return transmittance_common(c, n, a3, b3, seed, stream, idx, n_trials, out, false);
}

int pf_transmittance_ratio_batch(pf_ctx *c, size_t n, const double *a3, const double *b3, uint64_t seed,
                                 uint64_t stream, const uint64_t *idx, int n_trials, double *out) {
    return transmittance_common(c, n, a3, b3, seed, stream, idx, n_trials, out, true);
}

int pf_rng_doubles(pf_ctx *c, size_t n, uint64_t seed, uint64_t stream, const uint64_t *idx, int n_draws,
                   double *out) {
    if (!c || (n && (!idx || !out)) || n_draws <= 0) return set_err(PF_ERR_INVALID, "pf_rng_doubles: bad argument");
    if (n == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    BatchParams B;
    std::memset(&B, 0, sizeof(B));
    B.n = n;
    B.n_trials = n_draws;
    B.initstate = stream_initstate(seed, stream);
    const void *di;
    PF_CUDA(c->stage_in(0, idx, n * 8, &di));
    B.idx = (const uint64_t *)di;
    void *dout;
    bool ho;
    PF_CUDA(c->out_ptr(1, out, n * n_draws * 8, &dout, &ho));
    B.out = (double *)dout;
    PF_CUDA(launch_rng_doubles(B, c->stream));
    if (ho) {
        PF_CUDA(cudaMemcpyAsync(out, dout, n * n_draws * 8, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
    }
    return PF_OK;
}

// --------------------------------------------------------- photon trace --
// Scratch deposits are 44 B each (record + owning photon); bound the first
// attempt's scratch by this budget, retrace with the exact size on overflow.
static constexpr size_t kTraceScratchBudget = size_t(4) << 30;

int pf_trace_photons(pf_ctx *c, const pf_trace_desc *d, size_t *n_photons, uint64_t *emitted) {
    if (!c || !d || (d->n_phases > 0 && !d->phase_set)) return set_err(PF_ERR_INVALID, "pf_trace_photons: null argument");
    if (c->lights.empty()) return set_err(PF_ERR_INVALID, "TraceConfig: at least one light required");
    if (d->n_phases < 1) return set_err(PF_ERR_INVALID, "TraceConfig: phase set must be non-empty");
    if (d->n_phases > PF_MAX_TRACE_PHASES)
        return set_err(PF_ERR_INVALID, "TraceConfig: at most %d phases", PF_MAX_TRACE_PHASES);
    for (int g = 0; g < d->n_phases; ++g) {
        if (!(d->phase_set[g] >= -1.0 && d->phase_set[g] <= 1.0))
            return set_err(PF_ERR_INVALID, "TraceConfig: phase values must lie in [-1,1]");
        for (int h = 0; h < g; ++h)
            if (d->phase_set[h] == d->phase_set[g]) return set_err(PF_ERR_INVALID, "TraceConfig: phase values must be distinct");
    }
    if (d->max_bounces < 1) return set_err(PF_ERR_INVALID, "TraceConfig: max_bounces must be positive");
    if (d->max_bounces > 65536)  // deposit ordinals travel in 16 bits (pf_photon.cu)
        return set_err(PF_ERR_INVALID, "TraceConfig: max_bounces must be <= 65536");
    if (d->rr_start_bounce < 0) return set_err(PF_ERR_INVALID, "TraceConfig: rr_start_bounce must be >= 0");
    if (!(d->rr_min_survival > 0.0 && d->rr_min_survival <= d->rr_max_survival && d->rr_max_survival <= 1.0))
        return set_err(PF_ERR_INVALID, "TraceConfig: need 0 < rr_min_survival <= rr_max_survival <= 1");
    if (d->n_total >= 0xFFFFFFFFull) return set_err(PF_ERR_INVALID, "TraceConfig: n_total must be < 2^32");
    if (!c->vol_tex || !c->has_medium) return set_err(PF_ERR_INVALID, "pf_trace_photons: volume/medium not set");
    PF_CUDA(cudaSetDevice(c->device));
    const uint64_t n = d->n_total;
    const uint64_t pairs = (uint64_t)(c->lights.size() / 6) * (uint64_t)d->n_phases;
    if (emitted)
        for (uint64_t p = 0; p < pairs; ++p) emitted[p] = n / pairs + (p < n % pairs ? 1u : 0u);
    c->has_trace = false;
    c->t_n = 0;
    c->t_total = n;
    if (n_photons) *n_photons = 0;
    if (n == 0) {
        c->has_trace = true;
        return PF_OK;
    }
    PhotonTraceParams P;
    std::memset(&P, 0, sizeof(P));
    P.n_total = n;
    P.initstate = stream_initstate(d->seed, 1 /* Stream::Trace, rng.hpp:63 */);
    P.n_phases = d->n_phases;
    P.max_bounces = d->max_bounces;
    P.rr_start = d->rr_start_bounce;
    P.rr_min = d->rr_min_survival;
    P.rr_max = d->rr_max_survival;
    for (int g = 0; g < d->n_phases; ++g) P.g[g] = d->phase_set[g];
    PF_CUDA(c->t_counts.ensure(n * 4));
    PF_CUDA(c->t_ctr.ensure(16));
    P.counts = (uint32_t *)c->t_counts.p;
    P.counter = (unsigned long long *)c->t_ctr.p;
    P.steps = P.counter + 1;
    const uint64_t max_dep = n * (uint64_t)(d->max_bounces - 1);
    uint64_t cap = std::min<uint64_t>(max_dep, std::max<uint64_t>(n * 4, 1024));
    cap = std::min<uint64_t>(cap, kTraceScratchBudget / 44);
    const DevScene S = c->scene();
    unsigned long long hc[2] = {0, 0};
    for (int attempt = 0; attempt < 2; ++attempt) {
        PF_CUDA(c->t_rec.ensure(std::max<uint64_t>(cap, 1) * sizeof(PhotonOut)));
        PF_CUDA(c->t_rec_photon.ensure(std::max<uint64_t>(cap, 1) * 4));
        P.rec = (PhotonOut *)c->t_rec.p;
        P.rec_photon = (uint32_t *)c->t_rec_photon.p;
        P.cap = cap;
        PF_CUDA(cudaMemsetAsync(c->t_ctr.p, 0, 16, c->stream));
        if (c->timing) cudaEventRecord(c->ev[0], c->stream);
        PF_CUDA(launch_trace_photons(S, P, c->stream));
        if (c->timing) cudaEventRecord(c->ev[1], c->stream);
        PF_CUDA(cudaMemcpyAsync(hc, c->t_ctr.p, 16, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
        if (hc[0] <= cap) break;
        cap = hc[0];  // deterministic: the retrace deposits exactly hc[0]
    }
    const uint64_t total = hc[0];
    if (total >= 0xFFFFFFFFull) return set_err(PF_ERR_RUNTIME, "trace_photons: more than 2^32 deposits");
    size_t tmp_bytes = 0;
    PF_CUDA(photon_scan_bytes(n, &tmp_bytes));
    PF_CUDA(c->t_tmp.ensure(tmp_bytes));
    PF_CUDA(c->t_offs.ensure(n * 4));
    PF_CUDA(c->t_out.ensure(std::max<uint64_t>(total, 1) * sizeof(PhotonOut)));
    if (c->timing) cudaEventRecord(c->ev[3], c->stream);
    PF_CUDA(launch_photon_compact(P.counts, (uint32_t *)c->t_offs.p, n, c->t_tmp.p, tmp_bytes, P.rec,
                                  P.rec_photon, total, (PhotonOut *)c->t_out.p, c->stream));
    if (c->timing) cudaEventRecord(c->ev[2], c->stream);
    c->t_n = total;
    c->trace_steps = hc[1];
    c->has_trace = true;
    if (n_photons) *n_photons = total;
    return PF_OK;
}

int pf_trace_fetch(pf_ctx *c, pf_photon *out, size_t n) {
    if (!c || (n && !out)) return set_err(PF_ERR_INVALID, "pf_trace_fetch: null argument");
    if (!c->has_trace) return set_err(PF_ERR_INVALID, "pf_trace_fetch: call pf_trace_photons first");
    if (n != c->t_n) return set_err(PF_ERR_INVALID, "pf_trace_fetch: expected %zu records", c->t_n);
    if (n == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    const bool dev = is_device_ptr(out);
    PF_CUDA(cudaMemcpyAsync(out, c->t_out.p, n * sizeof(pf_photon),
                            dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
    if (!dev) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_trace_path_counts(pf_ctx *c, uint32_t *out, uint64_t n_total) {
    if (!c || (n_total && !out)) return set_err(PF_ERR_INVALID, "pf_trace_path_counts: null argument");
    if (!c->has_trace) return set_err(PF_ERR_INVALID, "pf_trace_path_counts: call pf_trace_photons first");
    if (n_total != c->t_total) return set_err(PF_ERR_INVALID, "pf_trace_path_counts: expected %llu photons",
                                              (unsigned long long)c->t_total);
    if (n_total == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    const bool dev = is_device_ptr(out);
    PF_CUDA(cudaMemcpyAsync(out, c->t_counts.p, n_total * 4, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                            c->stream));
    if (!dev) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_trace_stats(pf_ctx *c, double *ms_trace, double *ms_compact, uint64_t *tentative_collisions) {
    if (!c || !c->has_trace) return set_err(PF_ERR_INVALID, "pf_trace_stats: call pf_trace_photons first");
    if (tentative_collisions) *tentative_collisions = c->trace_steps;
    float a = 0.f, b = 0.f;
    if (c->timing && c->t_n > 0) {
        PF_CUDA(cudaEventSynchronize(c->ev[2]));
        PF_CUDA(cudaEventElapsedTime(&a, c->ev[0], c->ev[1]));
        PF_CUDA(cudaEventElapsedTime(&b, c->ev[3], c->ev[2]));
    }
    if (ms_trace) *ms_trace = a;
    if (ms_compact) *ms_compact = b;
    return PF_OK;
}

int pf_knn_build_traced(pf_ctx *c, int n_phases, const double *phase_set) {
    if (!c || !c->has_trace) return set_err(PF_ERR_INVALID, "pf_knn_build_traced: call pf_trace_photons first");
    return pf_knn_build(c, (const pf_photon *)c->t_out.p, c->t_n, n_phases, phase_set);
}

// ------------------------------------------------------------------ knn --
int pf_knn_build(pf_ctx *c, const pf_photon *photons, size_t n, int n_phases, const double *phase_set) {
    if (!c || (n && !photons) || !phase_set) return set_err(PF_ERR_INVALID, "pf_knn_build: null argument");
    if (n_phases < 1 || n_phases > PF_MAX_PHASES)
        return set_err(PF_ERR_INVALID, "pf_knn_build: 1..%d phases", PF_MAX_PHASES);
    if (n >= 0xFFFFFFFFull) return set_err(PF_ERR_INVALID, "pf_knn_build: too many photons");
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(c->k_photons.ensure(n * sizeof(PhotonRec)));
    if (n) {
        if (is_device_ptr(photons))
            PF_CUDA(cudaMemcpyAsync(c->k_photons.p, photons, n * 40, cudaMemcpyDeviceToDevice, c->stream));
        else
            PF_CUDA(cudaMemcpyAsync(c->k_photons.p, photons, n * 40, cudaMemcpyHostToDevice, c->stream));
    }
    // per-phase bounding boxes + counts
    PF_CUDA(c->k_bbox.ensure(PF_MAX_PHASES * 7 * 4));
    uint32_t init[PF_MAX_PHASES * 7];
    for (int i = 0; i < PF_MAX_PHASES * 3; ++i) init[i] = 0xFFFFFFFFu;
    for (int i = PF_MAX_PHASES * 3; i < PF_MAX_PHASES * 7; ++i) init[i] = 0u;
    PF_CUDA(cudaMemcpyAsync(c->k_bbox.p, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    uint32_t *mins = (uint32_t *)c->k_bbox.p, *maxs = mins + PF_MAX_PHASES * 3, *cnts = mins + PF_MAX_PHASES * 6;
    PF_CUDA(knn_bbox((const PhotonRec *)c->k_photons.p, n, n_phases, mins, maxs, cnts, c->stream));
    uint32_t hb[PF_MAX_PHASES * 7];
    PF_CUDA(cudaMemcpyAsync(hb, c->k_bbox.p, sizeof(hb), cudaMemcpyDeviceToHost, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    auto ord2f = [](uint32_t u) {
        uint32_t b = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
        float f;
        std::memcpy(&f, &b, 4);
        return f;
    };
    KnnParams K;
    std::memset(&K, 0, sizeof(K));
    K.n_phases = n_phases;
    uint32_t base = 0;
    for (int g = 0; g < n_phases; ++g) {
        KnnGrid &G = K.grid[g];
        K.phase[g] = phase_set[g];
        G.n = hb[PF_MAX_PHASES * 6 + g];
        G.cell_base = base;
        if (G.n == 0) {
            for (int a = 0; a < 3; ++a) {
                G.lo[a] = 0.0;
                G.h[a] = 1.0;
                G.inv_h[a] = 1.0;
                G.R[a] = 1;
            }
            G.hmin = 1.0;
            G.eps = 0.0;
            base += 1;
            continue;
        }
        double lo[3], ext[3], vol = 1.0;
        for (int a = 0; a < 3; ++a) {
            lo[a] = (double)ord2f(hb[3 * g + a]);
            const double hi = (double)ord2f(hb[PF_MAX_PHASES * 3 + 3 * g + a]);
            ext[a] = std::max(hi - lo[a], 1e-6);
            vol *= ext[a];
        }
        // ~8 photons of this phase per cell (K=64 reaches its K-th within ~1.2 cells)
        double h = std::cbrt(knn_photons_per_cell() * vol / (double)G.n);
        uint64_t cells = 1;
        for (int a = 0; a < 3; ++a) {
            G.R[a] = (int)std::min(1024.0, std::max(1.0, std::ceil(ext[a] / h)));
            cells *= (uint64_t)G.R[a];
        }
        while (cells > 4ull * G.n + 64) {  // degenerate extents: coarsen
            cells = 1;
            for (int a = 0; a < 3; ++a) {
                G.R[a] = std::max(1, G.R[a] / 2);
                cells *= (uint64_t)G.R[a];
            }
        }
        G.hmin = 1e300;
        for (int a = 0; a < 3; ++a) {
            G.lo[a] = lo[a];
            G.h[a] = ext[a] / G.R[a];
            G.inv_h[a] = 1.0 / G.h[a];
            G.hmin = std::min(G.hmin, G.h[a]);
        }
        G.eps = 1e-6 * std::max(ext[0], std::max(ext[1], ext[2])) + 1e-30;
        base += (uint32_t)cells;
    }
    K.total_cells = base;
    if (int e = (int)knn_sort((const PhotonRec *)c->k_photons.p, n, K, c->kb, c->stream))
        return set_err(PF_ERR_RUNTIME, "knn build: %s", cudaGetErrorString((cudaError_t)e));
    K.spos = (const float4 *)c->kb.spos.p;
    K.spay = (const float4 *)c->kb.spay.p;
    K.inv = (const uint32_t *)c->kb.inv.p;
    K.cell_start = (const uint32_t *)c->kb.cell_start.p;
    K.photons = (const PhotonRec *)c->k_photons.p;
    c->knn = K;
    c->k_n = n;
    c->has_knn = true;
    return PF_OK;
}

static int knn_run(pf_ctx *c, size_t nq, const float *x3, const double *w3, const uint8_t *gidx, int K,
                   float r_max, double psi, double *out3, uint32_t *ids, float *d2, int32_t *counts) {
    if (!c->has_knn) return set_err(PF_ERR_INVALID, "knn: call pf_knn_build first");
    if (K < 1 || K > 1024) return set_err(PF_ERR_INVALID, "KnnQuery: K must be in [1, 1024]");
    if (!(r_max > 0.0f)) return set_err(PF_ERR_INVALID, "KnnQuery: r_max must be > 0");
    if (nq == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    KnnParams P = c->knn;
    const void *dx, *dg, *dw = nullptr;
    PF_CUDA(c->stage_in(0, x3, nq * 12, &dx));
    PF_CUDA(c->stage_in(1, gidx, nq, &dg));
    if (w3) PF_CUDA(c->stage_in(2, w3, nq * 24, &dw));
    void *dids = nullptr, *dd2 = nullptr, *dcnt = nullptr, *dout = nullptr;
    bool hi = false, hd = false, hc = false, ho = false;
    if (ids) PF_CUDA(c->out_ptr(3, ids, nq * K * 4, &dids, &hi));
    if (d2) PF_CUDA(c->out_ptr(4, d2, nq * K * 4, &dd2, &hd));
    if (counts) PF_CUDA(c->out_ptr(5, counts, nq * 4, &dcnt, &hc));
    if (out3) PF_CUDA(c->out_ptr(6, out3, nq * 24, &dout, &ho));
    P.nq = nq;
    P.qx = (const float *)dx;
    P.qg = (const uint8_t *)dg;
    P.qw = (const double *)dw;
    P.K = K;
    P.r2 = r_max * r_max;
    P.psi = psi;
    P.enc_threshold = std::pow(10.0, -psi);
    P.out_ids = (uint32_t *)dids;
    P.out_d2 = (float *)dd2;
    P.out_counts = (int32_t *)dcnt;
    P.out_targets = (double *)dout;
    P.order = nullptr;
    if (nq >= 4096) PF_CUDA(knn_order(P.qx, P.qg, nq, c->kb, &P.order, c->stream));
    PF_CUDA(knn_query_auto(P, c->kb, c->stream));
    if (hi) PF_CUDA(cudaMemcpyAsync(ids, dids, nq * K * 4, cudaMemcpyDeviceToHost, c->stream));
    if (hd) PF_CUDA(cudaMemcpyAsync(d2, dd2, nq * K * 4, cudaMemcpyDeviceToHost, c->stream));
    if (hc) PF_CUDA(cudaMemcpyAsync(counts, dcnt, nq * 4, cudaMemcpyDeviceToHost, c->stream));
    if (ho) PF_CUDA(cudaMemcpyAsync(out3, dout, nq * 24, cudaMemcpyDeviceToHost, c->stream));
    if (hi || hd || hc || ho) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_knn_query(pf_ctx *c, size_t nq, const float *x3, const uint8_t *gidx, int K, float r_max, uint32_t *ids,
                 float *d2, int32_t *counts) {
    if (!c || (nq && (!x3 || !gidx || !ids))) return set_err(PF_ERR_INVALID, "pf_knn_query: null argument");
    return knn_run(c, nq, x3, nullptr, gidx, K, r_max, 5.0, nullptr, ids, d2, counts);
}

int pf_knn_targets(pf_ctx *c, size_t nq, const float *x3, const double *w3, const uint8_t *gidx, int K,
                   float r_max, double psi, double *out3, uint32_t *ids, float *d2, int32_t *counts) {
    if (!c || (nq && (!x3 || !w3 || !gidx || !out3))) return set_err(PF_ERR_INVALID, "pf_knn_targets: null argument");
    if (!(psi > 0.0)) return set_err(PF_ERR_INVALID, "EncodingConfig: psi must be positive");
    return knn_run(c, nq, x3, w3, gidx, K, r_max, psi, out3, ids, d2, counts);
}

int pf_make_batch(pf_ctx *c, uint64_t seed, uint64_t step, size_t batch, int K, float r_max, double psi, float *x3,
                  double *w3, uint8_t *gidx, double *targets3) {
    if (!c || (batch && (!x3 || !w3 || !gidx || !targets3))) return set_err(PF_ERR_INVALID, "pf_make_batch: null argument");
    if (!c->has_knn) return set_err(PF_ERR_INVALID, "make_batch: call pf_knn_build first");
    if (batch == 0) return PF_OK;
    PF_CUDA(cudaSetDevice(c->device));
    void *dx, *dw, *dg;
    bool hx, hw, hg;
    PF_CUDA(c->out_ptr(0, x3, batch * 12, &dx, &hx));
    PF_CUDA(c->out_ptr(1, w3, batch * 24, &dw, &hw));
    PF_CUDA(c->out_ptr(2, gidx, batch, &dg, &hg));
    PF_CUDA(knn_make_queries(stream_initstate(seed, PF_STREAM_TRAIN), step * (uint64_t)batch, batch,
                             c->knn.n_phases, (float *)dx, (double *)dw, (uint8_t *)dg, c->stream));
    if (int e = knn_run(c, batch, (const float *)dx, (const double *)dw, (const uint8_t *)dg, K, r_max, psi,
                        targets3, nullptr, nullptr, nullptr))
        return e;
    if (hx) PF_CUDA(cudaMemcpyAsync(x3, dx, batch * 12, cudaMemcpyDeviceToHost, c->stream));
    if (hw) PF_CUDA(cudaMemcpyAsync(w3, dw, batch * 24, cudaMemcpyDeviceToHost, c->stream));
    if (hg) PF_CUDA(cudaMemcpyAsync(gidx, dg, batch, cudaMemcpyDeviceToHost, c->stream));
    if (hx || hw || hg) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

// ------------------------------------------------------------- training --
static void adam_defaults(pf_adam_desc &a) {
    a.lr = 9e-4;
    a.beta1 = 0.9;
    a.beta2 = 0.99;
    a.eps = 1e-8;
    a.decay = 0.92;
    a.decay_start = 0.7;
    a.decay_interval = 25;
    a.eps_rel = 0.01;
}

int pf_train_init(pf_ctx *c, const pf_field_desc *d, const float *params, size_t n, const pf_adam_desc *adam) {
    if (!c || !d || !params) return set_err(PF_ERR_INVALID, "pf_train_init: null argument");
    FieldDesc f = to_fdesc(d);
    if (const char *m = field_validate(f)) return set_err(PF_ERR_INVALID, "%s", m);
    if (n != field_param_count(f))
        return set_err(PF_ERR_INVALID, "pf_train_init: expected %zu params, got %zu", field_param_count(f), n);
    pf_adam_desc a;
    adam_defaults(a);
    if (adam) a = *adam;
    if (!(a.lr > 0.0) || !(a.beta1 >= 0.0 && a.beta1 < 1.0) || !(a.beta2 >= 0.0 && a.beta2 < 1.0) || !(a.eps > 0.0) ||
        !(a.decay > 0.0 && a.decay <= 1.0) || !(a.decay_start >= 0.0) || a.decay_interval < 1 || !(a.eps_rel > 0.0))
        return set_err(PF_ERR_INVALID, "AdamState: invalid hyper-parameters");
    // the inference field shares the layout: load it too (render/query see the initial field)
    if (int e = field_load(c, f, params, n)) return e;
    PF_CUDA(cudaSetDevice(c->device));
    TrainState &S = c->train;
    S.lr = a.lr;
    S.beta1 = a.beta1;
    S.beta2 = a.beta2;
    S.eps = a.eps;
    S.decay = a.decay;
    S.decay_start = a.decay_start;
    S.decay_interval = a.decay_interval;
    S.eps_rel = a.eps_rel;
    const void *dp;
    PF_CUDA(c->stage_in(0, params, n * 4, &dp));
    PF_CUDA(train_init(S, f, c->fhost.levels, (const float *)dp, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

static int train_common(pf_ctx *c, size_t n, const float *x3, const float *w2, const float *g, const float *t3,
                        uint64_t step, uint64_t total, bool update, double *loss, float *grad, uint8_t *touched) {
    if (!c || (n && (!x3 || !w2 || !g || !t3))) return set_err(PF_ERR_INVALID, "train_step: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "train_step: call pf_train_init first");
    if (n == 0) return set_err(PF_ERR_INVALID, "train_step: empty batch");
    if (update && (total == 0 || step >= total)) return set_err(PF_ERR_INVALID, "train_step: need 0 <= step < total");
    PF_CUDA(cudaSetDevice(c->device));
    TrainState &S = c->train;
    const void *dx, *dw, *dg, *dt;
    PF_CUDA(c->stage_in(0, x3, n * 12, &dx));
    PF_CUDA(c->stage_in(1, w2, n * 8, &dw));
    PF_CUDA(c->stage_in(2, g, n * 4, &dg));
    PF_CUDA(c->stage_in(3, t3, n * 12, &dt));
    void *dgrad = nullptr, *dtouch = nullptr;
    bool hgrad = false, htouch = false;
    if (grad) PF_CUDA(c->out_ptr(4, grad, S.n_params * 4, &dgrad, &hgrad));
    if (touched) PF_CUDA(c->out_ptr(5, touched, S.n_entries, &dtouch, &htouch));
    PF_CUDA(S.loss_dev.ensure(8));
    PF_CUDA(train_step(S, n, (const float *)dx, (const float *)dw, (const float *)dg, (const float *)dt, step, total,
                       update, (float *)dgrad, (uint8_t *)dtouch, 0, c->sms, c->stream));
    if (hgrad) PF_CUDA(cudaMemcpyAsync(grad, dgrad, S.n_params * 4, cudaMemcpyDeviceToHost, c->stream));
    if (htouch) PF_CUDA(cudaMemcpyAsync(touched, dtouch, S.n_entries, cudaMemcpyDeviceToHost, c->stream));
    if (loss) {
        PF_CUDA(cudaMemcpyAsync(loss, S.loss_dev.p, 8, cudaMemcpyDeviceToHost, c->stream));
    }
    if (loss || hgrad || htouch) PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_train_step(pf_ctx *c, size_t n, const float *x3, const float *w_sph2, const float *g, const float *targets3,
                  uint64_t step, uint64_t total_steps, double *loss) {
    return train_common(c, n, x3, w_sph2, g, targets3, step, total_steps, true, loss, nullptr, nullptr);
}

int pf_train_grad(pf_ctx *c, size_t n, const float *x3, const float *w_sph2, const float *g, const float *targets3,
                  double *loss, float *grad, uint8_t *touched) {
    return train_common(c, n, x3, w_sph2, g, targets3, 0, 1, false, loss, grad, touched);
}

int pf_train_backward(pf_ctx *c, size_t n, const float *x3, const float *w_sph2, const float *g,
                      const float *targets3, size_t n_global, double *loss_part) {
    if (!c || (n && (!x3 || !w_sph2 || !g || !targets3))) return set_err(PF_ERR_INVALID, "train_backward: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "train_backward: call pf_train_init first");
    if (n == 0 || n_global < n) return set_err(PF_ERR_INVALID, "train_backward: need 0 < n <= n_global");
    PF_CUDA(cudaSetDevice(c->device));
    TrainState &S = c->train;
    const void *dx, *dw, *dg, *dt;
    PF_CUDA(c->stage_in(0, x3, n * 12, &dx));
    PF_CUDA(c->stage_in(1, w_sph2, n * 8, &dw));
    PF_CUDA(c->stage_in(2, g, n * 4, &dg));
    PF_CUDA(c->stage_in(3, targets3, n * 12, &dt));
    PF_CUDA(S.loss_dev.ensure(8));
    PF_CUDA(train_backward(S, n, (const float *)dx, (const float *)dw, (const float *)dg, (const float *)dt, n_global, 0,
                           c->stream));
    if (loss_part) {
        PF_CUDA(cudaMemcpyAsync(loss_part, S.loss_dev.p, 8, cudaMemcpyDeviceToHost, c->stream));
        PF_CUDA(cudaStreamSynchronize(c->stream));
    }
    return PF_OK;
}

int pf_train_grad_buffers(pf_ctx *c, void **gtab, size_t *n_tab, void **gmlp, size_t *n_mlp, void **touched,
                          size_t *n_entries) {
    if (!c || !gtab || !n_tab || !gmlp || !n_mlp || !touched || !n_entries)
        return set_err(PF_ERR_INVALID, "pf_train_grad_buffers: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_grad_buffers: call pf_train_init first");
    TrainState &S = c->train;
    *gtab = S.gtab.p;
    *n_tab = S.n_tab;
    *gmlp = S.gmlp.p;
    *n_mlp = S.n_params - S.n_tab;
    *touched = S.touched.p;
    *n_entries = S.n_entries;
    return PF_OK;
}

int pf_train_apply(pf_ctx *c, uint64_t step, uint64_t total_steps) {
    if (!c) return set_err(PF_ERR_INVALID, "null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_apply: call pf_train_init first");
    if (total_steps == 0 || step >= total_steps) return set_err(PF_ERR_INVALID, "train_step: need 0 <= step < total");
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(train_finish(c->train, step, total_steps, true, nullptr, nullptr, c->stream));
    return PF_OK;
}

int pf_train_counts(pf_ctx *c, size_t *n_params, size_t *n_entries) {
    if (!c || !n_params || !n_entries) return set_err(PF_ERR_INVALID, "null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "call pf_train_init first");
    *n_params = c->train.n_params;
    *n_entries = c->train.n_entries;
    return PF_OK;
}

int pf_train_params(pf_ctx *c, float *out, size_t n) {
    if (!c || !out) return set_err(PF_ERR_INVALID, "pf_train_params: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_params: call pf_train_init first");
    if (n != c->train.n_params) return set_err(PF_ERR_INVALID, "pf_train_params: expected %zu", c->train.n_params);
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(cudaMemcpyAsync(out, c->train.params.p, n * 4, cudaMemcpyDefault, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_train_commit(pf_ctx *c) {
    if (!c) return set_err(PF_ERR_INVALID, "null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_commit: call pf_train_init first");
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    return field_load(c, c->train.fd, (const float *)c->train.params.p, c->train.n_params);
}

int pf_train(pf_ctx *c, const pf_train_desc *d, double *loss_history, double *ms_knn, double *ms_step,
             double *ms_knn_steps, double *ms_step_steps) {
    if (!c || !d) return set_err(PF_ERR_INVALID, "pf_train: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train: call pf_train_init first");
    if (d->total_steps < 1 || d->batch < 1) return set_err(PF_ERR_INVALID, "TrainConfig: total_steps, batch >= 1");
    if (d->n_segments < 1 || !d->seg_end || !d->seg_radius)
        return set_err(PF_ERR_INVALID, "KnnSchedule: at least one segment");
    for (int i = 0; i < d->n_segments; ++i) {
        if (!(d->seg_end[i] > 0.0 && d->seg_end[i] <= 1.0) || (i && !(d->seg_end[i] > d->seg_end[i - 1])))
            return set_err(PF_ERR_INVALID, "KnnSchedule: fractions must be strictly increasing in (0, 1]");
        if (!(d->seg_radius[i] > 0.0) || (i && !(d->seg_radius[i] > d->seg_radius[i - 1])))
            return set_err(PF_ERR_INVALID, "KnnSchedule: radii must be positive and strictly increasing");
    }
    if (d->seg_end[d->n_segments - 1] != 1.0) return set_err(PF_ERR_INVALID, "KnnSchedule: last fraction must be 1");
    if (d->K < 1 || d->K > 1024) return set_err(PF_ERR_INVALID, "KnnQuery: K must be in [1, 1024]");
    if (!(d->psi > 0.0)) return set_err(PF_ERR_INVALID, "EncodingConfig: psi must be positive");
    if (!c->has_knn) return set_err(PF_ERR_INVALID, "pf_train: call pf_knn_build first");
    const uint64_t stop = d->stop_step ? d->stop_step : d->total_steps;
    if (stop > d->total_steps || d->start_step > stop)
        return set_err(PF_ERR_INVALID, "pf_train: need start_step <= stop_step <= total_steps");
    PF_CUDA(cudaSetDevice(c->device));
    TrainState &S = c->train;
    const size_t B = d->batch;
    PF_CUDA(c->tr_x.ensure(B * 12));
    PF_CUDA(c->tr_w3.ensure(B * 24));
    PF_CUDA(c->tr_gi.ensure(B));
    PF_CUDA(c->tr_t3d.ensure(B * 24));
    PF_CUDA(c->tr_w2.ensure(B * 8));
    PF_CUDA(c->tr_g.ensure(B * 4));
    PF_CUDA(c->tr_t.ensure(B * 12));
    PF_CUDA(S.loss_dev.ensure(d->total_steps * 8));
    cudaEvent_t ev[3];
    for (auto &e : ev) PF_CUDA(cudaEventCreate(&e));
    double knn_ms = 0.0, step_ms = 0.0;
    const uint64_t init = stream_initstate(d->seed, PF_STREAM_TRAIN);
    for (uint64_t step = d->start_step; step < stop; ++step) {
        // schedule_radius
        const double progress = (double)(step + 1) / (double)d->total_steps;
        double r = d->seg_radius[d->n_segments - 1];
        for (int i = 0; i < d->n_segments; ++i)
            if (d->seg_end[i] >= progress) {
                r = d->seg_radius[i];
                break;
            }
        cudaEventRecord(ev[0], c->stream);
        // make_batch on the device
        PF_CUDA(knn_make_queries(init, step * (uint64_t)B, B, c->knn.n_phases, (float *)c->tr_x.p,
                                 (double *)c->tr_w3.p, (uint8_t *)c->tr_gi.p, c->stream));
        if (int e = knn_run(c, B, (const float *)c->tr_x.p, (const double *)c->tr_w3.p, (const uint8_t *)c->tr_gi.p,
                            d->K, (float)r, d->psi, (double *)c->tr_t3d.p, nullptr, nullptr, nullptr))
            return e;
        cudaEventRecord(ev[1], c->stream);
        PF_CUDA(train_prep((const double *)c->tr_w3.p, (const uint8_t *)c->tr_gi.p, (const double *)c->tr_t3d.p,
                           c->knn.phase, c->knn.n_phases, B, (float *)c->tr_w2.p, (float *)c->tr_g.p,
                           (float *)c->tr_t.p, c->stream));
        PF_CUDA(train_step(S, B, (const float *)c->tr_x.p, (const float *)c->tr_w2.p, (const float *)c->tr_g.p,
                           (const float *)c->tr_t.p, step, d->total_steps, true, nullptr, nullptr, (size_t)step, c->sms,
                           c->stream));
        cudaEventRecord(ev[2], c->stream);
        PF_CUDA(cudaEventSynchronize(ev[2]));
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        knn_ms += a;
        step_ms += b;
        if (ms_knn_steps) ms_knn_steps[step] = a;
        if (ms_step_steps) ms_step_steps[step] = b;
    }
    for (auto &e : ev) cudaEventDestroy(e);
    if (loss_history && stop > d->start_step)
        PF_CUDA(cudaMemcpyAsync(loss_history + d->start_step, (const double *)S.loss_dev.p + d->start_step,
                                (stop - d->start_step) * 8, cudaMemcpyDefault, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    if (ms_knn) *ms_knn = knn_ms;
    if (ms_step) *ms_step = step_ms;
    // the renderer / field queries now use the trained field
    return field_load(c, S.fd, (const float *)S.params.p, S.n_params);
}

int pf_train_state_get(pf_ctx *c, float *params, float *m, float *v, size_t n) {
    if (!c) return set_err(PF_ERR_INVALID, "null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_state_get: call pf_train_init first");
    if (n != c->train.n_params) return set_err(PF_ERR_INVALID, "pf_train_state_get: expected %zu", c->train.n_params);
    PF_CUDA(cudaSetDevice(c->device));
    const void *src[3] = {c->train.params.p, c->train.m.p, c->train.v.p};
    float *dst[3] = {params, m, v};
    for (int k = 0; k < 3; ++k)
        if (dst[k]) PF_CUDA(cudaMemcpyAsync(dst[k], src[k], n * 4, cudaMemcpyDefault, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    return PF_OK;
}

int pf_train_state_set(pf_ctx *c, const float *params, const float *m, const float *v, size_t n) {
    if (!c || !params || !m || !v) return set_err(PF_ERR_INVALID, "pf_train_state_set: null argument");
    if (!c->train.ready) return set_err(PF_ERR_INVALID, "pf_train_state_set: call pf_train_init first");
    if (n != c->train.n_params) return set_err(PF_ERR_INVALID, "pf_train_state_set: expected %zu", c->train.n_params);
    PF_CUDA(cudaSetDevice(c->device));
    void *dst[3] = {c->train.params.p, c->train.m.p, c->train.v.p};
    const float *src[3] = {params, m, v};
    for (int k = 0; k < 3; ++k) PF_CUDA(cudaMemcpyAsync(dst[k], src[k], n * 4, cudaMemcpyDefault, c->stream));
    PF_CUDA(cudaStreamSynchronize(c->stream));
    return field_load(c, c->train.fd, (const float *)c->train.params.p, c->train.n_params);
}

// ----------------------------------------- multi-GPU frame over peer memory --
int pf_ipc_frame_create(pf_ctx *c, size_t bytes, void **dev_ptr, void *handle64) {
    if (!c || !dev_ptr || !handle64 || bytes == 0) return set_err(PF_ERR_INVALID, "pf_ipc_frame_create: bad argument");
    PF_CUDA(cudaSetDevice(c->device));
    void *p = nullptr;
    PF_CUDA(cudaMalloc(&p, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return set_err(PF_ERR_RUNTIME, "cudaIpcGetMemHandle failed: %s", cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, 64);
    PF_CUDA(cudaMemset(p, 0, bytes));
    *dev_ptr = p;
    return PF_OK;
}

int pf_ipc_frame_open(pf_ctx *c, const void *handle64, void **dev_ptr) {
    if (!c || !dev_ptr || !handle64) return set_err(PF_ERR_INVALID, "pf_ipc_frame_open: null argument");
    PF_CUDA(cudaSetDevice(c->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    PF_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return PF_OK;
}

int pf_ipc_frame_release(pf_ctx *c, void *dev_ptr, int owner) {
    if (!c || !dev_ptr) return set_err(PF_ERR_INVALID, "pf_ipc_frame_release: null argument");
    PF_CUDA(cudaSetDevice(c->device));
    PF_CUDA(owner ? cudaFree(dev_ptr) : cudaIpcCloseMemHandle(dev_ptr));
    return PF_OK;
}

}  // extern "C"
